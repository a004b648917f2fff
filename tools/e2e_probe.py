"""Where does the host-buffer (e2e) time of the cfg5 batch go?  Times gna_oscprob_batch_host
with pinned vs pageable outputs, several chunk sizes, and chi2-only (no spectra D2H)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07682_b200 as gna  # noqa: E402
import synth  # noqa: E402


def pinned(a):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).pin_memory()
    return t, t.numpy()


def main():
    torch.cuda.set_device(0)
    c = synth.config("cfg5")
    keep = []
    pts = {}
    for k, v in c["points"].items():
        t, a = pinned(v)
        keep.append(t)
        pts[k] = a
    te, edges = pinned(c["edges"])
    td, data = pinned(c["data"])
    ts, spectra = pinned(np.empty((1000, 10_000)))
    tx, chi2 = pinned(np.empty(1000))
    keep += [te, td, ts, tx]
    spectra_pageable = np.empty((1000, 10_000))

    def run(label, reps=5, **kw):
        gna.oscprob_batch_host(pts, c["L_km"], c["omega"], edges, c["order"], data=data, **kw)
        t0 = time.perf_counter()
        for _ in range(reps):
            gna.oscprob_batch_host(pts, c["L_km"], c["omega"], edges, c["order"], data=data, **kw)
        dt = (time.perf_counter() - t0) / reps
        print("%-40s %.3f ms/step  %.1f G energy points/s" % (label, dt * 1e3, 8e8 / dt / 1e9))

    run("pinned, default chunk", spectra=spectra, chi2=chi2)
    for cp in (25, 50, 200, 500, 1000):
        run("pinned, chunk %d points" % cp, spectra=spectra, chi2=chi2, chunk_points=cp)
    run("pageable spectra, default chunk", spectra=spectra_pageable, chi2=chi2)
    run("chi2 only (no spectra D2H)", spectra=False, chi2=chi2)
    # raw D2H bandwidth of 80 MB from device to the pinned buffer (torch copy)
    d = torch.empty((1000, 10_000), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        ts.copy_(d)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print("torch D2H 80 MB into pinned: %.3f ms (%.1f GB/s)" % (dt * 1e3, 80e6 / dt / 1e9))


if __name__ == "__main__":
    main()

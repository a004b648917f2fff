"""Where do the ~0.25 ms between the chunked host call with spectra (2.17 ms) and the chi^2-only
call (1.92 ms) go on cfg5?  (a) the batch split into device-only chunk calls (kernel efficiency
of chunking); (b) an 80 MB D2H alone and while the full batch kernel runs on another stream."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07682_b200 as gna  # noqa: E402
import synth  # noqa: E402


def ev_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    c = synth.config("cfg5")
    f64 = dict(dtype=torch.float64, device="cuda")
    pts = {k: torch.tensor(v, **f64) for k, v in c["points"].items()}
    edges, data = torch.tensor(c["edges"], **f64), torch.tensor(c["data"], **f64)
    P, nb = 1000, c["edges"].size - 1
    sp = torch.empty((P, nb), **f64)
    x2 = torch.empty(P, **f64)
    ws = torch.empty(gna.oscprob_batch_workspace_size(P, 8, nb, 10) // 8 + 2, **f64)
    L, om = c["L_km"], c["omega"]

    def full():
        gna.oscprob_batch(pts, L, om, edges, 10, data=data, spectra=sp, chi2=x2, workspace=ws)
    print("device, one call of 1000 points: %.3f ms" % ev_time(full))
    for ch in (101, 200, 250):
        def chunked():
            for i, a in enumerate(range(0, P, ch)):
                b = min(P, a + ch)
                gna.oscprob_batch({k: v[a:b] for k, v in pts.items()}, L, om, edges, 10, data=data,
                                  spectra=sp[a:b], chi2=x2[a:b], workspace=ws, tables_valid=i > 0)
        print("device, chunks of %d points: %.3f ms" % (ch, ev_time(chunked)))
    host = torch.empty((P, nb), dtype=torch.float64).pin_memory()
    print("D2H 80 MB alone: %.3f ms" % ev_time(lambda: host.copy_(sp, non_blocking=True)))
    s2 = torch.cuda.Stream()

    def both():
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s2):
            host.copy_(sp, non_blocking=True)
        full()
        torch.cuda.current_stream().wait_stream(s2)
    print("D2H 80 MB on a 2nd stream + the full kernel: %.3f ms" % ev_time(both))
    hp = {k: np.ascontiguousarray(v) for k, v in c["points"].items()}
    he, hd = np.ascontiguousarray(c["edges"]), np.ascontiguousarray(c["data"])
    tp = [torch.from_numpy(v).pin_memory() for v in hp.values()]
    hp = dict(zip(hp.keys(), [t.numpy() for t in tp]))
    hs, hx = host.numpy(), torch.empty(P, dtype=torch.float64).pin_memory().numpy()
    for ch in (0, 101, 200, 250, 334):
        t = ev_time(lambda: gna.oscprob_batch_host(hp, L, om, he, 10, data=hd, spectra=hs, chi2=hx,
                                                   chunk_points=ch))
        print("host call, chunk_points=%d: %.3f ms" % (ch, t))


if __name__ == "__main__":
    main()

"""SHA-256 of the spectra and chi2 bytes of one batch workload, for bitwise comparison of
library builds (kernel variants must agree bit for bit).

usage: python tools/batch_digest.py [--lib path] [--workload cfg4|cfg5|...] [--points N]
"""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07682_b200 as gna  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--points", type=int, default=0, help="first N points only (0 = all)")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "mixed"])
    a = ap.parse_args()
    gna.load(a.lib)
    c = synth.config(a.workload)
    pts = c["points"]
    if a.points:
        pts = {k: v[:a.points] for k, v in pts.items()}
    dev = torch.device("cuda", 0)
    t = {k: torch.tensor(v, dtype=torch.float64, device=dev) for k, v in pts.items()}
    sp, x2 = gna.oscprob_batch(t, c["L_km"], c["omega"],
                               torch.tensor(c["edges"], dtype=torch.float64, device=dev),
                               c["order"], data=torch.tensor(c["data"], dtype=torch.float64,
                                                             device=dev),
                               precision=a.precision)
    torch.cuda.synchronize()
    hs = hashlib.sha256(sp.cpu().numpy().tobytes()).hexdigest()[:16]
    hx = hashlib.sha256(x2.cpu().numpy().tobytes()).hexdigest()[:16]
    print("%s %s %s points=%d spectra=%s chi2=%s" % (a.lib or "default", a.workload, a.precision,
                                                  sp.shape[0], hs, hx))


if __name__ == "__main__":
    main()

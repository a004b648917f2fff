"""The paper's own GPU design, re-expressed with stock torch fp64 kernels on the B200, for
comparison with the fused kernel: "a set of transformations for each formula item"
 — one elementwise kernel per item (phase, sin, square, weight, sum), every
intermediate round-tripping through HBM.  cfg3: 1e8 energies, canonical point.  Not a product
path (torch.sin, libdevice accuracy); a measurement of what fusion buys."""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07682_b200 as gna  # noqa: E402
import synth  # noqa: E402


def per_item(E, p, L):
    w21 = math.cos(p["theta13"]) ** 4 * math.sin(2 * p["theta12"]) ** 2
    w31 = math.sin(2 * p["theta13"]) ** 2 * math.cos(p["theta12"]) ** 2
    w32 = math.sin(2 * p["theta13"]) ** 2 * math.sin(p["theta12"]) ** 2
    out = torch.ones_like(E)
    for dm2, w in ((p["dm2_21"], w21), (p["dm2_31"], w31), (p["dm2_31"] - p["dm2_21"], w32)):
        D = (1.26693268 * dm2 * L) / (E / 1000.0)   # phase item
        s = torch.sin(D)                            # sin item
        out -= w * (s * s)                          # square, weight, sum items
    return out


def timed(fn, reps=20):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    return float(np.median([x.elapsed_time(y) for x, y in ts]))


def main():
    c = synth.config("cfg3")
    E = torch.linspace(c["lo"], c["hi"], c["n"], dtype=torch.float64, device="cuda")
    out = torch.empty_like(E)
    p, L = c["params"], c["L_km"]
    for _ in range(3):
        per_item(E, p, L)
        gna.oscprob_eval(p, L, E, out=out)
    t_items = timed(lambda: per_item(E, p, L))
    t_fused = timed(lambda: gna.oscprob_eval(p, L, E, out=out))
    ref = per_item(E, p, L)
    diff = float((ref - out).abs().max())
    print("cfg3 1e8 energies: per-item torch kernels %.3f ms (%.1f G/s); fused gna kernel %.3f ms "
          "(%.1f G/s); speed-up %.1fx; max |diff| %.2e" % (
              t_items, c["n"] / t_items / 1e6, t_fused, c["n"] / t_fused / 1e6, t_items / t_fused,
              diff))


if __name__ == "__main__":
    main()

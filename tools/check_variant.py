"""Parity of a tuning-variant library (bench.py --lib) against the oracle, on the eval path
(ragged sizes around the TMA tile and the cfg3 size, sampled)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1804_07682_b200 as gna  # noqa: E402
import synth  # noqa: E402


def main(lib):
    gna.load(lib)
    g = synth.rng(5)
    worst = 0.0
    for n in (4096, 4097, 5000, 1 << 20, 1_000_003, 100_000_000):
        p = synth.random_params(g)
        E = torch.linspace(1.0, 10.0, n, dtype=torch.float64, device="cuda") if n == 100_000_000 \
            else torch.tensor(synth.random_energies(g, n), device="cuda")
        P = gna.oscprob_eval(p, 52.5, E)
        idx = np.r_[0:min(n, 64), g.integers(0, n, 5000), max(0, n - 64):n]
        it = torch.tensor(idx, device="cuda")
        Pr = oracle.prob_array(p, 52.5, E[it].cpu().numpy())
        d = float(np.max(np.abs(P[it].cpu().numpy() - Pr)))
        worst = max(worst, d)
        assert d <= 1e-12, (n, d)
    print("variant %s eval parity ok, worst %.3g" % (os.path.basename(lib), worst))


if __name__ == "__main__":
    main(sys.argv[1])

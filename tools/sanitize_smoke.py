"""Small invocation of every kernel/entry point, for compute-sanitizer (memcheck / racecheck /
synccheck) runs on the GPU box.  Sizes are ragged on purpose (partial TMA tiles, partial warps,
partial node groups)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07682_b200 as gna  # noqa: E402
import synth  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    g = synth.rng(9)
    p = synth.random_params(g)
    t = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)  # noqa
    for n in (1, 33, 4097, 3 * 1024 * 4 + 77):
        gna.oscprob_eval(p, 52.5, t(synth.random_energies(g, n)))
    for order in (1, 5, 10, 13, 32):
        gna.gl_integrate(p, 52.5, t(np.sort(g.uniform(1, 10, 70))), order)
    pts = synth.points_uniform(g, 9, dict(theta12=(0.5, 0.6), theta13=(0.1, 0.2)))
    edges = np.sort(g.uniform(1, 10, 45))
    data = synth.pseudo_data(g, edges, 2.0)
    for nbase, order in ((1, 10), (3, 7), (8, 4)):
        L = g.uniform(1, 300, nbase)
        om = np.ones(nbase)
        gna.oscprob_batch({k: t(v) for k, v in pts.items()}, L, om, t(edges), order, data=t(data))
        gna.oscprob_batch({k: t(v) for k, v in pts.items()}, L, om, t(edges), order, spectra=True)
    gna.oscprob_eval_host(p, 52.5, synth.random_energies(g, 10_001), chunk=4096)
    gna.oscprob_batch_host(pts, [52.5, 200.0], [1.0, 0.1], edges, 5, data=data, chunk_points=4)
    torch.cuda.synchronize()
    gna.release()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()

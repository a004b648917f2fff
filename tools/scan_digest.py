"""Digest (sha256 prefix) of gna_oscprob_scan's spectra and chi^2 on five seeded grids at GL10
with 1-8 baselines: run under different build or environment settings of stage A to check that
they give the same bits."""
import sys, hashlib
import numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch
import paper_1804_07682_b200 as gna
import synth
h = hashlib.sha256()
for seed, nmix, nmass, nbase in ((61, 9, 9, 8), (62, 5, 7, 3), (63, 3, 2, 2), (64, 4, 5, 6), (65, 9, 9, 1)):
    g = synth.rng(seed)
    grid = dict(theta12=g.uniform(0.5, 0.65, nmix), theta13=g.uniform(0.1, 0.2, nmix),
                dm2_21=g.uniform(6e-5, 9e-5, nmass), dm2_31=g.uniform(2.2e-3, 2.8e-3, nmass))
    grid = synth.invert_ordering(g, grid)
    L, om = g.uniform(1.0, 300.0, nbase), g.uniform(0.1, 2.0, nbase)
    edges = np.sort(g.uniform(1.0, 10.0, 1001))
    data = synth.pseudo_data(g, edges, om.sum())
    sp, x2 = gna.oscprob_scan({k: torch.tensor(v, device="cuda") for k, v in grid.items()}, L,
                              om, torch.tensor(edges, device="cuda"), 10,
                              data=torch.tensor(data, device="cuda"))
    h.update(sp.cpu().numpy().tobytes()); h.update(x2.cpu().numpy().tobytes())
print("DIGEST", h.hexdigest()[:16])

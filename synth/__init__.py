"""Seeded synthetic inputs for the five BASELINE.json configs.

Shared by the tests, bench.py and smoke(); holds NONE of the method's arithmetic
(no phases, no probabilities, no quadrature) — only the shapes, ranges and
distributions of the paper's workloads:

* energies in MeV over the reactor window 1-10 MeV (P:600 energy vector E_nu;
  SURVEY §8(d)); 10^4 elements is "the JUNO experiment's case", 10^6 the
  other Table-1 size;
* baselines: the JUNO-like 52.5 km of SPEC S:280 plus a near cluster and two far
  baselines (the multiple OscProb instances of P:596-603);
* parameter points uniform over physical ranges around the SPEC canonical point
  S:280, seed 1804;
* pseudo-data for chi^2: a positive spectrum proportional to bin width with
  seeded fluctuations (not computed from the method).
"""
from __future__ import annotations

import numpy as np

SEED = 1804

# SPEC S:280 canonical point.  theta23/delta do not enter P_ee (R2).
CANONICAL = dict(theta12=0.5838, theta13=0.1496, theta23=0.7854, delta_cp=0.0,
                 dm2_21=7.53e-5, dm2_31=2.52e-3, antineutrino=0)
L_JUNO = 52.5  # km

# Parity domain (R7): the 1e-12 absolute claim is made here.
PARITY_DOMAIN = dict(theta12=(0.5, 0.65), theta13=(0.1, 0.2), dm2_21=(6e-5, 9e-5),
                     dm2_31=(2.2e-3, 2.8e-3), L_km=(0.0, 300.0), E=(1.0, 10.0))

CFG5_BASELINES = np.array([52.1, 52.2, 52.4, 52.5, 52.6, 52.8, 215.0, 265.0])


def rng(seed: int = SEED) -> np.random.Generator:
    return np.random.default_rng(seed)


def uniform_edges(nbins: int, lo: float = 1.0, hi: float = 10.0) -> np.ndarray:
    return np.linspace(lo, hi, nbins + 1)


def random_params(g: np.random.Generator, domain=PARITY_DOMAIN, ordering_sign=True) -> dict:
    """One parameter point drawn uniformly from `domain` (theta23, delta arbitrary)."""
    p = dict(CANONICAL)
    for k in ("theta12", "theta13", "dm2_21", "dm2_31"):
        lo, hi = domain[k]
        p[k] = float(g.uniform(lo, hi))
    if ordering_sign and g.random() < 0.25:
        p["dm2_31"] = -p["dm2_31"]  # inverted ordering, S:328 signed dm2_31
    p["theta23"] = float(g.uniform(0.0, np.pi / 2))
    p["delta_cp"] = float(g.uniform(0.0, 2 * np.pi))
    p["antineutrino"] = int(g.random() < 0.5)
    return p


def random_energies(g: np.random.Generator, n: int, lo=1.0, hi=10.0) -> np.ndarray:
    return g.uniform(lo, hi, size=n)


def points_uniform(g: np.random.Generator, npoints: int, ranges: dict) -> dict:
    """SoA parameter points; keys theta12, theta13, dm2_21, dm2_31."""
    out = {}
    for k in ("theta12", "theta13", "dm2_21", "dm2_31"):
        if k in ranges:
            lo, hi = ranges[k]
            out[k] = g.uniform(lo, hi, size=npoints)
        else:
            out[k] = np.full(npoints, CANONICAL[k])
    return out


def invert_ordering(g: np.random.Generator, points: dict, frac: float = 0.25) -> dict:
    """Copy of `points` with dm2_31 sign-flipped on a random `frac` of them: inverted mass
    ordering (S:328 signed dm2_31), the DESIGN.md parity-draw recipe.  Works on point lists
    and on a scan grid's mass axis alike (only the dm2_31 array is touched)."""
    out = {k: np.array(v, dtype=np.float64, copy=True) for k, v in points.items()}
    flip = g.random(out["dm2_31"].size) < frac
    if out["dm2_31"].size >= 2 and not flip.any():
        flip[-1] = True  # every multi-point draw holds at least one inverted point
    out["dm2_31"][flip] = -out["dm2_31"][flip]
    return out


def pseudo_data(g: np.random.Generator, edges: np.ndarray, total_weight: float) -> np.ndarray:
    """Positive pseudo-data spectrum: bin width x total baseline weight x U(0.4, 0.9)."""
    width = np.diff(edges)
    return width * total_weight * g.uniform(0.4, 0.9, size=width.size)


def config(name: str) -> dict:
    """The five BASELINE.json configs as concrete seeded inputs (DESIGN.md Input recipe)."""
    g = rng()
    if name == "cfg1":
        return dict(name=name, params=dict(CANONICAL), L_km=L_JUNO,
                    E=np.linspace(1.0, 10.0, 1000), edges=uniform_edges(100), order=5)
    if name == "cfg2":
        return dict(name=name, params=dict(CANONICAL), L_km=L_JUNO,
                    edges=uniform_edges(100_000), order=10)
    if name == "cfg3":
        # E = linspace(1, 10, 1e8) is built on the device by bench.py (800 MB);
        # this records the recipe only.
        return dict(name=name, params=dict(CANONICAL), L_km=L_JUNO, n=100_000_000,
                    lo=1.0, hi=10.0)
    if name == "cfg4":
        pts = points_uniform(g, 10_000, dict(theta13=(0.10, 0.20), dm2_31=(2.3e-3, 2.7e-3)))
        edges = uniform_edges(1000)
        L = np.array([L_JUNO])
        omega = np.array([1.0])
        return dict(name=name, points=pts, L_km=L, omega=omega, edges=edges, order=10,
                    data=pseudo_data(g, edges, float(omega.sum())))
    if name == "cfg5":
        pts = points_uniform(g, 1000, dict(theta12=(0.55, 0.62), theta13=(0.13, 0.17),
                                           dm2_21=(7.0e-5, 8.0e-5), dm2_31=(2.4e-3, 2.6e-3)))
        edges = uniform_edges(10_000)
        L = CFG5_BASELINES.copy()
        omega = (L_JUNO / L) ** 2
        return dict(name=name, points=pts, L_km=L, omega=omega, edges=edges, order=10,
                    data=pseudo_data(g, edges, float(omega.sum())))
    if name == "cfg4grid":
        # the cfg4 scan as a structured 100 x 100 grid (SURVEY §8(d) "secondary"): mixing
        # points (theta13) x mass points (dm2_31); the separable path (NEXT-1) runs it
        n13, n31 = 100, 100
        grid = dict(theta12=np.full(n13, CANONICAL["theta12"]),
                    theta13=np.linspace(0.10, 0.20, n13),
                    dm2_21=np.full(n31, CANONICAL["dm2_21"]),
                    dm2_31=np.linspace(2.3e-3, 2.7e-3, n31))
        edges = uniform_edges(1000)
        L = np.array([L_JUNO])
        omega = np.array([1.0])
        return dict(name=name, grid=grid, L_km=L, omega=omega, edges=edges, order=10,
                    data=pseudo_data(g, edges, float(omega.sum())))
    raise KeyError(name)


def expand_grid(grid: dict) -> dict:
    """Point list of a separable grid in the scan's order: p = c * nmix + a."""
    nmix, nmass = grid["theta12"].size, grid["dm2_21"].size
    return dict(theta12=np.tile(grid["theta12"], nmass), theta13=np.tile(grid["theta13"], nmass),
                dm2_21=np.repeat(grid["dm2_21"], nmix), dm2_31=np.repeat(grid["dm2_31"], nmix))


def subset_points(points: dict, idx) -> dict:
    return {k: np.ascontiguousarray(v[idx]) for k, v in points.items()}

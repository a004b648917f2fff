"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Tolerances (BASELINE.json north_star; R7): 1e-12 absolute on
probabilities, 1e-11 relative on bin integrals and spectra; chi^2 within the
bound that the 1e-11 spectra tolerance propagates to.  Inputs are the seeded
synthetic workloads of synth/ (DESIGN.md "Input recipe").  Run on a B200 via
gpurun: python -m pytest tests -m gpu
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL_P = 1e-12
TOL_BIN = 1e-11
EPS = np.finfo(np.float64).eps
# sin^2 minimax error (degree 7, tests/test_abi_cpu.py) times sum_ij w_ij <= 2, plus 1e-15 of
# final rounding: the phase-independent part of the conditioning bound (R7)
POLY_P = 2 * 1.12e-15 + 1e-15


@pytest.fixture(scope="module")
def gna():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1804_07682_b200 import _build
    _build.build()
    import paper_1804_07682_b200 as g
    g.load()
    torch.cuda.set_device(0)
    return g


def _t(a):
    import torch
    return torch.tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def _np(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _nt():
    return oracle.max_threads()


def _chi2_bound(T, D):
    d = np.abs(T - D)
    return np.sum((2 * d * TOL_BIN * np.abs(T) + d * d * 8 * EPS) / D, axis=-1) + 1e-300


# ------------------------------------------------------------------------ (a3) eval
def test_eval_cfg1(gna):
    c = synth.config("cfg1")
    P = _np(gna.oscprob_eval(c["params"], c["L_km"], _t(c["E"])))
    Pr = oracle.prob_array(c["params"], c["L_km"], c["E"])
    assert np.max(np.abs(P - Pr)) <= TOL_P


@pytest.mark.parametrize("n", [1, 2, 3, 31, 257, 1000, 4097, 100_003])
def test_eval_random_params_ragged(gna, n):
    g = synth.rng(100 + n)
    for _ in range(6):
        p = synth.random_params(g)
        L = g.uniform(0, 300)
        E = synth.random_energies(g, n)
        P = _np(gna.oscprob_eval(p, L, _t(E)))
        Pr = oracle.prob_array(p, L, E, nthreads=_nt())
        assert np.max(np.abs(P - Pr)) <= TOL_P, (p, L)


def test_eval_misaligned_scalar_path(gna):
    import torch
    g = synth.rng(7)
    E = synth.random_energies(g, 1001)
    buf = _t(np.r_[0.0, E])
    Ein = buf[1:]                      # 8-byte aligned only -> scalar kernel
    out = torch.empty(1002, dtype=torch.float64, device="cuda")[1:]
    p = dict(synth.CANONICAL)
    P = _np(gna.oscprob_eval(p, 52.5, Ein, out=out))
    assert np.max(np.abs(P - oracle.prob_array(p, 52.5, E))) <= TOL_P


def test_eval_special_cases(gna):
    E = np.linspace(1, 10, 999)
    p0 = dict(synth.CANONICAL, theta12=0.0, theta13=0.0)
    assert np.all(_np(gna.oscprob_eval(p0, 52.5, _t(E))) == 1.0)       # zero mixing
    P = _np(gna.oscprob_eval(synth.CANONICAL, 0.0, _t(E)))             # L = 0
    assert np.max(np.abs(P - 1.0)) <= 2 * EPS
    # theta13 = 0: two-flavour limit via the oracle's two_flavor
    p1 = dict(synth.CANONICAL, theta13=0.0)
    P = _np(gna.oscprob_eval(p1, 52.5, _t(E)))
    ref = np.array([oracle.two_flavor(p1["theta12"], p1["dm2_21"], 52.5, e) for e in E])
    assert np.max(np.abs(P - ref)) <= TOL_P
    # theta23, delta, antineutrino do not change P_ee (R2): bitwise
    pa = dict(synth.CANONICAL, theta23=0.1, delta_cp=2.0, antineutrino=1)
    assert np.array_equal(_np(gna.oscprob_eval(pa, 52.5, _t(E))),
                          _np(gna.oscprob_eval(synth.CANONICAL, 52.5, _t(E))))


def test_eval_stress_domain_within_conditioning_bound(gna):
    # angles over [0, pi/2], L up to 300 km: agreement within the rounding bound
    # of the phases (R7): sum_ij w_ij |2 Delta_ij| * 8 eps
    g = synth.rng(9)
    for _ in range(10):
        p = synth.random_params(g, domain=dict(synth.PARITY_DOMAIN, theta12=(0, np.pi / 2),
                                               theta13=(0, np.pi / 2)))
        L = g.uniform(0, 300)
        E = synth.random_energies(g, 20_000)
        P = _np(gna.oscprob_eval(p, L, _t(E)))
        Pr = oracle.prob_array(p, L, E, nthreads=_nt())
        dm = np.array([p["dm2_21"], p["dm2_31"], p["dm2_31"] - p["dm2_21"]])
        ph = np.abs(1.26693268 * dm[:, None] * L / (E[None, :] / 1000.0))
        bound = POLY_P + np.sum(2 * ph * 8 * EPS, axis=0)  # w_ij <= 1, sum_ij w_ij <= 2
        assert np.all(np.abs(P - Pr) <= bound)


@pytest.mark.parametrize("L", [1_000.0, 12_000.0])
def test_eval_huge_phases_within_conditioning_bound(gna, L):
    """Phases far beyond the reactor domain (atmospheric-like L, E down to 0.1 MeV: |Delta| up
    to ~3e5 rad): the reduction stays exact (R10), so GPU and oracle differ only by the
    rounding of the phase itself, bounded by sum_ij |2 Delta_ij| * 8 eps."""
    g = synth.rng(int(L))
    for _ in range(4):
        p = synth.random_params(g)
        E = g.uniform(0.1, 10.0, 50_000)
        P = _np(gna.oscprob_eval(p, L, _t(E)))
        Pr = oracle.prob_array(p, L, E, nthreads=_nt())
        dm = np.array([p["dm2_21"], p["dm2_31"], p["dm2_31"] - p["dm2_21"]])
        ph = np.abs(1.26693268 * dm[:, None] * L / (E[None, :] / 1000.0))
        bound = POLY_P + np.sum(2 * ph * 8 * EPS, axis=0)
        assert np.all(np.abs(P - Pr) <= bound)
        assert np.max(np.abs(P - Pr)) > 0  # (the bound, not luck, is what is being tested)


def test_eval_cfg3_full_size_sampled(gna):
    """cfg3: 1e8 energies streamed from HBM, as bench.py launches it; sampled parity."""
    import torch
    c = synth.config("cfg3")
    E = torch.linspace(c["lo"], c["hi"], c["n"], dtype=torch.float64, device="cuda")
    P = gna.oscprob_eval(c["params"], c["L_km"], E)
    idx = np.r_[0:64, synth.rng(3).integers(0, c["n"], 10_000), c["n"] - 64:c["n"]]
    it = torch.tensor(idx, device="cuda")
    Es, Ps = _np(E[it]), _np(P[it])
    Pr = oracle.prob_array(c["params"], c["L_km"], Es)
    assert np.max(np.abs(Ps - Pr)) <= TOL_P
    assert float(P.min()) >= 0.0 and float(P.max()) <= 1.0 + TOL_P
    del E, P
    torch.cuda.empty_cache()


# ------------------------------------------------------------------------ NEXT-2 any channel
@pytest.mark.parametrize("n", [5, 4097, 100_003])
def test_eval_ab_all_channels_vs_oracle(gna, n):
    g = synth.rng(600 + n)
    for _ in range(3):
        p = synth.random_params(g)  # random theta23, delta, nu/nubar: they matter here
        L = g.uniform(0, 300)
        E = synth.random_energies(g, n)
        Et = _t(E)
        rows = []
        for a in range(3):
            row = []
            for b in range(3):
                P = _np(gna.oscprob_eval_ab(a, b, p, L, Et))
                Pr = oracle.prob_array(p, L, E, alpha=a, beta=b, nthreads=_nt())
                assert np.max(np.abs(P - Pr)) <= TOL_P, (a, b, p, L)
                row.append(P)
            rows.append(row)
        M = np.array(rows)  # [alpha][beta][n]
        assert np.max(np.abs(M.sum(axis=1) - 1)) <= 4 * TOL_P  # unitarity
        assert np.max(np.abs(M.sum(axis=0) - 1)) <= 4 * TOL_P
        # the e->e channel of the general path agrees with the P_ee hot path
        Pee = _np(gna.oscprob_eval(p, L, Et))
        assert np.max(np.abs(M[0, 0] - Pee)) <= 1e-14


@pytest.mark.parametrize("nbins,order", [(1, 1), (37, 5), (1000, 10), (100_003, 10), (50, 32)])
def test_gl_integrate_ab_all_channels_vs_oracle(gna, nbins, order):
    g = synth.rng(700 + nbins + order)
    p = synth.random_params(g)
    L = g.uniform(1, 300)
    edges = np.sort(g.uniform(1.0, 10.0, nbins + 1))
    de = _t(edges)
    tot = [np.zeros(nbins) for _ in range(3)]
    for a in range(3):
        for b in range(3):
            S = _np(gna.gl_integrate_ab(a, b, p, L, de, order))
            Sr = oracle.gl_integrate_ab(a, b, p, L, edges, order, nthreads=_nt())
            # appearance bins can be ~0: absolute tolerance relative to the bin width
            assert np.max(np.abs(S - Sr) / np.diff(edges)) <= TOL_BIN, (a, b)
            tot[a] += S
    for a in range(3):
        assert np.max(np.abs(tot[a] / np.diff(edges) - 1)) <= 1e-12


def test_eval_ab_cpt_and_L0(gna):
    g = synth.rng(61)
    p = synth.random_params(g)
    p["antineutrino"] = 0
    E = synth.random_energies(g, 5000)
    Et = _t(E)
    pm = dict(p, delta_cp=-p["delta_cp"])
    for a in range(3):
        for b in range(3):
            # CPT: P_ab(delta) = P_ba(-delta)
            assert np.max(np.abs(_np(gna.oscprob_eval_ab(a, b, p, 80.0, Et))
                                 - _np(gna.oscprob_eval_ab(b, a, pm, 80.0, Et)))) <= 2 * TOL_P
            # L = 0 -> delta_ab
            P0 = _np(gna.oscprob_eval_ab(a, b, p, 0.0, Et))
            assert np.max(np.abs(P0 - (1.0 if a == b else 0.0))) <= 4 * EPS


# ------------------------------------------------------------------------ 64-bit indexing
def test_eval_beyond_int32_elements(gna):
    """n = 2^31 + 123 energies (17 GB in, 17 GB out on the 180 GB B200): 64-bit tile and tail indexing."""
    import torch
    n = (1 << 31) + 123
    E = torch.linspace(1.0, 10.0, n, dtype=torch.float64, device="cuda")
    P = gna.oscprob_eval(synth.CANONICAL, 52.5, E)
    idx = np.r_[0:8, (1 << 31) - 4:(1 << 31) + 4, n - 130:n, synth.rng(8).integers(0, n, 2000)]
    it = torch.tensor(idx, device="cuda")
    Es, Ps = _np(E[it]), _np(P[it])
    assert np.max(np.abs(Ps - oracle.prob_array(synth.CANONICAL, 52.5, Es))) <= TOL_P
    del E, P, it
    torch.cuda.empty_cache()


def test_batch_spectra_beyond_int32_elements(gna):
    """P x nbins = 2.2e9 > 2^31 spectra elements (17.6 GB): 64-bit output indexing."""
    import torch
    P, nbins = 220_000, 10_000
    g = synth.rng(31)
    pts = synth.points_uniform(g, P, dict(theta13=(0.1, 0.2), dm2_31=(2.3e-3, 2.7e-3)))
    edges = synth.uniform_edges(nbins)
    data = synth.pseudo_data(g, edges, 1.0)
    sp, x2 = gna.oscprob_batch({k: _t(v) for k, v in pts.items()}, [52.5], [1.0], _t(edges), 1,
                               data=_t(data))
    rows = np.array([0, 1, 214_748, 214_749, P - 1])  # rows around p * nbins = 2^31
    sps = _np(sp[torch.tensor(rows, device="cuda")])
    x2s = _np(x2)[rows]
    spr, x2r = oracle.batch(synth.subset_points(pts, rows), [52.5], [1.0], edges, 1, data=data,
                            nthreads=_nt())
    assert np.max(np.abs(sps - spr) / np.abs(spr)) <= TOL_BIN
    assert np.all(np.abs(x2s - x2r) <= _chi2_bound(spr, data))
    del sp, x2
    torch.cuda.empty_cache()


# ------------------------------------------------------------------------ (a4) GL
def test_gl_cfg1(gna):
    c = synth.config("cfg1")
    S = _np(gna.gl_integrate(c["params"], c["L_km"], _t(c["edges"]), c["order"]))
    Sr = oracle.gl_integrate(c["params"], c["L_km"], c["edges"], c["order"])
    assert np.max(np.abs(S - Sr) / np.abs(Sr)) <= TOL_BIN


def test_gl_cfg2_full(gna):
    c = synth.config("cfg2")
    S = _np(gna.gl_integrate(c["params"], c["L_km"], _t(c["edges"]), c["order"]))
    Sr = oracle.gl_integrate(c["params"], c["L_km"], c["edges"], c["order"], nthreads=_nt())
    assert np.max(np.abs(S - Sr) / np.abs(Sr)) <= TOL_BIN


@pytest.mark.parametrize("order", list(range(1, 33)))
def test_gl_all_orders(gna, order):
    g = synth.rng(200 + order)
    p = synth.random_params(g)
    L = g.uniform(1, 300)
    edges = np.sort(g.uniform(1.0, 10.0, 38))
    S = _np(gna.gl_integrate(p, L, _t(edges), order))
    Sr = oracle.gl_integrate(p, L, edges, order)
    assert np.max(np.abs(S - Sr) / np.abs(Sr)) <= TOL_BIN


@pytest.mark.parametrize("nbins", [1, 63, 64, 65, 1000, 100_003])
def test_gl_ragged_sizes(gna, nbins):
    g = synth.rng(300 + nbins)
    p = synth.random_params(g)
    edges = synth.uniform_edges(nbins, 1.0, 10.0)
    S = _np(gna.gl_integrate(p, 52.5, _t(edges), 7))
    Sr = oracle.gl_integrate(p, 52.5, edges, 7, nthreads=_nt())
    assert np.max(np.abs(S - Sr) / np.abs(Sr)) <= TOL_BIN


@pytest.mark.parametrize("order", [1, 2, 3, 4, 5, 7, 10, 11, 13, 16, 29, 32])
def test_gl_thread_per_bin_path_all_group_shapes(gna, order):
    # fp64 P_ee runs the thread-per-bin kernel at every nbins (gl_tb_min_bins); node groups of
    # 5/4/3 and the ragged last group (orders 7, 11, 13, 29)
    g = synth.rng(1300 + order)
    p = synth.random_params(g)
    L = g.uniform(1, 300)
    nbins = 40_001
    edges = np.sort(g.uniform(1.0, 10.0, nbins + 1))
    S = _np(gna.gl_integrate(p, L, _t(edges), order))
    Sr = oracle.gl_integrate(p, L, edges, order, nthreads=_nt())
    assert np.max(np.abs(S - Sr) / np.abs(Sr)) <= TOL_BIN


@pytest.mark.parametrize("order", [1, 7, 10, 13, 29, 32])
@pytest.mark.parametrize("mode", ["fp64", "mixed", "ab"])
def test_gl_bin_value_independent_of_nbins_across_kernels(gna, mode, order):
    """The small-grid kernels (fp64 P_ee: node halves in two warps; mixed tier and general
    channel: lane pairs) and the thread-per-bin kernel (large nbins) form a bin's value
    identically: 300 000 bins in one call equal the same edges in 1 000-bin calls, bit for
    bit, at odd and ragged orders (halves of unequal length, ragged node groups)."""
    g = synth.rng(1900 + order)
    p = synth.random_params(g)
    edges = np.sort(g.uniform(1.0, 10.0, 300_001))
    de = _t(edges)

    def run(e):
        if mode == "ab":
            return _np(gna.gl_integrate_ab(0, 1, p, 60.0, e, order))
        return _np(gna.gl_integrate(p, 60.0, e, order, precision=mode))
    full = run(de)
    parts = np.concatenate([run(de[k:k + 1001]) for k in range(0, 300_000, 1000)])
    assert np.array_equal(full, parts)
    if mode == "fp64":  # and both equal the oracle within the tier tolerance
        Sr = oracle.gl_integrate(p, 60.0, edges[:2001], order, nthreads=_nt())
        assert np.max(np.abs(full[:2000] - Sr) / np.abs(Sr)) <= TOL_BIN


def test_gl_zero_mixing_is_bin_width(gna):
    e = synth.uniform_edges(333, 1.0, 10.0)
    p0 = dict(synth.CANONICAL, theta12=0.0, theta13=0.0)
    S = _np(gna.gl_integrate(p0, 52.5, _t(e), 10))
    assert np.max(np.abs(S / np.diff(e) - 1)) <= 4 * EPS


# ------------------------------------------------------------------------ (a5) batch
def _batch_case(g, P, nbase, nbins, order):
    pts = synth.points_uniform(g, P, dict(theta12=(0.5, 0.65), theta13=(0.1, 0.2),
                                          dm2_21=(6e-5, 9e-5), dm2_31=(2.2e-3, 2.8e-3)))
    pts = synth.invert_ordering(g, pts)  # 25 % inverted ordering
    L = g.uniform(1.0, 300.0, nbase)
    om = g.uniform(0.1, 2.0, nbase)
    edges = np.sort(g.uniform(1.0, 10.0, nbins + 1))
    data = synth.pseudo_data(g, edges, om.sum())
    return pts, L, om, edges, data


def _run_batch(gna, pts, L, om, edges, order, data, spectra=True, precision="fp64"):
    sp, x2 = gna.oscprob_batch({k: _t(v) for k, v in pts.items()}, L, om, _t(edges), order,
                               data=_t(data) if data is not None else None, spectra=spectra,
                               precision=precision)
    return (_np(sp) if sp is not None else None), (_np(x2) if x2 is not None else None)


@pytest.mark.parametrize("P,nbase,nbins,order", [
    (7, 3, 37, 4), (1, 1, 1, 1), (3, 2, 128, 10), (5, 8, 129, 10), (2, 64, 50, 32),
    (33, 1, 300, 5)])
def test_batch_small_vs_oracle(gna, P, nbase, nbins, order):
    g = synth.rng(400 + P * nbase + nbins)
    pts, L, om, edges, data = _batch_case(g, P, nbase, nbins, order)
    sp, x2 = _run_batch(gna, pts, L, om, edges, order, data)
    spr, x2r = oracle.batch(pts, L, om, edges, order, data=data, nthreads=_nt())
    assert np.max(np.abs(sp - spr) / np.abs(spr)) <= TOL_BIN
    assert np.all(np.abs(x2 - x2r) <= _chi2_bound(spr, data))
    # chi2-only and spectra-only runs give the same bits
    sp2, _ = _run_batch(gna, pts, L, om, edges, order, None)
    _, x22 = _run_batch(gna, pts, L, om, edges, order, data, spectra=False)
    assert np.array_equal(sp, sp2) and np.array_equal(x2, x22)


@pytest.mark.parametrize("order", [10, 7])
def test_batch_points_inner_path_vs_oracle(gna, order):
    """Single baseline, many points: the launcher packs several points per warp and runs
    the node-outer/points-inner kernel; all points compared with the oracle."""
    g = synth.rng(90 + order)
    pts, L, om, edges, data = _batch_case(g, 2003, 1, 1000, order)
    sp, x2 = _run_batch(gna, pts, L, om, edges, order, data)
    spr, x2r = oracle.batch(pts, L, om, edges, order, data=data, nthreads=_nt())
    assert np.max(np.abs(sp - spr) / np.abs(spr)) <= TOL_BIN
    assert np.all(np.abs(x2 - x2r) <= _chi2_bound(spr, data))


# ------------------------------------------------------------------------ NEXT-3 mixed tier
# fp64 phases/reduction, fp32 polynomial and per-node term sums (GNA_PREC_MIXED).  Tier
# tolerance: 1e-5 relative on spectra; chi^2 within the bound it propagates.
TOL_MIXED = 1e-5


def _chi2_bound_tol(T, D, tol):
    d = np.abs(T - D)
    return np.sum((2 * d * tol * np.abs(T) + (tol * T) ** 2) / D, axis=-1) + 1e-300


@pytest.mark.parametrize("P,nbase,nbins,order", [
    (7, 3, 37, 4), (1, 1, 1, 1), (3, 2, 128, 10), (5, 8, 129, 10), (2, 64, 50, 32),
    (33, 1, 300, 5), (40, 1, 1000, 10)])
def test_batch_mixed_vs_oracle(gna, P, nbase, nbins, order):
    g = synth.rng(900 + P * nbase + nbins)
    pts, L, om, edges, data = _batch_case(g, P, nbase, nbins, order)
    sp, x2 = _run_batch(gna, pts, L, om, edges, order, data, precision="mixed")
    spr, x2r = oracle.batch(pts, L, om, edges, order, data=data, nthreads=_nt())
    err = np.max(np.abs(sp - spr) / np.abs(spr))
    assert err <= TOL_MIXED
    assert np.all(np.abs(x2 - x2r) <= _chi2_bound_tol(spr, data, TOL_MIXED))
    # it really is the fp32 path (the fp64 path is ~1e-15 from the oracle)
    sp64, _ = _run_batch(gna, pts, L, om, edges, order, data)
    assert np.max(np.abs(sp64 - spr) / np.abs(spr)) <= TOL_BIN
    if nbins * order >= 10:
        assert np.max(np.abs(sp - sp64)) > 0
    # chi2-only and spectra-only runs give the same bits
    sp2, _ = _run_batch(gna, pts, L, om, edges, order, None, precision="mixed")
    _, x22 = _run_batch(gna, pts, L, om, edges, order, data, spectra=False, precision="mixed")
    assert np.array_equal(sp, sp2) and np.array_equal(x2, x22)


TOL_P_MIXED = 1e-6


@pytest.mark.parametrize("n", [1, 2, 3, 1001, 100_003])
def test_eval_mixed_vs_oracle(gna, n):
    """NEXT-3 tier of the elementwise path (gna_oscprob_eval_ex, GNA_PREC_MIXED): 1e-6 absolute,
    over the parity domain and the stress domain (angles up to pi/2, sum w <= 2)."""
    g = synth.rng(950 + n)
    for dom in (synth.PARITY_DOMAIN, dict(synth.PARITY_DOMAIN, theta12=(0, np.pi / 2),
                                          theta13=(0, np.pi / 2))):
        p = synth.random_params(g, domain=dom)
        L = g.uniform(0, 300)
        E = synth.random_energies(g, n)
        P = _np(gna.oscprob_eval(p, L, _t(E), precision="mixed"))
        Pr = oracle.prob_array(p, L, E, nthreads=_nt())
        assert np.max(np.abs(P - Pr)) <= TOL_P_MIXED, (p, L)


def test_eval_mixed_cfg3_full_size_sampled(gna):
    """cfg3 through the TMA-fed stream in the mixed tier (FFMA2 pairs of energies)."""
    import torch
    c = synth.config("cfg3")
    E = torch.linspace(c["lo"], c["hi"], c["n"], dtype=torch.float64, device="cuda")
    P = gna.oscprob_eval(c["params"], c["L_km"], E, precision="mixed")
    idx = np.r_[0:64, synth.rng(3).integers(0, c["n"], 10_000), c["n"] - 64:c["n"]]
    it = torch.tensor(idx, device="cuda")
    Es, Ps = _np(E[it]), _np(P[it])
    assert np.max(np.abs(Ps - oracle.prob_array(c["params"], c["L_km"], Es))) <= TOL_P_MIXED
    del E, P
    torch.cuda.empty_cache()


@pytest.mark.parametrize("nbins,order", [(1, 1), (37, 5), (1000, 10), (100_003, 10), (50, 32),
                                         (64, 7)])
def test_gl_integrate_mixed_vs_oracle(gna, nbins, order):
    g = synth.rng(970 + nbins + order)
    p = synth.random_params(g)
    L = g.uniform(0, 300)
    edges = np.sort(g.uniform(1.0, 10.0, nbins + 1))
    S = _np(gna.gl_integrate(p, L, _t(edges), order, precision="mixed"))
    Sr = oracle.gl_integrate(p, L, edges, order, nthreads=_nt())
    assert np.max(np.abs(S - Sr) / np.abs(Sr)) <= TOL_MIXED


@pytest.mark.parametrize("cfg,idx", [("cfg5", [0, 417, 999]), ("cfg4", [0, 1, 5000, 9999])])
def test_batch_mixed_full_size_sampled_and_split_invariant(gna, cfg, idx):
    """The mixed tier at the bench launch configuration (cfg5: per-point kernel; cfg4:
    points-inner kernel): sampled parity at the tier tolerance, and a point's result does not
    depend on the other points of the call (bitwise), as for the fp64 path."""
    c = synth.config(cfg)
    sp, x2 = _run_batch(gna, c["points"], c["L_km"], c["omega"], c["edges"], c["order"],
                        c["data"], precision="mixed")
    idx = np.array(idx)
    sub = synth.subset_points(c["points"], idx)
    spr, x2r = oracle.batch(sub, c["L_km"], c["omega"], c["edges"], c["order"], data=c["data"],
                            nthreads=_nt())
    assert np.max(np.abs(sp[idx] - spr) / np.abs(spr)) <= TOL_MIXED
    assert np.all(np.abs(x2[idx] - x2r) <= _chi2_bound_tol(spr, c["data"], TOL_MIXED))
    n = sp.shape[0]
    for lo, hi in ((0, n // 7), (n // 7, n)):
        s2 = synth.subset_points(c["points"], np.arange(lo, hi))
        sps, x2s = _run_batch(gna, s2, c["L_km"], c["omega"], c["edges"], c["order"], c["data"],
                              precision="mixed")
        assert np.array_equal(sps, sp[lo:hi]) and np.array_equal(x2s, x2[lo:hi])


@pytest.mark.parametrize("nbase,nbins,order", [(1, 1000, 10), (1, 257, 7), (2, 300, 5),
                                               (1, 33, 32), (2, 1, 1)])
def test_batch_points_across_lanes_path_vs_oracle_and_bitwise(gna, nbase, nbins, order):
    """>= 256 points and <= 2 baselines: the points-across-lanes kernel.  Sampled parity with
    the oracle, and bitwise equality with the other batch kernels (a 100-point call runs the
    points-inner or per-point kernel), incl. chi2 (same xor-tree order)."""
    g = synth.rng(1500 + nbase * nbins + order)
    pts, L, om, edges, data = _batch_case(g, 611, nbase, nbins, order)
    sp, x2 = _run_batch(gna, pts, L, om, edges, order, data)
    idx = np.array([0, 31, 32, 300, 607, 610])
    spr, x2r = oracle.batch(synth.subset_points(pts, idx), L, om, edges, order, data=data,
                            nthreads=_nt())
    assert np.max(np.abs(sp[idx] - spr) / np.abs(spr)) <= TOL_BIN
    assert np.all(np.abs(x2[idx] - x2r) <= _chi2_bound(spr, data))
    for lo, hi in ((0, 100), (100, 611), (1, 2)):
        s2 = synth.subset_points(pts, np.arange(lo, hi))
        sps, x2s = _run_batch(gna, s2, L, om, edges, order, data)
        assert np.array_equal(sps, sp[lo:hi]) and np.array_equal(x2s, x2[lo:hi]), (lo, hi)
    # chi2-only / spectra-only give the same bits
    sp2, _ = _run_batch(gna, pts, L, om, edges, order, None)
    _, x22 = _run_batch(gna, pts, L, om, edges, order, data, spectra=False)
    assert np.array_equal(sp, sp2) and np.array_equal(x2, x22)


@pytest.mark.parametrize("precision", ["fp64", "mixed"])
@pytest.mark.parametrize("nbase,nbins,order,odd_every", [(1, 1000, 10, 0), (2, 300, 5, 0),
                                                         (1, 257, 7, 41), (2, 33, 32, 97),
                                                         (1, 1, 1, 0)])
def test_batch_points_across_lanes_shared_dm2_21_bitwise_and_vs_oracle(gna, nbase, nbins, order,
                                                                        odd_every, precision):
    """A scan over (theta13, dm2_31) with the solar parameters fixed (cfg4's structure): the
    points-across-lanes kernel evaluates sin^2 Delta_21 once per warp instead of once per
    point.  Every point must keep its bits (equal to the per-point / points-inner kernels of
    100-point calls) and match the oracle; with odd_every > 0 some points carry another dm2_21,
    so their warps take the general path and the rest the shared one within one call."""
    g = synth.rng(2600 + nbins + order + odd_every)
    P = 611
    pts = synth.points_uniform(g, P, dict(theta13=(0.1, 0.2), dm2_31=(2.3e-3, 2.7e-3)))
    pts = synth.invert_ordering(g, pts)
    if odd_every:
        pts["dm2_21"] = pts["dm2_21"].copy()
        pts["dm2_21"][::odd_every] = 7.9e-5
    L = g.uniform(1.0, 300.0, nbase)
    om = g.uniform(0.1, 2.0, nbase)
    edges = np.sort(g.uniform(1.0, 10.0, nbins + 1))
    data = synth.pseudo_data(g, edges, om.sum())
    sp, x2 = _run_batch(gna, pts, L, om, edges, order, data, precision=precision)
    idx = np.array([0, 31, 32, 41, 300, 610])
    spr, x2r = oracle.batch(synth.subset_points(pts, idx), L, om, edges, order, data=data,
                            nthreads=_nt())
    tol = TOL_BIN if precision == "fp64" else TOL_MIXED
    assert np.max(np.abs(sp[idx] - spr) / np.abs(spr)) <= tol
    bound = (_chi2_bound(spr, data) if precision == "fp64" else
             _chi2_bound_tol(spr, data, TOL_MIXED))
    assert np.all(np.abs(x2[idx] - x2r) <= bound)
    for lo, hi in ((0, 100), (100, 200), (500, 611)):
        s2 = synth.subset_points(pts, np.arange(lo, hi))
        sps, x2s = _run_batch(gna, s2, L, om, edges, order, data, precision=precision)
        assert np.array_equal(sps, sp[lo:hi]) and np.array_equal(x2s, x2[lo:hi]), (lo, hi)


@pytest.mark.parametrize("nbase,nbins,order", [(1, 257, 7), (2, 300, 5), (1, 100, 10),
                                               (2, 33, 32), (1, 1, 1)])
def test_batch_mixed_points_across_lanes_vs_oracle_and_bitwise(gna, nbase, nbins, order):
    """Mixed tier with >= 256 points and <= 2 baselines: the points-across-lanes kernel with
    packed node pairs (odd groups end in a scalar chain).  Sampled parity at the tier
    tolerance, and bitwise equality with the points-inner mixed kernel (100-point calls)."""
    g = synth.rng(1700 + nbase * nbins + order)
    pts, L, om, edges, data = _batch_case(g, 411, nbase, nbins, order)
    sp, x2 = _run_batch(gna, pts, L, om, edges, order, data, precision="mixed")
    idx = np.array([0, 33, 205, 410])
    spr, x2r = oracle.batch(synth.subset_points(pts, idx), L, om, edges, order, data=data,
                            nthreads=_nt())
    assert np.max(np.abs(sp[idx] - spr) / np.abs(spr)) <= TOL_MIXED
    assert np.all(np.abs(x2[idx] - x2r) <= _chi2_bound_tol(spr, data, TOL_MIXED))
    for lo, hi in ((0, 100), (100, 411)):
        s2 = synth.subset_points(pts, np.arange(lo, hi))
        sps, x2s = _run_batch(gna, s2, L, om, edges, order, data, precision="mixed")
        assert np.array_equal(sps, sp[lo:hi]) and np.array_equal(x2s, x2[lo:hi]), (lo, hi)


@pytest.mark.parametrize("P,nbase,nbins,order,precision", [
    (300, 8, 1000, 10, "fp64"), (611, 1, 257, 7, "fp64"), (2003, 1, 300, 5, "fp64"),
    (300, 8, 1000, 10, "mixed"), (611, 2, 100, 10, "mixed")])
def test_batch_tables_valid_chunks_bitwise(gna, P, nbase, nbins, order, precision):
    """GNA_WS_TABLES_VALID: a batch split into chunks, only the first building the node
    tables in a shared workspace (sized for the largest chunk), gives the bits of one call
    over all points — every kernel family (per-point, points-across-lanes, points-inner)."""
    import torch
    g = synth.rng(2100 + P + nbins)
    pts, L, om, edges, data = _batch_case(g, P, nbase, nbins, order)
    full_sp, full_x2 = _run_batch(gna, pts, L, om, edges, order, data, precision=precision)
    de, dd = _t(edges), _t(data)
    dp = {k: _t(v) for k, v in pts.items()}
    sp = torch.empty((P, nbins), dtype=torch.float64, device="cuda")
    x2 = torch.empty(P, dtype=torch.float64, device="cuda")
    bounds = [0, P // 3, P // 3 + 1, P - 7, P]
    biggest = max(b - a for a, b in zip(bounds, bounds[1:]))
    ws = torch.empty(gna.oscprob_batch_workspace_size(biggest, nbase, nbins, order) // 8 + 2,
                     dtype=torch.float64, device="cuda")
    for c, (a, b) in enumerate(zip(bounds, bounds[1:])):
        sub = {k: v[a:b] for k, v in dp.items()}
        gna.oscprob_batch(sub, L, om, de, order, data=dd, spectra=sp[a:b], chi2=x2[a:b],
                          workspace=ws, precision=precision, tables_valid=c > 0)
    assert np.array_equal(_np(sp), full_sp) and np.array_equal(_np(x2), full_x2)


def test_batch_single_baseline_matches_gl_integrate(gna):
    g = synth.rng(41)
    pts, _, _, edges, _ = _batch_case(g, 4, 1, 200, 10)
    sp, _ = _run_batch(gna, pts, [52.5], [1.0], edges, 10, None)
    for p in range(4):
        pp = dict(synth.CANONICAL, **{k: float(v[p]) for k, v in pts.items()})
        S = _np(gna.gl_integrate(pp, 52.5, _t(edges), 10))
        assert np.max(np.abs(sp[p] - S) / S) <= 1e-14


def _check_sampled(sp, x2, c, idx):
    sub = synth.subset_points(c["points"], idx)
    spr, x2r = oracle.batch(sub, c["L_km"], c["omega"], c["edges"], c["order"], data=c["data"],
                            nthreads=_nt())
    assert np.max(np.abs(sp[idx] - spr) / np.abs(spr)) <= TOL_BIN
    assert np.all(np.abs(x2[idx] - x2r) <= _chi2_bound(spr, c["data"]))


def test_batch_cfg4_full_size_sampled(gna):
    c = synth.config("cfg4")
    sp, x2 = _run_batch(gna, c["points"], c["L_km"], c["omega"], c["edges"], c["order"],
                        c["data"])
    assert sp.shape == (10_000, 1000) and np.all(np.isfinite(sp)) and np.all(x2 >= 0)
    _check_sampled(sp, x2, c, np.r_[0, 1, synth.rng(4).integers(0, 10_000, 6), 9999])


def test_batch_cfg5_full_size_sampled_and_split_invariant(gna):
    c = synth.config("cfg5")
    sp, x2 = _run_batch(gna, c["points"], c["L_km"], c["omega"], c["edges"], c["order"],
                        c["data"])
    assert sp.shape == (1000, 10_000) and np.all(np.isfinite(sp)) and np.all(x2 >= 0)
    _check_sampled(sp, x2, c, np.array([0, 417, 999]))
    # deterministic, and a point's result does not depend on the other points
    # in the call (the multi-GPU shard property)
    sp_b, x2_b = _run_batch(gna, c["points"], c["L_km"], c["omega"], c["edges"], c["order"],
                            c["data"])
    assert np.array_equal(sp, sp_b) and np.array_equal(x2, x2_b)
    for lo, hi in ((0, 125), (125, 563), (563, 1000)):
        sub = synth.subset_points(c["points"], np.arange(lo, hi))
        sps, x2s = _run_batch(gna, sub, c["L_km"], c["omega"], c["edges"], c["order"],
                              c["data"])
        assert np.array_equal(sps, sp[lo:hi]) and np.array_equal(x2s, x2[lo:hi])


@pytest.mark.parametrize("cfg,precision", [("cfg5", "fp64"), ("cfg4", "fp64"), ("cfg5", "mixed"),
                                           ("cfg4", "mixed")])
def test_batch_cfg_inverted_ordering_full_size_sampled(gna, cfg, precision):
    """cfg4 / cfg5 at full size with every dm2_31 sign-flipped (inverted ordering), in
    the bench launch configuration (cfg5: per-point kernel; cfg4: points-across-lanes kernel),
    sampled against the oracle at the tier tolerance; a mixed set (every 4th point flipped)
    must give the same bits per point as the all-inverted and all-normal runs."""
    c = synth.config(cfg)
    inv = dict(c["points"], dm2_31=-c["points"]["dm2_31"])
    sp, x2 = _run_batch(gna, inv, c["L_km"], c["omega"], c["edges"], c["order"], c["data"],
                        precision=precision)
    n = sp.shape[0]
    idx = np.r_[0, 1, 31, 32, synth.rng(44).integers(0, n, 3), n - 1]
    spr, x2r = oracle.batch(synth.subset_points(inv, idx), c["L_km"], c["omega"], c["edges"],
                            c["order"], data=c["data"], nthreads=_nt())
    tol = TOL_BIN if precision == "fp64" else TOL_MIXED
    assert np.max(np.abs(sp[idx] - spr) / np.abs(spr)) <= tol
    bound = (_chi2_bound(spr, c["data"]) if precision == "fp64" else
             _chi2_bound_tol(spr, c["data"], TOL_MIXED))
    assert np.all(np.abs(x2[idx] - x2r) <= bound)
    # mixed ordering within one call: each point's bits equal its all-one-sign run
    flip = np.arange(n) % 4 == 1
    mix = dict(c["points"], dm2_31=np.where(flip, -c["points"]["dm2_31"], c["points"]["dm2_31"]))
    spm, x2m = _run_batch(gna, mix, c["L_km"], c["omega"], c["edges"], c["order"], c["data"],
                          precision=precision)
    assert np.array_equal(spm[flip], sp[flip]) and np.array_equal(x2m[flip], x2[flip])
    spn, x2n = _run_batch(gna, c["points"], c["L_km"], c["omega"], c["edges"], c["order"],
                          c["data"], precision=precision)
    assert np.array_equal(spm[~flip], spn[~flip]) and np.array_equal(x2m[~flip], x2n[~flip])


# ------------------------------------------------------------------------ NEXT-1 separable scan
def _scan_case(g, nmix, nmass, nbase, nbins, order):
    grid = dict(theta12=g.uniform(0.5, 0.65, nmix), theta13=g.uniform(0.1, 0.2, nmix),
                dm2_21=g.uniform(6e-5, 9e-5, nmass), dm2_31=g.uniform(2.2e-3, 2.8e-3, nmass))
    grid = synth.invert_ordering(g, grid)  # 25 % inverted mass points
    L = g.uniform(1.0, 300.0, nbase)
    om = g.uniform(0.1, 2.0, nbase)
    edges = np.sort(g.uniform(1.0, 10.0, nbins + 1))
    data = synth.pseudo_data(g, edges, om.sum())
    return grid, L, om, edges, data


@pytest.mark.parametrize("nmix,nmass,nbase,nbins,order", [
    (1, 1, 1, 1, 1), (7, 5, 3, 37, 4), (3, 4, 8, 300, 10), (2, 2, 64, 50, 32), (33, 1, 1, 257, 5),
    # GL10 (stage A compiled for the order) with 2..7 baselines and ragged grids
    (5, 3, 2, 51, 10), (4, 3, 3, 77, 10), (2, 7, 5, 129, 10), (6, 1, 7, 13, 10),
    # a small grid over more bins than one stage-B chunk: chi^2 from chunk partials (ragged)
    (3, 2, 2, 1100, 10)])
def test_scan_vs_oracle_on_expanded_grid(gna, nmix, nmass, nbase, nbins, order):
    g = synth.rng(500 + nmix * nmass + nbins)
    grid, L, om, edges, data = _scan_case(g, nmix, nmass, nbase, nbins, order)
    sp, x2 = gna.oscprob_scan({k: _t(v) for k, v in grid.items()}, L, om, _t(edges), order,
                              data=_t(data))
    sp, x2 = _np(sp).reshape(nmass * nmix, nbins), _np(x2).ravel()
    spr, x2r = oracle.batch(synth.expand_grid(grid), L, om, edges, order, data=data,
                            nthreads=_nt())
    assert np.max(np.abs(sp - spr) / np.abs(spr)) <= TOL_BIN
    assert np.all(np.abs(x2 - x2r) <= _chi2_bound(spr, data))
    # same quantity as the per-point batch path on the expanded points
    spb, x2b = _run_batch(gna, synth.expand_grid(grid), L, om, edges, order, data)
    assert np.max(np.abs(sp - spb) / np.abs(spb)) <= 1e-13


@pytest.mark.parametrize("sign", [1.0, -1.0])
def test_scan_cfg4grid_full_size_sampled(gna, sign):
    c = synth.config("cfg4grid")
    c["grid"]["dm2_31"] = sign * c["grid"]["dm2_31"]  # -1: inverted ordering
    sp, x2 = gna.oscprob_scan({k: _t(v) for k, v in c["grid"].items()}, c["L_km"], c["omega"],
                              _t(c["edges"]), c["order"], data=_t(c["data"]))
    sp, x2 = _np(sp).reshape(-1, c["edges"].size - 1), _np(x2).ravel()
    pts = synth.expand_grid(c["grid"])
    idx = np.array([0, 1, 99, 100, 5050, 9999])
    spr, x2r = oracle.batch(synth.subset_points(pts, idx), c["L_km"], c["omega"], c["edges"],
                            c["order"], data=c["data"], nthreads=_nt())
    assert np.max(np.abs(sp[idx] - spr) / np.abs(spr)) <= TOL_BIN
    assert np.all(np.abs(x2[idx] - x2r) <= _chi2_bound(spr, c["data"]))
    # chi2-only run gives the same bits
    _, x2o = gna.oscprob_scan({k: _t(v) for k, v in c["grid"].items()}, c["L_km"], c["omega"],
                              _t(c["edges"]), c["order"], data=_t(c["data"]), spectra=False)
    assert np.array_equal(_np(x2o).ravel(), x2)


# ------------------------------------------------------------------------ host-buffer path
def test_eval_host_bitwise_equals_device(gna):
    g = synth.rng(51)
    E = synth.random_energies(g, 1_000_003)
    p = synth.random_params(g)
    Ph = gna.oscprob_eval_host(p, 80.0, E, chunk=65_536)
    Pd = _np(gna.oscprob_eval(p, 80.0, _t(E)))
    assert np.array_equal(Ph, Pd)


def test_gl_integrate_host_bitwise_equals_device(gna):
    g = synth.rng(53)
    p = synth.random_params(g)
    edges = np.sort(g.uniform(1.0, 10.0, 100_001))
    for order in (5, 10, 17):
        bh = gna.gl_integrate_host(p, 60.0, edges, order, chunk=7_777)
        bd = _np(gna.gl_integrate(p, 60.0, _t(edges), order))
        assert np.array_equal(bh, bd)


@pytest.mark.parametrize("P,nbase", [(300, 3), (7, 8), (300, 1)])
def test_batch_host_pinned_spectra_bitwise_equals_device(gna, P, nbase):
    """Page-locked spectra: the per-point / points-inner kernels store the spectra straight
    into mapped host memory (GNA_HOST_DIRECT, one launch); the points-across-lanes case
    (300 x 1) stays staged.  Both give the device call's bits."""
    import torch
    g = synth.rng(55 + P + nbase)
    pts, L, om, edges, data = _batch_case(g, P, nbase, 257, 6)
    spec = torch.empty((P, 257), dtype=torch.float64).pin_memory()
    chi2 = torch.empty(P, dtype=torch.float64).pin_memory()
    spec.numpy().fill(np.nan)
    sph, x2h = gna.oscprob_batch_host(pts, L, om, edges, 6, data=data, spectra=spec.numpy(),
                                      chi2=chi2.numpy())
    spd, x2d = _run_batch(gna, pts, L, om, edges, 6, data)
    assert np.array_equal(sph, spd) and np.array_equal(x2h, x2d)


def test_batch_host_bitwise_equals_device(gna):
    g = synth.rng(52)
    pts, L, om, edges, data = _batch_case(g, 11, 3, 257, 6)
    sph, x2h = gna.oscprob_batch_host(pts, L, om, edges, 6, data=data, chunk_points=3)
    spd, x2d = _run_batch(gna, pts, L, om, edges, 6, data)
    assert np.array_equal(sph, spd) and np.array_equal(x2h, x2d)
    _, x2h2 = gna.oscprob_batch_host(pts, L, om, edges, 6, data=data, spectra=False)
    assert np.array_equal(x2h2, x2d)


_HOST_RING_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, %(root)r)
import torch
import paper_1804_07682_b200 as gna
import synth
g = synth.rng(54)
P, nb, order = 300, 257, 6
pts = synth.invert_ordering(g, synth.points_uniform(g, P, dict(
    theta12=(0.5, 0.65), theta13=(0.1, 0.2), dm2_21=(6e-5, 9e-5), dm2_31=(2.2e-3, 2.8e-3))))
L, om = np.array([52.5, 215.0, 1.0]), np.array([1.0, 0.1, 0.3])
edges = np.sort(g.uniform(1.0, 10.0, nb + 1))
data = synth.pseudo_data(g, edges, om.sum())
for cp in (40, 7, 300):  # tapered tails through a 3-slot ring; a single chunk
    sph, x2h = gna.oscprob_batch_host(pts, L, om, edges, order, data=data, chunk_points=cp)
    spd, x2d = gna.oscprob_batch({k: torch.tensor(v, device="cuda") for k, v in pts.items()}, L,
                                 om, torch.tensor(edges, device="cuda"), order,
                                 data=torch.tensor(data, device="cuda"))
    assert np.array_equal(sph, spd.cpu().numpy()) and np.array_equal(x2h, x2d.cpu().numpy()), cp
print("RING_OK")
"""


@pytest.mark.parametrize("spectra_max", ["1", "0"])
def test_batch_host_ring_and_tapered_chunks_bitwise(gna, spectra_max):
    """Host-buffer batch with tapered chunk plans, through the 3-slot spectra ring (forced by
    GNA_HOST_SPECTRA_MAX=1 byte, as for spectra larger than 2 GiB) and through the per-point
    staging regions (GNA_HOST_SPECTRA_MAX unset): bitwise equal to the device call.  Runs in a
    subprocess because the library reads the variable once."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    if spectra_max != "0":
        env["GNA_HOST_SPECTRA_MAX"] = spectra_max
    else:
        env.pop("GNA_HOST_SPECTRA_MAX", None)
    r = subprocess.run([sys.executable, "-c", _HOST_RING_SCRIPT % dict(root=root)],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0 and "RING_OK" in r.stdout, r.stderr[-3000:]


# ------------------------------------------------------------------------ streams and graphs
def test_batch_capturable_in_cuda_graph(gna):
    """The device entry points are stream-ordered and allocation-free: they can be captured
    in a CUDA graph and replayed (bench.py does this); replay == eager, bitwise."""
    import torch
    g = synth.rng(71)
    pts, L, om, edges, data = _batch_case(g, 9, 4, 300, 10)
    dp = {k: _t(v) for k, v in pts.items()}
    de, dd = _t(edges), _t(data)
    sp = torch.empty((9, 300), dtype=torch.float64, device="cuda")
    x2 = torch.empty(9, dtype=torch.float64, device="cuda")
    ws = torch.empty(gna.oscprob_batch_workspace_size(9, 4, 300, 10) // 8 + 2,
                     dtype=torch.float64, device="cuda")
    gna.oscprob_batch(dp, L, om, de, 10, data=dd, spectra=sp, chi2=x2, workspace=ws)
    ref_sp, ref_x2 = _np(sp).copy(), _np(x2).copy()
    sp.zero_()
    x2.zero_()
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            gna.oscprob_batch(dp, L, om, de, 10, data=dd, spectra=sp, chi2=x2, workspace=ws)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        graph.replay()
    assert np.array_equal(_np(sp), ref_sp) and np.array_equal(_np(x2), ref_x2)


def test_points_inner_batch_first_call_under_capture(gna):
    """The points-inner launch (one baseline) sizes its grid with the occupancy API on
    first use; in a fresh process the very first call happens inside graph capture, and
    the replay must equal a later eager call bitwise and match the oracle."""
    import subprocess
    import sys
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = r"""
import numpy as np, torch, sys
sys.path.insert(0, %r)
import paper_1804_07682_b200 as gna, synth
g = synth.rng(72)
P, nbins, order = 300, 1000, 10
pts = synth.points_uniform(g, P, dict(theta12=(0.5, 0.7), theta13=(0.1, 0.2),
                                      dm2_21=(6e-5, 9e-5), dm2_31=(2.2e-3, 2.8e-3)))
edges = np.sort(g.uniform(1.0, 10.0, nbins + 1))
data = synth.pseudo_data(g, edges, 1.0)
t = lambda a: torch.tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")
dp = {k: t(v) for k, v in pts.items()}
de, dd = t(edges), t(data)
sp = torch.empty((P, nbins), dtype=torch.float64, device="cuda")
x2 = torch.empty(P, dtype=torch.float64, device="cuda")
ws = torch.empty(gna.oscprob_batch_workspace_size(P, 1, nbins, order) // 8 + 2,
                 dtype=torch.float64, device="cuda")
graph = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    with torch.cuda.graph(graph, stream=s):
        gna.oscprob_batch(dp, [52.5], [1.0], de, order, data=dd, spectra=sp, chi2=x2,
                          workspace=ws)
torch.cuda.current_stream().wait_stream(s)
graph.replay()
torch.cuda.synchronize()
a, b = sp.cpu().numpy().copy(), x2.cpu().numpy().copy()
sp2, x22 = gna.oscprob_batch(dp, [52.5], [1.0], de, order, data=dd)
assert np.array_equal(a, sp2.cpu().numpy()) and np.array_equal(b, x22.cpu().numpy())
np.save(%r, a[[0, 151, 299]])
np.save(%r, b[[0, 151, 299]])
""" % (root, "/tmp/gna_cap_sp.npy", "/tmp/gna_cap_x2.npy")
    r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    g = synth.rng(72)
    pts = synth.points_uniform(g, 300, dict(theta12=(0.5, 0.7), theta13=(0.1, 0.2),
                                            dm2_21=(6e-5, 9e-5), dm2_31=(2.2e-3, 2.8e-3)))
    edges = np.sort(g.uniform(1.0, 10.0, 1001))
    data = synth.pseudo_data(g, edges, 1.0)
    idx = np.array([0, 151, 299])
    spr, x2r = oracle.batch(synth.subset_points(pts, idx), [52.5], [1.0], edges, 10, data=data,
                            nthreads=_nt())
    sp, x2 = np.load("/tmp/gna_cap_sp.npy"), np.load("/tmp/gna_cap_x2.npy")
    assert np.max(np.abs(sp - spr) / np.abs(spr)) <= TOL_BIN
    assert np.all(np.abs(x2 - x2r) <= _chi2_bound(spr, data))


def test_concurrent_calls_on_two_streams(gna):
    """Concurrent calls on disjoint outputs on two non-default streams."""
    import torch
    g = synth.rng(72)
    p1, p2 = synth.random_params(g), synth.random_params(g)
    E = _t(synth.random_energies(g, 300_000))
    edges = _t(np.sort(g.uniform(1, 10, 20_001)))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        a = gna.oscprob_eval(p1, 100.0, E)
        b = gna.gl_integrate(p1, 100.0, edges, 7)
    with torch.cuda.stream(s2):
        c = gna.oscprob_eval(p2, 30.0, E)
        d = gna.gl_integrate(p2, 30.0, edges, 9)
    torch.cuda.synchronize()
    assert np.array_equal(_np(a), _np(gna.oscprob_eval(p1, 100.0, E)))
    assert np.array_equal(_np(b), _np(gna.gl_integrate(p1, 100.0, edges, 7)))
    assert np.array_equal(_np(c), _np(gna.oscprob_eval(p2, 30.0, E)))
    assert np.array_equal(_np(d), _np(gna.gl_integrate(p2, 30.0, edges, 9)))


def test_repeated_calls_bitwise_deterministic(gna):
    g = synth.rng(73)
    p = synth.random_params(g)
    E = _t(synth.random_energies(g, 1_000_003))
    r0 = _np(gna.oscprob_eval(p, 52.5, E)).copy()
    for _ in range(3):
        assert np.array_equal(_np(gna.oscprob_eval(p, 52.5, E)), r0)


# ------------------------------------------------------------------------ NEXT-4 fused gather
@pytest.mark.parametrize("P,nbase", [(13, 3), (300, 1)])
def test_fused_gather_epilogue_single_rank(gna, P, nbase):
    """gna_oscprob_batch_ex writing through symmetric memory (1-rank group on this one
    GPU): peer-window stores and, where the fabric allows it, multicast stores give the
    same bits as the plain batch (per-point kernel; points-across-lanes kernel at 300x1)."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_1804_07682_b200 import dist as gdist
    g = synth.rng(81)
    pts, L, om, edges, data = _batch_case(g, P, nbase, 200, 10)
    dp = {k: _t(v) for k, v in pts.items()}
    de, dd = _t(edges), _t(data)
    ref_sp, ref_x2 = gna.oscprob_batch(dp, L, om, de, 10, data=dd)
    ref_sp, ref_x2 = _np(ref_sp).copy(), _np(ref_x2).copy()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%d" % port, rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        modes = [False, True]
        seen = []
        for prefer_mc in modes:
            fg = gdist.FusedGather(P, 200, "cuda", prefer_multicast=prefer_mc)
            if prefer_mc and not fg.multicast:
                continue
            fg.spectra.fill_(float("nan"))
            fg.chi2.fill_(float("nan"))
            sp_ptr, x2_ptr, flags = fg.out_ptrs()
            gna.oscprob_batch_ex(dp, L, om, de, 10, sp_ptr, x2_ptr, flags, data=dd)
            fg.barrier()
            sp, x2 = fg.result()
            assert np.array_equal(_np(sp), ref_sp) and np.array_equal(_np(x2), ref_x2)
            seen.append(flags)
        assert gna.GNA_OUT_PEER in seen
        # and the window's contents against the oracle (not only against the CUDA batch)
        idx = np.unique(np.r_[0, P // 2, P - 1])
        spr, x2r = oracle.batch(synth.subset_points(pts, idx), L, om, edges, 10, data=data,
                                nthreads=_nt())
        assert np.max(np.abs(ref_sp[idx] - spr) / np.abs(spr)) <= TOL_BIN
        assert np.all(np.abs(ref_x2[idx] - x2r) <= _chi2_bound(spr, data))
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------------ on-GPU fit loop
def _fit_case(sign=1.0, nbins=500):
    # sign = -1: inverted-ordering truth (signed dm2_31)
    truth = np.array([0.5838, 0.1496, 7.53e-5, sign * 2.52e-3])
    L, om = np.array([52.5, 53.0]), np.array([1.0, 0.98])
    edges = synth.uniform_edges(nbins, 1.0, 10.0)
    pts = dict(theta12=truth[:1], theta13=truth[1:2], dm2_21=truth[2:3], dm2_31=truth[3:4])
    data, _ = oracle.batch(pts, L, om, edges, 5, nthreads=_nt())  # pseudo-data = oracle at truth
    return truth, L, om, edges, data[0]


@pytest.mark.parametrize("sign", [1.0, -1.0])
def test_fit_pattern_search_recovers_truth(gna, sign):
    truth, L, om, edges, data = _fit_case(sign)
    step = np.array([0.01, 0.005, 2e-6, 5e-5])
    # start inside the truth's basin (chi^2 in dm2_31 is multimodal: the fast oscillation)
    start = truth + np.array([0.7, -0.6, 0.8, -0.5]) * step
    state = _t(np.r_[start, step])
    hist = _np(gna.fit_pattern_search(state, L, om, _t(edges), 5, _t(data), 120))
    x = _np(state)[:4]
    assert np.all(np.diff(hist) <= 0)          # best chi^2 never increases
    assert hist[-1] < 1e-12 * hist[0]
    assert np.all(np.abs(x - truth) <= 1e-6 * np.abs(truth)), (x, truth)


# nbins 500: stage B in one bin chunk; 1500: three chunks (chi^2 from partials); 501: odd, the
# scalar stage B + the update kernel — the argmin/update runs in stage B's last block otherwise
@pytest.mark.parametrize("sign,nbins", [(1.0, 500), (-1.0, 500), (1.0, 1500), (1.0, 501)])
def test_fit_pattern_search_steps_match_host_compass_search_on_oracle_chi2(gna, sign, nbins):
    """Each GPU iteration (niter = 1 calls) equals one compass step computed on the host:
    the 81 candidates centre + step * {-1, 0, 1}^4 (first coordinate fastest), their chi^2 from
    the oracle, argmin with ties to the lowest index; move there if it beats the centre, else
    halve the steps.  The state after every step must match bit for bit (normal and inverted
    ordering)."""
    truth, L, om, edges, data = _fit_case(sign, nbins)
    step = np.array([0.01, 0.005, 2e-6, 5e-5])
    st = np.r_[truth + np.array([0.7, -0.6, 0.8, -0.5]) * step, step]
    de, dd = _t(edges), _t(data)
    offs = np.array([[(c // 3 ** d) % 3 - 1 for d in range(4)] for c in range(81)], dtype=float)
    moved = halved = 0
    for _ in range(6):
        gpu = _t(st)
        hist = _np(gna.fit_pattern_search(gpu, L, om, de, 5, dd, 1))
        cand = st[:4][None, :] + offs * st[4:][None, :]
        pts = dict(theta12=cand[:, 0], theta13=cand[:, 1], dm2_21=cand[:, 2], dm2_31=cand[:, 3])
        _, x2 = oracle.batch(pts, L, om, edges, 5, data=data, want_spectra=False, nthreads=_nt())
        best = int(np.argmin(x2))
        gaps = np.sort(np.unique(x2))
        assert gaps.size < 2 or gaps[1] - gaps[0] > 1e-9 * gaps[1]  # decision not at the tolerance
        new = st.copy()
        if best != 40 and x2[best] < x2[40]:
            new[:4] = cand[best]
            moved += 1
        else:
            new[4:] *= 0.5
            halved += 1
        assert np.array_equal(_np(gpu), new)
        assert abs(hist[0] - min(x2[best], x2[40])) <= 1e-9 * x2[40]
        st = new
    assert moved and halved


def test_fit_pattern_search_deterministic_and_graph_capturable(gna):
    import torch
    truth, L, om, edges, data = _fit_case()
    step = np.array([0.01, 0.005, 2e-6, 5e-5])
    s0 = np.r_[truth + 0.6 * step, step]
    de, dd = _t(edges), _t(data)
    a = _t(s0)
    gna.fit_pattern_search(a, L, om, de, 5, dd, 30)
    b = _t(s0)
    ws = torch.empty(gna.fit_workspace_size(2, 500, 5) // 8 + 2, dtype=torch.float64, device="cuda")
    hist = torch.empty(30, dtype=torch.float64, device="cuda")
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            gna.fit_pattern_search(b, L, om, de, 5, dd, 30, hist=hist, workspace=ws)
    torch.cuda.current_stream().wait_stream(s)
    b.copy_(_t(s0))
    graph.replay()
    assert np.array_equal(_np(a), _np(b))


# ------------------------------------------------------------------------ ABI on the GPU
def test_host_pointer_to_device_entry_is_einval(gna):
    import ctypes
    E = np.linspace(1, 10, 100)
    P = np.empty(100)
    p = gna.OscParams()._c()
    rc = gna.load().gna_oscprob_eval(ctypes.byref(p), 52.5, E.ctypes.data, 100, P.ctypes.data,
                                     None)
    assert rc == gna.GNA_EINVAL


def test_launch_count_increments(gna):
    n0 = gna.launch_count()
    gna.gl_integrate(synth.CANONICAL, 52.5, _t(synth.uniform_edges(10)), 5)
    assert gna.launch_count() == n0 + 1


def test_c_abi_example_runs(gna, tmp_path):
    """examples/gl_integrate.c: the ABI from plain C (cudaMalloc'd buffers, gna_gl_integrate,
    gna_gl_integrate_host, EINVAL checks) exits 0."""
    import subprocess

    from test_abi_cpu import compile_c_example
    exe = compile_c_example(tmp_path / "gl_integrate_c")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("ok")


_MC_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, %(root)r)
import torch
from cuda.bindings import driver as d
import paper_1804_07682_b200 as gna
import synth


def ck(r):
    err, *rest = r if isinstance(r, tuple) else (r,)
    if err != d.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return rest[0] if len(rest) == 1 else rest


torch.zeros(1, device="cuda")  # torch's primary context is current
dev = ck(d.cuDeviceGet(0))
if not ck(d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)):
    print("NO_MULTICAST")
    sys.exit(0)
g = synth.rng(8100)
P, nb, order = %(P)d, 300, 10
pts = synth.invert_ordering(g, synth.points_uniform(g, P, dict(
    theta12=(0.5, 0.65), theta13=(0.1, 0.2), dm2_21=(6e-5, 9e-5), dm2_31=(2.2e-3, 2.8e-3))))
L, om = np.array([52.5, 215.0, 265.0])[:%(nbase)d], np.array([1.0, 0.06, 0.04])[:%(nbase)d]
edges = synth.uniform_edges(nb)
data = synth.pseudo_data(g, edges, om.sum())
need = P * nb * 8 + P * 8
H = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
prop = d.CUmulticastObjectProp()
prop.numDevices = 1
prop.handleTypes = H
prop.size = need
gran = ck(d.cuMulticastGetGranularity(
    prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
aprop = d.CUmemAllocationProp()
aprop.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
aprop.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
aprop.location.id = 0
aprop.requestedHandleTypes = H
agran = ck(d.cuMemGetAllocationGranularity(
    aprop, d.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))
gr = max(int(gran), int(agran))
size = -(-need // gr) * gr
prop.size = size
try:
    mc = ck(d.cuMulticastCreate(prop))
    ck(d.cuMulticastAddDevice(mc, dev))
except RuntimeError as exc:
    print("NO_MULTICAST", exc)
    sys.exit(0)
mem = ck(d.cuMemCreate(size, aprop, 0))
ck(d.cuMulticastBindMem(mc, 0, mem, 0, size, 0))
acc = d.CUmemAccessDesc()
acc.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
acc.location.id = 0
acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
uc = ck(d.cuMemAddressReserve(size, gr, 0, 0))
ck(d.cuMemMap(uc, size, 0, mem, 0))
ck(d.cuMemSetAccess(uc, size, [acc], 1))
mva = ck(d.cuMemAddressReserve(size, gr, 0, 0))
ck(d.cuMemMap(mva, size, 0, mc, 0))
ck(d.cuMemSetAccess(mva, size, [acc], 1))
ck(d.cuMemsetD8(uc, 0xff, size))  # NaN pattern: every output must be written
f64 = dict(dtype=torch.float64, device="cuda")
dp = {k: torch.tensor(v, **f64) for k, v in pts.items()}
de, dd = torch.tensor(edges, **f64), torch.tensor(data, **f64)
base = int(mva)
gna.oscprob_batch_ex(dp, L, om, de, order, base, base + P * nb * 8, gna.GNA_OUT_MULTICAST, data=dd)
torch.cuda.synchronize()
out = np.empty(P * nb + P)
ck(d.cuMemcpyDtoH(out.ctypes.data, uc, need))
sp, x2 = out[:P * nb].reshape(P, nb), out[P * nb:]
ref_sp, ref_x2 = gna.oscprob_batch(dp, L, om, de, order, data=dd)
assert np.array_equal(sp, ref_sp.cpu().numpy()) and np.array_equal(x2, ref_x2.cpu().numpy())
np.save(%(out)r, out)
print("MULTICAST_OK")
"""


@pytest.mark.parametrize("P,nbase", [(5, 3), (300, 1)])
def test_fused_epilogue_multicast_stores_single_gpu_nvls_object(gna, P, nbase, tmp_path):
    """NEXT-4 multicast epilogue on real NVLS hardware: a one-device multicast object
    (cuMulticastCreate + cuMulticastBindMem, driver API) mapped at a multicast VA; the batch
    kernel's multimem.st epilogue writes through it and the bound memory, read back through
    its unicast mapping, equals the plain batch bit for bit and the oracle on every point
    (per-point kernel at 5 x 3 baselines; points-across-lanes kernel at 300 x 1).  Runs in a
    subprocess so that a fault cannot poison this test process; skips where the fabric has
    no multicast support."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outp = str(tmp_path / "mc.npy")
    r = subprocess.run([sys.executable, "-c", _MC_SCRIPT % dict(root=root, P=P, nbase=nbase,
                                                                 out=outp)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    if "NO_MULTICAST" in r.stdout:
        pytest.skip("no NVLS multicast on this device: " + r.stdout.strip()[:200])
    assert "MULTICAST_OK" in r.stdout
    g = synth.rng(8100)
    pts = synth.invert_ordering(g, synth.points_uniform(g, P, dict(
        theta12=(0.5, 0.65), theta13=(0.1, 0.2), dm2_21=(6e-5, 9e-5), dm2_31=(2.2e-3, 2.8e-3))))
    L, om = np.array([52.5, 215.0, 265.0])[:nbase], np.array([1.0, 0.06, 0.04])[:nbase]
    edges = synth.uniform_edges(300)
    data = synth.pseudo_data(g, edges, om.sum())
    out = np.load(outp)
    sp, x2 = out[:P * 300].reshape(P, 300), out[P * 300:]
    idx = np.unique(np.r_[0, P // 2, P - 1])
    spr, x2r = oracle.batch(synth.subset_points(pts, idx), L, om, edges, 10, data=data,
                            nthreads=_nt())
    assert np.max(np.abs(sp[idx] - spr) / np.abs(spr)) <= TOL_BIN
    assert np.all(np.abs(x2[idx] - x2r) <= _chi2_bound(spr, data))

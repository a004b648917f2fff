"""CPU-side checks of the C-ABI library (no GPU needed).

* libgna_b200.so loads and exports every function include/gna_b200.h declares;
* every invalid-argument path returns GNA_EINVAL before any CUDA call;
* the library's Gauss-Legendre table equals an independent rule (oracle
  Newton and numpy leggauss);
* the sin^2 polynomial of the kernels meets its accuracy claim when evaluated
  exactly as the kernel does (fp64 FMA Horner, emulated with Fractions).
"""
from __future__ import annotations

import ctypes
import os
import re
from fractions import Fraction

import mpmath as mp
import numpy as np
import pytest

import oracle
import paper_1804_07682_b200 as gna
from paper_1804_07682_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gna_b200.h")


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return gna.load()


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gna_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    declared = _declared_functions()
    assert len(declared) >= 10
    assert sorted(declared) == sorted(gna.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_sm100a_only_cubin(lib):
    # the fatbin carries sm_100a SASS and no other architecture
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_strerror_and_version(lib):
    assert gna.abi_version() == 1
    for code in (0, -1, -2, -3, -4):
        assert lib.gna_strerror(code).startswith(b"GNA_")
    assert lib.gna_strerror(7) == b"unknown gna_status"
    assert lib.gna_last_cuda_error() == 0


BAD = ctypes.c_void_p(0x10000)    # non-null fake addresses: validation must reject
BAD2 = ctypes.c_void_p(0x900000)  # before touching them


def _params(**kw):
    p = gna.OscParams(**kw)._c()
    return ctypes.byref(p)


@pytest.mark.parametrize("case", [
    dict(n=0), dict(n=-5), dict(E=None), dict(P=None), dict(L=-1.0), dict(L=float("nan")),
    dict(L=float("inf")), dict(theta12=float("nan")), dict(dm2_31=float("inf")),
    dict(P=ctypes.c_void_p(0x10000 + 8)),  # overlaps E
])
def test_eval_einval(lib, case):
    n = case.get("n", 100)
    E = case.get("E", BAD)
    P = case.get("P", BAD2)
    L = case.get("L", 52.5)
    pk = {k: v for k, v in case.items() if k in ("theta12", "dm2_31")}
    for f in (lambda: lib.gna_oscprob_eval(_params(**pk), L, E, n, P, None),
              lambda: lib.gna_oscprob_eval_host(_params(**pk), L, E, n, P, 0, None)):
        assert f() == gna.GNA_EINVAL


@pytest.mark.parametrize("ab", [(-1, 0), (0, 3), (3, 3), (0, -2)])
def test_eval_ab_einval(lib, ab):
    assert lib.gna_oscprob_eval_ab(ab[0], ab[1], _params(), 52.5, BAD, 10, BAD2, None) == \
        gna.GNA_EINVAL
    # and the shared validation
    assert lib.gna_oscprob_eval_ab(0, 1, _params(), -1.0, BAD, 10, BAD2, None) == gna.GNA_EINVAL
    assert lib.gna_oscprob_eval_ab(0, 1, _params(), 1.0, BAD, 0, BAD2, None) == gna.GNA_EINVAL
    assert lib.gna_gl_integrate_ab(ab[0], ab[1], _params(), 52.5, BAD, 10, 5, BAD2, None) == \
        gna.GNA_EINVAL
    assert lib.gna_gl_integrate_ab(0, 1, _params(), 52.5, BAD, 10, 33, BAD2, None) == \
        gna.GNA_EINVAL


def test_eval_null_params(lib):
    assert lib.gna_oscprob_eval(None, 1.0, BAD, 10, BAD2, None) == gna.GNA_EINVAL


@pytest.mark.parametrize("case", [
    dict(nbins=0), dict(order=0), dict(order=33), dict(edges=None), dict(bins=None),
    dict(L=-0.5), dict(bins=ctypes.c_void_p(0x10000 + 16)),
])
def test_gl_einval(lib, case):
    r = lib.gna_gl_integrate(_params(), case.get("L", 52.5), case.get("edges", BAD),
                             case.get("nbins", 10), case.get("order", 5), case.get("bins", BAD2),
                             None)
    assert r == gna.GNA_EINVAL
    r = lib.gna_gl_integrate_host(_params(), case.get("L", 52.5), case.get("edges", BAD),
                                  case.get("nbins", 10), case.get("order", 5),
                                  case.get("bins", BAD2), 0, None)
    assert r == gna.GNA_EINVAL


def _batch(lib, host=False, **kw):
    P = kw.get("npoints", 4)
    pts = gna._CBatch(0x100000, 0x200000, 0x300000, kw.get("d31", 0x400000), P)
    nb = kw.get("nbase", 2)
    L = np.asarray(kw.get("L", [52.5, 1.0][:max(nb, 0)] + [1.0] * max(nb - 2, 0)), dtype=float)
    om = np.ones(max(nb, 1))
    if L.size < max(nb, 1):
        L = np.resize(L, max(nb, 1))
    args = [ctypes.byref(pts), L.ctypes.data, om.ctypes.data, nb, kw.get("edges", 0x500000),
            kw.get("nbins", 10), kw.get("order", 5), kw.get("spectra", 0x600000),
            kw.get("data", 0x700000), kw.get("chi2", 0x800000)]
    if host:
        return lib.gna_oscprob_batch_host(*args, 0, None)
    if "flags" in kw:
        return lib.gna_oscprob_batch_ex(*args, kw.get("ws", 0x900000), kw.get("wsb", 1 << 20),
                                        kw["flags"], None)
    return lib.gna_oscprob_batch(*args, kw.get("ws", 0x900000), kw.get("wsb", 1 << 20), None)


@pytest.mark.parametrize("case", [
    dict(npoints=0), dict(nbase=0), dict(nbase=65), dict(nbins=0), dict(order=0),
    dict(order=33), dict(spectra=None, chi2=None), dict(data=None), dict(edges=None),
    dict(d31=None), dict(L=[52.5, -1.0]), dict(L=[float("nan"), 1.0]),
    dict(chi2=0x600000 + 8),          # chi2 inside spectra
    dict(spectra=0x100000 - 8),       # spectra overlaps theta12
    dict(ws=None), dict(wsb=8),       # workspace missing or too small
    dict(ws=0x900008),                # workspace not 16-byte aligned
    dict(ws=0x100000 - 64),           # workspace overlaps theta12
])
def test_batch_einval(lib, case):
    assert _batch(lib, **case) == gna.GNA_EINVAL
    # the mixed tier (NEXT-3) validates exactly like the fp64 batch
    assert _batch(lib, flags=gna.GNA_PREC_MIXED, **case) == gna.GNA_EINVAL
    assert _batch(lib, flags=gna.GNA_WS_TABLES_VALID, **case) == gna.GNA_EINVAL
    if "ws" not in case and "wsb" not in case:
        assert _batch(lib, host=True, **case) == gna.GNA_EINVAL


@pytest.mark.parametrize("flags", [1, 2, 1 | 4, 2 | 4])
@pytest.mark.parametrize("ws", [0x100000 - 64, 0x500000 - 64, 0x700000 + 8])
def test_batch_ex_remote_outputs_workspace_overlap_einval(lib, flags, ws):
    """Peer / multicast outputs: the workspace still must not alias the local inputs
    (points, edges, data), or k_batch_setup would overwrite them."""
    assert _batch(lib, flags=flags, ws=ws) == gna.GNA_EINVAL


@pytest.mark.parametrize("flags", [16, 16 | 4, 1 | 2, 1 | 2 | 4, 1 | 2 | 8, 0xffffffff])
def test_batch_ex_bad_flags(lib, flags):
    assert _batch(lib, flags=flags) == gna.GNA_EINVAL


@pytest.mark.parametrize("flags", [1, 2, 8, 1 | 4, 0xffffffff])
def test_eval_gl_ex_bad_flags(lib, flags):
    """The single-point _ex calls accept only GNA_PREC_MIXED (NEXT-3)."""
    assert lib.gna_oscprob_eval_ex(_params(), 1.0, BAD, 10, BAD2, flags, None) == gna.GNA_EINVAL
    assert lib.gna_gl_integrate_ex(_params(), 1.0, BAD, 10, 5, BAD2, flags,
                                   None) == gna.GNA_EINVAL


def test_eval_gl_ex_mixed_validates_like_fp64(lib):
    m = gna.GNA_PREC_MIXED
    assert lib.gna_oscprob_eval_ex(_params(), -1.0, BAD, 10, BAD2, m, None) == gna.GNA_EINVAL
    assert lib.gna_oscprob_eval_ex(_params(), 1.0, BAD, 0, BAD2, m, None) == gna.GNA_EINVAL
    assert lib.gna_oscprob_eval_ex(None, 1.0, BAD, 10, BAD2, m, None) == gna.GNA_EINVAL
    assert lib.gna_gl_integrate_ex(_params(), 1.0, BAD, 10, 33, BAD2, m, None) == gna.GNA_EINVAL
    assert lib.gna_gl_integrate_ex(_params(), 1.0, BAD, 0, 5, BAD2, m, None) == gna.GNA_EINVAL


def test_header_constants_match_binding():
    """The Python binding's constants are the header's #defines."""
    src = open(HEADER).read()
    for name in ("GNA_OUT_PEER", "GNA_OUT_MULTICAST", "GNA_PREC_MIXED", "GNA_WS_TABLES_VALID",
                 "GNA_MAX_ORDER",
                 "GNA_MAX_NBASE", "GNA_OK", "GNA_EINVAL", "GNA_ECUDA", "GNA_ENODEV",
                 "GNA_ENOMEM"):
        m = (re.search(r"#define %s \(?(-?\d+)u?\)?" % name, src) or
             re.search(r"\b%s = (-?\d+)" % name, src))  # enum gna_status
        assert m, name
        assert int(m.group(1)) == getattr(gna, name), name


def _scan(lib, **kw):
    g = gna._CScan(0x100000, 0x200000, kw.get("nmix", 4), 0x300000, kw.get("d31", 0x400000),
                   kw.get("nmass", 3))
    nb = kw.get("nbase", 1)
    L = np.full(max(nb, 1), kw.get("L", 52.5))
    om = np.ones(max(nb, 1))
    return lib.gna_oscprob_scan(ctypes.byref(g), L.ctypes.data, om.ctypes.data, nb,
                                kw.get("edges", 0x500000), kw.get("nbins", 10),
                                kw.get("order", 5), kw.get("spectra", 0x600000),
                                kw.get("data", 0x700000), kw.get("chi2", 0x800000),
                                kw.get("ws", 0x900000), kw.get("wsb", 1 << 20), None)


@pytest.mark.parametrize("case", [
    dict(nmix=0), dict(nmass=0), dict(nbase=0), dict(nbase=65), dict(nbins=0), dict(order=0),
    dict(order=33), dict(spectra=None, chi2=None), dict(data=None), dict(edges=None),
    dict(d31=None), dict(L=-1.0), dict(L=float("inf")), dict(ws=None), dict(wsb=64),
    dict(ws=0x900010),                # not 32-byte aligned
    dict(chi2=0x600000 + 8),          # chi2 inside spectra
    dict(ws=0x100000 - 64),           # workspace overlaps theta12
])
def test_scan_einval(lib, case):
    assert _scan(lib, **case) == gna.GNA_EINVAL


def test_scan_workspace_size(lib):
    assert gna.oscprob_scan_workspace_size(0, 1, 10) == 0
    assert gna.oscprob_scan_workspace_size(1, 0, 10) == 0
    assert gna.oscprob_scan_workspace_size(1, 1, 0) == 0
    w = gna.oscprob_scan_workspace_size(100, 100, 1000)
    assert w >= 100 * 3 * 1000 * 8 + 2 * 1000 * 8 + 100 * 32 and w % 32 == 0


def test_fit_einval(lib):
    L = np.array([52.5])
    om = np.ones(1)
    args = dict(L=L.ctypes.data, om=om.ctypes.data, nbase=1, edges=0x500000, nbins=10, order=5,
                data=0x700000, state=0x800000, niter=5, hist=None, ws=0x900000, wsb=1 << 20)
    def call(**kw):
        a = dict(args, **kw)
        return lib.gna_fit_pattern_search(a["L"], a["om"], a["nbase"], a["edges"], a["nbins"],
                                          a["order"], a["data"], a["state"], a["niter"],
                                          a["hist"], a["ws"], a["wsb"], None)
    for kw in (dict(L=None), dict(nbase=0), dict(edges=None), dict(nbins=0), dict(order=40),
               dict(data=None), dict(state=None), dict(niter=-1), dict(ws=None), dict(wsb=8),
               dict(ws=0x900008)):
        assert call(**kw) == gna.GNA_EINVAL, kw
    assert gna.fit_workspace_size(1, 10, 5) > 0 and gna.fit_workspace_size(0, 10, 5) == 0


def test_batch_workspace_size(lib):
    assert gna.oscprob_batch_workspace_size(0, 1, 10, 5) == 0
    assert gna.oscprob_batch_workspace_size(10, 1, 0, 5) == 0
    assert gna.oscprob_batch_workspace_size(10, 0, 10, 5) == 0
    assert gna.oscprob_batch_workspace_size(10, 65, 10, 5) == 0
    assert gna.oscprob_batch_workspace_size(10, 1, 10, 33) == 0
    ws = gna.oscprob_batch_workspace_size(1000, 8, 10_000, 10)
    # coefficients + c0 + two node tables + chi2 partials
    assert ws >= 1000 * 8 * 3 * 16 + 1000 * 8 + 2 * 10 * 10_000 * 8 + 1000 * 313 * 8
    assert ws % 16 == 0


def test_valid_call_without_gpu_does_not_crash(lib):
    # on the CPU box there is no device: a valid call reports ECUDA/ENODEV/EINVAL, never crashes
    r = lib.gna_oscprob_eval(_params(), 52.5, BAD, 10, BAD2, None)
    assert r in (gna.GNA_ECUDA, gna.GNA_ENODEV, gna.GNA_EINVAL, gna.GNA_OK)


@pytest.mark.parametrize("n", list(range(1, 33)))
def test_library_gl_rule_matches_independent_rules(lib, n):
    t, w = gna.gl_rule(n)
    to, wo = oracle.gauleg(n)
    tn, wn = np.polynomial.legendre.leggauss(n)
    assert np.max(np.abs(t - to)) <= 2.3e-16 and np.max(np.abs(w - wo)) <= 4.5e-16
    assert np.max(np.abs(t - tn)) <= 4e-16 and np.max(np.abs(w - wn)) <= 6e-15
    assert np.array_equal(t, -t[::-1])


def test_gl_rule_einval(lib):
    buf = np.zeros(40)
    assert lib.gna_gl_rule(0, buf.ctypes.data, buf.ctypes.data) == gna.GNA_EINVAL
    assert lib.gna_gl_rule(33, buf.ctypes.data, buf.ctypes.data) == gna.GNA_EINVAL


def _sin2_coeffs(prefix="GNA_SIN2_C"):
    src = open(os.path.join(_build.CSRC, "sin2_poly.h")).read()
    cs = dict(re.findall(r"#define %s(\d) \(([-0-9a-fx.p+]+)\)" % prefix, src))
    return [float.fromhex(cs[str(j)]) for j in range(len(cs))]


def _sinpi_coeffs():
    src = open(os.path.join(_build.CSRC, "sinpi_poly.h")).read()
    cs = dict(re.findall(r"#define GNA_SINPI_C(\d) \(([-0-9a-fx.p+]+)\)", src))
    return [float.fromhex(cs[str(j)]) for j in range(len(cs))]


def test_kernel_sinpi_polynomial_accuracy():
    """sin(pi (q + f)) = (-1)^q f S(f^2) with the kernel's fp64 Horner: |err| <= 2.5e-16."""
    cf = _sinpi_coeffs()
    assert len(cf) == 9
    mp.mp.dps = 40
    fs = np.r_[np.linspace(-0.5, 0.5, 801), np.random.default_rng(4).uniform(-0.5, 0.5, 400)]
    worst = 0.0
    for f in fs:
        u = float(f) * float(f)
        p = cf[-1]
        for c in reversed(cf[:-1]):
            p = _fma(p, u, c)
        got = float(f) * p
        for q in (0, 3):
            ref = mp.sin(mp.pi * (q + mp.mpf(float(f))))
            worst = max(worst, abs((got if q % 2 == 0 else -got) - float(ref)))
    assert worst <= 2.5e-16


def _fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


@pytest.mark.parametrize("prefix,ncoef,bound", [("GNA_SIN2_C", 9, 1.2e-16),
                                                ("GNA_SIN2_D7_C", 8, 1.12e-15)])
def test_kernel_sin2_polynomial_accuracy(prefix, ncoef, bound):
    """sin^2((pi/2)(q+f)) = 1/2 + (-1)^q V(f^2) with the kernel's fp64 Horner: |err| <= bound
    (degree 8: 1.2e-16; degree 7, the default: 1.12e-15 — DESIGN.md R7), plus the final
    half-ulp of 1/2 +- v.  Both pin V(0) = -1/2, so sin^2 is exactly 0 at even q, f = 0."""
    cf = _sin2_coeffs(prefix)
    assert len(cf) == ncoef and cf[0] == -0.5
    mp.mp.dps = 40
    g = np.random.default_rng(3)
    fs = np.r_[np.linspace(-0.5, 0.5, 801), g.uniform(-0.5, 0.5, 400)]
    worst = 0.0
    for f in fs:
        u = float(f) * float(f)
        p = cf[-1]
        for c in reversed(cf[:-1]):
            p = _fma(p, u, c)
        for q in (0, 1, 7, 100):
            got = 0.5 + (p if q % 2 == 0 else -p)
            ref = mp.sin(mp.pi / 2 * (q + mp.mpf(float(f)))) ** 2
            worst = max(worst, abs(float(got - ref)))
    assert worst <= bound + 1.2e-16  # polynomial + final half-ulp of 1/2 +- v


def test_mixed_tier_fp32_polynomial_accuracy():
    """NEXT-3 mixed tier: -cos(pi y)/2 = W(h^2), y = 2m + 2h, with h rounded to fp32 (F2F, round
    to nearest) and W evaluated by the kernel's fp32 FMA Horner chain (GNA_COS2F_*): within
    1.3e-7 of the polynomial and 2.3e-7 of the exact value, for every residue class of y."""
    src = open(os.path.join(_build.CSRC, "sin2_poly.h")).read()
    cs = dict(re.findall(r"#define GNA_COS2F_C(\d) \(\(float\)([-0-9a-fx.p+]+)\)", src))
    cf = [float.fromhex(cs[str(j)]) for j in range(len(cs))]
    assert len(cf) == 7 and cf[0] == -0.5
    f32 = lambda x: float(np.float32(x))  # noqa: E731
    mp.mp.dps = 30
    g = np.random.default_rng(8)
    worst_poly = worst = 0.0
    for h in np.r_[np.linspace(-0.5, 0.5, 601), g.uniform(-0.5, 0.5, 300)]:
        hs = f32(h)
        u = f32(Fraction(hs) * Fraction(hs))
        p = cf[-1]
        for c in reversed(cf[:-1]):
            p = f32(Fraction(p) * Fraction(u) + Fraction(c))
        worst_poly = max(worst_poly, abs(p - float(-mp.cos(2 * mp.pi * mp.mpf(hs)) / 2)))
        for m in (0, 1, 37):  # y = 2m + 2h: the value does not depend on m
            ref = -mp.cos(mp.pi * (2 * m + 2 * mp.mpf(float(h)))) / 2
            worst = max(worst, abs(p - float(ref)))
    assert worst_poly <= 1.3e-7 and worst <= 2.3e-7


def test_kernel_sin2_small_phase_error_vanishes():
    """With V(0) = -1/2 pinned, the degree-7 error is O(u): for |f| <= 1e-3 the Horner result
    stays at the rounding level (<= 1.2e-16 (1 + 1e6 u)) instead of the 1.1e-15 worst case, so
    small phases (short baselines, L -> 0) are exact to rounding."""
    cf = _sin2_coeffs("GNA_SIN2_D7_C")
    mp.mp.dps = 40
    for f in np.linspace(-1e-3, 1e-3, 101):
        u = float(f) * float(f)
        p = cf[-1]
        for c in reversed(cf[:-1]):
            p = _fma(p, u, c)
        ref = -mp.cos(mp.pi * mp.mpf(float(f))) / 2
        assert abs(float(p - ref)) <= 1.2e-16 * (1 + 1e6 * u)


def compile_c_example(out_path):
    """Build examples/gl_integrate.c: include/gna_b200.h must be valid C11 and the library
    must link from plain C (no torch, no Python)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(root, "paper_1804_07682_b200")
    cuda = "/usr/local/cuda"
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-Werror",
           "-I" + os.path.join(root, "include"), "-I" + os.path.join(cuda, "include"),
           os.path.join(root, "examples", "gl_integrate.c"), "-L" + pkg, "-lgna_b200",
           "-L" + os.path.join(cuda, "lib64"), "-lcudart", "-lm", "-Wl,-rpath," + pkg,
           "-o", str(out_path)]
    subprocess.check_call(cmd)
    return str(out_path)


def test_c_abi_example_compiles_and_links(lib, tmp_path):
    import shutil
    if shutil.which("gcc") is None or not os.path.exists("/usr/local/cuda/include/cuda_runtime_api.h"):
        pytest.skip("gcc or the CUDA headers are not available")
    exe = compile_c_example(tmp_path / "gl_integrate_c")
    assert os.path.exists(exe)


def test_binding_checks_lengths_before_any_call(lib):
    """The binding rejects mismatched host array lengths before the C ABI (which reads nbase
    omegas and P values of every point array) could read past a numpy buffer."""
    import torch
    P = 4
    pts = {k: np.full(P, v) for k, v in dict(theta12=0.58, theta13=0.15, dm2_21=7.5e-5,
                                               dm2_31=2.5e-3).items()}
    edges = np.linspace(1.0, 10.0, 11)
    data = np.ones(10)
    short = dict(pts, theta13=np.full(P - 1, 0.15))
    with pytest.raises(ValueError):
        gna.oscprob_batch_host(short, [52.5], [1.0], edges, 5, data=data)
    with pytest.raises(ValueError):
        gna.oscprob_batch_host(pts, [52.5, 215.0], [1.0], edges, 5, data=data)
    with pytest.raises(ValueError):
        gna.oscprob_batch_host(pts, [52.5], 1.0 * np.ones(3), edges, 5, data=data)
    tp = {k: torch.tensor(v) for k, v in pts.items()}
    with pytest.raises(ValueError):
        gna.oscprob_batch_ex(tp, [52.5, 215.0], [1.0], torch.tensor(edges), 5, None, None, 0)
    with pytest.raises(ValueError):
        gna.fit_pattern_search(torch.zeros(8, dtype=torch.float64), [52.5, 215.0], [1.0],
                               torch.tensor(edges), 5, torch.tensor(data), 1)


def test_tables_valid_needs_a_workspace(lib):
    """tables_valid=True without the workspace that holds the tables is refused before any
    call (a fresh scratch workspace would hold no tables)."""
    import torch
    pts = {k: torch.zeros(3, dtype=torch.float64) for k in ("theta12", "theta13", "dm2_21",
                                                           "dm2_31")}
    with pytest.raises(ValueError):
        gna.oscprob_batch(pts, [52.5], [1.0], torch.linspace(1, 10, 11, dtype=torch.float64), 5,
                          tables_valid=True)

"""B200-native GNA hot path (arXiv:1804.07682): thin ctypes binding of libgna_b200.so.

Argument marshalling only — every step of the computation runs in the CUDA
kernels of ``csrc/gna_b200.cu`` behind the C ABI declared in
``include/gna_b200.h``.  There is no CPU fallback: if the library is missing or
the device is not a B200 the calls raise.  PyTorch supplies device memory and
streams only (tensors in, tensors out).

Names follow the C ABI: ``oscprob_eval``, ``gl_integrate``, ``oscprob_batch``
(device tensors) and ``oscprob_eval_host``, ``oscprob_batch_host`` (host numpy
arrays, the end-to-end path with overlapped copies).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, fields

import numpy as np

from . import _build

__all__ = [
    "GnaError", "OscParams", "load", "oscprob_eval", "gl_integrate", "oscprob_batch",
    "oscprob_batch_workspace_size", "oscprob_eval_host", "gl_integrate_host",
    "oscprob_batch_host", "gl_rule",
    "release", "launch_count", "abi_version", "EXPORTS", "GNA_MAX_ORDER", "GNA_MAX_NBASE",
    "oscprob_scan", "oscprob_scan_workspace_size", "oscprob_eval_ab", "oscprob_batch_ex",
    "gl_integrate_ab", "fit_pattern_search", "fit_workspace_size",
    "GNA_OUT_PEER", "GNA_OUT_MULTICAST", "GNA_PREC_MIXED", "GNA_WS_TABLES_VALID",
]

GNA_OK, GNA_EINVAL, GNA_ECUDA, GNA_ENODEV, GNA_ENOMEM = 0, -1, -2, -3, -4
GNA_MAX_ORDER = 32
GNA_MAX_NBASE = 64

# every symbol include/gna_b200.h declares
EXPORTS = (
    "gna_oscprob_eval", "gna_gl_integrate", "gna_oscprob_batch_workspace_size",
    "gna_oscprob_batch", "gna_oscprob_eval_host", "gna_gl_integrate_host",
    "gna_oscprob_batch_host", "gna_release",
    "gna_gl_rule", "gna_strerror", "gna_last_cuda_error", "gna_abi_version", "gna_launch_count",
    "gna_sin2_poly_degree", "gna_oscprob_eval_ex", "gna_gl_integrate_ex",
    "gna_oscprob_scan_workspace_size", "gna_oscprob_scan", "gna_oscprob_eval_ab",
    "gna_oscprob_batch_ex", "gna_gl_integrate_ab", "gna_fit_workspace_size",
    "gna_fit_pattern_search",
)

GNA_OUT_PEER = 1
GNA_OUT_MULTICAST = 2
GNA_PREC_MIXED = 4
GNA_WS_TABLES_VALID = 8


class GnaError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        msg = _lib.gna_strerror(code).decode() if _lib is not None else str(code)
        if code == GNA_ECUDA and _lib is not None:
            msg += " (cudaError %d)" % _lib.gna_last_cuda_error()
        super().__init__("%s: %s" % (what, msg))


class _CParams(ctypes.Structure):
    _fields_ = [("theta12", ctypes.c_double), ("theta13", ctypes.c_double),
                ("theta23", ctypes.c_double), ("delta_cp", ctypes.c_double),
                ("dm2_21", ctypes.c_double), ("dm2_31", ctypes.c_double),
                ("antineutrino", ctypes.c_int32)]


class _CScan(ctypes.Structure):
    _fields_ = [("theta12", ctypes.c_void_p), ("theta13", ctypes.c_void_p),
                ("nmix", ctypes.c_int64), ("dm2_21", ctypes.c_void_p),
                ("dm2_31", ctypes.c_void_p), ("nmass", ctypes.c_int64)]


class _CBatch(ctypes.Structure):
    _fields_ = [("theta12", ctypes.c_void_p), ("theta13", ctypes.c_void_p),
                ("dm2_21", ctypes.c_void_p), ("dm2_31", ctypes.c_void_p),
                ("npoints", ctypes.c_int64)]


@dataclass
class OscParams:
    """SPEC OscParams; angles in rad, dm2 in eV^2."""
    theta12: float = 0.5838
    theta13: float = 0.1496
    theta23: float = 0.7854
    delta_cp: float = 0.0
    dm2_21: float = 7.53e-5
    dm2_31: float = 2.52e-3
    antineutrino: int = 0

    @classmethod
    def of(cls, p) -> "OscParams":
        if isinstance(p, OscParams):
            return p
        names = {f.name for f in fields(cls)}
        return cls(**{k: v for k, v in dict(p).items() if k in names})

    def _c(self) -> _CParams:
        return _CParams(float(self.theta12), float(self.theta13), float(self.theta23),
                        float(self.delta_cp), float(self.dm2_21), float(self.dm2_31),
                        int(self.antineutrino))


_lib = None


def load(path: str | None = None) -> ctypes.CDLL:
    """Load libgna_b200.so (built by ``__graft_entry__.build()``); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or _build.LIB
    if not os.path.exists(path):
        raise ImportError("libgna_b200.so not built (%s); run `python -c 'import __graft_entry__ "
                          "as g; g.build()'` — there is no CPU fallback" % path)
    L = ctypes.CDLL(path)
    d, i32, i64, vp, sz = (ctypes.c_double, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p,
                           ctypes.c_size_t)
    P = ctypes.POINTER(_CParams)
    B = ctypes.POINTER(_CBatch)
    L.gna_oscprob_eval.argtypes = [P, d, vp, i64, vp, vp]
    L.gna_gl_integrate.argtypes = [P, d, vp, i64, i32, vp, vp]
    L.gna_oscprob_eval_ex.argtypes = [P, d, vp, i64, vp, ctypes.c_uint32, vp]
    L.gna_gl_integrate_ex.argtypes = [P, d, vp, i64, i32, vp, ctypes.c_uint32, vp]
    L.gna_oscprob_eval_ex.restype = ctypes.c_int
    L.gna_gl_integrate_ex.restype = ctypes.c_int
    L.gna_oscprob_eval_ab.argtypes = [i32, i32, P, d, vp, i64, vp, vp]
    L.gna_oscprob_batch_ex.argtypes = [B, vp, vp, i32, vp, i64, i32, vp, vp, vp, vp, sz,
                                       ctypes.c_uint32, vp]
    L.gna_oscprob_batch_ex.restype = ctypes.c_int
    L.gna_oscprob_eval_ab.restype = ctypes.c_int
    L.gna_gl_integrate_ab.argtypes = [i32, i32, P, d, vp, i64, i32, vp, vp]
    L.gna_gl_integrate_ab.restype = ctypes.c_int
    L.gna_fit_workspace_size.argtypes = [i32, i64, i32]
    L.gna_fit_workspace_size.restype = sz
    L.gna_fit_pattern_search.argtypes = [vp, vp, i32, vp, i64, i32, vp, vp, i32, vp, vp, sz, vp]
    L.gna_fit_pattern_search.restype = ctypes.c_int
    L.gna_oscprob_batch_workspace_size.argtypes = [i64, i32, i64, i32]
    L.gna_oscprob_batch_workspace_size.restype = sz
    L.gna_oscprob_batch.argtypes = [B, vp, vp, i32, vp, i64, i32, vp, vp, vp, vp, sz, vp]
    L.gna_oscprob_eval_host.argtypes = [P, d, vp, i64, vp, i64, vp]
    L.gna_oscprob_batch_host.argtypes = [B, vp, vp, i32, vp, i64, i32, vp, vp, vp, i64, vp]
    L.gna_gl_integrate_host.argtypes = [P, d, vp, i64, i32, vp, i64, vp]
    S = ctypes.POINTER(_CScan)
    L.gna_oscprob_scan_workspace_size.argtypes = [i64, i64, i64]
    L.gna_oscprob_scan_workspace_size.restype = sz
    L.gna_oscprob_scan.argtypes = [S, vp, vp, i32, vp, i64, i32, vp, vp, vp, vp, sz, vp]
    L.gna_oscprob_scan.restype = ctypes.c_int
    L.gna_release.argtypes = []
    L.gna_release.restype = None
    L.gna_gl_rule.argtypes = [i32, vp, vp]
    L.gna_strerror.argtypes = [ctypes.c_int]
    L.gna_strerror.restype = ctypes.c_char_p
    L.gna_last_cuda_error.argtypes = []
    L.gna_abi_version.argtypes = []
    L.gna_sin2_poly_degree.argtypes = []
    L.gna_launch_count.argtypes = []
    L.gna_launch_count.restype = i64
    for name in ("gna_oscprob_eval", "gna_gl_integrate", "gna_oscprob_batch",
                 "gna_oscprob_eval_host", "gna_gl_integrate_host", "gna_oscprob_batch_host",
                 "gna_gl_rule",
                 "gna_last_cuda_error", "gna_abi_version", "gna_sin2_poly_degree"):
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _check(rc: int, what: str):
    if rc != GNA_OK:
        raise GnaError(rc, what)


# ---------------------------------------------------------------- marshalling helpers
def _dev(t, name: str, n: int | None = None) -> int:
    """Pointer of a contiguous fp64 CUDA tensor (no copies, no conversions)."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("%s must be a CUDA tensor" % name)
    if t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError("%s must be a contiguous float64 tensor" % name)
    if n is not None and t.numel() != n:
        raise ValueError("%s must have %d elements, has %d" % (name, n, t.numel()))
    return t.data_ptr()


def _host(a, name: str, n: int | None = None, writable=False) -> np.ndarray:
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous:
        raise TypeError("%s must be a C-contiguous float64 numpy array" % name)
    if writable and not a.flags.writeable:
        raise TypeError("%s must be writable" % name)
    if n is not None and a.size != n:
        raise ValueError("%s must have %d elements, has %d" % (name, n, a.size))
    return a


def _stream(stream) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream) if hasattr(s, "cuda_stream") else int(s)


def _small(a, name) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).ravel())


def _baselines(L_km, omega):
    """Host arrays L_km[nbase], omega[nbase] of equal length (the C ABI reads nbase of each)."""
    Lh, om = _small(L_km, "L_km"), _small(omega, "omega")
    if Lh.size != om.size:
        raise ValueError("L_km and omega must have the same length (%d vs %d)"
                         % (Lh.size, om.size))
    return Lh, om


def _scratch(nbytes: int, dev, stream, align: int = 8):
    """Caller-side workspace for one call.  It is allocated on torch's current stream; when the
    call is enqueued on another `stream`, the block is recorded on that stream so the caching
    allocator cannot hand it to other work before the kernels that use it have finished."""
    import torch
    extra = align // 8
    ws = torch.empty(max((nbytes + 7) // 8, 2) + extra, dtype=torch.float64, device=dev)
    if stream is not None:
        if not isinstance(stream, torch.cuda.Stream):
            raise TypeError("pass workspace= explicitly when stream is a raw handle")
        ws.record_stream(stream)
    off = (-ws.data_ptr()) % align // 8
    return ws[off:]


# ---------------------------------------------------------------- device entry points
def _prec_flags(precision: str) -> int:
    if precision not in ("fp64", "mixed"):
        raise ValueError("precision must be 'fp64' or 'mixed'")
    return GNA_PREC_MIXED if precision == "mixed" else 0


def oscprob_eval(params, L_km: float, E, out=None, stream=None, precision: str = "fp64"):
    """P_ee over a device energy tensor (gna_oscprob_eval; precision="mixed":
    gna_oscprob_eval_ex with GNA_PREC_MIXED, the NEXT-3 1e-6 tier)."""
    import torch
    L = load()
    n = E.numel()
    flags = _prec_flags(precision)
    if out is None:
        out = torch.empty_like(E)
    p = OscParams.of(params)._c()
    if flags:
        _check(L.gna_oscprob_eval_ex(ctypes.byref(p), float(L_km), _dev(E, "E"), n,
                                     _dev(out, "out", n), flags, _stream(stream)),
               "gna_oscprob_eval_ex")
    else:
        _check(L.gna_oscprob_eval(ctypes.byref(p), float(L_km), _dev(E, "E"), n,
                                  _dev(out, "out", n), _stream(stream)), "gna_oscprob_eval")
    return out


def oscprob_eval_ab(alpha: int, beta: int, params, L_km: float, E, out=None, stream=None):
    """P(nu_alpha -> nu_beta) over a device energy tensor (gna_oscprob_eval_ab, NEXT-2);
    alpha, beta in {0: e, 1: mu, 2: tau}."""
    import torch
    L = load()
    n = E.numel()
    if out is None:
        out = torch.empty_like(E)
    p = OscParams.of(params)._c()
    _check(L.gna_oscprob_eval_ab(int(alpha), int(beta), ctypes.byref(p), float(L_km),
                                 _dev(E, "E"), n, _dev(out, "out", n), _stream(stream)),
           "gna_oscprob_eval_ab")
    return out


def gl_integrate_ab(alpha: int, beta: int, params, L_km: float, edges, order: int, out=None,
                    stream=None):
    """Per-bin GL integrals of P(nu_alpha -> nu_beta) (gna_gl_integrate_ab, NEXT-2)."""
    import torch
    L = load()
    nbins = edges.numel() - 1
    if out is None:
        out = torch.empty(max(nbins, 0), dtype=torch.float64, device=edges.device)
    p = OscParams.of(params)._c()
    _check(L.gna_gl_integrate_ab(int(alpha), int(beta), ctypes.byref(p), float(L_km),
                                 _dev(edges, "edges"), nbins, int(order),
                                 _dev(out, "out", max(nbins, 0)), _stream(stream)),
           "gna_gl_integrate_ab")
    return out


def gl_integrate(params, L_km: float, edges, order: int, out=None, stream=None,
                 precision: str = "fp64"):
    """Per-bin Gauss-Legendre integrals of P_ee (gna_gl_integrate; precision="mixed":
    gna_gl_integrate_ex with GNA_PREC_MIXED, the NEXT-3 1e-5 tier)."""
    import torch
    L = load()
    nbins = edges.numel() - 1
    flags = _prec_flags(precision)
    if out is None:
        out = torch.empty(max(nbins, 0), dtype=torch.float64, device=edges.device)
    p = OscParams.of(params)._c()
    args = (ctypes.byref(p), float(L_km), _dev(edges, "edges"), nbins, int(order),
            _dev(out, "out", max(nbins, 0)))
    if flags:
        _check(L.gna_gl_integrate_ex(*args, flags, _stream(stream)), "gna_gl_integrate_ex")
    else:
        _check(L.gna_gl_integrate(*args, _stream(stream)), "gna_gl_integrate")
    return out


def oscprob_batch_workspace_size(npoints: int, nbase: int, nbins: int, order: int) -> int:
    return int(load().gna_oscprob_batch_workspace_size(int(npoints), int(nbase), int(nbins),
                                                       int(order)))


def oscprob_batch(points: dict, L_km, omega, edges, order: int, data=None, spectra=True,
                  chi2=None, workspace=None, stream=None, precision: str = "fp64",
                  tables_valid: bool = False):
    """Batched spectra and chi^2 (gna_oscprob_batch).

    points: dict of CUDA float64 tensors theta12, theta13, dm2_21, dm2_31 [P].
    spectra: True to allocate, a [P, nbins] tensor to fill, or None/False.
    chi2: computed when `data` is given (a [P] tensor may be passed to fill).
    precision: "fp64" (gna_oscprob_batch, the 1e-11 tier) or "mixed" (gna_oscprob_batch_ex
    with GNA_PREC_MIXED: fp64 phases, fp32 polynomial and term sums; 1e-5 tier).
    tables_valid: the caller's `workspace` already holds the node tables of an earlier call
    with the same edges and order (GNA_WS_TABLES_VALID; bitwise the same result).
    Returns (spectra or None, chi2 or None).
    """
    _prec_flags(precision)
    import torch
    L = load()
    P = points["theta12"].numel()
    nbins = edges.numel() - 1
    dev = edges.device
    if spectra is True:
        spectra = torch.empty((P, max(nbins, 0)), dtype=torch.float64, device=dev)
    elif spectra is False:
        spectra = None
    if data is not None and chi2 is None:
        chi2 = torch.empty(P, dtype=torch.float64, device=dev)
    Lh, om = _baselines(L_km, omega)
    if tables_valid and workspace is None:
        raise ValueError("tables_valid needs the workspace that holds the tables")
    b = _CBatch(*(_dev(points[k], k, P) for k in ("theta12", "theta13", "dm2_21", "dm2_31")), P)
    if workspace is None:
        workspace = _scratch(oscprob_batch_workspace_size(P, Lh.size, nbins, order), dev, stream)
    args = (ctypes.byref(b), Lh.ctypes.data, om.ctypes.data, Lh.size, _dev(edges, "edges"),
            nbins, int(order), _dev(spectra, "spectra", P * nbins) if spectra is not None else None,
            _dev(data, "data", nbins) if data is not None else None,
            _dev(chi2, "chi2", P) if chi2 is not None else None,
            _dev(workspace, "workspace"), workspace.numel() * 8)
    flags = _prec_flags(precision) | (GNA_WS_TABLES_VALID if tables_valid else 0)
    if flags:
        _check(L.gna_oscprob_batch_ex(*args, flags, _stream(stream)), "gna_oscprob_batch_ex")
    else:
        _check(L.gna_oscprob_batch(*args, _stream(stream)), "gna_oscprob_batch")
    return spectra, chi2


def oscprob_scan_workspace_size(nmix: int, nmass: int, nbins: int) -> int:
    return int(load().gna_oscprob_scan_workspace_size(int(nmix), int(nmass), int(nbins)))


def oscprob_scan(grid: dict, L_km, omega, edges, order: int, data=None, spectra=True, chi2=None,
                 workspace=None, stream=None):
    """Separable grid scan (gna_oscprob_scan): mixing points theta12/theta13 [nmix] x
    mass points dm2_21/dm2_31 [nmass] (CUDA float64 tensors).  Returns (spectra
    [nmass, nmix, nbins] or None, chi2 [nmass, nmix] or None)."""
    import torch
    L = load()
    nmix = grid["theta12"].numel()
    nmass = grid["dm2_21"].numel()
    nbins = edges.numel() - 1
    dev = edges.device
    if spectra is True:
        spectra = torch.empty((nmass, nmix, max(nbins, 0)), dtype=torch.float64, device=dev)
    elif spectra is False:
        spectra = None
    if data is not None and chi2 is None:
        chi2 = torch.empty((nmass, nmix), dtype=torch.float64, device=dev)
    Lh, om = _baselines(L_km, omega)
    if workspace is None:  # 32-byte aligned
        workspace = _scratch(oscprob_scan_workspace_size(nmix, nmass, nbins), dev, stream, 32)
    g = _CScan(_dev(grid["theta12"], "theta12", nmix), _dev(grid["theta13"], "theta13", nmix),
               nmix, _dev(grid["dm2_21"], "dm2_21", nmass), _dev(grid["dm2_31"], "dm2_31", nmass),
               nmass)
    _check(L.gna_oscprob_scan(
        ctypes.byref(g), Lh.ctypes.data, om.ctypes.data, Lh.size, _dev(edges, "edges"), nbins,
        int(order),
        _dev(spectra, "spectra", nmass * nmix * nbins) if spectra is not None else None,
        _dev(data, "data", nbins) if data is not None else None,
        _dev(chi2, "chi2", nmass * nmix) if chi2 is not None else None,
        workspace.data_ptr(), workspace.numel() * 8, _stream(stream)), "gna_oscprob_scan")
    return spectra, chi2


def oscprob_batch_ex(points: dict, L_km, omega, edges, order: int, spectra_ptr: int | None,
                     chi2_ptr: int | None, flags: int, data=None, workspace=None, stream=None):
    """gna_oscprob_batch_ex (NEXT-4): outputs are raw addresses of a remote window (peer or
    NVLS multicast VA from symmetric memory, see dist.FusedGather); inputs are local tensors."""
    import torch
    L = load()
    P = points["theta12"].numel()
    nbins = edges.numel() - 1
    Lh, om = _baselines(L_km, omega)
    if workspace is None:
        workspace = _scratch(oscprob_batch_workspace_size(P, Lh.size, nbins, order),
                             edges.device, stream)
    b = _CBatch(*(_dev(points[k], k, P) for k in ("theta12", "theta13", "dm2_21", "dm2_31")), P)
    _check(L.gna_oscprob_batch_ex(
        ctypes.byref(b), Lh.ctypes.data, om.ctypes.data, Lh.size, _dev(edges, "edges"), nbins,
        int(order), spectra_ptr, _dev(data, "data", nbins) if data is not None else None,
        chi2_ptr, _dev(workspace, "workspace"), workspace.numel() * 8, int(flags),
        _stream(stream)), "gna_oscprob_batch_ex")


def fit_workspace_size(nbase: int, nbins: int, order: int) -> int:
    return int(load().gna_fit_workspace_size(int(nbase), int(nbins), int(order)))


def fit_pattern_search(state, L_km, omega, edges, order: int, data, niter: int, hist=None,
                       workspace=None, stream=None):
    """On-GPU chi^2 pattern search (gna_fit_pattern_search).  state: CUDA float64 [8] =
    centre (theta12, theta13, dm2_21, dm2_31) + steps, updated in place; returns hist."""
    import torch
    L = load()
    nbins = edges.numel() - 1
    Lh, om = _baselines(L_km, omega)
    if hist is None and niter > 0:
        hist = torch.empty(niter, dtype=torch.float64, device=edges.device)
    if workspace is None:
        workspace = _scratch(fit_workspace_size(Lh.size, nbins, order), edges.device, stream)
    _check(L.gna_fit_pattern_search(
        Lh.ctypes.data, om.ctypes.data, Lh.size, _dev(edges, "edges"), nbins, int(order),
        _dev(data, "data", nbins), _dev(state, "state", 8), int(niter),
        _dev(hist, "hist", niter) if hist is not None else None, _dev(workspace, "workspace"),
        workspace.numel() * 8, _stream(stream)), "gna_fit_pattern_search")
    return hist


# ---------------------------------------------------------------- host-buffer entry points
def oscprob_eval_host(params, L_km: float, E: np.ndarray, out: np.ndarray | None = None,
                      chunk: int = 0, stream=None) -> np.ndarray:
    """P_ee over a HOST energy array: chunked H2D / kernel / D2H on three streams (copies overlap kernels)."""
    L = load()
    E = _host(E, "E")
    if out is None:
        out = np.empty_like(E)
    _host(out, "out", E.size, writable=True)
    p = OscParams.of(params)._c()
    _check(L.gna_oscprob_eval_host(ctypes.byref(p), float(L_km), E.ctypes.data, E.size,
                                   out.ctypes.data, int(chunk), _stream(stream)),
           "gna_oscprob_eval_host")
    return out


def gl_integrate_host(params, L_km: float, edges: np.ndarray, order: int,
                      out: np.ndarray | None = None, chunk: int = 0, stream=None) -> np.ndarray:
    """Per-bin GL integrals over HOST bin edges (chunked H2D / kernel / D2H)."""
    L = load()
    edges = _host(edges, "edges")
    nbins = edges.size - 1
    if out is None:
        out = np.empty(max(nbins, 0))
    _host(out, "out", max(nbins, 0), writable=True)
    p = OscParams.of(params)._c()
    _check(L.gna_gl_integrate_host(ctypes.byref(p), float(L_km), edges.ctypes.data, nbins,
                                   int(order), out.ctypes.data, int(chunk), _stream(stream)),
           "gna_gl_integrate_host")
    return out


def oscprob_batch_host(points: dict, L_km, omega, edges: np.ndarray, order: int,
                       data: np.ndarray | None = None, spectra=True, chi2=None,
                       chunk_points: int = 0, stream=None):
    """Batch over HOST arrays (end-to-end path); returns (spectra, chi2) numpy arrays."""
    L = load()
    P = _host(points["theta12"], "theta12").size
    pts = {k: _host(points[k], k, P) for k in ("theta12", "theta13", "dm2_21", "dm2_31")}
    edges = _host(edges, "edges")
    nbins = edges.size - 1
    if spectra is True:
        spectra = np.empty((P, max(nbins, 0)))
    elif spectra is False:
        spectra = None
    if spectra is not None:
        _host(spectra, "spectra", P * nbins, writable=True)
    if data is not None:
        _host(data, "data", nbins)
        if chi2 is None:
            chi2 = np.empty(P)
    if chi2 is not None:
        _host(chi2, "chi2", P, writable=True)
    b = _CBatch(*(pts[k].ctypes.data for k in ("theta12", "theta13", "dm2_21", "dm2_31")), P)
    Lh, om = _baselines(L_km, omega)
    _check(L.gna_oscprob_batch_host(
        ctypes.byref(b), Lh.ctypes.data, om.ctypes.data, Lh.size, edges.ctypes.data, nbins,
        int(order), spectra.ctypes.data if spectra is not None else None,
        data.ctypes.data if data is not None else None,
        chi2.ctypes.data if chi2 is not None else None, int(chunk_points), _stream(stream)),
        "gna_oscprob_batch_host")
    return spectra, chi2


# ---------------------------------------------------------------- misc
def gl_rule(order: int):
    t = np.zeros(max(order, 1))
    w = np.zeros(max(order, 1))
    _check(load().gna_gl_rule(int(order), t.ctypes.data, w.ctypes.data), "gna_gl_rule")
    return t, w


def release() -> None:
    load().gna_release()


def launch_count() -> int:
    return int(load().gna_launch_count())


def abi_version() -> int:
    return int(load().gna_abi_version())


def sin2_poly_degree() -> int:
    """Degree of the sin^2 minimax compiled into the library (gna_sin2_poly_degree)."""
    return int(load().gna_sin2_poly_degree())

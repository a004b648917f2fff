"""CPU oracle for the GNA hot path (arXiv:1804.07682) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product package
``paper_1804_07682_b200`` never imports it, and the two share no code.

This module is argument marshalling (ctypes) around ``oracle.c``; every line of
arithmetic lives in ``oracle.c`` and cites the passage it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# -O2, no FMA contraction, no fast-math (R9); OpenMP only over
# independent outputs, so results are bitwise identical for any thread count.
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        d, i, i64, p = ctypes.c_double, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
        L.oracle_pmns.argtypes = [d, d, d, d, i, p]
        L.oracle_pmns.restype = None
        L.oracle_phase.argtypes = [d, d, d]
        L.oracle_phase.restype = d
        L.oracle_prob.argtypes = [i, i, p, d, d, d, d]
        L.oracle_prob.restype = d
        L.oracle_prob_amplitude.argtypes = [i, i, p, d, d, d, d]
        L.oracle_prob_amplitude.restype = d
        L.oracle_two_flavor.argtypes = [d, d, d, d]
        L.oracle_two_flavor.restype = d
        L.oracle_prob_array.argtypes = [i, i, d, d, d, d, i, d, d, d, p, i64, p, i]
        L.oracle_prob_array.restype = i
        L.oracle_gauleg.argtypes = [i, p, p]
        L.oracle_gauleg.restype = i
        L.oracle_gl_integrate.argtypes = [d, d, d, d, i, d, d, d, p, i64, i, p, i]
        L.oracle_gl_integrate.restype = i
        L.oracle_batch.argtypes = [p, p, p, p, i64, d, d, i, p, p, i, p, i64, i, p, p, p, i]
        L.oracle_gl_integrate_ab.argtypes = [i, i, d, d, d, d, i, d, d, d, p, i64, i, p, i]
        L.oracle_gl_integrate_ab.restype = i
        L.oracle_batch.restype = i
        L.oracle_max_threads.argtypes = []
        L.oracle_max_threads.restype = i
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# Canonical oscillation parameters of SPEC S:280 (theta23 and delta do not
# change P_ee but the general formula takes them).
CANONICAL = dict(theta12=0.5838, theta13=0.1496, theta23=0.7854, delta_cp=0.0,
                 dm2_21=7.53e-5, dm2_31=2.52e-3, antineutrino=0)


def pmns(theta12, theta13, theta23, delta_cp, antineutrino=0) -> np.ndarray:
    V = np.zeros(9, dtype=np.complex128)
    lib().oracle_pmns(theta12, theta13, theta23, delta_cp, int(antineutrino), _ptr(V))
    return V.reshape(3, 3)


def phase(dm2, L_km, E_MeV) -> float:
    return lib().oracle_phase(dm2, L_km, E_MeV)


def prob(alpha, beta, params: dict, L_km, E_MeV, amplitude=False) -> float:
    V = np.ascontiguousarray(pmns(params["theta12"], params["theta13"], params["theta23"],
                                  params["delta_cp"], params.get("antineutrino", 0)).ravel())
    f = lib().oracle_prob_amplitude if amplitude else lib().oracle_prob
    return f(alpha, beta, _ptr(V), params["dm2_21"], params["dm2_31"], L_km, E_MeV)


def two_flavor(theta, dm2, L_km, E_MeV) -> float:
    return lib().oracle_two_flavor(theta, dm2, L_km, E_MeV)


def prob_array(params: dict, L_km, E, alpha=0, beta=0, nthreads=1) -> np.ndarray:
    E = _f64(E)
    P = np.empty_like(E)
    lib().oracle_prob_array(alpha, beta, params["theta12"], params["theta13"],
                            params["theta23"], params["delta_cp"],
                            int(params.get("antineutrino", 0)), params["dm2_21"],
                            params["dm2_31"], L_km, _ptr(E), E.size, _ptr(P), nthreads)
    return P


def gauleg(n: int):
    t = np.zeros(n)
    w = np.zeros(n)
    if lib().oracle_gauleg(n, _ptr(t), _ptr(w)) != 0:
        raise ValueError("order must be >= 1")
    return t, w


def gl_integrate(params: dict, L_km, edges, order: int, nthreads=1) -> np.ndarray:
    edges = _f64(edges)
    nbins = edges.size - 1
    bins = np.empty(max(nbins, 0))
    rc = lib().oracle_gl_integrate(params["theta12"], params["theta13"], params["theta23"],
                                   params["delta_cp"], int(params.get("antineutrino", 0)),
                                   params["dm2_21"], params["dm2_31"], L_km, _ptr(edges),
                                   nbins, order, _ptr(bins), nthreads)
    if rc < 0:
        raise ValueError("bad order")
    return bins


def gl_integrate_ab(alpha, beta, params: dict, L_km, edges, order: int, nthreads=1) -> np.ndarray:
    edges = _f64(edges)
    nbins = edges.size - 1
    bins = np.empty(max(nbins, 0))
    rc = lib().oracle_gl_integrate_ab(alpha, beta, params["theta12"], params["theta13"],
                                      params["theta23"], params["delta_cp"],
                                      int(params.get("antineutrino", 0)), params["dm2_21"],
                                      params["dm2_31"], L_km, _ptr(edges), nbins, order,
                                      _ptr(bins), nthreads)
    if rc < 0:
        raise ValueError("bad order")
    return bins


def batch(points: dict, L_km, omega, edges, order: int, data=None, want_spectra=True,
          theta23=CANONICAL["theta23"], delta_cp=0.0, antineutrino=0, nthreads=1):
    """Returns (spectra [P][nbins] or None, chi2 [P] or None)."""
    th12, th13 = _f64(points["theta12"]), _f64(points["theta13"])
    d21, d31 = _f64(points["dm2_21"]), _f64(points["dm2_31"])
    P = th12.size
    L_km, omega, edges = _f64(L_km), _f64(omega), _f64(edges)
    nbins = edges.size - 1
    spectra = np.empty((P, nbins)) if want_spectra else None
    chi2 = np.empty(P) if data is not None else None
    data_a = _f64(data) if data is not None else None
    rc = lib().oracle_batch(_ptr(th12), _ptr(th13), _ptr(d21), _ptr(d31), P, theta23, delta_cp,
                            int(antineutrino), _ptr(L_km), _ptr(omega), L_km.size, _ptr(edges),
                            nbins, order, _ptr(spectra) if spectra is not None else None,
                            _ptr(data_a) if data_a is not None else None,
                            _ptr(chi2) if chi2 is not None else None, nthreads)
    if rc < 0:
        raise ValueError("bad order")
    return spectra, chi2


def max_threads() -> int:
    return lib().oracle_max_threads()

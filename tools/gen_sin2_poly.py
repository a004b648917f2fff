"""Generate the minimax polynomial used by the CUDA path for sin^2.

The kernel writes Delta = (pi/2) * y, y = q + f with q = rint(y), |f| <= 1/2, so
    sin^2(Delta) = 1/2 + (-1)^q * v(f),   v(f) = -cos(pi f) / 2,
and v is an even function: v(f) = V(u), u = f^2 in [0, 1/4].  This script fits V
by Chebyshev interpolation in 60-digit mpmath, refines it with a few Remez-style
exchange steps (relative to absolute error), rounds the coefficients to fp64 and
checks the fp64-FMA Horner evaluation (emulated exactly with Fractions) against
mpmath on a dense grid.  Output: paper_1804_07682_b200/csrc/sin2_poly.h.

This is a constant generator of the CUDA path only; the oracle uses libm sin
and never sees these numbers.
"""
from __future__ import annotations

import os
import sys
from fractions import Fraction

import mpmath as mp

mp.mp.dps = 60
A, B = mp.mpf(0), mp.mpf(1) / 4


def V(u):
    return -mp.cos(mp.pi * mp.sqrt(u)) / 2


def cheb_fit(deg):
    # interpolate at Chebyshev nodes of the first kind, return monomial coeffs c0..cdeg
    n = deg + 1
    xs = [(A + B) / 2 + (B - A) / 2 * mp.cos(mp.pi * (2 * k + 1) / (2 * n)) for k in range(n)]
    M = mp.matrix([[x ** j for j in range(n)] for x in xs])
    y = mp.matrix([V(x) for x in xs])
    c = mp.lu_solve(M, y)
    return [c[j] for j in range(n)]


def remez(deg, iters=8):
    n = deg + 2
    # start from Chebyshev extrema
    xs = [(A + B) / 2 - (B - A) / 2 * mp.cos(mp.pi * k / (n - 1)) for k in range(n)]
    c = None
    for _ in range(iters):
        M = mp.matrix([[x ** j for j in range(deg + 1)] + [(-1) ** k] for k, x in enumerate(xs)])
        y = mp.matrix([V(x) for x in xs])
        sol = mp.lu_solve(M, y)
        c = [sol[j] for j in range(deg + 1)]
        # locate extrema of the error on a fine grid, one per alternation interval
        grid = [A + (B - A) * mp.mpf(i) / 4000 for i in range(4001)]
        err = [sum(c[j] * g ** j for j in range(deg + 1)) - V(g) for g in grid]
        # pick sign-alternating extrema
        ext = []
        i = 0
        while i < len(grid):
            s = mp.sign(err[i]) or 1
            j = i
            best = i
            while j < len(grid) and (mp.sign(err[j]) or 1) == s:
                if abs(err[j]) > abs(err[best]):
                    best = j
                j += 1
            ext.append(best)
            i = j
        if len(ext) < n:
            break
        # keep the n largest consecutive set
        while len(ext) > n:
            if abs(err[ext[0]]) < abs(err[ext[-1]]):
                ext.pop(0)
            else:
                ext.pop()
        xs = [grid[k] for k in ext]
    return c


def remez_c0(deg, iters=12):
    """Minimax of V on [0, 1/4] with the constant term pinned to V(0) = -1/2 exactly, so that
    sin^2 is exactly 0 at every even multiple of pi/2 (f = 0) and the error vanishes like u
    near there.  Unknowns c1..cdeg and the levelled error E; alternation points in (0, 1/4]."""
    n = deg + 1
    xs = [B * (1 - mp.cos(mp.pi * (k + 1) / n)) / 2 for k in range(n)]
    c = None
    for _ in range(iters):
        M = mp.matrix([[x ** j for j in range(1, deg + 1)] + [(-1) ** k] for k, x in enumerate(xs)])
        y = mp.matrix([V(x) + mp.mpf(1) / 2 for x in xs])
        sol = mp.lu_solve(M, y)
        c = [mp.mpf(-1) / 2] + [sol[j] for j in range(deg)]
        grid = [A + (B - A) * mp.mpf(i) / 4000 for i in range(1, 4001)]
        err = [sum(c[j] * g ** j for j in range(deg + 1)) - V(g) for g in grid]
        ext = []
        i = 0
        while i < len(grid):
            s = mp.sign(err[i]) or 1
            j = i
            best = i
            while j < len(grid) and (mp.sign(err[j]) or 1) == s:
                if abs(err[j]) > abs(err[best]):
                    best = j
                j += 1
            ext.append(best)
            i = j
        if len(ext) < n:
            break
        while len(ext) > n:
            if abs(err[ext[0]]) < abs(err[ext[-1]]):
                ext.pop(0)
            else:
                ext.pop()
        xs = [grid[k] for k in ext]
    return c


def fma(a: float, b: float, c: float) -> float:
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def horner_fp64(cf, u):
    p = cf[-1]
    for c in reversed(cf[:-1]):
        p = fma(p, u, c)
    return p


def r32(x) -> float:
    """Nearest fp32 value (as a Python float) of a float or Fraction."""
    import numpy as np
    return float(np.float32(float(x)))


def max_err_fp32(cf, npts=4000):
    """Mixed tier (NEXT-3): the reduced argument rounded to fp32, u = f*f and the Horner chain
    in fp32 FMA (error against the current V at the rounded argument)."""
    worst = 0.0
    for i in range(npts + 1):
        f = r32(0.5 * i / npts)
        u = r32(Fraction(f) * Fraction(f))
        p = cf[-1]
        for c in reversed(cf[:-1]):
            p = r32(Fraction(p) * Fraction(u) + Fraction(c))
        worst = max(worst, abs(float(p - V(mp.mpf(f) ** 2))))
    return worst


def max_err(cf, npts=4000):
    worst = 0.0
    for i in range(npts + 1):
        f = 0.5 * i / npts
        u = f * f  # fp64 product, as the kernel forms it
        got = horner_fp64(cf, u)
        ref = V(mp.mpf(u))
        worst = max(worst, abs(float(got - ref)))
    return worst


def S(u):
    """sin(pi sqrt(u)) / sqrt(u): sin(pi f) = f * S(f^2) (appearance channels, NEXT-2)."""
    if u == 0:
        return mp.pi
    r = mp.sqrt(u)
    return mp.sin(mp.pi * r) / r


def main_sinpi(out):
    global V
    V0 = V
    V = S
    try:
        best = None
        for deg in (7, 8, 9):
            c = remez(deg)
            cf = [float(x) for x in c]
            worst = 0.0
            for i in range(4001):
                f = 0.5 * i / 4000
                u = f * f
                got = f * horner_fp64(cf, u)
                ref = mp.sin(mp.pi * mp.mpf(f))
                worst = max(worst, abs(float(got - ref)))
            print("sinpi degree", deg, "max |err|:", worst, file=sys.stderr)
            if best is None or worst < best[1]:
                best = (deg, worst, cf)
        deg, err, cf = best
        lines = ["// GENERATED by tools/gen_sin2_poly.py — do not edit.",
                 "// S(u) = sin(pi*sqrt(u))/sqrt(u) on u in [0, 1/4], minimax degree %d; sin(pi f) = f S(f^2)." % deg,
                 "// Max abs error of f * (fp64 FMA Horner) vs 60-digit mpmath on 4001 points: %.3e." % err,
                 "#pragma once", "#define GNA_SINPI_POLY_DEG %d" % deg]
        for j, x in enumerate(cf):
            lines.append("#define GNA_SINPI_C%d (%s)  /* %.17g */" % (j, x.hex(), x))
        open(out, "w").write("\n".join(lines) + "\n")
    finally:
        V = V0


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--sinpi":
        return main_sinpi(os.path.join(os.path.dirname(__file__), "..", "paper_1804_07682_b200",
                                       "csrc", "sinpi_poly.h"))
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(
        os.path.dirname(__file__), "..", "paper_1804_07682_b200", "csrc", "sin2_poly.h")
    results = {}
    for deg in (7, 8, 9):
        c = remez(deg)
        cf = [float(x) for x in c]
        results[deg] = (cf, max_err(cf))
        print("degree", deg, "max |err| fp64 Horner:", results[deg][1], file=sys.stderr)
    cf, err = results[8]
    cf7 = [float(x) for x in remez_c0(7)]
    err7 = max_err(cf7)
    print("degree 7 (c0 = -1/2 pinned) max |err| fp64 Horner:", err7, file=sys.stderr)
    # full-period form for the packed (FFMA2) mixed kernels: reducing y modulo 2,
    # y = 2m + 2h with |h| <= 1/2, gives (-1)^q v(f) = -cos(pi y)/2 = -cos(2 pi h)/2 with no
    # sign flip; W(u) = -cos(2 pi sqrt u)/2 on u = h^2 in [0, 1/4], degree 6 in fp32
    global V
    V0 = V
    V = lambda u: -mp.cos(2 * mp.pi * mp.sqrt(u)) / 2  # noqa: E731
    try:
        cfw = [r32(x) for x in remez_c0(6)]
        errw = max_err_fp32(cfw)
    finally:
        V = V0
    print("fp32 full-period degree 6 max |err| fp32 Horner:", errw, file=sys.stderr)
    lines = [
        "// GENERATED by tools/gen_sin2_poly.py — do not edit.",
        "// v(u) = -cos(pi*sqrt(u))/2 on u in [0, 1/4] (u = f^2, |f| <= 1/2), minimax.",
        "// sin^2((pi/2)(q+f)) = 1/2 + (-1)^q v(f^2).  Max abs error of the fp64 FMA Horner",
        "// evaluation vs 60-digit mpmath on 4001 points: degree 8 %.3e, degree 7 %.3e." % (err, err7),
        "// Degree 7 (GNA_SIN2_D7_*) has c0 = -1/2 pinned: sin^2 = 0 exactly at f = 0.",
        "#pragma once",
        "#define GNA_SIN2_ERR8 %.3e" % err,
        "#define GNA_SIN2_ERR7 %.3e" % err7,
    ]
    for j, x in enumerate(cf):
        lines.append("#define GNA_SIN2_C%d (%s)  /* %.17g */" % (j, x.hex(), x))
    for j, x in enumerate(cf7):
        lines.append("#define GNA_SIN2_D7_C%d (%s)  /* %.17g */" % (j, x.hex(), x))
    lines.append("// Mixed tier (NEXT-3): W(u) = -cos(2 pi sqrt(u))/2 on u = h^2 in [0, 1/4] (y reduced")
    lines.append("// modulo 2, no sign flip), fp32 degree 6, c0 = -1/2 pinned; max abs error with h rounded")
    lines.append("// to fp32 and an fp32 FMA Horner chain: %.3e." % errw)
    lines.append("#define GNA_COS2F_ERR %.3e" % errw)
    for j, x in enumerate(cfw):
        lines.append("#define GNA_COS2F_C%d ((float)%s)  /* %.9g */" % (j, x.hex(), x))
    open(out, "w").write("\n".join(lines) + "\n")
    print("wrote", out, "err", err, file=sys.stderr)


if __name__ == "__main__":
    main()

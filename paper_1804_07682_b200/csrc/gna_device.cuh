// gna_device.cuh — device building blocks of the fused P_ee / GL path (sm_100a, fp64).
//
// Arithmetic per sin^2 term, all on the FP64 pipe:
//   t  = kq * invE + 1.5*2^52   DFMA  (rounds y = kq/E to the nearest integer q, in t's low word)
//   q  = t - 1.5*2^52           DADD  (exact)
//   f  = kq * invE - q          DFMA  (one rounding of the exact product minus q, |f| <= 1/2)
//   u  = f * f                  DMUL
//   v  = V(u)                   8 DFMA (minimax, |err| <= 1.1e-16; sin2_poly.h)
//   acc += w * ((-1)^q v)       DFMA  (sign of v flipped with 2 integer ops on its hi word)
// = 13 FP64-pipe instructions, exploiting sin^2((pi/2)(q+f)) = 1/2 + (-1)^q v(f),
// v(f) = -cos(pi f)/2, so that sum_ij w_ij sin^2 = sum w_ij / 2 + sum w_ij (-1)^q v.
// The reduction is exact for |y| < 2^51; the only error beyond the polynomial's is
// the rounding of kq and invE (R7, R9).
#pragma once
#include <cstdint>

#include "sin2_poly.h"

namespace gna {

constexpr double kRoundMagic = 6755399441055744.0;  // 1.5 * 2^52

// minimax coefficients in the constant bank: DFMA takes c[][] operands directly,
// so the Horner chain needs no register or uniform-register moves.
__constant__ double c_sin2[9] = {GNA_SIN2_C0, GNA_SIN2_C1, GNA_SIN2_C2, GNA_SIN2_C3, GNA_SIN2_C4,
                                 GNA_SIN2_C5, GNA_SIN2_C6, GNA_SIN2_C7, GNA_SIN2_C8};

// (-1)^q * V(f^2) for y = kq * invE = q + f  (y itself is never rounded separately)
__device__ __forceinline__ double sin2c(double kq, double invE) {
  const double t = fma(kq, invE, kRoundMagic);
  const double q = t - kRoundMagic;
  const double f = fma(kq, invE, -q);
  const double u = f * f;
  double p = fma(u, c_sin2[8], c_sin2[7]);
  p = fma(p, u, c_sin2[6]);
  p = fma(p, u, c_sin2[5]);
  p = fma(p, u, c_sin2[4]);
  p = fma(p, u, c_sin2[3]);
  p = fma(p, u, c_sin2[2]);
  p = fma(p, u, c_sin2[1]);
  p = fma(p, u, c_sin2[0]);
  // parity of q = bit 0 of t's low word -> sign bit of p
  const int odd = __double2loint(t) << 31;
  return __hiloint2double(__double2hiint(p) ^ odd, __double2loint(p));
}

// 1/x for x > 0 (normal): MUFU.RCP64H seed (measured 20 bits, tools/probe_rcp.cu,
// profiles/r01_probe_rcp.jsonl) + one cubically convergent step r(1 + e + e^2),
// e = 1 - x r: 3 DFMA, max error 1 ulp (2.2e-16 relative) over 1-10 MeV.
__device__ __forceinline__ double rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// Per-call coefficients of one (parameter point, baseline).
struct PeeCoef {
  double kq[3];  // phase slopes in units of pi/2 per (1/MeV): y_ij = kq_ij / E
  double w[3];   // mixing weights w21, w31, w32 (optionally times a baseline weight)
  double c0;     // 1 - (w21 + w31 + w32)/2 (times the same baseline weight)
};

__device__ __forceinline__ double pee_inv(const PeeCoef& c, double invE) {
  double acc = c.w[0] * sin2c(c.kq[0], invE);
  acc = fma(c.w[1], sin2c(c.kq[1], invE), acc);
  acc = fma(c.w[2], sin2c(c.kq[2], invE), acc);
  return c.c0 - acc;
}

}  // namespace gna

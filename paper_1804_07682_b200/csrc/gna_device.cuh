// gna_device.cuh — device building blocks of the fused P_ee / GL path (sm_100a, fp64).
//
// Arithmetic per sin^2 term, all on the FP64 pipe:
//   y  = kq * invE          DMUL   (kq = 1.26693268*dm2*L*1000 * 2/pi, so Delta = (pi/2) y)
//   t  = y + 1.5*2^52       DADD   (rounds y to the nearest integer q, held in t's low word)
//   q  = t - 1.5*2^52       DADD   (exact)
//   f  = y - q              DADD   (exact, |f| <= 1/2)
//   u  = f * f              DMUL
//   v  = V(u)               8 DFMA (minimax, |err| <= 1.1e-16; sin2_poly.h)
//   acc += (-1)^q w v       DFMA   (sign applied to w with 2 integer ops on the hi word)
// = 14 FP64-pipe instructions, exploiting sin^2((pi/2)(q+f)) = 1/2 + (-1)^q v(f),
// v(f) = -cos(pi f)/2.  The reduction is exact for |y| < 2^51, so the only error
// beyond the polynomial's is the rounding of y itself (R7, R9).
#pragma once
#include <cstdint>

#include "sin2_poly.h"

namespace gna {

constexpr double kRoundMagic = 6755399441055744.0;  // 1.5 * 2^52

// (-1)^q * v(f) * w  accumulated into acc, for y = q + f.
__device__ __forceinline__ double sin2c_acc(double y, double w, double acc) {
  const double t = y + kRoundMagic;
  const double q = t - kRoundMagic;
  const double f = y - q;
  const double u = f * f;
  double p = GNA_SIN2_C8;
  p = fma(p, u, GNA_SIN2_C7);
  p = fma(p, u, GNA_SIN2_C6);
  p = fma(p, u, GNA_SIN2_C5);
  p = fma(p, u, GNA_SIN2_C4);
  p = fma(p, u, GNA_SIN2_C3);
  p = fma(p, u, GNA_SIN2_C2);
  p = fma(p, u, GNA_SIN2_C1);
  p = fma(p, u, GNA_SIN2_C0);
  // parity of q = bit 0 of t's low word; flip the sign of w when q is odd
  const uint32_t odd = static_cast<uint32_t>(__double2loint(t)) << 31;
  const double ws = __hiloint2double(__double2hiint(w) ^ static_cast<int>(odd), __double2loint(w));
  return fma(ws, p, acc);
}

// 1/x for x > 0 (normal): MUFU.RCP64H seed + two Newton steps (4 DFMA).
__device__ __forceinline__ double rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  return r;
}

// Per-call coefficients of one (parameter point, baseline).
struct PeeCoef {
  double kq[3];  // phase slopes in units of pi/2 per (1/MeV): y_ij = kq_ij / E
  double w[3];   // mixing weights w21, w31, w32 (optionally times a baseline weight)
  double c0;     // 1 - (w21 + w31 + w32)/2 (times the same baseline weight)
};

__device__ __forceinline__ double pee_inv(const PeeCoef& c, double invE) {
  double acc = sin2c_acc(c.kq[0] * invE, c.w[0], 0.0);
  acc = sin2c_acc(c.kq[1] * invE, c.w[1], acc);
  acc = sin2c_acc(c.kq[2] * invE, c.w[2], acc);
  return c.c0 - acc;
}

}  // namespace gna

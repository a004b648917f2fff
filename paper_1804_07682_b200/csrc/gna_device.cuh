// gna_device.cuh — device building blocks of the fused P_ee / GL path (sm_100a, fp64).
//
// Arithmetic per sin^2 term, all on the FP64 pipe:
//   t  = kq * invE + 1.5*2^52   DFMA  (rounds y = kq/E to the nearest integer q, in t's low word)
//   q  = t - 1.5*2^52           DADD  (exact)
//   f  = kq * invE - q          DFMA  (one rounding of the exact product minus q, |f| <= 1/2)
//   u  = f * f                  DMUL
//   v  = V(u)                   7 DFMA (minimax of degree 7 in u, |err| <= 1.11e-15, V(0) = -1/2
//                               exactly; sin2_poly.h.  GNA_SIN2_DEG 8: 8 DFMA, |err| <= 1.1e-16)
//   acc += w * ((-1)^q v)       DFMA  (sign of v flipped by one IMAD on its hi word, flip_by_parity)
// = 12 (13) FP64-pipe instructions, exploiting sin^2((pi/2)(q+f)) = 1/2 + (-1)^q v(f),
// v(f) = -cos(pi f)/2, so that sum_ij w_ij sin^2 = sum w_ij / 2 + sum w_ij (-1)^q v.
// The reduction is exact for |y| < 2^51, i.e. |Delta| < pi * 2^50 (t then lies in
// [2^52, 2^53), where the ulp is 1 and t's low mantissa bit is the parity of q); the only
// error beyond the polynomial's is the rounding of kq and invE (R7, R9, R10).
#pragma once
#include <cstdint>

#include "sin2_poly.h"
#include "sinpi_poly.h"

namespace gna {

constexpr double kRoundMagic = 6755399441055744.0;  // 1.5 * 2^52

// Degree of the v(u) minimax (sin2_poly.h): 8 (|err| 1.1e-16) or 7 (|err| 1.1e-15, c0 = -1/2
// pinned; one DFMA fewer per term).  DESIGN.md §6.1 and R7.
#ifndef GNA_SIN2_DEG
#define GNA_SIN2_DEG 7
#endif

// minimax coefficients in the constant bank: DFMA takes c[][] operands directly,
// so the Horner chain needs no register or uniform-register moves.
#if GNA_SIN2_DEG == 7
__constant__ double c_sin2[8] = {GNA_SIN2_D7_C0, GNA_SIN2_D7_C1, GNA_SIN2_D7_C2, GNA_SIN2_D7_C3,
                                 GNA_SIN2_D7_C4, GNA_SIN2_D7_C5, GNA_SIN2_D7_C6, GNA_SIN2_D7_C7};
#elif GNA_SIN2_DEG == 8
__constant__ double c_sin2[9] = {GNA_SIN2_C0, GNA_SIN2_C1, GNA_SIN2_C2, GNA_SIN2_C3, GNA_SIN2_C4,
                                 GNA_SIN2_C5, GNA_SIN2_C6, GNA_SIN2_C7, GNA_SIN2_C8};
#else
#error "GNA_SIN2_DEG must be 7 or 8"
#endif
// sin(pi f) = f S(f^2), S minimax of degree 8 (sinpi_poly.h; appearance channels, NEXT-2)
__constant__ double c_sinpi[9] = {GNA_SINPI_C0, GNA_SINPI_C1, GNA_SINPI_C2, GNA_SINPI_C3,
                                  GNA_SINPI_C4, GNA_SINPI_C5, GNA_SINPI_C6, GNA_SINPI_C7,
                                  GNA_SINPI_C8};

// v(u) = -cos(pi sqrt(u)) / 2 by Horner on the constant bank
__device__ __forceinline__ double sin2_poly(double u) {
#if GNA_SIN2_DEG == 8
  double p = fma(u, c_sin2[8], c_sin2[7]);
  p = fma(p, u, c_sin2[6]);
#else
  double p = fma(u, c_sin2[7], c_sin2[6]);
#endif
  p = fma(p, u, c_sin2[5]);
  p = fma(p, u, c_sin2[4]);
  p = fma(p, u, c_sin2[3]);
  p = fma(p, u, c_sin2[2]);
  p = fma(p, u, c_sin2[1]);
  return fma(p, u, c_sin2[0]);
}

// (-1)^q p, the parity of q being bit 0 of t's low word: hi(p) + lo(t) * 2^31 (mod 2^32) adds
// 2^31 to p's high word — toggles its sign bit and nothing else — exactly when q is odd.  One
// IMAD instead of a shift and an XOR (GNA_SIGN_IMAD; the same bits either way).
#ifndef GNA_SIGN_IMAD
#define GNA_SIGN_IMAD 1
#endif
__device__ __forceinline__ double flip_by_parity(double p, double t) {
#if GNA_SIGN_IMAD
  unsigned hi;
  asm("mad.lo.u32 %0, %1, 0x80000000, %2;"
      : "=r"(hi)
      : "r"((unsigned)__double2loint(t)), "r"((unsigned)__double2hiint(p)));
  return __hiloint2double((int)hi, __double2loint(p));
#else
  const int odd = __double2loint(t) << 31;
  return __hiloint2double(__double2hiint(p) ^ odd, __double2loint(p));
#endif
}

// (-1)^q * V(f^2) for y = kq * invE = q + f  (y itself is never rounded separately)
__device__ __forceinline__ double sin2c(double kq, double invE) {
  const double t = fma(kq, invE, kRoundMagic);
  const double q = t - kRoundMagic;
  const double f = fma(kq, invE, -q);
  const double u = f * f;
  // parity of q = bit 0 of t's low word -> sign bit of p
  return flip_by_parity(sin2_poly(u), t);
}

// Mixed tier.  The phase y = kq/E and its reduction stay
// fp64 — they need it: y reaches ~1e3 and fp32 would lose the phase (ulp(550) = 6e-5).  The
// reduction is taken modulo 2, y = 2m + 2h with m = rint(y/2), |h| <= 1/2 (three FP64
// instructions on kqh = kq/2, staged exactly), so that (-1)^q v(f) = -cos(pi y)/2 =
// -cos(2 pi h)/2 = W(h^2) needs no sign flip; h is rounded to fp32 (F2F) and W is a degree-6
// fp32 minimax (|err| 1.3e-7, sin2_poly.h).  Two chains are evaluated per instruction with
// sm_100a's packed FP32 FMA (FFMA2): per pair of terms 2 x (3 FP64 + F2F) + FMUL2 + 6 FFMA2
// + the accumulating FFMA2 = 16 instructions, 8 per term (the fp64 path: 12).
__constant__ float c_cos2f[7] = {GNA_COS2F_C0, GNA_COS2F_C1, GNA_COS2F_C2, GNA_COS2F_C3,
                                 GNA_COS2F_C4, GNA_COS2F_C5, GNA_COS2F_C6};

typedef unsigned long long f32x2;  // two fp32 lanes in one 64-bit register pair

__device__ __forceinline__ f32x2 f2_pack(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float f2_lo(f32x2 v) { return __int_as_float((int)(unsigned)v); }
__device__ __forceinline__ float f2_hi(f32x2 v) { return __int_as_float((int)(unsigned)(v >> 32)); }
__device__ __forceinline__ f32x2 f2_fma(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f32x2 f2_mul(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// h = y/2 - rint(y/2) for y/2 = kqh * invE, rounded to fp32 (F2F, XU pipe)
__device__ __forceinline__ float mixed_h1(double kqh, double invE) {
  const double t = fma(kqh, invE, kRoundMagic);
  const double m = t - kRoundMagic;
  return __double2float_rn(fma(kqh, invE, -m));
}

// W(h^2) = -cos(2 pi h)/2 for one chain
__device__ __forceinline__ float cos2_w(float h) {
  const float u = h * h;
  float p = fmaf(u, c_cos2f[6], c_cos2f[5]);
  p = fmaf(p, u, c_cos2f[4]);
  p = fmaf(p, u, c_cos2f[3]);
  p = fmaf(p, u, c_cos2f[2]);
  p = fmaf(p, u, c_cos2f[1]);
  return fmaf(p, u, c_cos2f[0]);
}

__device__ __forceinline__ f32x2 mixed_h2(double kqa, double iEa, double kqb, double iEb) {
  return f2_pack(mixed_h1(kqa, iEa), mixed_h1(kqb, iEb));
}

// the same for two chains packed in one register pair
__device__ __forceinline__ f32x2 cos2_w2(f32x2 h2) {
  const f32x2 u = f2_mul(h2, h2);
  f32x2 p = f2_fma(u, f2_pack(c_cos2f[6], c_cos2f[6]), f2_pack(c_cos2f[5], c_cos2f[5]));
  p = f2_fma(p, u, f2_pack(c_cos2f[4], c_cos2f[4]));
  p = f2_fma(p, u, f2_pack(c_cos2f[3], c_cos2f[3]));
  p = f2_fma(p, u, f2_pack(c_cos2f[2], c_cos2f[2]));
  p = f2_fma(p, u, f2_pack(c_cos2f[1], c_cos2f[1]));
  return f2_fma(p, u, f2_pack(c_cos2f[0], c_cos2f[0]));
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

// General term of P:633-636 for one pair: with y = kq/E = q + f,
//   a sin^2(Delta) + b sin(2 Delta) = a/2 + (-1)^q (a v(f) + b sin(pi f)),
// a = -4 Re X_ij, b = 2 Im X_ij.  Shares the reduction with sin2c; 24 FP64 instructions.
__device__ __forceinline__ double sin2_sin_c(double kq, double invE, double a, double b) {
  const double t = fma(kq, invE, kRoundMagic);
  const double q = t - kRoundMagic;
  const double f = fma(kq, invE, -q);
  const double u = f * f;
#if GNA_SIN2_DEG == 8
  double p = fma(u, c_sin2[8], c_sin2[7]);
  p = fma(p, u, c_sin2[6]);
#else
  double p = fma(u, c_sin2[7], c_sin2[6]);
#endif
  double r = fma(u, c_sinpi[8], c_sinpi[7]);
  r = fma(r, u, c_sinpi[6]);
  p = fma(p, u, c_sin2[5]);
  r = fma(r, u, c_sinpi[5]);
  p = fma(p, u, c_sin2[4]);
  r = fma(r, u, c_sinpi[4]);
  p = fma(p, u, c_sin2[3]);
  r = fma(r, u, c_sinpi[3]);
  p = fma(p, u, c_sin2[2]);
  r = fma(r, u, c_sinpi[2]);
  p = fma(p, u, c_sin2[1]);
  r = fma(r, u, c_sinpi[1]);
  p = fma(p, u, c_sin2[0]);
  r = fma(r, u, c_sinpi[0]);
  return flip_by_parity(fma(b * f, r, a * p), t);
}

// Per-call coefficients of one (parameter point, baseline): P_ee (the hot path).
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

// NEXT-3 mixed tier of the single-point paths (eval, GL): phase slopes halved (modulo-2
// reduction, see mixed_h), weights in fp32, the term sum of one energy in fp32.
struct PeeMixCoef {
  double kqh[3];  // kq / 2
  float w[3];
  double c0;
};

__device__ __forceinline__ double prob_inv(const PeeMixCoef& c, double invE) {
  float acc = c.w[0] * cos2_w(mixed_h1(c.kqh[0], invE));
  acc = fmaf(c.w[1], cos2_w(mixed_h1(c.kqh[1], invE)), acc);
  acc = fmaf(c.w[2], cos2_w(mixed_h1(c.kqh[2], invE)), acc);
  return c.c0 - (double)acc;
}

// two energies per packed FFMA2 chain (the elementwise kernels' double2 pairs)
__device__ __forceinline__ double2 prob_pair(const PeeMixCoef& c, double iE0, double iE1) {
  f32x2 acc = 0ull;
#pragma unroll
  for (int j = 0; j < 3; ++j)
    acc = f2_fma(f2_pack(c.w[j], c.w[j]), cos2_w2(mixed_h2(c.kqh[j], iE0, c.kqh[j], iE1)), acc);
  return make_double2(c.c0 - (double)f2_lo(acc), c.c0 - (double)f2_hi(acc));
}

// Any channel alpha -> beta (NEXT-2): P = c0 + sum_ij (-1)^q (a_ij v + b_ij sin(pi f)),
// c0 = delta_ab + sum_ij a_ij / 2.
struct PabCoef {
  double kq[3];
  double a[3];  // -4 Re X_ij
  double b[3];  //  2 Im X_ij
  double c0;
};

__device__ __forceinline__ double pab_inv(const PabCoef& c, double invE) {
  double acc = sin2_sin_c(c.kq[0], invE, c.a[0], c.b[0]);
  acc += sin2_sin_c(c.kq[1], invE, c.a[1], c.b[1]);
  acc += sin2_sin_c(c.kq[2], invE, c.a[2], c.b[2]);
  return c.c0 + acc;
}

__device__ __forceinline__ double prob_inv(const PeeCoef& c, double invE) { return pee_inv(c, invE); }
__device__ __forceinline__ double prob_inv(const PabCoef& c, double invE) { return pab_inv(c, invE); }

// a pair of energies (the elementwise kernels' double2): two independent evaluations
template <class Coef>
__device__ __forceinline__ double2 prob_pair(const Coef& c, double iE0, double iE1) {
  return make_double2(prob_inv(c, iE0), prob_inv(c, iE1));
}

// H energies at once, term-major: every coefficient feeds H independent chains (ILP = H).
// Round 1 kept the term loop rolled (one basic block per term, the coefficient picked with
// selects) because ptxas serialised the H chains of the unrolled form in the lane-pair kernel;
// with the one-IMAD sign flip the unrolled form (GNA_PROB_TERM_UNROLL 3) is faster for the
// thread-per-bin and warp-split GL kernels — the rolled loop spent ~14 instructions per term on
// loop control and coefficient selects (10^5 bins x GL10 back to back 4.01 -> 3.94 us, 10^6
// bins 27.8 -> 26.2 us; elementwise unchanged; profiles/variants_r02/term_unroll/).
#ifndef GNA_PROB_TERM_UNROLL
#define GNA_PROB_TERM_UNROLL 3
#endif
constexpr int kProbTermUnroll = GNA_PROB_TERM_UNROLL;
template <int H>
__device__ __forceinline__ void prob_inv_n(const PeeCoef& c, const double (&iE)[H], double (&P)[H]) {
  double acc[H];
#pragma unroll
  for (int i = 0; i < H; ++i) acc[i] = 0.0;
#pragma unroll kProbTermUnroll
  for (int j = 0; j < 3; ++j) {
    const double kq = j == 0 ? c.kq[0] : (j == 1 ? c.kq[1] : c.kq[2]);
    const double w = j == 0 ? c.w[0] : (j == 1 ? c.w[1] : c.w[2]);
#pragma unroll
    for (int i = 0; i < H; ++i) acc[i] = fma(w, sin2c(kq, iE[i]), acc[i]);
  }
#pragma unroll
  for (int i = 0; i < H; ++i) P[i] = c.c0 - acc[i];
}

template <int H>
__device__ __forceinline__ void prob_inv_n(const PeeMixCoef& c, const double (&iE)[H],
                                           double (&P)[H]) {
  constexpr int NP = H / 2;
  f32x2 acc2[NP > 0 ? NP : 1];
  float acc1 = 0.0f;
#pragma unroll
  for (int k = 0; k < NP; ++k) acc2[k] = 0ull;
#pragma unroll 1
  for (int j = 0; j < 3; ++j) {
    const double kqh = j == 0 ? c.kqh[0] : (j == 1 ? c.kqh[1] : c.kqh[2]);
    const float w = j == 0 ? c.w[0] : (j == 1 ? c.w[1] : c.w[2]);
#pragma unroll
    for (int k = 0; k < NP; ++k)
      acc2[k] = f2_fma(f2_pack(w, w), cos2_w2(mixed_h2(kqh, iE[2 * k], kqh, iE[2 * k + 1])), acc2[k]);
    if constexpr (H & 1) acc1 = fmaf(w, cos2_w(mixed_h1(kqh, iE[H - 1])), acc1);
  }
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    P[2 * k] = c.c0 - (double)f2_lo(acc2[k]);
    P[2 * k + 1] = c.c0 - (double)f2_hi(acc2[k]);
  }
  if constexpr (H & 1) P[H - 1] = c.c0 - (double)acc1;
}

template <int H>
__device__ __forceinline__ void prob_inv_n(const PabCoef& c, const double (&iE)[H], double (&P)[H]) {
  double acc[H];
#pragma unroll
  for (int i = 0; i < H; ++i) acc[i] = 0.0;
#pragma unroll 1
  for (int j = 0; j < 3; ++j) {
    const double kq = j == 0 ? c.kq[0] : (j == 1 ? c.kq[1] : c.kq[2]);
    const double a = j == 0 ? c.a[0] : (j == 1 ? c.a[1] : c.a[2]);
    const double b = j == 0 ? c.b[0] : (j == 1 ? c.b[1] : c.b[2]);
#pragma unroll
    for (int i = 0; i < H; ++i) acc[i] += sin2_sin_c(kq, iE[i], a, b);
  }
#pragma unroll
  for (int i = 0; i < H; ++i) P[i] = c.c0 + acc[i];
}

}  // namespace gna

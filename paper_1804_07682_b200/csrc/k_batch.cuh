// k_batch.cuh — (a1)-(a5) batch kernels: setup, per-point / points-inner main pass, chi2 reduce
// Part of libgna_b200.so: included once, from gna_b200.cu (single translation unit).
#pragma once
#include "gna_common.cuh"

namespace {

struct BatchSetupArgs {
  double L[GNA_MAX_NBASE];
  double omega[GNA_MAX_NBASE];
  double omega_sum;  // sum_b omega_b (left to right)
  int nbase;
  int order;
  int64_t nbins;
  int64_t npoints;
  int tables;  // 1: also build the per-node tables invE / hw (0: the caller's are valid)
};

// Workspace layout of the batch path (all offsets 16-byte aligned), see
// gna_oscprob_batch_workspace_size:  invE [order][nbins], hw [order][nbins] first (their
// offsets do not depend on the number of points, so a caller that splits its points over
// several calls can keep one set of node tables: GNA_WS_TABLES_VALID), then coef
// [P][nbase][3] double2 (kq, omega_b w_ij), c0 [P], partial [P][wpp][S] (S = 1 except for
// k_oscprob_batch_pt sub-tiles; sized for S = kPtSubMax).
struct BatchWs {
  double2* coef;
  double* c0;
  double* invE;
  double* hw;
  double* partial;
};

// chi2 partials per (point, 32-bin tile); the points-across-lanes kernel may split a tile
// into up to kPtSubMax sub-tiles, each with its own partial (k_oscprob_batch_pt)
constexpr int kPtSubMax = 4;

size_t batch_tables_bytes(int64_t nbins, int order) {
  return 2 * align16((size_t)order * nbins * sizeof(double));
}

size_t batch_ws_bytes(int64_t P, int nbase, int64_t nbins, int order, bool chi2) {
  size_t b = batch_tables_bytes(nbins, order);
  b += align16((size_t)P * nbase * 3 * sizeof(double2));
  b += align16((size_t)P * sizeof(double));
  if (chi2) b += align16((size_t)P * warps_per_point(nbins) * kPtSubMax * sizeof(double));
  return b;
}

BatchWs batch_ws_carve(void* base, int64_t P, int nbase, int64_t nbins, int order, bool chi2) {
  char* c = (char*)base;
  BatchWs w;
  w.invE = (double*)c;
  c += align16((size_t)order * nbins * sizeof(double));
  w.hw = (double*)c;
  c += align16((size_t)order * nbins * sizeof(double));
  w.coef = (double2*)c;
  c += align16((size_t)P * nbase * 3 * sizeof(double2));
  w.c0 = (double*)c;
  c += align16((size_t)P * sizeof(double));
  w.partial = chi2 ? (double*)c : nullptr;
  return w;
}

// (a1)+(a2) setup: per-(point, baseline) coefficients and the per-node tables
//   invE[i][k] = 1 / (c_k + h_k t_i),  hw[i][k] = h_k w_i   (shared by every point).
__global__ void __launch_bounds__(256) k_batch_setup(BatchSetupArgs a,
                                                     const double* __restrict__ th12,
                                                     const double* __restrict__ th13,
                                                     const double* __restrict__ d21,
                                                     const double* __restrict__ d31,
                                                     const double* __restrict__ edges, BatchWs w) {
  pdl_launch_dependents();  // the main pass may be scheduled now; it waits in pdl_wait()
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n1 = a.npoints * a.nbase;
  const int64_t n2 = a.tables ? (int64_t)a.order * a.nbins : 0;
  if (t < n1) {
    const int64_t p = t / a.nbase;
    const int b = (int)(t - p * a.nbase);
    double s12, c12, s13, c13, w21, w31, w32;
    sincos(th12[p], &s12, &c12);
    sincos(th13[p], &s13, &c13);
    mixing_weights(s12, c12, s13, c13, &w21, &w31, &w32);
    const double m21 = d21[p], m31 = d31[p];
    const double m32 = m31 - m21;
    const double L = a.L[b], om = a.omega[b];
    double2* c = w.coef + t * 3;
    c[0] = make_double2(phase_slope(m21, L), om * w21);
    c[1] = make_double2(phase_slope(m31, L), om * w31);
    c[2] = make_double2(phase_slope(m32, L), om * w32);
    if (b == 0) w.c0[p] = a.omega_sum * (1.0 - 0.5 * ((w21 + w31) + w32));
  } else if (t < n1 + n2) {
    const int64_t idx = t - n1;
    const int i = (int)(idx / a.nbins);
    const int64_t k = idx - (int64_t)i * a.nbins;
    const int off = GNA_GL_OFF(a.order);
    const double e0 = edges[k], e1 = edges[k + 1];
    const double ctr = 0.5 * (e0 + e1);
    const double h = 0.5 * (e1 - e0);
    w.invE[idx] = 1.0 / fma(h, c_gl_t[off + i], ctr);
    w.hw[idx] = h * c_gl_w[off + i];
  }
}

#define GNA_PRAGMA(x) _Pragma(#x)
#define GNA_UNROLL(n) GNA_PRAGMA(unroll n)
#ifndef GNA_BATCH_PI
#define GNA_BATCH_PI 1
#endif
#ifndef GNA_BATCH_PI_Q2
#define GNA_BATCH_PI_Q2 1
#endif
#ifndef GNA_BATCH_PI_MAX_TERMS
#define GNA_BATCH_PI_MAX_TERMS 6
#endif
#ifndef GNA_BATCH_PPW_WORK_BIG
#define GNA_BATCH_PPW_WORK_BIG 480
#endif
#ifndef GNA_BATCH_PPW_MIN_WAVES
#define GNA_BATCH_PPW_MIN_WAVES 32
#endif
#ifndef GNA_BATCH_PPW_WORK
#define GNA_BATCH_PPW_WORK 480
#endif
#ifndef GNA_BATCH_JUNROLL
#define GNA_BATCH_JUNROLL 2
#endif
#ifndef GNA_BATCH_MINB
#define GNA_BATCH_MINB 1
#endif
#ifndef GNA_BATCH_N10_FP64
#define GNA_BATCH_N10_FP64 1  // fp64: 10 nodes per coefficient load when the order allows (cfg5 +0.3 %)
#endif
#ifndef GNA_MIXED_N10
#define GNA_MIXED_N10 1
#endif
#ifndef GNA_MIXED_JUNROLL
#define GNA_MIXED_JUNROLL 1
#endif
#ifndef GNA_BATCH_PI_NT
#define GNA_BATCH_PI_NT 1
#endif
#ifndef GNA_BATCH_PI_MINB
#define GNA_BATCH_PI_MINB GNA_BATCH_MINB
#endif

// N GL nodes of one bin at a time: each (kq, omega*w) coefficient load from
// shared memory feeds N independent sin^2 chains (ILP across nodes).
template <int N, bool kMixed = false>
__device__ __forceinline__ void batch_nodes(const double2* __restrict__ sc, int nterm,
                                            const double* __restrict__ invE,
                                            const double* __restrict__ hw, int64_t nbins, int i,
                                            double& W, double& A) {
  double iE[N], a[N];
#pragma unroll
  for (int n = 0; n < N; ++n) {
    iE[n] = invE[(int64_t)(i + n) * nbins];
    a[n] = 0.0;
  }
  if constexpr (kMixed) {
    // NEXT-3 mixed tier: y/2 reduced in fp64, W(h^2) and the per-node term sum in fp32, two
    // nodes per packed FFMA2 (an odd last node runs scalar); one conversion to fp64 per node.
    // Rows are staged as (kq/2, omega w as fp32 in both halves of .y).
    constexpr int NP = N / 2;
    gna::f32x2 acc2[NP > 0 ? NP : 1];
    float acc1 = 0.0f;
#pragma unroll
    for (int k = 0; k < NP; ++k) acc2[k] = 0ull;
    GNA_UNROLL(GNA_MIXED_JUNROLL)
    for (int j = 0; j < nterm; ++j) {
      const double2 cw = sc[j];
      const gna::f32x2 w2 = (gna::f32x2)__double_as_longlong(cw.y);
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const gna::f32x2 h2 = gna::mixed_h2(cw.x, iE[2 * k], cw.x, iE[2 * k + 1]);
        acc2[k] = gna::f2_fma(w2, gna::cos2_w2(h2), acc2[k]);
      }
      if constexpr (N & 1)
        acc1 = fmaf(__int_as_float(__double2loint(cw.y)), gna::cos2_w(gna::mixed_h1(cw.x, iE[N - 1])),
                    acc1);
    }
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      a[2 * k] = (double)gna::f2_lo(acc2[k]);
      a[2 * k + 1] = (double)gna::f2_hi(acc2[k]);
    }
    if constexpr (N & 1) a[N - 1] = (double)acc1;
  } else {
  GNA_UNROLL(GNA_BATCH_JUNROLL)
  for (int j = 0; j < nterm; ++j) {
    const double2 cw = sc[j];
#pragma unroll
    for (int n = 0; n < N; ++n) a[n] = fma(cw.y, gna::sin2c(cw.x, iE[n]), a[n]);
  }
  }
#pragma unroll
  for (int n = 0; n < N; ++n) {
    const double h = hw[(int64_t)(i + n) * nbins];
    W += h;
    A = fma(h, a[n], A);
  }
}

// remainder of r < N nodes, compile-time group size
template <int N, bool kMixed = false>
__device__ __forceinline__ void batch_tail(int r, const double2* __restrict__ sc, int nterm,
                                           const double* __restrict__ invE,
                                           const double* __restrict__ hw, int64_t nbins, int i,
                                           double& W, double& A) {
  if constexpr (N > 1) {
    if (r == N - 1) {
      batch_nodes<N - 1, kMixed>(sc, nterm, invE, hw, nbins, i, W, A);
      return;
    }
    batch_tail<N - 1, kMixed>(r, sc, nterm, invE, hw, nbins, i, W, A);
  }
}

// coefficient row entry as staged in shared memory: fp64 (kq, omega w), or for the mixed
// tier kq/2 in fp64 and omega w as fp32 in both 32-bit halves of .y (a packed pair)
template <bool kMixed>
__device__ __forceinline__ double2 stage_coef(double2 c) {
  if constexpr (kMixed) {
    const int wb = __float_as_int(__double2float_rn(c.y));
    c = make_double2(0.5 * c.x, __hiloint2double(wb, wb));  // kq/2 is exact
  }
  return c;
}

// Output stores of the batch epilogue (NEXT-4, fused gather):
//   kOutLocal     plain stores to this GPU's memory;
//   kOutPeer      plain stores to a peer GPU's memory mapped into this address space
//                 (symmetric memory over NVLink), system-scope fence at the end;
//   kOutMulticast multimem.st to an NVLink-SHARP (NVLS) multicast address: one store
//                 lands in every participating GPU's buffer (all-gather in the epilogue).
enum { kOutLocal = 0, kOutPeer = 1, kOutMulticast = 2 };

template <int kOut>
__device__ __forceinline__ void out_store(double* p, double v) {
  if constexpr (kOut == kOutMulticast)
    asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
  else
    *p = v;
}

// (a3)+(a4)+(a5) main pass.  Block = (point p, kWarps x 32 bins); every warp is
// independent (no block barrier): it copies its point's coefficient row into a
// warp-private smem slice, then each lane integrates one bin, N GL nodes at a time
// (N divides the order when possible, so no group runs with reduced ILP).
template <int kWarps, int N, int kOut, bool kMixed = false>
__global__ void __launch_bounds__(kWarps * 32, GNA_BATCH_MINB) k_oscprob_batch(
    int nterm, int order, int64_t nbins, int64_t npoints, int64_t bpp, int ppw, BatchWs w,
    double* __restrict__ spectra, const double* __restrict__ data) {
  extern __shared__ double2 s_coef[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pg = blockIdx.x / bpp;                          // point group
  const int64_t wt = (blockIdx.x - pg * bpp) * kWarps + warp;  // warp tile within a point
  const int64_t k0 = wt * 32;
  if (k0 >= nbins) return;  // whole warp
  double2* sc = s_coef + warp * nterm;
  const int64_t k = k0 + lane;
  const bool active = k < nbins;
  const int64_t kk = active ? k : nbins - 1;
  const double* __restrict__ invE = w.invE + kk;
  const double* __restrict__ hw = w.hw + kk;
  const double D = (data && active) ? data[k] : 1.0;
  const double iD = 1.0 / D;  // once per lane: chi2 terms d^2 / D as d^2 * iD (no per-point divide)
  const int64_t wpp = warps_per_point_dev(nbins);
  pdl_wait();  // the setup kernel's tables are complete and visible
  // ppw points per warp, same bins: the node tables stay in L1 across points
  const int64_t pend = min(npoints, (pg + 1) * (int64_t)ppw);
  for (int64_t p = pg * (int64_t)ppw; p < pend; ++p) {
    const double2* __restrict__ gc = w.coef + p * nterm;
    __syncwarp();  // previous point's reads of sc are done
    for (int j = lane; j < nterm; j += 32) {
      sc[j] = stage_coef<kMixed>(gc[j]);
    }
    __syncwarp();
    // bin = sum_n h w_n (c0 - a_n) = c0 W - A,  W = sum_n h w_n,  A = sum_n h w_n a_n
    // (one FP64 op per node instead of two)
    double W = 0.0, A = 0.0;
    int i = 0;
    for (; i + N <= order; i += N) batch_nodes<N, kMixed>(sc, nterm, invE, hw, nbins, i, W, A);
    if (i < order) batch_tail<N, kMixed>(order - i, sc, nterm, invE, hw, nbins, i, W, A);
    const double s = fma(w.c0[p], W, -A);
    double x2 = 0.0;
    if (active) {
      if (spectra) out_store<kOut>(spectra + p * nbins + k, s);
      const double d = s - D;
      x2 = d * d * iD;
    }
    if (w.partial) {  // chi2 requested: fixed xor tree, deterministic
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x2 += __shfl_xor_sync(0xffffffffu, x2, o);
      if (lane == 0) w.partial[p * wpp + wt] = x2;
    }
  }
  if constexpr (kOut != kOutLocal) __threadfence_system();  // remote stores before completion
}

// Small-nbase variant (few terms per node, several points per warp, e.g. cfg4's
// single-baseline scan): the loops are interchanged so the node group is outer and the
// warp's points inner — 1/E and h*w of a node group are loaded once for all ppw points
// instead of once per point.  Per point the node sums are accumulated in the same order
// as k_oscprob_batch, so the results are bitwise identical.
constexpr int kMaxPPW = 16;

template <int N, int kOut, int NT = 0, bool kMixed = false>
__global__ void __launch_bounds__(32, GNA_BATCH_PI_MINB) k_oscprob_batch_pi(
    int nterm_rt, int order, int64_t nbins, int64_t npoints, int64_t bpp, int ppw, BatchWs w,
    double* __restrict__ spectra, const double* __restrict__ data) {
  extern __shared__ double2 s_dyn[];
  const int nterm = NT ? NT : nterm_rt;  // NT > 0: term loop unrolled at compile time
  double2* sc = s_dyn;                                          // [ppw][nterm]
  double* s_acc = reinterpret_cast<double*>(s_dyn + ppw * nterm);  // [ppw][32]
  double* s_c0 = s_acc + ppw * 32;                               // [ppw]
  const int lane = threadIdx.x & 31;
  const int64_t pg = blockIdx.x / bpp;
  const int64_t wt = blockIdx.x - pg * bpp;
  const int64_t k0 = wt * 32;
  if (k0 >= nbins) return;
  const int64_t p0 = pg * (int64_t)ppw;
  const int np = (int)min((int64_t)ppw, npoints - p0);
  pdl_wait();  // the setup kernel's tables are complete and visible
  for (int j = lane; j < np * nterm; j += 32) sc[j] = stage_coef<kMixed>(w.coef[p0 * nterm + j]);
  for (int j = lane; j < np; j += 32) s_c0[j] = w.c0[p0 + j];
  for (int q = 0; q < np; ++q) s_acc[q * 32 + lane] = 0.0;
  __syncwarp();
  const int64_t k = k0 + lane;
  const bool active = k < nbins;
  const int64_t kk = active ? k : nbins - 1;
  const double* __restrict__ invE = w.invE + kk;
  const double* __restrict__ hw = w.hw + kk;
  double W = 0.0;  // sum_n h w_n of this lane's bin, same order as k_oscprob_batch
  for (int i = 0; i < order; i += N) {
    const int nn = min(N, order - i);
    double iE[N], hv[N];
#pragma unroll
    for (int n = 0; n < N; ++n) {
      iE[n] = n < nn ? invE[(int64_t)(i + n) * nbins] : 1.0;
      hv[n] = n < nn ? hw[(int64_t)(i + n) * nbins] : 0.0;
    }
#pragma unroll
    for (int n = 0; n < N; ++n)
      if (n < nn) W += hv[n];
    int q = 0;
#if GNA_BATCH_PI_Q2
    // two points at a time: 2N independent sin^2 chains per coefficient step
    for (; q + 1 < np; q += 2) {
      const double2* __restrict__ cq = sc + q * nterm;
      const double2* __restrict__ cr = cq + nterm;
      double a[N], b[N];
      if constexpr (kMixed) {
        // the two points' chains of one node share a packed FFMA2 pair
        gna::f32x2 ab[N];
#pragma unroll
        for (int n = 0; n < N; ++n) ab[n] = 0ull;
        GNA_UNROLL((NT ? NT : 1))
        for (int j = 0; j < nterm; ++j) {
          const double2 cw = cq[j], cv = cr[j];
          const gna::f32x2 w2 = gna::f2_pack(__int_as_float(__double2loint(cw.y)),
                                             __int_as_float(__double2loint(cv.y)));
#pragma unroll
          for (int n = 0; n < N; ++n) {
            const gna::f32x2 h2 = gna::mixed_h2(cw.x, iE[n], cv.x, iE[n]);
            ab[n] = gna::f2_fma(w2, gna::cos2_w2(h2), ab[n]);
          }
        }
#pragma unroll
        for (int n = 0; n < N; ++n) {
          a[n] = (double)gna::f2_lo(ab[n]);
          b[n] = (double)gna::f2_hi(ab[n]);
        }
      } else {
#pragma unroll
        for (int n = 0; n < N; ++n) a[n] = b[n] = 0.0;
        GNA_UNROLL((NT ? NT : 1))
        for (int j = 0; j < nterm; ++j) {
          const double2 cw = cq[j], cv = cr[j];
#pragma unroll
          for (int n = 0; n < N; ++n) {
            a[n] = fma(cw.y, gna::sin2c(cw.x, iE[n]), a[n]);
            b[n] = fma(cv.y, gna::sin2c(cv.x, iE[n]), b[n]);
          }
        }
      }
      double sa = s_acc[q * 32 + lane], sb = s_acc[(q + 1) * 32 + lane];
#pragma unroll
      for (int n = 0; n < N; ++n)
        if (n < nn) {
          sa = fma(hv[n], a[n], sa);
          sb = fma(hv[n], b[n], sb);
        }
      s_acc[q * 32 + lane] = sa;
      s_acc[(q + 1) * 32 + lane] = sb;
    }
#endif
    for (; q < np; ++q) {
      const double2* __restrict__ cq = sc + q * nterm;
      double a[N];
      if constexpr (kMixed) {
        float af[N];
#pragma unroll
        for (int n = 0; n < N; ++n) af[n] = 0.0f;
        GNA_UNROLL((NT ? NT : 1))
        for (int j = 0; j < nterm; ++j) {
          const double2 cw = cq[j];
          const float wa = __int_as_float(__double2loint(cw.y));
#pragma unroll
          for (int n = 0; n < N; ++n) af[n] = fmaf(wa, gna::cos2_w(gna::mixed_h1(cw.x, iE[n])), af[n]);
        }
#pragma unroll
        for (int n = 0; n < N; ++n) a[n] = (double)af[n];
      } else {
#pragma unroll
        for (int n = 0; n < N; ++n) a[n] = 0.0;
        GNA_UNROLL((NT ? NT : 1))
        for (int j = 0; j < nterm; ++j) {
          const double2 cw = cq[j];
#pragma unroll
          for (int n = 0; n < N; ++n) a[n] = fma(cw.y, gna::sin2c(cw.x, iE[n]), a[n]);
        }
      }
      double sv = s_acc[q * 32 + lane];
#pragma unroll
      for (int n = 0; n < N; ++n)
        if (n < nn) sv = fma(hv[n], a[n], sv);
      s_acc[q * 32 + lane] = sv;
    }
  }
  const double D = (data && active) ? data[k] : 1.0;
  const double iD = 1.0 / D;  // once per lane: chi2 terms d^2 / D as d^2 * iD (no per-point divide)
  const int64_t wpp = warps_per_point_dev(nbins);
  for (int q = 0; q < np; ++q) {
    const int64_t p = p0 + q;
    const double sv = fma(s_c0[q], W, -s_acc[q * 32 + lane]);  // c0 W - A
    double x2 = 0.0;
    if (active) {
      if (spectra) out_store<kOut>(spectra + p * nbins + k, sv);
      const double d = sv - D;
      x2 = d * d * iD;
    }
    if (w.partial) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x2 += __shfl_xor_sync(0xffffffffu, x2, o);
      if (lane == 0) w.partial[p * wpp + wt] = x2;
    }
  }
  if constexpr (kOut != kOutLocal) __threadfence_system();
}

// Points-across-lanes variant (few terms, many points: cfg4's single-baseline scan).  Block
// = one warp = 32 consecutive points x one 32-bin tile.  Each lane keeps its point's NT
// coefficients in registers; the tile's node tables (1/E, h w), W, D and 1/D are staged once
// into shared memory and read back as warp-uniform broadcasts, bin by bin.  Compared with
// k_oscprob_batch_pi this drops the per-bin chi2 shuffle tree, the per-point shared-memory
// accumulators and (fp64) the empty bins of a ragged last tile (nbins = 1000 = 31.25
// tiles).  Results are bitwise identical to k_oscprob_batch: the same operations in the
// same order per (point, bin), and the tile's chi2 partial is the same xor-tree sum — the
// bins are visited in bit-reversed order, which turns the tree into consecutive pairs,
// summed online with a 5-level binary counter (pt_tile).  The mixed tier runs the same
// kernel with the NEXT-3 arithmetic of batch_nodes (node pairs on packed FFMA2s).
// §6.2 has the measurements behind each choice.
#ifndef GNA_BATCH_PT
#define GNA_BATCH_PT 1
#endif
#ifndef GNA_BATCH_PT_MINB
#define GNA_BATCH_PT_MINB 24  // <= 80 registers: 24 warps per SM
#endif
#ifndef GNA_BATCH_PT_SHARED21
#define GNA_BATCH_PT_SHARED21 1  // sin^2 Delta_21 once per warp when dm2_21 and L are shared
#endif
#ifndef GNA_BATCH_PT_SUB
#define GNA_BATCH_PT_SUB 2  // sub-tiles per 32-bin tile: 1, 2 or 4
#endif
#ifndef GNA_BATCH_PT_MUNROLL
#define GNA_BATCH_PT_MUNROLL 1
#endif
#ifndef GNA_BATCH_PT_MIXED
#define GNA_BATCH_PT_MIXED 1  // the mixed tier also takes the points-across-lanes kernel
#endif
#ifndef GNA_BATCH_PT_MIXED_MINB
#define GNA_BATCH_PT_MIXED_MINB 1  // 72 registers; a cap of 64 (32 warps per SM) lost 3 %
#endif
#ifndef GNA_BATCH_PT_MIXED_N10
#define GNA_BATCH_PT_MIXED_N10 1
#endif
#ifndef GNA_BATCH_PT_N10
#define GNA_BATCH_PT_N10 0
#endif
#ifndef GNA_BATCH_PT_MIN_POINTS
#define GNA_BATCH_PT_MIN_POINTS 256
#endif
// GNA_BATCH_PT_EH: a node's 1/E and h w staged as one double2 (one 16-byte shared load per node
// instead of two 8-byte ones); GNA_BATCH_PT_ORD10: order 10 compiled as a constant (node loops
// unrolled, shared-memory offsets immediate).  Same arithmetic, same bits.
#ifndef GNA_BATCH_PT_EH
#define GNA_BATCH_PT_EH 0
#endif
#ifndef GNA_BATCH_PT_ORD10
#define GNA_BATCH_PT_ORD10 1
#endif
// node i of the tile's bin b in the staged node table: (1/E, h w) pairs or two planes
__device__ __forceinline__ double pt_iE(const double* __restrict__ sE, int i, int b) {
  return GNA_BATCH_PT_EH ? sE[2 * (i * 32 + b)] : sE[i * 32 + b];
}

// kShared (fp64 only): every point of the warp has the same (2,1) phase slope per baseline
// (the same dm2_21 and L: a scan over theta13 / dm2_31 with the solar parameters fixed, as in
// cfg4), so sin^2 Delta_21 of each (bin, node) was evaluated once per warp into sS
// [baseline][node][32 bins] and is read instead of recomputed by all 32 point-lanes — the
// paper's "computed only once ... re-computed only if ... modified" inside the
// batch.  The value read is the one sin2c returns for that bin and node, so the bits are
// unchanged.
template <int N, int NT, bool kMixed, bool kShared = false>
__device__ __forceinline__ void pt_nodes(const double (&kq)[NT], const double (&cw)[NT],
                                         const float (&wf)[NT], const double* __restrict__ sE,
                                         const double* __restrict__ sH, int b, int i, double& A,
                                         const double* __restrict__ sS = nullptr, int order = 0) {
  double iE[N], a[N], hw[N];
#pragma unroll
  for (int n = 0; n < N; ++n) {
    if constexpr (GNA_BATCH_PT_EH) {
      const double2 eh = reinterpret_cast<const double2*>(sE)[(i + n) * 32 + b];
      iE[n] = eh.x;
      hw[n] = eh.y;
    } else {
      iE[n] = sE[(i + n) * 32 + b];
      hw[n] = 0.0;
    }
    a[n] = 0.0;
  }
  if constexpr (kMixed) {
    // NEXT-3 mixed tier, as in batch_nodes: kq[] holds kq/2, the node pairs share FFMA2s
    constexpr int NP = N / 2;
    gna::f32x2 acc2[NP > 0 ? NP : 1];
    float acc1 = 0.0f;
#pragma unroll
    for (int k = 0; k < NP; ++k) acc2[k] = 0ull;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const gna::f32x2 w2 = gna::f2_pack(wf[j], wf[j]);
      if (kShared && j % 3 == 0) {
        // shared W(h^2) of term 21 (fp32, [baseline][node][32 bins]): the packed evaluation is
        // element-wise, so a node's value does not depend on which node it is paired with
        const float* sW = reinterpret_cast<const float*>(sS) + ((j / 3) * order + i) * 32 + b;
#pragma unroll
        for (int k = 0; k < NP; ++k)
          acc2[k] = gna::f2_fma(w2, gna::f2_pack(sW[(2 * k) * 32], sW[(2 * k + 1) * 32]), acc2[k]);
        if constexpr (N & 1) acc1 = fmaf(wf[j], sW[(N - 1) * 32], acc1);
        continue;
      }
#pragma unroll
      for (int k = 0; k < NP; ++k)
        acc2[k] = gna::f2_fma(w2, gna::cos2_w2(gna::mixed_h2(kq[j], iE[2 * k], kq[j], iE[2 * k + 1])),
                              acc2[k]);
      if constexpr (N & 1) acc1 = fmaf(wf[j], gna::cos2_w(gna::mixed_h1(kq[j], iE[N - 1])), acc1);
    }
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      a[2 * k] = (double)gna::f2_lo(acc2[k]);
      a[2 * k + 1] = (double)gna::f2_hi(acc2[k]);
    }
    if constexpr (N & 1) a[N - 1] = (double)acc1;
  } else {
#pragma unroll
    for (int j = 0; j < NT; ++j) {
#pragma unroll
      for (int n = 0; n < N; ++n) {
        if (kShared && j % 3 == 0)
          a[n] = fma(cw[j], sS[((j / 3) * order + i + n) * 32 + b], a[n]);
        else
          a[n] = fma(cw[j], gna::sin2c(kq[j], iE[n]), a[n]);
      }
    }
  }
#pragma unroll
  for (int n = 0; n < N; ++n) A = fma(GNA_BATCH_PT_EH ? hw[n] : sH[(i + n) * 32 + b], a[n], A);
}

template <int N, int NT, bool kMixed, bool kShared = false>
__device__ __forceinline__ void pt_tail(int r, const double (&kq)[NT], const double (&cw)[NT],
                                        const float (&wf)[NT], const double* __restrict__ sE,
                                        const double* __restrict__ sH, int b, int i, double& A,
                                        const double* __restrict__ sS = nullptr, int order = 0) {
  if constexpr (N > 1) {
    if (r == N - 1) {
      pt_nodes<N - 1, NT, kMixed, kShared>(kq, cw, wf, sE, sH, b, i, A, sS, order);
      return;
    }
    pt_tail<N - 1, NT, kMixed, kShared>(r, kq, cw, wf, sE, sH, b, i, A, sS, order);
  }
}

// One (sub-)tile of k_oscprob_batch_pt: the bins of visits [sub 2^lv, (sub + 1) 2^lv) in
// bit-reversed order.  chi2 partial of the tile = xor tree over its 32 bins (k_oscprob_batch);
// visited in bit-reversed order the tree pairs consecutive visits: r[l] holds the pending
// left operand of level l, and after the sub-tile's last visit x2 is its subtree sum.
// kMode 0: a full tile (no bounds checks); 1: bins at or past nbins are skipped; 2: every
// bin is computed and those at or past nbins are dropped (x2 = 0 for them in both cases, as
// in k_oscprob_batch).
template <int kMode, int N, int NT, int kOut, bool kMixed, bool kShared = false, int kOrd = 0>
__device__ __forceinline__ double pt_tile(const double (&kq)[NT], const double (&cw)[NT],
                                          const float (&wf)[NT], double c0,
                                          const double* __restrict__ sE,
                                          const double* __restrict__ sH,
                                          const double* __restrict__ sW,
                                          const double* __restrict__ sD,
                                          const double* __restrict__ sID, int order, int64_t k0,
                                          int64_t nbins, double* __restrict__ out, bool pact,
                                          int sub, int lv, const double* __restrict__ sS = nullptr) {
  double r[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  double x2 = 0.0;
  const int m0 = sub << lv;
  GNA_UNROLL(GNA_BATCH_PT_MUNROLL)
  for (int m = m0; m < m0 + (1 << lv); ++m) {
    const int b = (int)(__brev((unsigned)m) >> 27);
    x2 = 0.0;
    if (kMode != 1 || k0 + b < nbins) {
      double A = 0.0;
      if constexpr (kOrd > 0) {
        static_assert(kOrd % N == 0, "kOrd");
#pragma unroll
        for (int i = 0; i < kOrd; i += N)
          pt_nodes<N, NT, kMixed, kShared>(kq, cw, wf, sE, sH, b, i, A, sS, kOrd);
      } else {
        int i = 0;
        for (; i + N <= order; i += N)
          pt_nodes<N, NT, kMixed, kShared>(kq, cw, wf, sE, sH, b, i, A, sS, order);
        if (i < order)
          pt_tail<N, NT, kMixed, kShared>(order - i, kq, cw, wf, sE, sH, b, i, A, sS, order);
      }
      const double s = fma(c0, sW[b], -A);
      if (kMode != 2 || k0 + b < nbins) {
        if (out && pact) out_store<kOut>(out + k0 + b, s);
        const double d = s - sD[b];
        x2 = d * d * sID[b];
      }
    }
#pragma unroll
    for (int l = 0; l < 5; ++l) {
      if (l >= lv) break;
      if (!(m & (1 << l))) {
        r[l] = x2;
        break;
      }
      x2 = r[l] + x2;
    }
  }
  return x2;
}

// A tile may be split into S = 2^(5 - lv) sub-tiles of 2^lv consecutive visits (more,
// shorter warps: a smaller last wave); each sub-tile's tree sum is a chi2 sub-partial and
// k_chi2_reduce<S> finishes the tree's top levels.
template <int N, int NT, int kOut, bool kMixed = false, int kOrd = 0>
__global__ void __launch_bounds__(32, kMixed ? GNA_BATCH_PT_MIXED_MINB : GNA_BATCH_PT_MINB)
    k_oscprob_batch_pt(
    int order, int64_t nbins, int64_t npoints, int64_t bpp, int lv, BatchWs w,
    double* __restrict__ spectra, const double* __restrict__ data) {
  extern __shared__ double s_pt[];
  if constexpr (kOrd > 0) order = kOrd;
  // [order][32] 1/E and h w of the tile's nodes: interleaved pairs (GNA_BATCH_PT_EH) or planes
  double* sE = s_pt;
  double* sH = GNA_BATCH_PT_EH ? sE + 1 : sE + order * 32;
  double* sW = s_pt + 2 * order * 32;  // [32] sum_i h w_i (same order as k_oscprob_batch)
  double* sD = sW + 32;             // [32] data
  double* sID = sD + 32;            // [32] 1 / data
  double* sS = sID + 32;            // [NT/3][order][32] shared sin^2 Delta_21 (fp64) or W (fp32)
  const int lane = threadIdx.x & 31;
  const int S = 32 >> lv;
  const int64_t tile = blockIdx.x / S;  // (point group, bin tile)
  const int sub = (int)(blockIdx.x - tile * S);
  const int64_t pg = tile / bpp;
  const int64_t wt = tile - pg * bpp;
  const int64_t k0 = wt * 32;
  const int64_t p = pg * 32 + lane;
  const bool pact = p < npoints;
  const int64_t pp = pact ? p : npoints - 1;
  {
    const int64_t k = k0 + lane;
    const bool kact = k < nbins;
    const int64_t kk = kact ? k : nbins - 1;
    const double D = (data && kact) ? data[k] : 1.0;
    sD[lane] = D;
    sID[lane] = 1.0 / D;
    pdl_wait();  // the setup kernel's tables are complete and visible
    double W = 0.0;
    for (int i = 0; i < order; ++i) {
      const double h = w.hw[(int64_t)i * nbins + kk];
      const double iEk = w.invE[(int64_t)i * nbins + kk];
      if constexpr (GNA_BATCH_PT_EH) {
        reinterpret_cast<double2*>(sE)[i * 32 + lane] = make_double2(iEk, h);
      } else {
        sE[i * 32 + lane] = iEk;
        sH[i * 32 + lane] = h;
      }
      W += h;
    }
    sW[lane] = W;
  }
  double kq[NT], cw[NT];
  float wf[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const double2 c = w.coef[pp * NT + j];
    kq[j] = kMixed ? 0.5 * c.x : c.x;  // mixed tier: kq/2 (exact), weights in fp32
    cw[j] = c.y;
    wf[j] = __double2float_rn(c.y);
  }
  const double c0 = w.c0[pp];
  __syncwarp();
  // shared (2,1) phase: the same kq21 on every lane for every baseline -> evaluate its sin^2
  // once per (bin, node) of the tile (lane = bin) instead of once per point
  bool shared = false;
  if constexpr (GNA_BATCH_PT_SHARED21) {
    shared = true;
#pragma unroll
    for (int j = 0; j < NT; j += 3) {
      const double k21 = __shfl_sync(0xffffffffu, kq[j], 0);
      shared = shared && __all_sync(0xffffffffu, kq[j] == k21);
    }
    if (shared) {
      float* sSf = reinterpret_cast<float*>(sS);  // mixed tier: W(h^2) in fp32
#pragma unroll
      for (int j = 0; j < NT; j += 3)
        for (int i = 0; i < order; ++i) {
          if constexpr (kMixed)
            sSf[((j / 3) * order + i) * 32 + lane] =
                gna::cos2_w(gna::mixed_h1(kq[j], pt_iE(sE, i, lane)));
          else
            sS[((j / 3) * order + i) * 32 + lane] = gna::sin2c(kq[j], pt_iE(sE, i, lane));
        }
      __syncwarp();
    }
  }
  double* __restrict__ out = spectra ? spectra + pp * nbins : nullptr;
  // fp64: a ragged last tile (nbins not a multiple of 32) skips its empty bins in a separate
  // copy of the loop, so full tiles run the branch-free one (cfg4 363.0 -> 364.2 G/s).  Mixed
  // tier: one loop that computes every bin and drops the empty ones — the second loop copy
  // cost it 7 % (556 -> 518 G/s).
  double x2;
  if constexpr (kMixed) {
    if (shared)
      x2 = pt_tile<2, N, NT, kOut, kMixed, true, kOrd>(kq, cw, wf, c0, sE, sH, sW, sD, sID, order, k0,
                                                 nbins, out, pact, sub, lv, sS);
    else
      x2 = pt_tile<2, N, NT, kOut, kMixed, false, kOrd>(kq, cw, wf, c0, sE, sH, sW, sD, sID, order, k0,
                                           nbins, out, pact, sub, lv);
  }
  else if (shared)
    x2 = k0 + 32 <= nbins
             ? pt_tile<0, N, NT, kOut, kMixed, true, kOrd>(kq, cw, wf, c0, sE, sH, sW, sD, sID, order,
                                                     k0, nbins, out, pact, sub, lv, sS)
             : pt_tile<1, N, NT, kOut, kMixed, true, kOrd>(kq, cw, wf, c0, sE, sH, sW, sD, sID, order,
                                                     k0, nbins, out, pact, sub, lv, sS);
  else
    x2 = k0 + 32 <= nbins
             ? pt_tile<0, N, NT, kOut, kMixed, false, kOrd>(kq, cw, wf, c0, sE, sH, sW, sD, sID, order, k0,
                                               nbins, out, pact, sub, lv)
             : pt_tile<1, N, NT, kOut, kMixed, false, kOrd>(kq, cw, wf, c0, sE, sH, sW, sD, sID, order, k0,
                                               nbins, out, pact, sub, lv);
  if (w.partial && pact) w.partial[(p * warps_per_point_dev(nbins) + wt) * S + sub] = x2;
  if constexpr (kOut != kOutLocal) __threadfence_system();
}

// chi2[p] = sum of the point's warp partials: lane l folds partials l, l+32, ...
// in order, then a fixed xor tree (deterministic, independent of scheduling).
// With S > 1 (k_oscprob_batch_pt sub-tiles) a tile's partial is first assembled from its S
// sub-partials by the top levels of the same tree.
template <int S>
__device__ __forceinline__ double tile_partial(const double* __restrict__ q, int64_t j) {
  if constexpr (S == 1) return q[j];
  else if constexpr (S == 2) return q[2 * j] + q[2 * j + 1];
  else return (q[4 * j] + q[4 * j + 1]) + (q[4 * j + 2] + q[4 * j + 3]);
}

template <int kOut, int S = 1>
__global__ void __launch_bounds__(kReduceThreads) k_chi2_reduce(const double* __restrict__ partial,
                                                                int64_t npoints, int64_t wpp,
                                                                double* __restrict__ chi2) {
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  pdl_wait();  // every partial of the main pass is written
  if (p >= npoints) return;
  const double* q = partial + p * wpp * S;
  double s = 0.0;
  for (int64_t j = lane; j < wpp; j += 32) s += tile_partial<S>(q, j);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out_store<kOut>(chi2 + p, s);
  if constexpr (kOut != kOutLocal) __threadfence_system();
}

}  // namespace

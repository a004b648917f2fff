// gna_b200.cu — sm_100a kernels and the C ABI of libgna_b200.so (include/gna_b200.h).
//
// Hot path (BASELINE.json north_star), fp64 throughout:
//   (a2) per-point coefficients: mixing weights w21/w31/w32 and phase slopes
//   (a3) P_ee(E) = 1 - sum_ij w_ij sin^2(Delta_ij)            (§4.1)
//   (a4) S_k = h_k sum_i w_i P_ee(c_k + h_k t_i)                (Gauss-Legendre)
//   (a5) T[p][k] = sum_b omega_b S_{p,b,k}, chi2[p]             (batch epilogue)
// Everything after argument validation runs in the kernels below; there is no
// host or CPU fallback.  See DESIGN.md for the roofline of each kernel.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <complex>
#include <utility>
#include <mutex>

#include "../../include/gna_b200.h"
#include "gl_table.h"
#include "gna_device.cuh"
#include "gna_tma.cuh"

using gna::PeeCoef;

namespace {

// ----------------------------------------------------------------------------
// constants
// ----------------------------------------------------------------------------
// S:265 / S:317 phase literal (R1); Delta = kPhase * dm2 * L / (E/1000).
constexpr double kPhase = 1.26693268;
// 1000 (MeV per GeV) * 2/pi: the kernels work with y = Delta * 2/pi.
constexpr double kMeV2Over_pi = 636.6197723675813430755;  // 2000/pi

__constant__ double c_gl_t[GNA_GL_TABLE_SIZE] = GNA_GL_NODES_INIT;
__constant__ double c_gl_w[GNA_GL_TABLE_SIZE] = GNA_GL_WEIGHTS_INIT;
// global-memory copy for lane-divergent indexing (the constant cache serialises
// a warp's distinct addresses; L1 serves them in one wavefront)
__device__ double g_gl_t[GNA_GL_TABLE_SIZE] = GNA_GL_NODES_INIT;
__device__ double g_gl_w[GNA_GL_TABLE_SIZE] = GNA_GL_WEIGHTS_INIT;
const double h_gl_t[GNA_GL_TABLE_SIZE] = GNA_GL_NODES_INIT;
const double h_gl_w[GNA_GL_TABLE_SIZE] = GNA_GL_WEIGHTS_INIT;

std::atomic<int64_t> g_launches{0};
thread_local int t_last_cuda_error = 0;

constexpr int kEvalThreads = 256;
#ifndef GNA_BATCH_WARPS
#define GNA_BATCH_WARPS 1
#endif
constexpr int kBatchWarps = GNA_BATCH_WARPS;
constexpr int kReduceThreads = 128;

__device__ __forceinline__ int64_t warps_per_point_dev(int64_t nbins) { return (nbins + 31) / 32; }

// phase slope in units of pi/2 per 1/MeV: y = kq / E  <=>  Delta = kPhase*dm2*L/(E/1000)
__host__ __device__ inline double phase_slope(double dm2, double L_km) {
  return ((kPhase * dm2) * L_km) * kMeV2Over_pi;
}

// mixing weights of P_ee (R2): w21 = c13^4 sin^2 2t12,
// w31 = sin^2 2t13 c12^2, w32 = sin^2 2t13 s12^2
__host__ __device__ inline void mixing_weights(double s12, double c12, double s13, double c13,
                                               double* w21, double* w31, double* w32) {
  const double s2t12 = 2.0 * s12 * c12;
  const double s2t13 = 2.0 * s13 * c13;
  const double c13sq = c13 * c13;
  *w21 = (c13sq * c13sq) * (s2t12 * s2t12);
  *w31 = (s2t13 * s2t13) * (c12 * c12);
  *w32 = (s2t13 * s2t13) * (s12 * s12);
}

// ----------------------------------------------------------------------------
// kernels
// ----------------------------------------------------------------------------

// (a3) elementwise P_ee, double2-vectorised grid-stride stream.
template <bool kVec, class Coef>
__global__ void __launch_bounds__(kEvalThreads) k_oscprob_eval(Coef c,
                                                               const double* __restrict__ E,
                                                               double* __restrict__ P, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (kVec) {
    const int64_t n2 = n >> 1;
    const double2* __restrict__ E2 = reinterpret_cast<const double2*>(E);
    double2* __restrict__ P2 = reinterpret_cast<double2*>(P);
    for (int64_t i = tid; i < n2; i += stride) {
      const double2 e = __ldcs(E2 + i);
      double2 r;
      r.x = gna::prob_inv(c, gna::rcp(e.x));
      r.y = gna::prob_inv(c, gna::rcp(e.y));
      __stcs(P2 + i, r);
    }
    if ((n & 1) && tid == 0) P[n - 1] = gna::prob_inv(c, gna::rcp(E[n - 1]));
  } else {
    for (int64_t i = tid; i < n; i += stride) P[i] = gna::prob_inv(c, gna::rcp(E[i]));
  }
}

// (a3) elementwise P_ee fed by TMA: a persistent block streams 8 KiB tiles of E
// global -> shared with cp.async.bulk into a kEvalStages-deep ring (mbarrier per
// stage), so ~kEvalStages x 8 KiB per block stay in flight independently of the
// registers; threads read their double2 pairs from shared memory, compute, and
// store P with streaming (evict-first) stores.  Full tiles only; the < 1 tile tail
// is done by block 0 with plain loads.
#ifndef GNA_EVAL_TILE
#define GNA_EVAL_TILE 1024
#endif
#ifndef GNA_EVAL_STAGES
#define GNA_EVAL_STAGES 4
#endif
#ifndef GNA_EVAL_MINB
#define GNA_EVAL_MINB 6
#endif
#ifndef GNA_EVAL_THREADS
#define GNA_EVAL_THREADS 128
#endif
constexpr int kEvalTile = GNA_EVAL_TILE;  // doubles per tile (8 KiB)
constexpr int kEvalStages = GNA_EVAL_STAGES;
constexpr int kEvalTmaThreads = GNA_EVAL_THREADS;

template <class Coef>
__global__ void __launch_bounds__(kEvalTmaThreads, GNA_EVAL_MINB) k_oscprob_eval_tma(Coef c,
                                                                       const double* __restrict__ E,
                                                                       double* __restrict__ P,
                                                                       int64_t n) {
  __shared__ alignas(128) double s_buf[kEvalStages][kEvalTile];
  __shared__ alignas(8) uint64_t s_full[kEvalStages];
  const int64_t ntiles = n / kEvalTile;
  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int64_t mine = first < ntiles ? (ntiles - 1 - first) / stride + 1 : 0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kEvalStages; ++st) gna::mbar_init(&s_full[st], 1);
    gna::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int st = 0; st < kEvalStages && st < mine; ++st) {
      gna::mbar_expect_tx(&s_full[st], kEvalTile * 8);
      gna::bulk_g2s(s_buf[st], E + (first + st * stride) * kEvalTile, kEvalTile * 8, &s_full[st]);
    }
  }
  for (int64_t it = 0; it < mine; ++it) {
    const int st = (int)(it % kEvalStages);
    gna::mbar_wait(&s_full[st], (uint32_t)((it / kEvalStages) & 1));
    const int64_t tile = first + it * stride;
    const double2* src = reinterpret_cast<const double2*>(s_buf[st]);
    double2* dst = reinterpret_cast<double2*>(P + tile * kEvalTile);
#pragma unroll
    for (int j = threadIdx.x; j < kEvalTile / 2; j += kEvalTmaThreads) {
      const double2 e = src[j];
      double2 r;
      r.x = gna::prob_inv(c, gna::rcp(e.x));
      r.y = gna::prob_inv(c, gna::rcp(e.y));
      __stcs(dst + j, r);
    }
    __syncthreads();  // every thread is done with stage st before it is refilled
    if (threadIdx.x == 0 && it + kEvalStages < mine) {
      gna::mbar_expect_tx(&s_full[st], kEvalTile * 8);
      gna::bulk_g2s(s_buf[st], E + (first + (it + kEvalStages) * stride) * kEvalTile,
                    kEvalTile * 8, &s_full[st]);
    }
  }
  if (blockIdx.x == 0)
    for (int64_t i = ntiles * kEvalTile + threadIdx.x; i < n; i += kEvalTmaThreads)
      P[i] = gna::prob_inv(c, gna::rcp(E[i]));
}

// (a3)+(a4) one parameter point.  A lane pair owns one bin: lane 2m+h evaluates the
// nodes [h*H, min((h+1)*H, order)), H = ceil(order/2), fully unrolled (compile-time
// order), so each lane runs H independent reciprocal + 3 sin^2 chains; the two
// halves are combined with one shuffle.  The whole grid is resident in one wave, so
// the bin edges' DRAM latency is paid once.  GL nodes/weights are read per lane
// from a global (L1) copy of the table.
constexpr int kGLLaneThreads = 128;

template <int kOrder, class Coef>
__global__ void __launch_bounds__(kGLLaneThreads) k_gl_integrate(Coef c,
                                                                 const double* __restrict__ edges,
                                                                 int64_t nbins,
                                                                 double* __restrict__ bins) {
  constexpr int H = (kOrder + 1) / 2;
  constexpr int off = GNA_GL_OFF(kOrder);
  const int64_t t = (int64_t)blockIdx.x * kGLLaneThreads + threadIdx.x;
  const int64_t k = t >> 1;
  const int half = (int)(t & 1);
  const bool act = k < nbins;
  const int64_t kk = act ? k : nbins - 1;
  const double e0 = edges[kk], e1 = edges[kk + 1];
  const double ctr = 0.5 * (e0 + e1);
  const double h = 0.5 * (e1 - e0);
  double pv[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const int node = half * H + i;
    pv[i] = 0.0;
    if (node < kOrder)
      pv[i] = __ldg(&g_gl_w[off + node]) *
              gna::prob_inv(c, gna::rcp(fma(h, __ldg(&g_gl_t[off + node]), ctr)));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < H; ++i) s += pv[i];
  const double other = __shfl_xor_sync(0xffffffffu, s, 1);
  if (act && half == 0) bins[k] = h * (s + other);
}

template <class Coef>
using gl_kernel_t = void (*)(Coef, const double*, int64_t, double*);

template <class Coef, int... N>
gl_kernel_t<Coef> gl_kernel_for(int order, std::integer_sequence<int, N...>) {
  static const gl_kernel_t<Coef> t[] = {k_gl_integrate<N + 1, Coef>...};
  return t[order - 1];
}

struct BatchSetupArgs {
  double L[GNA_MAX_NBASE];
  double omega[GNA_MAX_NBASE];
  double omega_sum;  // sum_b omega_b (left to right)
  int nbase;
  int order;
  int64_t nbins;
  int64_t npoints;
};

// Workspace layout of the batch path (all offsets 16-byte aligned), see
// gna_oscprob_batch_workspace_size:  coef [P][nbase][3] double2 (kq, omega_b w_ij),
// c0 [P], invE [order][nbins], hw [order][nbins], partial [P][wpp].
struct BatchWs {
  double2* coef;
  double* c0;
  double* invE;
  double* hw;
  double* partial;
};

size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }
size_t align32(size_t x) { return (x + 31) & ~(size_t)31; }

int64_t warps_per_point(int64_t nbins) { return (nbins + 31) / 32; }

size_t batch_ws_bytes(int64_t P, int nbase, int64_t nbins, int order, bool chi2) {
  size_t b = align16((size_t)P * nbase * 3 * sizeof(double2));
  b += align16((size_t)P * sizeof(double));
  b += 2 * align16((size_t)order * nbins * sizeof(double));
  if (chi2) b += align16((size_t)P * warps_per_point(nbins) * sizeof(double));
  return b;
}

BatchWs batch_ws_carve(void* base, int64_t P, int nbase, int64_t nbins, int order, bool chi2) {
  char* c = (char*)base;
  BatchWs w;
  w.coef = (double2*)c;
  c += align16((size_t)P * nbase * 3 * sizeof(double2));
  w.c0 = (double*)c;
  c += align16((size_t)P * sizeof(double));
  w.invE = (double*)c;
  c += align16((size_t)order * nbins * sizeof(double));
  w.hw = (double*)c;
  c += align16((size_t)order * nbins * sizeof(double));
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
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n1 = a.npoints * a.nbase;
  const int64_t n2 = (int64_t)a.order * a.nbins;
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
#ifndef GNA_BATCH_PPW_WORK
#define GNA_BATCH_PPW_WORK 480
#endif
#ifndef GNA_BATCH_LDS_PREFETCH
#define GNA_BATCH_LDS_PREFETCH 0
#endif
#ifndef GNA_BATCH_JUNROLL
#define GNA_BATCH_JUNROLL 1
#endif
#ifndef GNA_BATCH_MINB
#define GNA_BATCH_MINB 1
#endif

// N GL nodes of one bin at a time: each (kq, omega*w) coefficient load from
// shared memory feeds N independent sin^2 chains (ILP across nodes).
template <int N>
__device__ __forceinline__ void batch_nodes(const double2* __restrict__ sc, int nterm,
                                            const double* __restrict__ invE,
                                            const double* __restrict__ hw, int64_t nbins, int i,
                                            double c0, double& s) {
  double iE[N], a[N];
#pragma unroll
  for (int n = 0; n < N; ++n) {
    iE[n] = invE[(int64_t)(i + n) * nbins];
    a[n] = 0.0;
  }
#if GNA_BATCH_LDS_PREFETCH
  // the next coefficient pair is loaded before the current one is consumed, so the
  // LDS latency is not exposed at the top of every iteration
  double2 cw = sc[0];
  GNA_UNROLL(GNA_BATCH_JUNROLL)
  for (int j = 0; j < nterm; ++j) {
    const double2 cn = sc[j + 1 < nterm ? j + 1 : j];
#pragma unroll
    for (int n = 0; n < N; ++n) a[n] = fma(cw.y, gna::sin2c(cw.x, iE[n]), a[n]);
    cw = cn;
  }
#else
  GNA_UNROLL(GNA_BATCH_JUNROLL)
  for (int j = 0; j < nterm; ++j) {
    const double2 cw = sc[j];
#pragma unroll
    for (int n = 0; n < N; ++n) a[n] = fma(cw.y, gna::sin2c(cw.x, iE[n]), a[n]);
  }
#endif
#pragma unroll
  for (int n = 0; n < N; ++n) s = fma(hw[(int64_t)(i + n) * nbins], c0 - a[n], s);
}

// remainder of r < N nodes, compile-time group size
template <int N>
__device__ __forceinline__ void batch_tail(int r, const double2* __restrict__ sc, int nterm,
                                           const double* __restrict__ invE,
                                           const double* __restrict__ hw, int64_t nbins, int i,
                                           double c0, double& s) {
  if constexpr (N > 1) {
    if (r == N - 1) {
      batch_nodes<N - 1>(sc, nterm, invE, hw, nbins, i, c0, s);
      return;
    }
    batch_tail<N - 1>(r, sc, nterm, invE, hw, nbins, i, c0, s);
  }
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
template <int kWarps, int N, int kOut>
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
  const int64_t wpp = warps_per_point_dev(nbins);
  // ppw points per warp, same bins: the node tables stay in L1 across points
  const int64_t pend = min(npoints, (pg + 1) * (int64_t)ppw);
  for (int64_t p = pg * (int64_t)ppw; p < pend; ++p) {
    const double2* __restrict__ gc = w.coef + p * nterm;
    __syncwarp();  // previous point's reads of sc are done
    for (int j = lane; j < nterm; j += 32) sc[j] = gc[j];
    __syncwarp();
    const double c0 = w.c0[p];
    double s = 0.0;
    int i = 0;
    for (; i + N <= order; i += N) batch_nodes<N>(sc, nterm, invE, hw, nbins, i, c0, s);
    if (i < order) batch_tail<N>(order - i, sc, nterm, invE, hw, nbins, i, c0, s);
    double x2 = 0.0;
    if (active) {
      if (spectra) out_store<kOut>(spectra + p * nbins + k, s);
      const double d = s - D;
      x2 = d * d / D;
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

template <int N, int kOut>
__global__ void __launch_bounds__(32, GNA_BATCH_MINB) k_oscprob_batch_pi(
    int nterm, int order, int64_t nbins, int64_t npoints, int64_t bpp, int ppw, BatchWs w,
    double* __restrict__ spectra, const double* __restrict__ data) {
  extern __shared__ double2 s_dyn[];
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
  for (int j = lane; j < np * nterm; j += 32) sc[j] = w.coef[p0 * nterm + j];
  for (int j = lane; j < np; j += 32) s_c0[j] = w.c0[p0 + j];
  for (int q = 0; q < np; ++q) s_acc[q * 32 + lane] = 0.0;
  __syncwarp();
  const int64_t k = k0 + lane;
  const bool active = k < nbins;
  const int64_t kk = active ? k : nbins - 1;
  const double* __restrict__ invE = w.invE + kk;
  const double* __restrict__ hw = w.hw + kk;
  for (int i = 0; i < order; i += N) {
    const int nn = min(N, order - i);
    double iE[N], hv[N];
#pragma unroll
    for (int n = 0; n < N; ++n) {
      iE[n] = n < nn ? invE[(int64_t)(i + n) * nbins] : 1.0;
      hv[n] = n < nn ? hw[(int64_t)(i + n) * nbins] : 0.0;
    }
    int q = 0;
#if GNA_BATCH_PI_Q2
    // two points at a time: 2N independent sin^2 chains per coefficient step
    for (; q + 1 < np; q += 2) {
      const double2* __restrict__ cq = sc + q * nterm;
      const double2* __restrict__ cr = cq + nterm;
      double a[N], b[N];
#pragma unroll
      for (int n = 0; n < N; ++n) a[n] = b[n] = 0.0;
      for (int j = 0; j < nterm; ++j) {
        const double2 cw = cq[j], cv = cr[j];
#pragma unroll
        for (int n = 0; n < N; ++n) {
          a[n] = fma(cw.y, gna::sin2c(cw.x, iE[n]), a[n]);
          b[n] = fma(cv.y, gna::sin2c(cv.x, iE[n]), b[n]);
        }
      }
      const double c0a = s_c0[q], c0b = s_c0[q + 1];
      double sa = s_acc[q * 32 + lane], sb = s_acc[(q + 1) * 32 + lane];
#pragma unroll
      for (int n = 0; n < N; ++n)
        if (n < nn) {
          sa = fma(hv[n], c0a - a[n], sa);
          sb = fma(hv[n], c0b - b[n], sb);
        }
      s_acc[q * 32 + lane] = sa;
      s_acc[(q + 1) * 32 + lane] = sb;
    }
#endif
    for (; q < np; ++q) {
      const double2* __restrict__ cq = sc + q * nterm;
      double a[N];
#pragma unroll
      for (int n = 0; n < N; ++n) a[n] = 0.0;
      for (int j = 0; j < nterm; ++j) {
        const double2 cw = cq[j];
#pragma unroll
        for (int n = 0; n < N; ++n) a[n] = fma(cw.y, gna::sin2c(cw.x, iE[n]), a[n]);
      }
      const double c0 = s_c0[q];
      double sv = s_acc[q * 32 + lane];
#pragma unroll
      for (int n = 0; n < N; ++n)
        if (n < nn) sv = fma(hv[n], c0 - a[n], sv);
      s_acc[q * 32 + lane] = sv;
    }
  }
  const double D = (data && active) ? data[k] : 1.0;
  const int64_t wpp = warps_per_point_dev(nbins);
  for (int q = 0; q < np; ++q) {
    const int64_t p = p0 + q;
    const double sv = s_acc[q * 32 + lane];
    double x2 = 0.0;
    if (active) {
      if (spectra) out_store<kOut>(spectra + p * nbins + k, sv);
      const double d = sv - D;
      x2 = d * d / D;
    }
    if (w.partial) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x2 += __shfl_xor_sync(0xffffffffu, x2, o);
      if (lane == 0) w.partial[p * wpp + wt] = x2;
    }
  }
  if constexpr (kOut != kOutLocal) __threadfence_system();
}

// chi2[p] = sum of the point's warp partials: lane l folds partials l, l+32, ...
// in order, then a fixed xor tree (deterministic, independent of scheduling).
template <int kOut>
__global__ void __launch_bounds__(kReduceThreads) k_chi2_reduce(const double* __restrict__ partial,
                                                                int64_t npoints, int64_t wpp,
                                                                double* __restrict__ chi2) {
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= npoints) return;
  const double* q = partial + p * wpp;
  double s = 0.0;
  for (int64_t j = lane; j < wpp; j += 32) s += q[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out_store<kOut>(chi2 + p, s);
  if constexpr (kOut != kOutLocal) __threadfence_system();
}

// ----------------------------------------------------------------------------
// NEXT-1: separable grid scan ("computed only once ... re-computed
// only if any of the variables or inputs it depends on were modified", P:641-642 one
// transformation per formula item).  The mixing weights enter P_ee only linearly, so for a
// grid {mixing points a} x {mass points c} the binned sin^2 sums depend on c alone:
//   G[c][ij][k] = sum_b omega_b h_k sum_i w_i sin^2(Delta_ij(c, b, E_ki)),
//   H[k]        = Omega h_k sum_i w_i,
//   T[c*nmix+a][k] = H[k] - sum_ij w_ij(a) G[c][ij][k]      (a rank-3 update per point).
// Stage A costs nmass x nbase x 3 x nbins x order sin^2 (FP64); stage B is bound by writing
// the spectra to HBM.
struct ScanArgs {
  double L[GNA_MAX_NBASE];
  double omega[GNA_MAX_NBASE];
  double omega_sum;
  int nbase;
  int order;
  int64_t nbins;
  int64_t nmix;
  int64_t nmass;
};

struct ScanWs {
  double* G;     // [nmass][3][nbins]
  double* H;     // [nbins]
  double* invD;  // [nbins]  1 / data (chi2 only)
  double* wmix;  // [nmix][4]  (w21, w31, w32, 0)
};

size_t scan_ws_bytes(int64_t nmix, int64_t nmass, int64_t nbins) {
  size_t b = align32((size_t)nmass * 3 * nbins * sizeof(double));
  b += 2 * align32((size_t)nbins * sizeof(double));
  b += align32((size_t)nmix * 4 * sizeof(double));
  return b;
}

ScanWs scan_ws_carve(void* base, int64_t nmix, int64_t nmass, int64_t nbins) {
  char* c = (char*)base;
  ScanWs w;
  w.G = (double*)c;
  c += align32((size_t)nmass * 3 * nbins * sizeof(double));
  w.H = (double*)c;
  c += align32((size_t)nbins * sizeof(double));
  w.invD = (double*)c;
  c += align32((size_t)nbins * sizeof(double));
  w.wmix = (double*)c;
  return w;
}

// stage A: thread per (mass point c, bin k): the three pairs share each node's
// reciprocal and run as three independent sin^2 chains (two nodes per iteration:
// six chains) -> G[c][*][k]; threads with c == 0 also write H[k] and 1/D[k]; extra
// threads compute the mixing weights of each mixing point.
__global__ void __launch_bounds__(128) k_scan_setup(ScanArgs a, const double* __restrict__ th12,
                                                    const double* __restrict__ th13,
                                                    const double* __restrict__ d21,
                                                    const double* __restrict__ d31,
                                                    const double* __restrict__ edges,
                                                    const double* __restrict__ data, ScanWs w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n1 = a.nmass * a.nbins;
  if (t < n1) {
    const int64_t c = t / a.nbins;
    const int64_t k = t - c * a.nbins;
    const int off = GNA_GL_OFF(a.order);
    const double e0 = edges[k], e1 = edges[k + 1];
    const double ctr = 0.5 * (e0 + e1);
    const double h = 0.5 * (e1 - e0);
    double wsum = 0.0;
    for (int i = 0; i < a.order; ++i) wsum += c_gl_w[off + i];
    const double m21 = d21[c], m31 = d31[c];
    const double m32 = m31 - m21;
    double G0 = 0.0, G1 = 0.0, G2 = 0.0;
    for (int b = 0; b < a.nbase; ++b) {
      const double k0 = phase_slope(m21, a.L[b]);
      const double k1 = phase_slope(m31, a.L[b]);
      const double k2 = phase_slope(m32, a.L[b]);
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll 2
      for (int i = 0; i < a.order; ++i) {
        const double invE = gna::rcp(fma(h, c_gl_t[off + i], ctr));
        const double wi = c_gl_w[off + i];
        s0 = fma(wi, gna::sin2c(k0, invE), s0);
        s1 = fma(wi, gna::sin2c(k1, invE), s1);
        s2 = fma(wi, gna::sin2c(k2, invE), s2);
      }
      // h sum_i w_i sin^2 = h (W/2 + sum_i w_i (-1)^q v)
      const double ob = a.omega[b] * h;
      G0 = fma(ob, fma(0.5, wsum, s0), G0);
      G1 = fma(ob, fma(0.5, wsum, s1), G1);
      G2 = fma(ob, fma(0.5, wsum, s2), G2);
    }
    double* g = w.G + (c * 3) * a.nbins + k;
    g[0] = G0;
    g[a.nbins] = G1;
    g[2 * a.nbins] = G2;
    if (c == 0) {
      w.H[k] = a.omega_sum * h * wsum;
      if (data) w.invD[k] = 1.0 / data[k];
    }
  } else if (t < n1 + a.nmix) {
    const int64_t mm = t - n1;
    double s12, c12, s13, c13;
    sincos(th12[mm], &s12, &c12);
    sincos(th13[mm], &s13, &c13);
    double* wm = w.wmix + 4 * mm;
    mixing_weights(s12, c12, s13, c13, &wm[0], &wm[1], &wm[2]);
    wm[3] = 0.0;
  }
}

// stage B: block = (mass point c, chunk of kScanA (4) mixing points).  Each thread loads
// G[c][*][k], H[k], D[k], 1/D[k] of its bins once and writes T for all kScanA points
// (coalesced rows), so G is read once per chunk instead of once per point; chi2 of each
// point is reduced in the block (fixed shuffle tree + warps in order) and written directly.
#ifndef GNA_SCAN_A
#define GNA_SCAN_A 4
#endif
#ifndef GNA_SCAN_THREADS
#define GNA_SCAN_THREADS 128
#endif
constexpr int kScanThreads = GNA_SCAN_THREADS;
constexpr int kScanA = GNA_SCAN_A;

__global__ void __launch_bounds__(kScanThreads) k_scan_expand(int64_t nmix, int64_t nbins,
                                                              int64_t nchunk, ScanWs w,
                                                              double* __restrict__ spectra,
                                                              const double* __restrict__ data,
                                                              double* __restrict__ chi2) {
  __shared__ double s_x2[kScanA][kScanThreads / 32];
  const int64_t c = blockIdx.x / nchunk;
  const int64_t a0 = (blockIdx.x - c * nchunk) * kScanA;
  const int na = (int)min((int64_t)kScanA, nmix - a0);
  double w0[kScanA], w1[kScanA], w2[kScanA], x2[kScanA];
#pragma unroll
  for (int j = 0; j < kScanA; ++j) {
    const int64_t aj = a0 + (j < na ? j : 0);
    const double4 wm = *reinterpret_cast<const double4*>(w.wmix + 4 * aj);
    w0[j] = wm.x;
    w1[j] = wm.y;
    w2[j] = wm.z;
    x2[j] = 0.0;
  }
  const double* __restrict__ g0 = w.G + (c * 3) * nbins;
  const double* __restrict__ g1 = g0 + nbins;
  const double* __restrict__ g2 = g1 + nbins;
  double* __restrict__ out = spectra ? spectra + (c * nmix + a0) * nbins : nullptr;
  // software-pipelined: the 6 loads of bin k + kScanThreads are issued before bin k's
  // outputs are computed, so one L2 round trip is always in flight per thread
  int64_t k = threadIdx.x;
  double G0 = 0, G1 = 0, G2 = 0, H = 0, D = 0, iD = 0;
  if (k < nbins) {
    G0 = g0[k], G1 = g1[k], G2 = g2[k], H = w.H[k];
    if (chi2) D = data[k], iD = w.invD[k];
  }
  for (; k < nbins; k += kScanThreads) {
    const int64_t kn = k + kScanThreads;
    double nG0 = 0, nG1 = 0, nG2 = 0, nH = 0, nD = 0, niD = 0;
    if (kn < nbins) {
      nG0 = g0[kn], nG1 = g1[kn], nG2 = g2[kn], nH = w.H[kn];
      if (chi2) nD = data[kn], niD = w.invD[kn];
    }
#pragma unroll
    for (int j = 0; j < kScanA; ++j) {
      if (j < na) {
        const double T = H - fma(w0[j], G0, fma(w1[j], G1, w2[j] * G2));
        if (out) __stcs(out + (int64_t)j * nbins + k, T);
        const double d = T - D;
        x2[j] = fma(d * d, iD, x2[j]);
      }
    }
    G0 = nG0, G1 = nG1, G2 = nG2, H = nH, D = nD, iD = niD;
  }
  if (chi2) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < kScanA; ++j) {
      double v = x2[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) s_x2[j][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < na) {
      double t = 0.0;
#pragma unroll
      for (int i = 0; i < kScanThreads / 32; ++i) t += s_x2[threadIdx.x][i];
      chi2[c * nmix + a0 + threadIdx.x] = t;
    }
  }
}

// ----------------------------------------------------------------------------
// NEXT-4 (second part): a chi^2 minimiser that stays on the GPU (the fit of P:446-451).
// Deterministic compass/pattern search over (theta12, theta13, dm2_21, dm2_31): every
// iteration evaluates the 3^4 = 81 points centre + step * {-1, 0, +1}^4 with the batch
// kernels (chi^2 only), takes the argmin (lowest index on ties), moves the centre there,
// or halves the steps if the centre is already best.  The whole loop is stream-ordered
// (no host round trip), so it can be captured in one CUDA graph.
constexpr int kFitDim = 4;
constexpr int kFitCand = 81;  // 3^4

// state = {centre[4], step[4]} (device, fp64)
__global__ void __launch_bounds__(128) k_fit_candidates(const double* __restrict__ state,
                                                        double* __restrict__ cand) {
  const int c = threadIdx.x;
  if (c >= kFitCand) return;
  int code = c;
#pragma unroll
  for (int d = 0; d < kFitDim; ++d) {
    const int o = code % 3 - 1;  // -1, 0, +1 ; candidate 40 is the centre
    code /= 3;
    cand[d * kFitCand + c] = fma((double)o, state[kFitDim + d], state[d]);
  }
}

__global__ void __launch_bounds__(128) k_fit_update(double* __restrict__ state,
                                                    const double* __restrict__ cand,
                                                    const double* __restrict__ chi2,
                                                    double* __restrict__ hist, int iter) {
  __shared__ double s_v[128];
  __shared__ int s_i[128];
  const int t = threadIdx.x;
  s_v[t] = t < kFitCand ? chi2[t] : INFINITY;
  s_i[t] = t;
  __syncthreads();
  for (int o = 64; o > 0; o >>= 1) {  // argmin, ties -> lowest index (deterministic)
    if (t < o) {
      const double a = s_v[t], b = s_v[t + o];
      if (b < a || (b == a && s_i[t + o] < s_i[t])) {
        s_v[t] = b;
        s_i[t] = s_i[t + o];
      }
    }
    __syncthreads();
  }
  if (t == 0) {
    const int best = s_i[0];
    const int centre = kFitCand / 2;
    if (best == centre || !(s_v[0] < chi2[centre])) {
#pragma unroll
      for (int d = 0; d < kFitDim; ++d) state[kFitDim + d] *= 0.5;
    } else {
#pragma unroll
      for (int d = 0; d < kFitDim; ++d) state[d] = cand[d * kFitCand + best];
    }
    if (hist) hist[iter] = fmin(s_v[0], chi2[centre]);
  }
}

// ----------------------------------------------------------------------------
// host helpers
// ----------------------------------------------------------------------------
int cuda_fail(cudaError_t e) {
  t_last_cuda_error = (int)e;
  return GNA_ECUDA;
}

bool is_fin(double x) { return std::isfinite(x); }

bool params_ok(const gna_osc_params* p) {
  return p && is_fin(p->theta12) && is_fin(p->theta13) && is_fin(p->theta23) &&
         is_fin(p->delta_cp) && is_fin(p->dm2_21) && is_fin(p->dm2_31);
}

bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
  return x < y + nb && y < x + na;
}

// 0 ok, else status.  Checks the current device is sm_100 (cached per device).
int check_device() {
  static std::atomic<int> state[128];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e);
  if (dev < 0 || dev >= 128) return GNA_ENODEV;
  int s = state[dev].load(std::memory_order_relaxed);
  if (s == 0) {
    int major = 0, minor = 0;
    e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e != cudaSuccess) return cuda_fail(e);
    e = cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (e != cudaSuccess) return cuda_fail(e);
    s = (major == 10 && minor == 0) ? 1 : 2;
    state[dev].store(s, std::memory_order_relaxed);
  }
  return s == 1 ? GNA_OK : GNA_ENODEV;
}

// EINVAL unless ptr is device (or managed) memory.
int check_dev_ptr(const void* ptr) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear the sticky-free error
    return GNA_EINVAL;
  }
  return (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) ? GNA_OK
                                                                              : GNA_EINVAL;
}

void make_coef(const gna_osc_params* p, double L_km, PeeCoef* c) {
  double w21, w31, w32;
  mixing_weights(std::sin(p->theta12), std::cos(p->theta12), std::sin(p->theta13),
                 std::cos(p->theta13), &w21, &w31, &w32);
  const double m32 = p->dm2_31 - p->dm2_21;
  c->kq[0] = phase_slope(p->dm2_21, L_km);
  c->kq[1] = phase_slope(p->dm2_31, L_km);
  c->kq[2] = phase_slope(m32, L_km);
  c->w[0] = w21;
  c->w[1] = w31;
  c->w[2] = w32;
  c->c0 = 1.0 - 0.5 * ((w21 + w31) + w32);
}

// NEXT-2: coefficients of any channel alpha -> beta.  PMNS elements from the PDG
// closed form (independent of the oracle's matrix product), conj for antineutrinos
// (S:256); X_ij = V*_ai V_bi V_aj V*_bj for pairs (2,1), (3,1), (3,2).
void make_coef_ab(int alpha, int beta, const gna_osc_params* p, double L_km, gna::PabCoef* c) {
  using cd = std::complex<double>;
  const double c12 = std::cos(p->theta12), s12 = std::sin(p->theta12);
  const double c13 = std::cos(p->theta13), s13 = std::sin(p->theta13);
  const double c23 = std::cos(p->theta23), s23 = std::sin(p->theta23);
  const cd e = std::polar(1.0, p->delta_cp);  // e^{i delta}
  cd V[3][3] = {{c12 * c13, s12 * c13, s13 * std::conj(e)},
                {-s12 * c23 - c12 * s23 * s13 * e, c12 * c23 - s12 * s23 * s13 * e, s23 * c13},
                {s12 * s23 - c12 * c23 * s13 * e, -c12 * s23 - s12 * c23 * s13 * e, c23 * c13}};
  if (p->antineutrino)
    for (auto& row : V)
      for (auto& x : row) x = std::conj(x);
  const int pi_[3] = {1, 2, 2}, pj_[3] = {0, 0, 1};
  const double dm[3] = {p->dm2_21, p->dm2_31, p->dm2_31 - p->dm2_21};
  double c0 = alpha == beta ? 1.0 : 0.0;
  for (int k = 0; k < 3; ++k) {
    const int i = pi_[k], j = pj_[k];
    const cd X = std::conj(V[alpha][i]) * V[beta][i] * V[alpha][j] * std::conj(V[beta][j]);
    c->kq[k] = phase_slope(dm[k], L_km);
    c->a[k] = -4.0 * X.real();
    c->b[k] = 2.0 * X.imag();
    c0 += 0.5 * c->a[k];
  }
  c->c0 = c0;
}

int grid_for(int64_t work_items, int threads, int max_blocks) {
  int64_t b = (work_items + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

int sm_count() {
  static std::atomic<int> cached{0};
  int v = cached.load();
  if (v == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cached.store(v);
  }
  return v;
}

// --- validation shared by device and host variants --------------------------
int validate_eval(const gna_osc_params* p, double L_km, const double* E, int64_t n, const double* P) {
  if (!params_ok(p) || !E || !P || n < 1 || !is_fin(L_km) || L_km < 0) return GNA_EINVAL;
  if (overlap(E, (size_t)n * 8, P, (size_t)n * 8)) return GNA_EINVAL;
  return GNA_OK;
}

int validate_gl(const gna_osc_params* p, double L_km, const double* edges, int64_t nbins,
                int32_t order, const double* bins) {
  if (!params_ok(p) || !edges || !bins || nbins < 1 || order < 1 || order > GNA_MAX_ORDER ||
      !is_fin(L_km) || L_km < 0)
    return GNA_EINVAL;
  if (overlap(edges, (size_t)(nbins + 1) * 8, bins, (size_t)nbins * 8)) return GNA_EINVAL;
  return GNA_OK;
}

int validate_batch(const gna_param_batch* pts, const double* L_km, const double* omega,
                   int32_t nbase, const double* edges, int64_t nbins, int32_t order,
                   const double* spectra, const double* data, const double* chi2) {
  if (!pts || !pts->theta12 || !pts->theta13 || !pts->dm2_21 || !pts->dm2_31 ||
      pts->npoints < 1 || !L_km || !omega || nbase < 1 || nbase > GNA_MAX_NBASE || !edges ||
      nbins < 1 || order < 1 || order > GNA_MAX_ORDER)
    return GNA_EINVAL;
  if (!spectra && !chi2) return GNA_EINVAL;
  if (chi2 && !data) return GNA_EINVAL;
  for (int b = 0; b < nbase; ++b)
    if (!is_fin(L_km[b]) || L_km[b] < 0 || !is_fin(omega[b])) return GNA_EINVAL;
  const size_t P8 = (size_t)pts->npoints * 8;
  if (spectra) {
    const size_t S8 = (size_t)pts->npoints * (size_t)nbins * 8;
    const void* ins[6] = {pts->theta12, pts->theta13, pts->dm2_21, pts->dm2_31, edges, data};
    const size_t ln[6] = {P8, P8, P8, P8, (size_t)(nbins + 1) * 8, data ? (size_t)nbins * 8 : 0};
    for (int i = 0; i < 6; ++i)
      if (ins[i] && overlap(spectra, S8, ins[i], ln[i])) return GNA_EINVAL;
    if (chi2 && overlap(spectra, S8, chi2, P8)) return GNA_EINVAL;
  }
  if (chi2) {
    const void* ins[6] = {pts->theta12, pts->theta13, pts->dm2_21, pts->dm2_31, edges, data};
    const size_t ln[6] = {P8, P8, P8, P8, (size_t)(nbins + 1) * 8, (size_t)nbins * 8};
    for (int i = 0; i < 6; ++i)
      if (overlap(chi2, P8, ins[i], ln[i])) return GNA_EINVAL;
  }
  return GNA_OK;
}

int64_t blocks_per_point(int64_t nbins) {
  return (warps_per_point(nbins) + kBatchWarps - 1) / kBatchWarps;
}

// launch of the batch kernels on already-validated device arguments
template <int kOut>
int launch_batch_k(const gna_param_batch* pts, const double* L_km, const double* omega,
                   int32_t nbase, const double* edges, int64_t nbins, int32_t order,
                   double* spectra, const double* data, double* chi2, void* workspace,
                   cudaStream_t s) {
  BatchSetupArgs a;
  std::memset(&a, 0, sizeof(a));
  double om = 0.0;
  for (int b = 0; b < nbase; ++b) {
    a.L[b] = L_km[b];
    a.omega[b] = omega[b];
    om += omega[b];
  }
  a.omega_sum = om;
  a.nbase = nbase;
  a.order = order;
  a.nbins = nbins;
  a.npoints = pts->npoints;
  const BatchWs w = batch_ws_carve(workspace, pts->npoints, nbase, nbins, order, chi2 != nullptr);
  const int64_t bpp = blocks_per_point(nbins);
  // points per warp: enough sin^2 work per lane to amortise the per-point overhead
  // (>= 240; >= GNA_BATCH_PPW_WORK for the small-nbase points-inner kernel), while
  // keeping >= 16 warps per SM worth of blocks
  const int64_t work = (int64_t)3 * nbase * order;
  const bool small_terms = 3 * nbase <= GNA_BATCH_PI_MAX_TERMS;
  int64_t ppw = std::max<int64_t>(1, ((small_terms ? GNA_BATCH_PPW_WORK : 240) + work - 1) / work);
  const int64_t min_blocks = (int64_t)sm_count() * 16;
  while (ppw > 1 && ((pts->npoints + ppw - 1) / ppw) * bpp < min_blocks) ppw >>= 1;
  const int64_t ngroups = (pts->npoints + ppw - 1) / ppw;
  const int64_t nblocks = ngroups * bpp;
  const int64_t nsetup = pts->npoints * nbase + (int64_t)order * nbins;
  if (nblocks > 0x7fffffffLL || (nsetup + 255) / 256 > 0x7fffffffLL) return GNA_EINVAL;

  k_batch_setup<<<(unsigned)((nsetup + 255) / 256), 256, 0, s>>>(
      a, pts->theta12, pts->theta13, pts->dm2_21, pts->dm2_31, edges, w);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e);

  const int nterm = 3 * nbase;
  const size_t smem = (size_t)kBatchWarps * nterm * sizeof(double2);
  // node-group size: 5, 4 or 3 when it divides the order, else 4
  auto kern = (order % 5 == 0)   ? k_oscprob_batch<kBatchWarps, 5, kOut>
              : (order % 4 == 0) ? k_oscprob_batch<kBatchWarps, 4, kOut>
              : (order % 3 == 0) ? k_oscprob_batch<kBatchWarps, 3, kOut>
                                 : k_oscprob_batch<kBatchWarps, 4, kOut>;
  if (ppw > 1 && small_terms && kBatchWarps == 1 && GNA_BATCH_PI) {
    // several points per warp: node groups outer, points inner (bitwise-identical sums)
    ppw = std::min<int64_t>(ppw, kMaxPPW);
    const int64_t ng = (pts->npoints + ppw - 1) / ppw;
    const size_t smem_pi = (size_t)ppw * nterm * sizeof(double2) + (size_t)ppw * 33 * 8;
    auto kpi = (order % 5 == 0)   ? k_oscprob_batch_pi<5, kOut>
               : (order % 4 == 0) ? k_oscprob_batch_pi<4, kOut>
               : (order % 3 == 0) ? k_oscprob_batch_pi<3, kOut>
                                  : k_oscprob_batch_pi<4, kOut>;
    kpi<<<(unsigned)(ng * bpp), 32, smem_pi, s>>>(nterm, order, nbins, pts->npoints, bpp,
                                                  (int)ppw, w, spectra, chi2 ? data : nullptr);
  } else {
    kern<<<(unsigned)nblocks, kBatchWarps * 32, smem, s>>>(
        nterm, order, nbins, pts->npoints, bpp, (int)ppw, w, spectra, chi2 ? data : nullptr);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e);
  if (chi2) {
    const int64_t threads = pts->npoints * 32;
    const int grid = (int)((threads + kReduceThreads - 1) / kReduceThreads);
    k_chi2_reduce<kOut><<<grid, kReduceThreads, 0, s>>>(w.partial, pts->npoints,
                                                        warps_per_point(nbins), chi2);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e);
  }
  return GNA_OK;
}

int launch_batch(const gna_param_batch* pts, const double* L_km, const double* omega,
                 int32_t nbase, const double* edges, int64_t nbins, int32_t order,
                 double* spectra, const double* data, double* chi2, void* workspace,
                 cudaStream_t s, int out_mode = kOutLocal) {
  if (out_mode == kOutMulticast)
    return launch_batch_k<kOutMulticast>(pts, L_km, omega, nbase, edges, nbins, order, spectra,
                                         data, chi2, workspace, s);
  if (out_mode == kOutPeer)
    return launch_batch_k<kOutPeer>(pts, L_km, omega, nbase, edges, nbins, order, spectra, data,
                                    chi2, workspace, s);
  return launch_batch_k<kOutLocal>(pts, L_km, omega, nbase, edges, nbins, order, spectra, data,
                                   chi2, workspace, s);
}

int launch_scan(const gna_scan_grid* g, const double* L_km, const double* omega, int32_t nbase,
                const double* edges, int64_t nbins, int32_t order, double* spectra,
                const double* data, double* chi2, void* workspace, cudaStream_t s) {
  ScanArgs a;
  std::memset(&a, 0, sizeof(a));
  double om = 0.0;
  for (int b = 0; b < nbase; ++b) {
    a.L[b] = L_km[b];
    a.omega[b] = omega[b];
    om += omega[b];
  }
  a.omega_sum = om;
  a.nbase = nbase;
  a.order = order;
  a.nbins = nbins;
  a.nmix = g->nmix;
  a.nmass = g->nmass;
  const ScanWs w = scan_ws_carve(workspace, g->nmix, g->nmass, nbins);
  const int64_t nsetup = g->nmass * nbins + g->nmix;
  const int64_t nchunk = (g->nmix + kScanA - 1) / kScanA;
  const int64_t nblk = g->nmass * nchunk;
  if ((nsetup + 127) / 128 > 0x7fffffffLL || nblk > 0x7fffffffLL) return GNA_EINVAL;
  k_scan_setup<<<(unsigned)((nsetup + 127) / 128), 128, 0, s>>>(
      a, g->theta12, g->theta13, g->dm2_21, g->dm2_31, edges, chi2 ? data : nullptr, w);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e);
  k_scan_expand<<<(unsigned)nblk, kScanThreads, 0, s>>>(g->nmix, nbins, nchunk, w, spectra,
                                                        chi2 ? data : nullptr, chi2);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  e = cudaGetLastError();
  return e == cudaSuccess ? GNA_OK : cuda_fail(e);
}

template <class Coef>
int launch_gl(const Coef& c, const double* edges, int64_t nbins, int order, double* bins,
              cudaStream_t s) {
  const int64_t grid = (2 * nbins + kGLLaneThreads - 1) / kGLLaneThreads;
  if (grid > 0x7fffffffLL) return GNA_EINVAL;
  const gl_kernel_t<Coef> kern =
      gl_kernel_for<Coef>(order, std::make_integer_sequence<int, GNA_MAX_ORDER>{});
  kern<<<(unsigned)grid, kGLLaneThreads, 0, s>>>(c, edges, nbins, bins);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GNA_OK : cuda_fail(e);
}

template <class Coef>
int launch_eval(const Coef& c, const double* E, int64_t n, double* P, cudaStream_t s) {
  const bool vec = ((((uintptr_t)E) | ((uintptr_t)P)) & 15) == 0;
  const int maxb = sm_count() * 8;
  if (vec && n >= (int64_t)kEvalTile * 4) {
    // persistent TMA-fed stream: GNA_EVAL_MINB blocks per SM (4 x 8 KiB smem ring each)
    const int64_t ntiles = n / kEvalTile;
    const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sm_count() * GNA_EVAL_MINB);
    k_oscprob_eval_tma<Coef><<<grid, kEvalTmaThreads, 0, s>>>(c, E, P, n);
  } else if (vec) {
    const int grid = grid_for((n + 1) / 2, kEvalThreads, maxb);
    k_oscprob_eval<true, Coef><<<grid, kEvalThreads, 0, s>>>(c, E, P, n);
  } else {
    const int grid = grid_for(n, kEvalThreads, maxb);
    k_oscprob_eval<false, Coef><<<grid, kEvalThreads, 0, s>>>(c, E, P, n);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GNA_OK : cuda_fail(e);
}

// ----------------------------------------------------------------------------
// staging for the *_host entry points (library-owned, per device)
// ----------------------------------------------------------------------------
struct Staging {
  bool init = false;
  cudaStream_t st[2] = {nullptr, nullptr};
  cudaEvent_t ev_in = nullptr;
  void* buf[2] = {nullptr, nullptr};  // per-stream chunk buffers
  size_t cap[2] = {0, 0};
  void* shared = nullptr;             // per-call shared inputs (edges, data)
  size_t shared_cap = 0;
};

std::mutex g_stage_mu;
Staging g_stage[128];

int ensure(void** p, size_t* cap, size_t need) {
  if (*cap >= need) return GNA_OK;
  if (*p) {
    cudaFree(*p);
    *p = nullptr;
    *cap = 0;
  }
  cudaError_t e = cudaMalloc(p, need);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return GNA_ENOMEM;
  }
  *cap = need;
  return GNA_OK;
}

int stage_init(Staging* S) {
  if (S->init) return GNA_OK;
  cudaError_t e;
  for (int i = 0; i < 2; ++i) {
    e = cudaStreamCreateWithFlags(&S->st[i], cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  e = cudaEventCreateWithFlags(&S->ev_in, cudaEventDisableTiming);
  if (e != cudaSuccess) return cuda_fail(e);
  S->init = true;
  return GNA_OK;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int gna_oscprob_eval(const gna_osc_params* p, double L_km, const double* d_E, int64_t n,
                     double* d_P, void* stream) {
  int rc = validate_eval(p, L_km, d_E, n, d_P);
  if (rc) return rc;
  if ((rc = check_device())) return rc;
  if (check_dev_ptr(d_E) || check_dev_ptr(d_P)) return GNA_EINVAL;
  PeeCoef c;
  make_coef(p, L_km, &c);
  return launch_eval(c, d_E, n, d_P, (cudaStream_t)stream);
}

int gna_oscprob_eval_ab(int32_t alpha, int32_t beta, const gna_osc_params* p, double L_km,
                        const double* d_E, int64_t n, double* d_P, void* stream) {
  if (alpha < 0 || alpha > 2 || beta < 0 || beta > 2) return GNA_EINVAL;
  int rc = validate_eval(p, L_km, d_E, n, d_P);
  if (rc) return rc;
  if ((rc = check_device())) return rc;
  if (check_dev_ptr(d_E) || check_dev_ptr(d_P)) return GNA_EINVAL;
  gna::PabCoef c;
  make_coef_ab(alpha, beta, p, L_km, &c);
  return launch_eval(c, d_E, n, d_P, (cudaStream_t)stream);
}

int gna_gl_integrate(const gna_osc_params* p, double L_km, const double* d_edges, int64_t nbins,
                     int32_t order, double* d_bins, void* stream) {
  int rc = validate_gl(p, L_km, d_edges, nbins, order, d_bins);
  if (rc) return rc;
  if ((rc = check_device())) return rc;
  if (check_dev_ptr(d_edges) || check_dev_ptr(d_bins)) return GNA_EINVAL;
  PeeCoef c;
  make_coef(p, L_km, &c);
  return launch_gl(c, d_edges, nbins, order, d_bins, (cudaStream_t)stream);
}

int gna_gl_integrate_ab(int32_t alpha, int32_t beta, const gna_osc_params* p, double L_km,
                        const double* d_edges, int64_t nbins, int32_t order, double* d_bins,
                        void* stream) {
  if (alpha < 0 || alpha > 2 || beta < 0 || beta > 2) return GNA_EINVAL;
  int rc = validate_gl(p, L_km, d_edges, nbins, order, d_bins);
  if (rc) return rc;
  if ((rc = check_device())) return rc;
  if (check_dev_ptr(d_edges) || check_dev_ptr(d_bins)) return GNA_EINVAL;
  gna::PabCoef c;
  make_coef_ab(alpha, beta, p, L_km, &c);
  return launch_gl(c, d_edges, nbins, order, d_bins, (cudaStream_t)stream);
}

int gna_gl_integrate_host(const gna_osc_params* p, double L_km, const double* h_edges,
                          int64_t nbins, int32_t order, double* h_bins, int64_t chunk,
                          void* stream) {
  int rc = validate_gl(p, L_km, h_edges, nbins, order, h_bins);
  if (rc) return rc;
  if ((rc = check_device())) return rc;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_stage_mu);
  Staging* S = &g_stage[dev];
  if ((rc = stage_init(S))) return rc;
  if (chunk <= 0) chunk = (int64_t)1 << 20;  // bins per chunk
  if (chunk > nbins) chunk = nbins;
  const size_t need = (size_t)(2 * chunk + 2) * 8;  // edges (chunk+1) + bins (chunk), aligned
  for (int i = 0; i < 2; ++i)
    if ((rc = ensure(&S->buf[i], &S->cap[i], need))) return rc;
  PeeCoef c;
  make_coef(p, L_km, &c);
  cudaError_t e = cudaEventRecord(S->ev_in, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e);
  for (int i = 0; i < 2; ++i)
    if ((e = cudaStreamWaitEvent(S->st[i], S->ev_in, 0)) != cudaSuccess) return cuda_fail(e);
  const int64_t nchunks = (nbins + chunk - 1) / chunk;
  for (int64_t ci = 0; ci < nchunks; ++ci) {
    const int si = (int)(ci & 1);
    cudaStream_t s = S->st[si];
    const int64_t o = ci * chunk;
    const int64_t m = (o + chunk <= nbins) ? chunk : nbins - o;
    double* dEd = (double*)S->buf[si];
    double* dB = dEd + chunk + 2;
    if ((e = cudaMemcpyAsync(dEd, h_edges + o, (size_t)(m + 1) * 8, cudaMemcpyHostToDevice, s)))
      return cuda_fail(e);
    if ((rc = launch_gl(c, dEd, m, order, dB, s))) return rc;
    if ((e = cudaMemcpyAsync(h_bins + o, dB, (size_t)m * 8, cudaMemcpyDeviceToHost, s)))
      return cuda_fail(e);
  }
  for (int i = 0; i < 2; ++i)
    if ((e = cudaStreamSynchronize(S->st[i])) != cudaSuccess) return cuda_fail(e);
  return GNA_OK;
}

size_t gna_oscprob_batch_workspace_size(int64_t npoints, int32_t nbase, int64_t nbins,
                                        int32_t order) {
  if (npoints < 1 || nbins < 1 || nbase < 1 || nbase > GNA_MAX_NBASE || order < 1 ||
      order > GNA_MAX_ORDER)
    return 0;
  return batch_ws_bytes(npoints, nbase, nbins, order, true);
}

int gna_oscprob_batch(const gna_param_batch* pts, const double* L_km, const double* omega,
                      int32_t nbase, const double* d_edges, int64_t nbins, int32_t order,
                      double* d_spectra, const double* d_data, double* d_chi2,
                      void* d_workspace, size_t workspace_bytes, void* stream) {
  int rc = validate_batch(pts, L_km, omega, nbase, d_edges, nbins, order, d_spectra, d_data,
                          d_chi2);
  if (rc) return rc;
  if (!d_workspace ||
      workspace_bytes < batch_ws_bytes(pts->npoints, nbase, nbins, order, d_chi2 != nullptr) ||
      ((uintptr_t)d_workspace & 15))
    return GNA_EINVAL;
  {
    const size_t W = batch_ws_bytes(pts->npoints, nbase, nbins, order, d_chi2 != nullptr);
    const size_t P8 = (size_t)pts->npoints * 8;
    const void* ins[8] = {pts->theta12, pts->theta13, pts->dm2_21, pts->dm2_31,
                          d_edges,      d_spectra,    d_data,     d_chi2};
    const size_t ln[8] = {P8, P8, P8, P8, (size_t)(nbins + 1) * 8,
                          (size_t)pts->npoints * (size_t)nbins * 8, (size_t)nbins * 8, P8};
    for (int i = 0; i < 8; ++i)
      if (ins[i] && overlap(d_workspace, W, ins[i], ln[i])) return GNA_EINVAL;
  }
  if ((rc = check_device())) return rc;
  const void* ptrs[9] = {pts->theta12, pts->theta13, pts->dm2_21, pts->dm2_31, d_edges,
                         d_spectra,    d_data,       d_chi2,      d_workspace};
  for (const void* q : ptrs)
    if (q && check_dev_ptr(q)) return GNA_EINVAL;
  return launch_batch(pts, L_km, omega, nbase, d_edges, nbins, order, d_spectra, d_data, d_chi2,
                      d_workspace, (cudaStream_t)stream);
}

size_t gna_oscprob_scan_workspace_size(int64_t nmix, int64_t nmass, int64_t nbins) {
  if (nmix < 1 || nmass < 1 || nbins < 1) return 0;
  return scan_ws_bytes(nmix, nmass, nbins);
}

int gna_oscprob_scan(const gna_scan_grid* g, const double* L_km, const double* omega,
                     int32_t nbase, const double* d_edges, int64_t nbins, int32_t order,
                     double* d_spectra, const double* d_data, double* d_chi2, void* d_workspace,
                     size_t workspace_bytes, void* stream) {
  if (!g || !g->theta12 || !g->theta13 || !g->dm2_21 || !g->dm2_31 || g->nmix < 1 ||
      g->nmass < 1 || !L_km || !omega || nbase < 1 || nbase > GNA_MAX_NBASE || !d_edges ||
      nbins < 1 || order < 1 || order > GNA_MAX_ORDER || (!d_spectra && !d_chi2) ||
      (d_chi2 && !d_data) || !d_workspace || ((uintptr_t)d_workspace & 31))
    return GNA_EINVAL;
  for (int b = 0; b < nbase; ++b)
    if (!is_fin(L_km[b]) || L_km[b] < 0 || !is_fin(omega[b])) return GNA_EINVAL;
  const size_t W = scan_ws_bytes(g->nmix, g->nmass, nbins);
  if (workspace_bytes < W) return GNA_EINVAL;
  const size_t P8 = (size_t)g->nmass * g->nmix * 8;
  const void* ins[9] = {g->theta12, g->theta13, g->dm2_21, g->dm2_31, d_edges, d_data,
                        d_spectra, d_chi2, d_workspace};
  const size_t ln[9] = {(size_t)g->nmix * 8, (size_t)g->nmix * 8, (size_t)g->nmass * 8,
                        (size_t)g->nmass * 8, (size_t)(nbins + 1) * 8, (size_t)nbins * 8,
                        P8 * (size_t)nbins, P8, W};
  for (int i = 5; i < 9; ++i)  // outputs and workspace vs everything else
    for (int j = 0; j < 9; ++j)
      if (i != j && ins[i] && ins[j] && overlap(ins[i], ln[i], ins[j], ln[j])) return GNA_EINVAL;
  int rc;
  if ((rc = check_device())) return rc;
  for (const void* q : ins)
    if (q && check_dev_ptr(q)) return GNA_EINVAL;
  return launch_scan(g, L_km, omega, nbase, d_edges, nbins, order, d_spectra, d_data, d_chi2,
                     d_workspace, (cudaStream_t)stream);
}

size_t gna_fit_workspace_size(int32_t nbase, int64_t nbins, int32_t order) {
  if (nbase < 1 || nbase > GNA_MAX_NBASE || nbins < 1 || order < 1 || order > GNA_MAX_ORDER)
    return 0;
  return align16((size_t)kFitDim * kFitCand * 8) + align16((size_t)kFitCand * 8) +
         batch_ws_bytes(kFitCand, nbase, nbins, order, true);
}

int gna_fit_pattern_search(const double* L_km, const double* omega, int32_t nbase,
                           const double* d_edges, int64_t nbins, int32_t order,
                           const double* d_data, double* d_state, int32_t niter, double* d_hist,
                           void* d_workspace, size_t workspace_bytes, void* stream) {
  if (!L_km || !omega || nbase < 1 || nbase > GNA_MAX_NBASE || !d_edges || nbins < 1 ||
      order < 1 || order > GNA_MAX_ORDER || !d_data || !d_state || niter < 0 || !d_workspace ||
      ((uintptr_t)d_workspace & 15) ||
      workspace_bytes < gna_fit_workspace_size(nbase, nbins, order))
    return GNA_EINVAL;
  for (int b = 0; b < nbase; ++b)
    if (!is_fin(L_km[b]) || L_km[b] < 0 || !is_fin(omega[b])) return GNA_EINVAL;
  int rc;
  if ((rc = check_device())) return rc;
  const void* ptrs[5] = {d_edges, d_data, d_state, d_hist, d_workspace};
  for (const void* q : ptrs)
    if (q && check_dev_ptr(q)) return GNA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  char* w = (char*)d_workspace;
  double* cand = (double*)w;
  w += align16((size_t)kFitDim * kFitCand * 8);
  double* chi2 = (double*)w;
  w += align16((size_t)kFitCand * 8);
  void* bws = w;
  const gna_param_batch pts = {cand, cand + kFitCand, cand + 2 * kFitCand, cand + 3 * kFitCand,
                               kFitCand};
  for (int it = 0; it < niter; ++it) {
    k_fit_candidates<<<1, 128, 0, s>>>(d_state, cand);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if ((rc = launch_batch(&pts, L_km, omega, nbase, d_edges, nbins, order, nullptr, d_data,
                           chi2, bws, s)))
      return rc;
    k_fit_update<<<1, 128, 0, s>>>(d_state, cand, chi2, d_hist, it);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e);
  }
  return GNA_OK;
}

int gna_oscprob_batch_ex(const gna_param_batch* pts, const double* L_km, const double* omega,
                         int32_t nbase, const double* d_edges, int64_t nbins, int32_t order,
                         double* d_spectra, const double* d_data, double* d_chi2,
                         void* d_workspace, size_t workspace_bytes, uint32_t flags,
                         void* stream) {
  const uint32_t known = GNA_OUT_PEER | GNA_OUT_MULTICAST;
  if ((flags & ~known) || ((flags & GNA_OUT_PEER) && (flags & GNA_OUT_MULTICAST)))
    return GNA_EINVAL;
  if (flags == 0)
    return gna_oscprob_batch(pts, L_km, omega, nbase, d_edges, nbins, order, d_spectra, d_data,
                             d_chi2, d_workspace, workspace_bytes, stream);
  int rc = validate_batch(pts, L_km, omega, nbase, d_edges, nbins, order, d_spectra, d_data,
                          d_chi2);
  if (rc) return rc;
  if (!d_workspace ||
      workspace_bytes < batch_ws_bytes(pts->npoints, nbase, nbins, order, d_chi2 != nullptr) ||
      ((uintptr_t)d_workspace & 15))
    return GNA_EINVAL;
  if ((rc = check_device())) return rc;
  // inputs and workspace must be this GPU's memory; the outputs are remote windows
  const void* ptrs[7] = {pts->theta12, pts->theta13, pts->dm2_21, pts->dm2_31, d_edges, d_data,
                         d_workspace};
  for (const void* q : ptrs)
    if (q && check_dev_ptr(q)) return GNA_EINVAL;
  return launch_batch(pts, L_km, omega, nbase, d_edges, nbins, order, d_spectra, d_data, d_chi2,
                      d_workspace, (cudaStream_t)stream,
                      (flags & GNA_OUT_MULTICAST) ? kOutMulticast : kOutPeer);
}

int gna_oscprob_eval_host(const gna_osc_params* p, double L_km, const double* h_E, int64_t n,
                          double* h_P, int64_t chunk, void* stream) {
  int rc = validate_eval(p, L_km, h_E, n, h_P);
  if (rc) return rc;
  if ((rc = check_device())) return rc;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_stage_mu);
  Staging* S = &g_stage[dev];
  if ((rc = stage_init(S))) return rc;
  if (chunk <= 0) chunk = (int64_t)1 << 22;  // 4 Mi elements = 32 MiB per direction
  if (chunk > n) chunk = n;
  chunk = (chunk + 1) & ~(int64_t)1;         // keep the double2 path aligned
  const size_t need = (size_t)chunk * 16;    // E and P halves
  for (int i = 0; i < 2; ++i)
    if ((rc = ensure(&S->buf[i], &S->cap[i], need))) return rc;
  PeeCoef c;
  make_coef(p, L_km, &c);
  cudaError_t e = cudaEventRecord(S->ev_in, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e);
  for (int i = 0; i < 2; ++i)
    if ((e = cudaStreamWaitEvent(S->st[i], S->ev_in, 0)) != cudaSuccess) return cuda_fail(e);
  int64_t nchunks = (n + chunk - 1) / chunk;
  for (int64_t ci = 0; ci < nchunks; ++ci) {
    const int si = (int)(ci & 1);
    cudaStream_t s = S->st[si];
    const int64_t o = ci * chunk;
    const int64_t m = (o + chunk <= n) ? chunk : n - o;
    double* dE = (double*)S->buf[si];
    double* dP = dE + chunk;
    if ((e = cudaMemcpyAsync(dE, h_E + o, (size_t)m * 8, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return cuda_fail(e);
    if ((rc = launch_eval(c, dE, m, dP, s))) return rc;
    if ((e = cudaMemcpyAsync(h_P + o, dP, (size_t)m * 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return cuda_fail(e);
  }
  for (int i = 0; i < 2; ++i)
    if ((e = cudaStreamSynchronize(S->st[i])) != cudaSuccess) return cuda_fail(e);
  return GNA_OK;
}

int gna_oscprob_batch_host(const gna_param_batch* h_pts, const double* L_km, const double* omega,
                           int32_t nbase, const double* h_edges, int64_t nbins, int32_t order,
                           double* h_spectra, const double* h_data, double* h_chi2,
                           int64_t chunk_points, void* stream) {
  int rc = validate_batch(h_pts, L_km, omega, nbase, h_edges, nbins, order, h_spectra, h_data,
                          h_chi2);
  if (rc) return rc;
  if ((rc = check_device())) return rc;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_stage_mu);
  Staging* S = &g_stage[dev];
  if ((rc = stage_init(S))) return rc;
  const int64_t P = h_pts->npoints;
  if (chunk_points <= 0) {
    // ~8 MiB of spectra per chunk, at least 1 point
    chunk_points = ((int64_t)8 << 20) / (nbins * 8);
    if (chunk_points < 1) chunk_points = 1;
  }
  if (chunk_points > P) chunk_points = P;
  // per-stream chunk buffer: workspace (16-aligned, first) + 4 param arrays + spectra + chi2
  const size_t ws_bytes = batch_ws_bytes(chunk_points, nbase, nbins, order, h_chi2 != nullptr);
  const size_t n_ws = ws_bytes / 8;
  const size_t n_par = 4 * (size_t)chunk_points;
  const size_t n_spec = h_spectra ? (size_t)chunk_points * nbins : 0;
  const size_t n_chi = h_chi2 ? (size_t)chunk_points : 0;
  const size_t need = (n_ws + n_par + n_spec + n_chi) * 8;
  for (int i = 0; i < 2; ++i)
    if ((rc = ensure(&S->buf[i], &S->cap[i], need))) return rc;
  const size_t n_shared = (size_t)(nbins + 1) + (h_data ? (size_t)nbins : 0);
  if ((rc = ensure(&S->shared, &S->shared_cap, n_shared * 8))) return rc;
  double* d_edges = (double*)S->shared;
  double* d_data = h_data ? d_edges + (nbins + 1) : nullptr;

  cudaError_t e;
  cudaStream_t s0 = S->st[0];
  if ((e = cudaEventRecord(S->ev_in, (cudaStream_t)stream)) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaStreamWaitEvent(s0, S->ev_in, 0)) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaMemcpyAsync(d_edges, h_edges, (size_t)(nbins + 1) * 8, cudaMemcpyHostToDevice, s0)))
    return cuda_fail(e);
  if (d_data &&
      (e = cudaMemcpyAsync(d_data, h_data, (size_t)nbins * 8, cudaMemcpyHostToDevice, s0)))
    return cuda_fail(e);
  if ((e = cudaEventRecord(S->ev_in, s0)) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaStreamWaitEvent(S->st[1], S->ev_in, 0)) != cudaSuccess) return cuda_fail(e);

  const double* hsrc[4] = {h_pts->theta12, h_pts->theta13, h_pts->dm2_21, h_pts->dm2_31};
  const int64_t nchunks = (P + chunk_points - 1) / chunk_points;
  for (int64_t ci = 0; ci < nchunks; ++ci) {
    const int si = (int)(ci & 1);
    cudaStream_t s = S->st[si];
    const int64_t o = ci * chunk_points;
    const int64_t m = (o + chunk_points <= P) ? chunk_points : P - o;
    double* base = (double*)S->buf[si];
    void* dws = base;
    double* dpar = base + n_ws;
    double* dspec = h_spectra ? dpar + n_par : nullptr;
    double* dchi = h_chi2 ? dpar + n_par + n_spec : nullptr;
    for (int a = 0; a < 4; ++a)
      if ((e = cudaMemcpyAsync(dpar + a * chunk_points, hsrc[a] + o, (size_t)m * 8,
                               cudaMemcpyHostToDevice, s)))
        return cuda_fail(e);
    gna_param_batch dp = {dpar, dpar + chunk_points, dpar + 2 * chunk_points,
                          dpar + 3 * chunk_points, m};
    if ((rc = launch_batch(&dp, L_km, omega, nbase, d_edges, nbins, order, dspec, d_data, dchi,
                           dws, s)))
      return rc;
    if (h_spectra && (e = cudaMemcpyAsync(h_spectra + o * nbins, dspec, (size_t)m * nbins * 8,
                                          cudaMemcpyDeviceToHost, s)))
      return cuda_fail(e);
    if (h_chi2 &&
        (e = cudaMemcpyAsync(h_chi2 + o, dchi, (size_t)m * 8, cudaMemcpyDeviceToHost, s)))
      return cuda_fail(e);
  }
  for (int i = 0; i < 2; ++i)
    if ((e = cudaStreamSynchronize(S->st[i])) != cudaSuccess) return cuda_fail(e);
  return GNA_OK;
}

void gna_release(void) {
  std::lock_guard<std::mutex> lk(g_stage_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (int d = 0; d < 128; ++d) {
    Staging* S = &g_stage[d];
    if (!S->init && !S->buf[0] && !S->buf[1] && !S->shared) continue;
    cudaSetDevice(d);
    for (int i = 0; i < 2; ++i) {
      if (S->st[i]) cudaStreamSynchronize(S->st[i]);
      if (S->buf[i]) cudaFree(S->buf[i]);
      if (S->st[i]) cudaStreamDestroy(S->st[i]);
      S->buf[i] = nullptr;
      S->cap[i] = 0;
      S->st[i] = nullptr;
    }
    if (S->shared) cudaFree(S->shared);
    if (S->ev_in) cudaEventDestroy(S->ev_in);
    *S = Staging();
  }
  cudaSetDevice(cur);
}

int gna_gl_rule(int32_t order, double* t, double* w) {
  if (order < 1 || order > GNA_MAX_ORDER || !t || !w) return GNA_EINVAL;
  const int off = GNA_GL_OFF(order);
  for (int i = 0; i < order; ++i) {
    t[i] = h_gl_t[off + i];
    w[i] = h_gl_w[off + i];
  }
  return GNA_OK;
}

const char* gna_strerror(int code) {
  switch (code) {
    case GNA_OK: return "GNA_OK: success";
    case GNA_EINVAL: return "GNA_EINVAL: invalid argument";
    case GNA_ECUDA: return "GNA_ECUDA: CUDA call or kernel launch failed (see gna_last_cuda_error)";
    case GNA_ENODEV: return "GNA_ENODEV: current device is not sm_100 (B200)";
    case GNA_ENOMEM: return "GNA_ENOMEM: staging allocation failed";
    default: return "unknown gna_status";
  }
}

int gna_last_cuda_error(void) { return t_last_cuda_error; }

int gna_abi_version(void) { return GNA_ABI_VERSION; }

int64_t gna_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

}  // extern "C"

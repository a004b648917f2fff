// k_gl.cuh — (a3)+(a4) single-point Gauss-Legendre kernel
// Part of libgna_b200.so: included once, from gna_b200.cu (single translation unit).
#pragma once
#include <type_traits>
#include <utility>

#include "gna_common.cuh"

namespace {

// (a3)+(a4) one parameter point.  A lane pair owns one bin: lane 2m+h evaluates the
// nodes [h*H, min((h+1)*H, order)), H = ceil(order/2), fully unrolled (compile-time
// order), so each lane runs H independent reciprocal + 3 sin^2 chains; the two
// halves are combined with one shuffle.  The whole grid is resident in one wave, so
// the bin edges' DRAM latency is paid once.  GL nodes/weights are read per lane
// from a global (L1) copy of the table.
#ifndef GNA_GL_MINB
#define GNA_GL_MINB 8
#endif
constexpr int kGLLaneThreads = 128;

template <int kOrder, class Coef>
__global__ void __launch_bounds__(kGLLaneThreads, GNA_GL_MINB) k_gl_integrate(Coef c,
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
  pdl_launch_dependents();
  pdl_wait();
  const double e0 = edges[kk], e1 = edges[kk + 1];
  const double ctr = 0.5 * (e0 + e1);
  const double h = 0.5 * (e1 - e0);
  double iE[H], pv[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const int node = half * H + i < kOrder ? half * H + i : kOrder - 1;
    iE[i] = gna::rcp(fma(h, __ldg(&g_gl_t[off + node]), ctr));
  }
  gna::prob_inv_n<H>(c, iE, pv);
  // s_half = sum over the lane's nodes, ascending, of w_i P_i (explicit FMAs: the same
  // arithmetic as k_gl_integrate_tb, so a bin's value does not depend on nbins)
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const int node = half * H + i;
    if (node < kOrder) s = fma(__ldg(&g_gl_w[off + node]), pv[i], s);
  }
  const double other = __shfl_xor_sync(0xffffffffu, s, 1);
  if (act && half == 0) bins[k] = h * (s + other);
}

// Large nbins: one thread per bin.  All lanes of a warp visit the same node index at the
// same time, so the GL nodes and weights come from the constant bank as uniform operands
// (no table loads); the nodes are taken G at a time (G divides the order when it can),
// each group's reciprocals and three sin^2 terms forming G independent chains.  The
// weighted node sum is formed exactly as in the lane-pair kernel (two ascending halves,
// then h (s0 + s1)), so both kernels give the same bits for a bin.  Measured against the
// lane-pair kernel (tools/gl_sweep.py, profiles/r01_gl_sweep.jsonl): equal up to 10^5 bins
// (both at the launch floor), 1.12x (GL10) / 1.38x (GL5) at 10^6 bins, 1.13x / 1.41x at 10^7.
#ifndef GNA_GL_TB_MINB
#define GNA_GL_TB_MINB 4
#endif
// nbins from which the thread-per-bin kernel is used, per coefficient type (below: lane
// pairs).  Back-to-back launch times, tools/gl_b2b.py (profiles/r01_gl_b2b.jsonl): P_ee fp64
// is faster (or equal) with thread per bin than with lane pairs at every size from 1 bin up
// (cfg1 1.79 -> 1.54 us, cfg2 4.76 -> 4.53 us), so the lane-pair kernel is not even built for
// it (launch_gl); small P_ee grids take the warp-split kernel below instead.  The mixed tier
// and the general channel are faster with lane pairs up to ~10^5 bins and with thread per bin
// at 10^6.
#ifndef GNA_GL_TB_MIN_BINS
#define GNA_GL_TB_MIN_BINS 1
#endif
#ifndef GNA_GL_TB_MIN_BINS_MIXED
#define GNA_GL_TB_MIN_BINS_MIXED 131072
#endif
#ifndef GNA_GL_TB_MIN_BINS_AB
#define GNA_GL_TB_MIN_BINS_AB 262144
#endif
template <class Coef>
constexpr int64_t gl_tb_min_bins() {
  return std::is_same<Coef, gna::PeeCoef>::value       ? (int64_t)GNA_GL_TB_MIN_BINS
         : std::is_same<Coef, gna::PeeMixCoef>::value ? (int64_t)GNA_GL_TB_MIN_BINS_MIXED
                                                       : (int64_t)GNA_GL_TB_MIN_BINS_AB;
}
#ifndef GNA_GL_TB_THREADS
#define GNA_GL_TB_THREADS 128
#endif
constexpr int kGLTbThreads = GNA_GL_TB_THREADS;

__host__ __device__ constexpr int gl_group(int order) {
  return order % 5 == 0 ? 5 : order % 4 == 0 ? 4 : order % 3 == 0 ? 3 : order < 5 ? order : 5;
}

template <int kOrder, class Coef>
__global__ void __launch_bounds__(kGLTbThreads, GNA_GL_TB_MINB) k_gl_integrate_tb(
    Coef c, const double* __restrict__ edges, int64_t nbins, double* __restrict__ bins) {
  constexpr int G = gl_group(kOrder);
  constexpr int off = GNA_GL_OFF(kOrder);
  const int64_t k = (int64_t)blockIdx.x * kGLTbThreads + threadIdx.x;
  pdl_launch_dependents();
  if (k >= nbins) return;
  pdl_wait();
  const double e0 = edges[k], e1 = edges[k + 1];
  const double ctr = 0.5 * (e0 + e1);
  const double h = 0.5 * (e1 - e0);
  constexpr int H = (kOrder + 1) / 2;
  double s0 = 0.0, s1 = 0.0;  // nodes [0, H) and [H, order): the lane-pair kernel's halves
#pragma unroll
  for (int i0 = 0; i0 < kOrder; i0 += G) {
    const int n = kOrder - i0 < G ? kOrder - i0 : G;
    double iE[G], pv[G];
#pragma unroll
    for (int i = 0; i < G; ++i) iE[i] = gna::rcp(fma(h, c_gl_t[off + (i < n ? i0 + i : i0)], ctr));
    gna::prob_inv_n<G>(c, iE, pv);
#pragma unroll
    for (int i = 0; i < G; ++i) {
      if (i < n) {
        if (i0 + i < H)
          s0 = fma(c_gl_w[off + i0 + i], pv[i], s0);
        else
          s1 = fma(c_gl_w[off + i0 + i], pv[i], s1);
      }
    }
  }
  bins[k] = h * (s0 + s1);
}

// Sum over the nodes [kLo, kHi) of one bin, ascending, w_i P(c + h t_i) accumulated with
// FMAs, the nodes taken G at a time (independent reciprocal + sin^2 chains).  A node's P does
// not depend on the group it is evaluated in, so any grouping gives the same bits.
template <int kOrder, int kLo, int kHi, class Coef>
__device__ __forceinline__ double gl_nodes_sum(const Coef& c, double ctr, double h) {
  constexpr int off = GNA_GL_OFF(kOrder);
  constexpr int G = gl_group(kHi - kLo > 0 ? kHi - kLo : 1);
  double s = 0.0;
#pragma unroll
  for (int i0 = kLo; i0 < kHi; i0 += G) {
    const int n = kHi - i0 < G ? kHi - i0 : G;
    double iE[G], pv[G];
#pragma unroll
    for (int i = 0; i < G; ++i) iE[i] = gna::rcp(fma(h, c_gl_t[off + (i < n ? i0 + i : i0)], ctr));
    gna::prob_inv_n<G>(c, iE, pv);
#pragma unroll
    for (int i = 0; i < G; ++i)
      if (i < n) s = fma(c_gl_w[off + i0 + i], pv[i], s);
  }
  return s;
}

// Grids smaller than a few waves (cfg2: 10^5 bins = 0.75 waves of the thread-per-bin kernel,
// 25 % of the warps active): the two node halves of a bin run in two different warps of one
// block — warp w < BW takes nodes [0, H) of 32 bins, warp BW + w nodes [H, order) of the same
// bins — and meet in shared memory: bins[k] = h (s0 + s1), the thread-per-bin kernel's
// arithmetic to the bit.  Twice the threads, half the dependent chain per thread, and node
// indices stay warp-uniform (constant-bank operands).
#ifndef GNA_GL_SPLIT
#define GNA_GL_SPLIT 1
#endif
#ifndef GNA_GL_SPLIT_BW
#define GNA_GL_SPLIT_BW 2
#endif
#ifndef GNA_GL_SPLIT_MINB
#define GNA_GL_SPLIT_MINB 4
#endif
// P_ee fp64 takes the split kernel for 2 <= order and nbins <= this (above: thread per bin)
#ifndef GNA_GL_SPLIT_MAX_BINS
#define GNA_GL_SPLIT_MAX_BINS 262144
#endif
constexpr int kGLSplitBW = GNA_GL_SPLIT_BW;
constexpr int kGLSplitThreads = 64 * kGLSplitBW;

template <int kOrder, class Coef>
__global__ void __launch_bounds__(kGLSplitThreads, GNA_GL_SPLIT_MINB) k_gl_integrate_split(
    Coef c, const double* __restrict__ edges, int64_t nbins, double* __restrict__ bins) {
  constexpr int H = (kOrder + 1) / 2;
  __shared__ double s_hi[32 * kGLSplitBW];
  const int warp = threadIdx.x >> 5;
  const int upper = warp >= kGLSplitBW;  // warp-uniform
  const int slot = (warp - upper * kGLSplitBW) * 32 + (threadIdx.x & 31);
  const int64_t k = (int64_t)blockIdx.x * (32 * kGLSplitBW) + slot;
  const int64_t kk = k < nbins ? k : nbins - 1;
  pdl_launch_dependents();
  pdl_wait();
  const double e0 = edges[kk], e1 = edges[kk + 1];
  const double ctr = 0.5 * (e0 + e1);
  const double h = 0.5 * (e1 - e0);
  double s;
  if (upper) {
    s = gl_nodes_sum<kOrder, H, kOrder>(c, ctr, h);
    s_hi[slot] = s;
  } else {
    s = gl_nodes_sum<kOrder, 0, H>(c, ctr, h);
  }
  __syncthreads();
  if (!upper && k < nbins) bins[k] = h * (s + s_hi[slot]);
}

template <class Coef>
using gl_kernel_t = void (*)(Coef, const double*, int64_t, double*);

template <class Coef, int... N>
gl_kernel_t<Coef> gl_split_kernel_for(int order, std::integer_sequence<int, N...>) {
  static const gl_kernel_t<Coef> t[] = {k_gl_integrate_split<N + 1, Coef>...};
  return t[order - 1];
}

template <class Coef, int... N>
gl_kernel_t<Coef> gl_kernel_for(int order, std::integer_sequence<int, N...>) {
  static const gl_kernel_t<Coef> t[] = {k_gl_integrate<N + 1, Coef>...};
  return t[order - 1];
}

template <class Coef, int... N>
gl_kernel_t<Coef> gl_tb_kernel_for(int order, std::integer_sequence<int, N...>) {
  static const gl_kernel_t<Coef> t[] = {k_gl_integrate_tb<N + 1, Coef>...};
  return t[order - 1];
}

}  // namespace

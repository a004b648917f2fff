// k_gl.cuh — (a3)+(a4) single-point Gauss-Legendre kernel
// Part of libgna_b200.so: included once, from gna_b200.cu (single translation unit).
#pragma once
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
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const int node = half * H + i;
    pv[i] = node < kOrder ? __ldg(&g_gl_w[off + node]) * pv[i] : 0.0;
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

}  // namespace

// k_fit.cuh — NEXT-4b on-GPU chi^2 pattern-search kernels
// Part of libgna_b200.so: included once, from gna_b200.cu (single translation unit).
#pragma once
#include "gna_common.cuh"

namespace {

// ----------------------------------------------------------------------------
// NEXT-4 (second part): a chi^2 minimiser that stays on the GPU (the fit of P:446-451).
// Deterministic compass/pattern search over (theta12, theta13, dm2_21, dm2_31): every
// iteration evaluates the 3^4 = 81 points centre + step * {-1, 0, +1}^4 with the batch
// kernels (chi^2 only), takes the argmin (lowest index on ties), moves the centre there,
// or halves the steps if the centre is already best.  The whole loop is stream-ordered
// (no host round trip), so it can be captured in one CUDA graph.
constexpr int kFitDim = 4;
constexpr int kFitCand = 81;  // 3^4

// state = {centre[4], step[4]} (device, fp64); candidate c of the current state
__device__ __forceinline__ void fit_candidate(const double* __restrict__ state,
                                              double* __restrict__ cand, int c) {
  int code = c;
#pragma unroll
  for (int d = 0; d < kFitDim; ++d) {
    const int o = code % 3 - 1;  // -1, 0, +1 ; candidate 40 is the centre
    code /= 3;
    cand[d * kFitCand + c] = fma((double)o, state[kFitDim + d], state[d]);
  }
}

// the first iteration's candidates (later ones are written by k_fit_update)
__global__ void __launch_bounds__(128) k_fit_candidates(const double* __restrict__ state,
                                                        double* __restrict__ cand) {
  if (threadIdx.x < kFitCand) fit_candidate(state, cand, threadIdx.x);
}

// argmin + move/halve, then (next_cand) the next iteration's candidates from the new state:
// one launch per iteration fewer than a separate candidates kernel
__global__ void __launch_bounds__(128) k_fit_update(double* __restrict__ state,
                                                    double* __restrict__ cand,
                                                    const double* __restrict__ chi2,
                                                    double* __restrict__ hist, int iter,
                                                    int next_cand) {
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
  if (next_cand) {
    __syncthreads();  // thread 0's state update (and its reads of cand) are complete
    if (t < kFitCand) fit_candidate(state, cand, t);
  }
}

// ----------------------------------------------------------------------------
// Separable stencil (GNA_FIT_SCAN, default): the 81 candidates are the Cartesian product of 9
// mixing points (theta12, theta13) and 9 mass points (dm2_21, dm2_31), and candidate
// c = i0 + 3 i1 + 9 i2 + 27 i3 is mixing point i0 + 3 i1 of mass point i2 + 3 i3 — exactly the
// NEXT-1 scan's point order (mass-major).  So one iteration is one gna_oscprob_scan over a
// 9 x 9 grid: the binned sin^2 sums are formed for 9 mass points instead of 81 candidates
// (P:439-440), and the mixing weights enter linearly.  Candidate coordinates are the same
// fma(o, step, centre) values as fit_candidate's, so the state sequence is unchanged whenever
// the argmin is.
#ifndef GNA_FIT_SCAN
#define GNA_FIT_SCAN 1
#endif
constexpr int kFitGrid = 9;  // 3^2 mixing points, 3^2 mass points

// grid arrays [theta12[9] | theta13[9] | dm2_21[9] | dm2_31[9]] of the current state
__device__ __forceinline__ void fit_grid(const double* __restrict__ state,
                                         double* __restrict__ grid, int t) {
  if (t < kFitGrid) {
    const int o0 = t % 3 - 1, o1 = t / 3 - 1;
    grid[t] = fma((double)o0, state[kFitDim + 0], state[0]);
    grid[kFitGrid + t] = fma((double)o1, state[kFitDim + 1], state[1]);
    grid[2 * kFitGrid + t] = fma((double)o0, state[kFitDim + 2], state[2]);
    grid[3 * kFitGrid + t] = fma((double)o1, state[kFitDim + 3], state[3]);
  }
}

__global__ void __launch_bounds__(128) k_fit_grid(const double* __restrict__ state,
                                                  double* __restrict__ grid) {
  pdl_launch_dependents();
  pdl_wait();  // launched with PDL (GNA_PDL_SCAN): the predecessor's writes are visible
  fit_grid(state, grid, threadIdx.x);
}

// argmin + move/halve as k_fit_update; the best candidate's coordinates are rebuilt from the
// old state (the same fma as fit_candidate), then the next grid is written
// GNA_FIT_FOLD: with partial != nullptr the chi^2 of candidate t is folded here from stage B's
// nbc bin-chunk partials in chunk order — k_scan_chi2_fold's sum, one launch per iteration fewer
#ifndef GNA_FIT_FOLD
#define GNA_FIT_FOLD 1
#endif
__global__ void __launch_bounds__(128) k_fit_update_grid(double* __restrict__ state,
                                                         double* __restrict__ grid,
                                                         const double* __restrict__ chi2,
                                                         const double* __restrict__ partial,
                                                         int64_t nbc,
                                                         double* __restrict__ hist, int iter,
                                                         int next_grid) {
  __shared__ double s_v[128];
  __shared__ double s_c[kFitCand];
  __shared__ int s_i[128];
  const int t = threadIdx.x;
  pdl_launch_dependents();
  pdl_wait();  // launched with PDL (GNA_PDL_SCAN): stage B's chi^2 is complete and visible
  double x = INFINITY;
  if (t < kFitCand) {
    if (partial) {
      x = 0.0;
      for (int64_t j = 0; j < nbc; ++j) x += partial[t * nbc + j];
    } else {
      x = chi2[t];
    }
    s_c[t] = x;
  }
  s_v[t] = x;
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
    if (best == centre || !(s_v[0] < s_c[centre])) {
#pragma unroll
      for (int d = 0; d < kFitDim; ++d) state[kFitDim + d] *= 0.5;
    } else {
      double nc[kFitDim];
      int code = best;
#pragma unroll
      for (int d = 0; d < kFitDim; ++d) {
        const int o = code % 3 - 1;
        code /= 3;
        nc[d] = fma((double)o, state[kFitDim + d], state[d]);
      }
#pragma unroll
      for (int d = 0; d < kFitDim; ++d) state[d] = nc[d];
    }
    if (hist) hist[iter] = fmin(s_v[0], s_c[centre]);
  }
  if (next_grid) {
    __syncthreads();  // thread 0's state update is complete
    fit_grid(state, grid, t);
  }
}

}  // namespace

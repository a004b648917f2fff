// k_eval.cuh — (a3) elementwise kernels: grid-stride and TMA-fed streaming
// Part of libgna_b200.so: included once, from gna_b200.cu (single translation unit).
#pragma once
#include "gna_common.cuh"
#include "gna_tma.cuh"

namespace {

template <bool kVec, class Coef>
__global__ void __launch_bounds__(kEvalThreads) k_oscprob_eval(Coef c,
                                                               const double* __restrict__ E,
                                                               double* __restrict__ P, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  pdl_launch_dependents();
  pdl_wait();
  if (kVec) {
    const int64_t n2 = n >> 1;
    const double2* __restrict__ E2 = reinterpret_cast<const double2*>(E);
    double2* __restrict__ P2 = reinterpret_cast<double2*>(P);
    for (int64_t i = tid; i < n2; i += stride) {
      const double2 e = __ldcs(E2 + i);
      const double2 r = gna::prob_pair(c, gna::rcp(e.x), gna::rcp(e.y));
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
#ifndef GNA_EVAL_BULK_STORE
#define GNA_EVAL_BULK_STORE 0
#endif
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
  pdl_launch_dependents();
  pdl_wait();  // before the first read of E (a predecessor may have written it)
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
#if GNA_EVAL_BULK_STORE
    // results overwrite the inputs in the same stage (each thread owns its slots), then one
    // thread hands the whole 8 KiB tile to the bulk-copy engine (no per-thread stores)
    double2* buf = reinterpret_cast<double2*>(s_buf[st]);
#pragma unroll
    for (int j = threadIdx.x; j < kEvalTile / 2; j += kEvalTmaThreads) {
      const double2 e = buf[j];
      const double2 r = gna::prob_pair(c, gna::rcp(e.x), gna::rcp(e.y));
      buf[j] = r;
    }
    gna::fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      gna::bulk_s2g(P + tile * kEvalTile, s_buf[st], kEvalTile * 8);
      gna::bulk_commit();
      if (it + kEvalStages < mine) {
        gna::bulk_wait_read<0>();  // the store has read stage st before it is refilled
        gna::mbar_expect_tx(&s_full[st], kEvalTile * 8);
        gna::bulk_g2s(s_buf[st], E + (first + (it + kEvalStages) * stride) * kEvalTile,
                      kEvalTile * 8, &s_full[st]);
      }
    }
  }
  if (threadIdx.x == 0) gna::bulk_wait_all();
#else
    const double2* src = reinterpret_cast<const double2*>(s_buf[st]);
    double2* dst = reinterpret_cast<double2*>(P + tile * kEvalTile);
#pragma unroll
    for (int j = threadIdx.x; j < kEvalTile / 2; j += kEvalTmaThreads) {
      const double2 e = src[j];
      const double2 r = gna::prob_pair(c, gna::rcp(e.x), gna::rcp(e.y));
      __stcs(dst + j, r);
    }
    __syncthreads();  // every thread is done with stage st before it is refilled
    if (threadIdx.x == 0 && it + kEvalStages < mine) {
      gna::mbar_expect_tx(&s_full[st], kEvalTile * 8);
      gna::bulk_g2s(s_buf[st], E + (first + (it + kEvalStages) * stride) * kEvalTile,
                    kEvalTile * 8, &s_full[st]);
    }
  }
#endif
  if (blockIdx.x == 0)
    for (int64_t i = ntiles * kEvalTile + threadIdx.x; i < n; i += kEvalTmaThreads)
      P[i] = gna::prob_inv(c, gna::rcp(E[i]));
}

}  // namespace

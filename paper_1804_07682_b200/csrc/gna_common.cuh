// gna_common.cuh — constants, GL tables, shared host/device helpers
// Part of libgna_b200.so: included once, from gna_b200.cu (single translation unit).
#pragma once
#include <atomic>
#include <cstdint>

#include "../../include/gna_b200.h"
#include "gl_table.h"
#include "gna_device.cuh"

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

// Programmatic dependent launch (sm_90+; GNA_PDL): a kernel launched with the
// programmatic-stream-serialization attribute may start while its predecessor on the stream
// finishes; it waits here (griddepcontrol.wait: the predecessor grid has completed and its
// memory is visible) before it reads anything a predecessor may have written.  The batch main
// pass and chi2 reduce wait for their setup / main pass; the single-point GL and elementwise
// kernels (GNA_PDL_SINGLE) wait before their first input load, so only launch latency and
// block rasterisation overlap the previous call — never a read of its outputs.  Without a
// programmatic dependency both instructions are no-ops.
#ifndef GNA_PDL
#define GNA_PDL 1
#endif
#ifndef GNA_PDL_SINGLE
#define GNA_PDL_SINGLE 1
#endif
__device__ __forceinline__ void pdl_wait() {
#if GNA_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_launch_dependents() {
#if GNA_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// ----------------------------------------------------------------------------
// kernels
size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }
size_t align32(size_t x) { return (x + 31) & ~(size_t)31; }

int64_t warps_per_point(int64_t nbins) { return (nbins + 31) / 32; }

}  // namespace

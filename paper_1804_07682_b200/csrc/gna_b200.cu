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
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <complex>
#include <utility>
#include <mutex>
#include <vector>

#include "../../include/gna_b200.h"
#include "gna_common.cuh"
#include "k_batch.cuh"
#include "k_eval.cuh"
#include "k_fit.cuh"
#include "k_gl.cuh"
#include "k_scan.cuh"

using gna::PeeCoef;

namespace {

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

// NEXT-3 mixed tier: the same coefficients with kq halved (exact) and the weights in fp32
void make_coef_mix(const gna_osc_params* p, double L_km, gna::PeeMixCoef* c) {
  PeeCoef d;
  make_coef(p, L_km, &d);
  for (int j = 0; j < 3; ++j) {
    c->kqh[j] = 0.5 * d.kq[j];
    c->w[j] = (float)d.w[j];
  }
  c->c0 = d.c0;
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

// SM count of the current device (cached per device; 148 on B200)
int sm_count() {
  static std::atomic<int> cached[128];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 128) return 148;
  int v = cached[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cached[dev].store(v, std::memory_order_relaxed);
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

// <<<grid, block, smem, s>>> with the programmatic-stream-serialization attribute (PDL): the
// kernel may start while its predecessor on the stream finishes; it synchronises in-kernel
// (pdl_wait) before touching the predecessor's outputs.
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = GNA_PDL ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// scan and scan-fit kernels (k_scan_*, k_fit_grid, k_fit_update_grid): PDL when GNA_PDL_SCAN;
// each of them executes pdl_launch_dependents + pdl_wait on entry, before any load or store,
// so only the next kernel's launch and block rasterisation overlap this one's tail (stage B
// after stage A, and the fit's five kernels per iteration)
#ifndef GNA_PDL_SCAN
#define GNA_PDL_SCAN 1
#endif
template <class... KArgs, class... Args>
cudaError_t launch_pdl_scan(void (*kern)(KArgs...), unsigned grid, unsigned block,
                            cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (GNA_PDL && GNA_PDL_SCAN) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// single-point kernels (GL, elementwise): PDL when GNA_PDL_SINGLE (they wait before their
// first input load, gna_common.cuh), else a plain stream-ordered launch
template <class... KArgs, class... Args>
cudaError_t launch_pdl_single(void (*kern)(KArgs...), unsigned grid, unsigned block,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (GNA_PDL && GNA_PDL_SINGLE) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

#ifndef GNA_BATCH_PT_BPSM
#define GNA_BATCH_PT_BPSM 0
#endif
// launch of the batch kernels on already-validated device arguments
template <int kOut, bool kMixed>
int launch_batch_k(const gna_param_batch* pts, const double* L_km, const double* omega,
                   int32_t nbase, const double* edges, int64_t nbins, int32_t order,
                   double* spectra, const double* data, double* chi2, void* workspace,
                   cudaStream_t s, const double* tables) {
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
  BatchWs w = batch_ws_carve(workspace, pts->npoints, nbase, nbins, order, chi2 != nullptr);
  // tables: node tables built earlier (invE at tables, hw right after, batch_ws_carve's
  // layout); the setup kernel then only forms the per-point coefficients
  a.tables = tables == nullptr;
  if (tables) {
    w.invE = const_cast<double*>(tables);
    w.hw = (double*)((char*)w.invE + align16((size_t)order * nbins * sizeof(double)));
  }
  const int64_t bpp = blocks_per_point(nbins);
  // points per warp: enough sin^2 work per lane to amortise the per-point overhead
  // (>= GNA_BATCH_PPW_WORK_BIG; >= GNA_BATCH_PPW_WORK for the small-nbase points-inner
  // kernel), while keeping >= 16 warps per SM worth of blocks — for the per-point kernel
  // >= GNA_BATCH_PPW_MIN_WAVES such waves, so the longer warps do not leave a costly last
  // wave (cfg5: ppw 2, +0.5 %; the 81-point fit step stays at ppw 1, where ppw 2 lost 2 %)
  const int64_t work = (int64_t)3 * nbase * order;
  const bool small_terms = 3 * nbase <= GNA_BATCH_PI_MAX_TERMS;
  int64_t ppw = std::max<int64_t>(
      1, ((small_terms ? GNA_BATCH_PPW_WORK : GNA_BATCH_PPW_WORK_BIG) + work - 1) / work);
  const int64_t min_blocks =
      (int64_t)sm_count() * 16 * (small_terms ? 1 : GNA_BATCH_PPW_MIN_WAVES);
  while (ppw > 1 && ((pts->npoints + ppw - 1) / ppw) * bpp < min_blocks) ppw >>= 1;
  const int64_t ngroups = (pts->npoints + ppw - 1) / ppw;
  const int64_t nblocks = ngroups * bpp;
  const int64_t nsetup = pts->npoints * nbase + (a.tables ? (int64_t)order * nbins : 0);
  if (nblocks > 0x7fffffffLL || (nsetup + 255) / 256 > 0x7fffffffLL) return GNA_EINVAL;

  k_batch_setup<<<(unsigned)((nsetup + 255) / 256), 256, 0, s>>>(
      a, pts->theta12, pts->theta13, pts->dm2_21, pts->dm2_31, edges, w);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e);

  const int nterm = 3 * nbase;
  const size_t smem = (size_t)kBatchWarps * nterm * sizeof(double2);
  // node-group size: 5, 4 or 3 when it divides the order, else 4
  auto kern = (order % 5 == 0)   ? k_oscprob_batch<kBatchWarps, 5, kOut, kMixed>
              : (order % 4 == 0) ? k_oscprob_batch<kBatchWarps, 4, kOut, kMixed>
              : (order % 3 == 0) ? k_oscprob_batch<kBatchWarps, 3, kOut, kMixed>
                                 : k_oscprob_batch<kBatchWarps, 4, kOut, kMixed>;
#if GNA_MIXED_N10
  // mixed tier: 10 nodes (5 packed pairs) per coefficient load when the order allows
  if (kMixed && order % 10 == 0) kern = k_oscprob_batch<kBatchWarps, 10, kOut, kMixed>;
#endif
#if GNA_BATCH_N10_FP64
  if (!kMixed && order % 10 == 0) kern = k_oscprob_batch<kBatchWarps, 10, kOut, kMixed>;
#endif
  int pt_sub = 1;  // chi2 sub-partials per tile (k_oscprob_batch_pt)
  if ((GNA_BATCH_PT_MIXED || !kMixed) && GNA_BATCH_PT && kBatchWarps == 1 &&
      (nterm == 3 || nterm == 6) && pts->npoints >= GNA_BATCH_PT_MIN_POINTS) {
    // many points, few terms: points across lanes, 32-bin tiles (bitwise-identical sums)
    auto kpt = (order % 5 == 0)   ? k_oscprob_batch_pt<5, 3, kOut, kMixed>
               : (order % 4 == 0) ? k_oscprob_batch_pt<4, 3, kOut, kMixed>
               : (order % 3 == 0) ? k_oscprob_batch_pt<3, 3, kOut, kMixed>
                                  : k_oscprob_batch_pt<4, 3, kOut, kMixed>;
    if (nterm == 6)
      kpt = (order % 5 == 0)   ? k_oscprob_batch_pt<5, 6, kOut, kMixed>
            : (order % 4 == 0) ? k_oscprob_batch_pt<4, 6, kOut, kMixed>
            : (order % 3 == 0) ? k_oscprob_batch_pt<3, 6, kOut, kMixed>
                               : k_oscprob_batch_pt<4, 6, kOut, kMixed>;
#if GNA_BATCH_PT_MIXED_N10
    if (kMixed && order % 10 == 0)
      kpt = nterm == 3 ? k_oscprob_batch_pt<10, 3, kOut, kMixed> : k_oscprob_batch_pt<10, 6, kOut, kMixed>;
#if GNA_BATCH_PT_ORD10
    if (kMixed && order == 10)
      kpt = nterm == 3 ? k_oscprob_batch_pt<10, 3, kOut, kMixed, 10>
                       : k_oscprob_batch_pt<10, 6, kOut, kMixed, 10>;
#endif
#endif
#if GNA_BATCH_PT_N10
    if (order % 10 == 0)
      kpt = nterm == 3 ? k_oscprob_batch_pt<10, 3, kOut, kMixed> : k_oscprob_batch_pt<10, 6, kOut, kMixed>;
#endif
#if GNA_BATCH_PT_ORD10
    // GL10 (the reactor configurations): the order as a compile-time constant
    if (!kMixed && order == 10)
      kpt = nterm == 3 ? k_oscprob_batch_pt<5, 3, kOut, kMixed, 10>
                       : k_oscprob_batch_pt<5, 6, kOut, kMixed, 10>;
#endif
    const int64_t ng = (pts->npoints + 31) / 32;
    size_t smem_pt = (size_t)(2 * order + 3) * 32 * sizeof(double);
    if (GNA_BATCH_PT_SHARED21)  // shared sin^2 Delta_21 per baseline (k_batch.cuh)
      smem_pt += (size_t)(nterm / 3) * order * 32 * (kMixed ? sizeof(float) : sizeof(double));
#if GNA_BATCH_PT_BPSM
    // wave shaping (experiment): pad shared memory so that at most GNA_BATCH_PT_BPSM one-warp
    // blocks fit on an SM (228 KiB per SM, 1 KiB reserved per block)
    smem_pt = std::max<size_t>(smem_pt, (size_t)233472 / GNA_BATCH_PT_BPSM - 1024);
    if (smem_pt > 48 * 1024)
      cudaFuncSetAttribute(kpt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_pt);
#endif
    pt_sub = GNA_BATCH_PT_SUB;
    const int lv = pt_sub == 4 ? 3 : pt_sub == 2 ? 4 : 5;
    if (ng * bpp * pt_sub > 0x7fffffffLL) return GNA_EINVAL;
    e = launch_pdl(kpt, (unsigned)(ng * bpp * pt_sub), 32, smem_pt, s, (int)order, nbins,
                   pts->npoints, bpp, lv, w, spectra, chi2 ? data : nullptr);
    if (e != cudaSuccess) return cuda_fail(e);
  } else if (ppw > 1 && small_terms && kBatchWarps == 1 && GNA_BATCH_PI) {
    // several points per warp: node groups outer, points inner (bitwise-identical sums)
    ppw = std::min<int64_t>(ppw, kMaxPPW);
    auto kpi = (order % 5 == 0)   ? k_oscprob_batch_pi<5, kOut, 0, kMixed>
               : (order % 4 == 0) ? k_oscprob_batch_pi<4, kOut, 0, kMixed>
               : (order % 3 == 0) ? k_oscprob_batch_pi<3, kOut, 0, kMixed>
                                  : k_oscprob_batch_pi<4, kOut, 0, kMixed>;
#if GNA_BATCH_PI_NT
    // single baseline (3 terms): term loop unrolled at compile time
    if (nterm == 3)
      kpi = (order % 5 == 0)   ? k_oscprob_batch_pi<5, kOut, 3, kMixed>
            : (order % 4 == 0) ? k_oscprob_batch_pi<4, kOut, 3, kMixed>
            : (order % 3 == 0) ? k_oscprob_batch_pi<3, kOut, 3, kMixed>
                               : k_oscprob_batch_pi<4, kOut, 3, kMixed>;
#endif
    const int64_t ng = (pts->npoints + ppw - 1) / ppw;
    const size_t smem_pi = (size_t)ppw * nterm * sizeof(double2) + (size_t)ppw * 33 * 8;
    e = launch_pdl(kpi, (unsigned)(ng * bpp), 32, smem_pi, s, nterm, order, nbins, pts->npoints,
                   bpp, (int)ppw, w, spectra, chi2 ? data : nullptr);
    if (e != cudaSuccess) return cuda_fail(e);
  } else {
    e = launch_pdl(kern, (unsigned)nblocks, kBatchWarps * 32, smem, s, nterm, order, nbins,
                   pts->npoints, bpp, (int)ppw, w, spectra, chi2 ? data : nullptr);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e);
  if (chi2) {
    const int64_t threads = pts->npoints * 32;
    const int grid = (int)((threads + kReduceThreads - 1) / kReduceThreads);
    auto kred = pt_sub == 4 ? k_chi2_reduce<kOut, 4>
                : pt_sub == 2 ? k_chi2_reduce<kOut, 2> : k_chi2_reduce<kOut, 1>;
    e = launch_pdl(kred, (unsigned)grid, kReduceThreads, 0, s,
                   (const double*)w.partial, pts->npoints, warps_per_point(nbins), chi2);
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e);
  }
  return GNA_OK;
}

// tables_only: k_batch_setup building just the node tables (invE, hw) at `tables`
int launch_batch_tables(const double* edges, int64_t nbins, int32_t order, double* tables,
                        cudaStream_t s) {
  BatchSetupArgs a;
  std::memset(&a, 0, sizeof(a));
  a.order = order;
  a.nbins = nbins;
  a.npoints = 0;
  a.tables = 1;
  BatchWs w;
  std::memset(&w, 0, sizeof(w));
  w.invE = tables;
  w.hw = (double*)((char*)tables + align16((size_t)order * nbins * sizeof(double)));
  const int64_t n = (int64_t)order * nbins;
  if ((n + 255) / 256 > 0x7fffffffLL) return GNA_EINVAL;
  k_batch_setup<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, nullptr, nullptr, nullptr,
                                                             nullptr, edges, w);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GNA_OK : cuda_fail(e);
}

int launch_batch(const gna_param_batch* pts, const double* L_km, const double* omega,
                 int32_t nbase, const double* edges, int64_t nbins, int32_t order,
                 double* spectra, const double* data, double* chi2, void* workspace,
                 cudaStream_t s, int out_mode = kOutLocal, bool mixed = false,
                 const double* tables = nullptr) {
#define GNA_LB(M, X) launch_batch_k<M, X>(pts, L_km, omega, nbase, edges, nbins, order, spectra, \
                                          data, chi2, workspace, s, tables)
  if (mixed) {
    if (out_mode == kOutMulticast) return GNA_LB(kOutMulticast, true);
    if (out_mode == kOutPeer) return GNA_LB(kOutPeer, true);
    return GNA_LB(kOutLocal, true);
  }
  if (out_mode == kOutMulticast) return GNA_LB(kOutMulticast, false);
  if (out_mode == kOutPeer) return GNA_LB(kOutPeer, false);
  return GNA_LB(kOutLocal, false);
#undef GNA_LB
}

// fold_out (the fit, GNA_FIT_FOLD): when stage B leaves chi^2 as bin-chunk partials, skip
// k_scan_chi2_fold and report the partials (and their count per point) so the caller's next
// kernel folds them itself, in the same order
int launch_scan(const gna_scan_grid* g, const double* L_km, const double* omega, int32_t nbase,
                const double* edges, int64_t nbins, int32_t order, double* spectra,
                const double* data, double* chi2, void* workspace, cudaStream_t s,
                const double** fold_out = nullptr, int64_t* fold_nbc = nullptr) {
  if (fold_out) *fold_out = nullptr;
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
  // node groups of 5 (4, 3) when they divide the order, else 4 with a ragged last group
  auto ksetup = (order % 5 == 0)   ? k_scan_setup<5>
                : (order % 4 == 0) ? k_scan_setup<4>
                : (order % 3 == 0) ? k_scan_setup<3>
                                   : k_scan_setup<GNA_SCAN_G_DEFAULT>;
  if (GNA_SCAN_ORD10 && order == 10) ksetup = k_scan_setup<5, 10>;
  const int64_t nthr = nsetup;
  cudaError_t e = launch_pdl_scan(ksetup, (unsigned)((nthr + 127) / 128), 128, s, a,
                                  g->theta12, g->theta13, g->dm2_21, g->dm2_31, edges,
                                  chi2 ? data : nullptr, w);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (e != cudaSuccess) return cuda_fail(e);
  const bool vec2 = (nbins & 1) == 0 && ((uintptr_t)spectra & 15) == 0 &&
                    (!chi2 || ((uintptr_t)data & 15) == 0);
  const double* dchi = chi2 ? data : nullptr;
  if (GNA_SCAN_EXPAND2 && vec2) {
    // bin chunks only when the grid gives fewer than 4 blocks per SM on its own
    const int64_t nbc = nblk < GNA_SCAN_CHUNK_BPSM * sm_count() ? scan_nbc(nbins) : 1;
    if (nblk * nbc > 0x7fffffffLL) return GNA_EINVAL;
    if (nbc > 1)
      e = launch_pdl_scan(k_scan_expand2<true>, (unsigned)(nblk * nbc), kScanThreads, s,
                          g->nmix, nbins, nchunk, w, spectra, dchi, chi2);
    else
      e = launch_pdl_scan(k_scan_expand2<false>, (unsigned)nblk, kScanThreads, s, g->nmix,
                          nbins, nchunk, w, spectra, dchi, chi2);
    if (e == cudaSuccess && chi2 && nbc > 1 && fold_out) {
      *fold_out = w.partial;
      *fold_nbc = nbc;
    } else if (e == cudaSuccess && chi2 && nbc > 1) {
      g_launches.fetch_add(1, std::memory_order_relaxed);
      const int64_t np = g->nmass * g->nmix;
      e = launch_pdl_scan(k_scan_chi2_fold, (unsigned)((np + 127) / 128), 128, s,
                          (const double*)w.partial, np, nbc, chi2);
    }
  } else
    e = launch_pdl_scan(k_scan_expand, (unsigned)nblk, kScanThreads, s, g->nmix, nbins, nchunk,
                        w, spectra, dchi, chi2);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (e != cudaSuccess) return cuda_fail(e);
  e = cudaGetLastError();
  return e == cudaSuccess ? GNA_OK : cuda_fail(e);
}

template <class Coef>
int launch_gl(const Coef& c, const double* edges, int64_t nbins, int order, double* bins,
              cudaStream_t s) {
  constexpr bool kPee = std::is_same<Coef, PeeCoef>::value;
  if (kPee && GNA_GL_SPLIT && order >= 2 && nbins <= GNA_GL_SPLIT_MAX_BINS) {
    // node halves in two warps (k_gl.cuh), the same bits as thread per bin
    const int64_t grid = (nbins + 32 * kGLSplitBW - 1) / (32 * kGLSplitBW);
    const gl_kernel_t<Coef> kern =
        gl_split_kernel_for<Coef>(order, std::make_integer_sequence<int, GNA_MAX_ORDER>{});
    cudaError_t e = launch_pdl_single(kern, (unsigned)grid, kGLSplitThreads, s, c, edges, nbins,
                                      bins);
    if (e != cudaSuccess) return cuda_fail(e);
  } else if (nbins >= gl_tb_min_bins<Coef>()) {
    // thread per bin, GL table as uniform constant-bank operands (k_gl.cuh)
    const int64_t grid = (nbins + kGLTbThreads - 1) / kGLTbThreads;
    if (grid > 0x7fffffffLL) return GNA_EINVAL;
    const gl_kernel_t<Coef> kern =
        gl_tb_kernel_for<Coef>(order, std::make_integer_sequence<int, GNA_MAX_ORDER>{});
    cudaError_t e = launch_pdl_single(kern, (unsigned)grid, kGLTbThreads, s, c, edges, nbins,
                                      bins);
    if (e != cudaSuccess) return cuda_fail(e);
  } else {
    // lane pairs (mixed tier and general channel only: not instantiated for P_ee fp64,
    // whose gl_tb_min_bins is 1)
    if constexpr (gl_tb_min_bins<Coef>() > 1) {
      const int64_t grid = (2 * nbins + kGLLaneThreads - 1) / kGLLaneThreads;
      if (grid > 0x7fffffffLL) return GNA_EINVAL;
      const gl_kernel_t<Coef> kern =
          gl_kernel_for<Coef>(order, std::make_integer_sequence<int, GNA_MAX_ORDER>{});
      cudaError_t e = launch_pdl_single(kern, (unsigned)grid, kGLLaneThreads, s, c, edges,
                                        nbins, bins);
      if (e != cudaSuccess) return cuda_fail(e);
    } else {
      return GNA_EINVAL;  // unreachable: nbins >= 1 was validated
    }
  }
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
    cudaError_t e = launch_pdl_single(k_oscprob_eval_tma<Coef>, (unsigned)grid, kEvalTmaThreads,
                                      s, c, E, P, n);
    if (e != cudaSuccess) return cuda_fail(e);
  } else if (vec) {
    const int grid = grid_for((n + 1) / 2, kEvalThreads, maxb);
    cudaError_t e = launch_pdl_single(k_oscprob_eval<true, Coef>, (unsigned)grid, kEvalThreads,
                                      s, c, E, P, n);
    if (e != cudaSuccess) return cuda_fail(e);
  } else {
    const int grid = grid_for(n, kEvalThreads, maxb);
    cudaError_t e = launch_pdl_single(k_oscprob_eval<false, Coef>, (unsigned)grid, kEvalThreads,
                                      s, c, E, P, n);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GNA_OK : cuda_fail(e);
}

// ----------------------------------------------------------------------------
// staging for the *_host entry points (library-owned, per device)
// ----------------------------------------------------------------------------
// Three streams per device: 0 = H2D, 1 = compute, 2 = D2H, and a ring of kRing chunk
// slots whose reuse is ordered by events, so chunk c's D2H, chunk c+1's kernel and chunk
// c+2's H2D run at the same time (the paper's "CUDA Streams ... overlapped execution,
// asynchronous memory copying") while every kernel still gets the whole GPU.
constexpr int kRing = 3;
#ifndef GNA_HOST_DIRECT
#define GNA_HOST_DIRECT 1  // batch spectra stored by the kernel into page-locked host memory
#endif
#ifndef GNA_HOST_SPECTRA_MAX
#define GNA_HOST_SPECTRA_MAX (1ull << 31)  // device bytes for un-ringed batch spectra staging
#endif
// the environment variable of the same name overrides it (read once; tests use it to run
// the ring path at small sizes)
size_t host_spectra_max() {
  static const size_t v = [] {
    const char* e = std::getenv("GNA_HOST_SPECTRA_MAX");
    return e ? (size_t)std::strtoull(e, nullptr, 10) : (size_t)GNA_HOST_SPECTRA_MAX;
  }();
  return v;
}
struct Staging {
  bool init = false;
  cudaStream_t st[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_in = nullptr;
  cudaEvent_t ev_h[kRing] = {}, ev_k[kRing] = {}, ev_d[kRing] = {};
  void* buf = nullptr;  // one device allocation, carved per call
  size_t cap = 0;
};

std::mutex g_stage_mu[128];  // one lock per device: host-buffer calls on different GPUs overlap
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
  for (int i = 0; i < 3; ++i) {
    e = cudaStreamCreateWithFlags(&S->st[i], cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  cudaEvent_t* evs[1 + 3 * kRing];
  int n = 0;
  evs[n++] = &S->ev_in;
  for (int r = 0; r < kRing; ++r) {
    evs[n++] = &S->ev_h[r];
    evs[n++] = &S->ev_k[r];
    evs[n++] = &S->ev_d[r];
  }
  for (int i = 0; i < n; ++i) {
    e = cudaEventCreateWithFlags(evs[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  S->init = true;
  return GNA_OK;
}

// Chunk pipeline of the host-buffer entry points: H2D(ci) on st[0] -> kernel(ci) on st[1]
// -> D2H(ci) on st[2], chunk ci in ring slot ci % kRing.  A slot's input is overwritten only
// after the kernel of chunk ci - kRing has read it, and its output only after the D2H of
// chunk ci - kRing has copied it out.  Waits for the caller's stream first; returns after
// all three streams are idle (also on error, so no copy outlives the call).
//   h2d_each = false: only chunk 0 has an H2D stage (the batch uploads everything at once), so
//     later kernels do not wait on the H2D stream;
//   out_ring = false: each chunk writes its own output region (no slot reuse), so the compute
//     stream never waits on the D2H stream and the kernels run back to back.
template <class FH, class FK, class FD>
int run_pipeline(Staging* S, cudaStream_t caller, int64_t nchunks, FH h2d, FK kern, FD d2h,
                 bool h2d_each = true, bool out_ring = true) {
  cudaError_t e = cudaSuccess;
  int rc = GNA_OK;
  auto fail = [&](int code) {
    for (int i = 0; i < 3; ++i) cudaStreamSynchronize(S->st[i]);
    return code;
  };
  if ((e = cudaEventRecord(S->ev_in, caller)) != cudaSuccess) return cuda_fail(e);
  if (nchunks == 1) {
    // nothing to overlap: the three stages in order on one stream, no cross-stream events
    // (small calls — cfg1/cfg2-sized single points, the chi^2-only fit step — are latency-bound)
    cudaStream_t s1 = S->st[1];
    if ((e = cudaStreamWaitEvent(s1, S->ev_in, 0)) != cudaSuccess) return cuda_fail(e);
    if ((rc = h2d(0, 0, s1)) || (rc = kern(0, 0, s1)) || (rc = d2h(0, 0, s1))) return fail(rc);
    if ((e = cudaStreamSynchronize(s1)) != cudaSuccess) return fail(cuda_fail(e));
    return GNA_OK;
  }
  for (int i = 0; i < 3; ++i)
    if ((e = cudaStreamWaitEvent(S->st[i], S->ev_in, 0)) != cudaSuccess) return cuda_fail(e);
  for (int64_t ci = 0; ci < nchunks; ++ci) {
    const int r = (int)(ci % kRing);
    const bool reuse = ci >= kRing;
    if (h2d_each || ci == 0) {
      if (reuse && (e = cudaStreamWaitEvent(S->st[0], S->ev_k[r], 0)) != cudaSuccess) break;
      if ((rc = h2d(ci, r, S->st[0]))) return fail(rc);
      if ((e = cudaEventRecord(S->ev_h[r], S->st[0])) != cudaSuccess) break;
      if ((e = cudaStreamWaitEvent(S->st[1], S->ev_h[r], 0)) != cudaSuccess) break;
    }
    if (out_ring && reuse && (e = cudaStreamWaitEvent(S->st[1], S->ev_d[r], 0)) != cudaSuccess)
      break;
    if ((rc = kern(ci, r, S->st[1]))) return fail(rc);
    if ((e = cudaEventRecord(S->ev_k[r], S->st[1])) != cudaSuccess) break;
    if ((e = cudaStreamWaitEvent(S->st[2], S->ev_k[r], 0)) != cudaSuccess) break;
    if ((rc = d2h(ci, r, S->st[2]))) return fail(rc);
    if ((e = cudaEventRecord(S->ev_d[r], S->st[2])) != cudaSuccess) break;
  }
  if (e != cudaSuccess) return fail(cuda_fail(e));
  for (int i = 0; i < 3; ++i)
    if ((e = cudaStreamSynchronize(S->st[i])) != cudaSuccess) return fail(cuda_fail(e));
  return GNA_OK;
}

int h2d_copy(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  return e == cudaSuccess ? GNA_OK : cuda_fail(e);
}
int d2h_copy(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
  return e == cudaSuccess ? GNA_OK : cuda_fail(e);
}

// Chunk boundaries over [0, total) for run_pipeline: chunks of `chunk` units, the first
// and / or last ones tapered (chunk/8, chunk/4, chunk/2) so that the pipeline's unhidden
// head (the first H2D) and tail (the last D2H) are short.  Sizes are multiples of `align`
// (except a ragged end) and never exceed `chunk`.  Returns the nchunks + 1 offsets.
std::vector<int64_t> plan_chunks(int64_t total, int64_t chunk, bool taper_head, bool taper_tail,
                                 int64_t align) {
  std::vector<int64_t> sizes, tail;
  auto al = [&](int64_t v) { return std::max<int64_t>(align, v / align * align); };
  int64_t rem = total;
  const int64_t tapered = (taper_head ? chunk - chunk / 8 : 0) + (taper_tail ? chunk - chunk / 8 : 0);
  if (total > 2 * chunk + tapered && chunk >= 8 * align) {
    if (taper_head)
      for (int64_t c = chunk / 8; c < chunk; c *= 2) {
        sizes.push_back(al(c));
        rem -= sizes.back();
      }
    if (taper_tail)
      for (int64_t c = chunk / 8; c < chunk; c *= 2) {
        tail.push_back(al(c));
        rem -= tail.back();
      }
  }
  const int64_t nmid = (rem + chunk - 1) / chunk;
  if (nmid > 0) {  // nmid near-equal chunks (<= chunk each; the last one takes the rest)
    int64_t msz = (rem + nmid - 1) / nmid;
    msz = std::min<int64_t>(chunk, (msz + align - 1) / align * align);
    for (int64_t i = 0; i + 1 < nmid; ++i) sizes.push_back(msz);
    sizes.push_back(rem - (nmid - 1) * msz);
  }
  for (auto it = tail.rbegin(); it != tail.rend(); ++it) sizes.push_back(*it);
  std::vector<int64_t> off(1, 0);
  for (int64_t m : sizes)
    if (m > 0) off.push_back(off.back() + m);
  return off;
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

int gna_oscprob_eval_ex(const gna_osc_params* p, double L_km, const double* d_E, int64_t n,
                        double* d_P, uint32_t flags, void* stream) {
  if (flags & ~GNA_PREC_MIXED) return GNA_EINVAL;
  if (!flags) return gna_oscprob_eval(p, L_km, d_E, n, d_P, stream);
  int rc = validate_eval(p, L_km, d_E, n, d_P);
  if (rc) return rc;
  if ((rc = check_device())) return rc;
  if (check_dev_ptr(d_E) || check_dev_ptr(d_P)) return GNA_EINVAL;
  gna::PeeMixCoef c;
  make_coef_mix(p, L_km, &c);
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

int gna_gl_integrate_ex(const gna_osc_params* p, double L_km, const double* d_edges, int64_t nbins,
                        int32_t order, double* d_bins, uint32_t flags, void* stream) {
  if (flags & ~GNA_PREC_MIXED) return GNA_EINVAL;
  if (!flags) return gna_gl_integrate(p, L_km, d_edges, nbins, order, d_bins, stream);
  int rc = validate_gl(p, L_km, d_edges, nbins, order, d_bins);
  if (rc) return rc;
  if ((rc = check_device())) return rc;
  if (check_dev_ptr(d_edges) || check_dev_ptr(d_bins)) return GNA_EINVAL;
  gna::PeeMixCoef c;
  make_coef_mix(p, L_km, &c);
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
  std::lock_guard<std::mutex> lk(g_stage_mu[dev]);
  Staging* S = &g_stage[dev];
  if ((rc = stage_init(S))) return rc;
  if (chunk <= 0) chunk = (int64_t)1 << 20;  // bins per chunk
  if (chunk > nbins) chunk = nbins;
  // slot r: edges (chunk + 1, padded to chunk + 2) then bins (chunk)
  const size_t slot = (size_t)(2 * chunk + 2);
  if ((rc = ensure(&S->buf, &S->cap, kRing * slot * 8))) return rc;
  double* base = (double*)S->buf;
  PeeCoef c;
  make_coef(p, L_km, &c);
  const std::vector<int64_t> off = plan_chunks(nbins, chunk, true, true, 1);
  auto rows = [&](int64_t ci) { return off[ci + 1] - off[ci]; };
  return run_pipeline(
      S, (cudaStream_t)stream, (int64_t)off.size() - 1,
      [&](int64_t ci, int r, cudaStream_t s) {
        return h2d_copy(base + r * slot, h_edges + off[ci], (size_t)(rows(ci) + 1) * 8, s);
      },
      [&](int64_t ci, int r, cudaStream_t s) {
        return launch_gl(c, base + r * slot, rows(ci), order, base + r * slot + chunk + 2, s);
      },
      [&](int64_t ci, int r, cudaStream_t s) {
        return d2h_copy(h_bins + off[ci], base + r * slot + chunk + 2, (size_t)rows(ci) * 8, s);
      });
}

size_t gna_oscprob_batch_workspace_size(int64_t npoints, int32_t nbase, int64_t nbins,
                                        int32_t order) {
  if (npoints < 1 || nbins < 1 || nbase < 1 || nbase > GNA_MAX_NBASE || order < 1 ||
      order > GNA_MAX_ORDER)
    return 0;
  return batch_ws_bytes(npoints, nbase, nbins, order, true);
}

// The batch workspace must not alias any input or local output: k_batch_setup writes the
// coefficient rows and node tables into it before the main kernel reads the inputs.  Remote
// outputs (peer / multicast windows) are other GPUs' memory and pass nullptr here.
static bool batch_ws_overlaps(const gna_param_batch* pts, const double* d_edges, int64_t nbins,
                              int32_t order, int32_t nbase, const double* d_data,
                              const double* d_spectra, const double* d_chi2, bool want_chi2,
                              const void* d_workspace) {
  const size_t W = batch_ws_bytes(pts->npoints, nbase, nbins, order, want_chi2);
  const size_t P8 = (size_t)pts->npoints * 8;
  const void* ins[8] = {pts->theta12, pts->theta13, pts->dm2_21, pts->dm2_31,
                        d_edges,      d_spectra,    d_data,     d_chi2};
  const size_t ln[8] = {P8, P8, P8, P8, (size_t)(nbins + 1) * 8,
                        (size_t)pts->npoints * (size_t)nbins * 8, (size_t)nbins * 8, P8};
  for (int i = 0; i < 8; ++i)
    if (ins[i] && overlap(d_workspace, W, ins[i], ln[i])) return true;
  return false;
}

// gna_oscprob_batch and the local-output case of gna_oscprob_batch_ex (fp64 or mixed tier)
static int batch_local(const gna_param_batch* pts, const double* L_km, const double* omega,
                       int32_t nbase, const double* d_edges, int64_t nbins, int32_t order,
                       double* d_spectra, const double* d_data, double* d_chi2,
                       void* d_workspace, size_t workspace_bytes, void* stream, bool mixed,
                       bool tables_valid = false) {
  int rc = validate_batch(pts, L_km, omega, nbase, d_edges, nbins, order, d_spectra, d_data,
                          d_chi2);
  if (rc) return rc;
  if (!d_workspace ||
      workspace_bytes < batch_ws_bytes(pts->npoints, nbase, nbins, order, d_chi2 != nullptr) ||
      ((uintptr_t)d_workspace & 15))
    return GNA_EINVAL;
  if (batch_ws_overlaps(pts, d_edges, nbins, order, nbase, d_data, d_spectra, d_chi2,
                        d_chi2 != nullptr, d_workspace))
    return GNA_EINVAL;
  if ((rc = check_device())) return rc;
  const void* ptrs[9] = {pts->theta12, pts->theta13, pts->dm2_21, pts->dm2_31, d_edges,
                         d_spectra,    d_data,       d_chi2,      d_workspace};
  for (const void* q : ptrs)
    if (q && check_dev_ptr(q)) return GNA_EINVAL;
  return launch_batch(pts, L_km, omega, nbase, d_edges, nbins, order, d_spectra, d_data, d_chi2,
                      d_workspace, (cudaStream_t)stream, kOutLocal, mixed,
                      tables_valid ? (const double*)d_workspace : nullptr);
}

int gna_oscprob_batch(const gna_param_batch* pts, const double* L_km, const double* omega,
                      int32_t nbase, const double* d_edges, int64_t nbins, int32_t order,
                      double* d_spectra, const double* d_data, double* d_chi2,
                      void* d_workspace, size_t workspace_bytes, void* stream) {
  return batch_local(pts, L_km, omega, nbase, d_edges, nbins, order, d_spectra, d_data, d_chi2,
                     d_workspace, workspace_bytes, stream, false);
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
  if (GNA_FIT_SCAN)  // grid [4][9] | chi2 [81] | scan workspace (32-byte aligned pieces)
    return align32((size_t)kFitDim * kFitGrid * 8) + align32((size_t)kFitCand * 8) +
           scan_ws_bytes(kFitGrid, kFitGrid, nbins) + 32;
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
  if (GNA_FIT_SCAN) {
    // one 9 x 9 separable scan per iteration (k_fit.cuh)
    char* w = (char*)(((uintptr_t)d_workspace + 31) & ~(uintptr_t)31);
    double* grid = (double*)w;
    w += align32((size_t)kFitDim * kFitGrid * 8);
    double* chi2 = (double*)w;
    w += align32((size_t)kFitCand * 8);
    void* sws = w;
    const gna_scan_grid g = {grid, grid + kFitGrid, kFitGrid, grid + 2 * kFitGrid,
                             grid + 3 * kFitGrid, kFitGrid};
    if (niter > 0) {
      cudaError_t e = launch_pdl_scan(k_fit_grid, 1, 128, s, (const double*)d_state, grid);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      if (e != cudaSuccess) return cuda_fail(e);
    }
    for (int it = 0; it < niter; ++it) {
      const double* part = nullptr;
      int64_t nbc = 0;
      if ((rc = launch_scan(&g, L_km, omega, nbase, d_edges, nbins, order, nullptr, d_data, chi2,
                            sws, s, GNA_FIT_FOLD ? &part : nullptr, &nbc)))
        return rc;
      cudaError_t e = launch_pdl_scan(k_fit_update_grid, 1, 128, s, d_state, grid,
                                      (const double*)chi2, part, nbc, d_hist, it,
                                      (int)(it + 1 < niter));
      g_launches.fetch_add(1, std::memory_order_relaxed);
      if (e != cudaSuccess) return cuda_fail(e);
    }
    return GNA_OK;
  }
  char* w = (char*)d_workspace;
  double* cand = (double*)w;
  w += align16((size_t)kFitDim * kFitCand * 8);
  double* chi2 = (double*)w;
  w += align16((size_t)kFitCand * 8);
  void* bws = w;
  const gna_param_batch pts = {cand, cand + kFitCand, cand + 2 * kFitCand, cand + 3 * kFitCand,
                               kFitCand};
  if (niter > 0) {
    k_fit_candidates<<<1, 128, 0, s>>>(d_state, cand);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    // the node tables depend only on the edges and the order: built once per fit
    if ((rc = launch_batch_tables(d_edges, nbins, order, (double*)bws, s))) return rc;
  }
  for (int it = 0; it < niter; ++it) {
    if ((rc = launch_batch(&pts, L_km, omega, nbase, d_edges, nbins, order, nullptr, d_data,
                           chi2, bws, s, kOutLocal, false, (const double*)bws)))
      return rc;
    k_fit_update<<<1, 128, 0, s>>>(d_state, cand, chi2, d_hist, it, it + 1 < niter);
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
  const uint32_t known = GNA_OUT_PEER | GNA_OUT_MULTICAST | GNA_PREC_MIXED | GNA_WS_TABLES_VALID;
  if ((flags & ~known) || ((flags & GNA_OUT_PEER) && (flags & GNA_OUT_MULTICAST)))
    return GNA_EINVAL;
  const bool mixed = (flags & GNA_PREC_MIXED) != 0;
  const bool tables_valid = (flags & GNA_WS_TABLES_VALID) != 0;
  if ((flags & (GNA_OUT_PEER | GNA_OUT_MULTICAST)) == 0)
    return batch_local(pts, L_km, omega, nbase, d_edges, nbins, order, d_spectra, d_data, d_chi2,
                       d_workspace, workspace_bytes, stream, mixed, tables_valid);
  int rc = validate_batch(pts, L_km, omega, nbase, d_edges, nbins, order, d_spectra, d_data,
                          d_chi2);
  if (rc) return rc;
  if (!d_workspace ||
      workspace_bytes < batch_ws_bytes(pts->npoints, nbase, nbins, order, d_chi2 != nullptr) ||
      ((uintptr_t)d_workspace & 15))
    return GNA_EINVAL;
  // remote outputs are excluded from the overlap check (they are not this GPU's memory)
  if (batch_ws_overlaps(pts, d_edges, nbins, order, nbase, d_data, nullptr, nullptr,
                        d_chi2 != nullptr, d_workspace))
    return GNA_EINVAL;
  if ((rc = check_device())) return rc;
  // inputs and workspace must be this GPU's memory; the outputs are remote windows
  const void* ptrs[7] = {pts->theta12, pts->theta13, pts->dm2_21, pts->dm2_31, d_edges, d_data,
                         d_workspace};
  for (const void* q : ptrs)
    if (q && check_dev_ptr(q)) return GNA_EINVAL;
  return launch_batch(pts, L_km, omega, nbase, d_edges, nbins, order, d_spectra, d_data, d_chi2,
                      d_workspace, (cudaStream_t)stream,
                      (flags & GNA_OUT_MULTICAST) ? kOutMulticast : kOutPeer, mixed,
                      tables_valid ? (const double*)d_workspace : nullptr);
}

int gna_oscprob_eval_host(const gna_osc_params* p, double L_km, const double* h_E, int64_t n,
                          double* h_P, int64_t chunk, void* stream) {
  int rc = validate_eval(p, L_km, h_E, n, h_P);
  if (rc) return rc;
  if ((rc = check_device())) return rc;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_stage_mu[dev]);
  Staging* S = &g_stage[dev];
  if ((rc = stage_init(S))) return rc;
  if (chunk <= 0) chunk = (int64_t)1 << 22;  // 4 Mi elements = 32 MiB per direction
  if (chunk > n) chunk = n;
  chunk = (chunk + 1) & ~(int64_t)1;         // keep the double2 path aligned
  const size_t slot = (size_t)chunk * 2;     // E then P
  if ((rc = ensure(&S->buf, &S->cap, kRing * slot * 8))) return rc;
  double* base = (double*)S->buf;
  PeeCoef c;
  make_coef(p, L_km, &c);
  const std::vector<int64_t> off = plan_chunks(n, chunk, true, true, 2);
  auto len = [&](int64_t ci) { return off[ci + 1] - off[ci]; };
  return run_pipeline(
      S, (cudaStream_t)stream, (int64_t)off.size() - 1,
      [&](int64_t ci, int r, cudaStream_t s) {
        return h2d_copy(base + r * slot, h_E + off[ci], (size_t)len(ci) * 8, s);
      },
      [&](int64_t ci, int r, cudaStream_t s) {
        return launch_eval(c, base + r * slot, len(ci), base + r * slot + chunk, s);
      },
      [&](int64_t ci, int r, cudaStream_t s) {
        return d2h_copy(h_P + off[ci], base + r * slot + chunk, (size_t)len(ci) * 8, s);
      });
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
  std::lock_guard<std::mutex> lk(g_stage_mu[dev]);
  Staging* S = &g_stage[dev];
  if ((rc = stage_init(S))) return rc;
  const int64_t P = h_pts->npoints;
  // Page-locked spectra (cudaHostAlloc / cudaHostRegister, mapped into the unified address
  // space): the kernel stores the spectra straight into host memory over PCIe while it
  // computes — one launch over all points, no staging copy to overlap (GNA_HOST_DIRECT)
  // Only for the kernels whose spectra stores are whole rows of consecutive bins (per-point
  // and points-inner); the points-across-lanes kernel (<= 2 baselines, >= GNA_BATCH_PT_MIN_POINTS
  // points) stores one bin of 32 different rows per warp instruction, which over PCIe is
  // ~30x slower than staging (cfg4: 5.4 vs 60 G energy points/s end to end).
  const bool pt_kernel = GNA_BATCH_PT && nbase <= 2 && h_pts->npoints >= GNA_BATCH_PT_MIN_POINTS;
  bool direct = false;
  if (GNA_HOST_DIRECT && h_spectra && chunk_points <= 0 && !pt_kernel) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, h_spectra) == cudaSuccess)
      direct = at.type == cudaMemoryTypeHost && at.devicePointer == (void*)h_spectra;
    else
      cudaGetLastError();  // pageable memory: clear the error, use the staged pipeline
  }
  if (direct) chunk_points = P;
  if (chunk_points <= 0) {
    // ~8 MiB of spectra per chunk (their D2H overlaps the next chunks' kernels), at least 1
    // point; without spectra there is nothing large to overlap: one launch over all points
    chunk_points = h_spectra ? ((int64_t)8 << 20) / (nbins * 8) : P;
    if (chunk_points < 1) chunk_points = 1;
  }
  if (chunk_points > P) chunk_points = P;
  // device layout (16-byte aligned pieces): node tables | edges | data | points [4][P] |
  // chi2 [P] | workspace (one chunk) | kRing spectra slots (one chunk each)
  const size_t tb = batch_tables_bytes(nbins, order);
  const size_t b_edges = align16((size_t)(nbins + 1) * 8);
  const size_t b_data = h_data ? align16((size_t)nbins * 8) : 0;
  const size_t b_pts = align16((size_t)4 * P * 8);
  const size_t b_chi = h_chi2 ? align16((size_t)P * 8) : 0;
  const size_t b_ws = batch_ws_bytes(chunk_points, nbase, nbins, order, h_chi2 != nullptr);
  // spectra: one region per point (no reuse, the kernels never wait for a copy) when all of
  // them fit in GNA_HOST_SPECTRA_MAX bytes, else a ring of kRing chunk slots
  const size_t b_all = align16((size_t)P * nbins * 8);
  const bool out_ring = h_spectra && b_all > host_spectra_max();
  const size_t b_slot = h_spectra ? align16((size_t)chunk_points * nbins * 8) : 0;
  const size_t b_spec = (!h_spectra || direct) ? 0 : out_ring ? kRing * b_slot : b_all;
  if ((rc = ensure(&S->buf, &S->cap, tb + b_edges + b_data + b_pts + b_chi + b_ws + b_spec)))
    return rc;
  char* q = (char*)S->buf;
  double* d_tables = (double*)q;
  q += tb;
  double* d_edges = (double*)q;
  q += b_edges;
  double* d_data = h_data ? (double*)q : nullptr;
  q += b_data;
  double* d_pts = (double*)q;
  q += b_pts;
  double* d_chi = h_chi2 ? (double*)q : nullptr;
  q += b_chi;
  void* d_ws = q;
  q += b_ws;
  char* d_slots = q;
  const double* hsrc[4] = {h_pts->theta12, h_pts->theta13, h_pts->dm2_21, h_pts->dm2_31};
  // tapered tail: the last D2H of spectra (not hidden by any kernel) stays short
  const std::vector<int64_t> off = plan_chunks(P, chunk_points, false, h_spectra != nullptr, 1);
  auto rows = [&](int64_t ci) { return off[ci + 1] - off[ci]; };
  return run_pipeline(
      S, (cudaStream_t)stream, (int64_t)off.size() - 1,
      [&](int64_t ci, int, cudaStream_t s) {
        if (ci > 0) return (int)GNA_OK;  // every input goes up with the first chunk
        int r2 = h2d_copy(d_edges, h_edges, (size_t)(nbins + 1) * 8, s);
        if (!r2 && d_data) r2 = h2d_copy(d_data, h_data, (size_t)nbins * 8, s);
        for (int a = 0; a < 4 && !r2; ++a) r2 = h2d_copy(d_pts + a * P, hsrc[a], (size_t)P * 8, s);
        return r2;
      },
      [&](int64_t ci, int r, cudaStream_t s) {
        int r2 = GNA_OK;
        if (ci == 0 && (r2 = launch_batch_tables(d_edges, nbins, order, d_tables, s))) return r2;
        const int64_t o = off[ci], m = rows(ci);
        const gna_param_batch dp = {d_pts + o, d_pts + P + o, d_pts + 2 * P + o,
                                    d_pts + 3 * P + o, m};
        double* dspec = !h_spectra ? nullptr
                        : direct   ? h_spectra + o * nbins  // mapped host memory
                        : out_ring ? (double*)(d_slots + r * b_slot)
                                   : (double*)d_slots + o * nbins;
        return launch_batch(&dp, L_km, omega, nbase, d_edges, nbins, order, dspec, d_data,
                            d_chi ? d_chi + o : nullptr, d_ws, s, kOutLocal, false, d_tables);
      },
      [&](int64_t ci, int r, cudaStream_t s) {
        const int64_t o = off[ci], m = rows(ci);
        int r2 = GNA_OK;
        if (h_spectra && !direct)
          r2 = d2h_copy(h_spectra + o * nbins,
                        out_ring ? (const void*)(d_slots + r * b_slot)
                                 : (const void*)((double*)d_slots + o * nbins),
                        (size_t)m * nbins * 8, s);
        if (!r2 && h_chi2) r2 = d2h_copy(h_chi2 + o, d_chi + o, (size_t)m * 8, s);
        return r2;
      },
      /*h2d_each=*/false, out_ring);
}

void gna_release(void) {
  int cur = 0;
  cudaGetDevice(&cur);
  for (int d = 0; d < 128; ++d) {
    std::lock_guard<std::mutex> lk(g_stage_mu[d]);
    Staging* S = &g_stage[d];
    if (!S->init && !S->buf) continue;
    cudaSetDevice(d);
    for (int i = 0; i < 3; ++i)
      if (S->st[i]) cudaStreamSynchronize(S->st[i]);
    if (S->buf) cudaFree(S->buf);
    for (int i = 0; i < 3; ++i)
      if (S->st[i]) cudaStreamDestroy(S->st[i]);
    if (S->ev_in) cudaEventDestroy(S->ev_in);
    for (int r = 0; r < kRing; ++r) {
      if (S->ev_h[r]) cudaEventDestroy(S->ev_h[r]);
      if (S->ev_k[r]) cudaEventDestroy(S->ev_k[r]);
      if (S->ev_d[r]) cudaEventDestroy(S->ev_d[r]);
    }
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

int gna_sin2_poly_degree(void) { return GNA_SIN2_DEG; }

}  // extern "C"


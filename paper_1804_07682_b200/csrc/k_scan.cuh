// k_scan.cuh — NEXT-1 separable grid-scan kernels
// Part of libgna_b200.so: included once, from gna_b200.cu (single translation unit).
#pragma once
#include "k_batch.cuh"

namespace {

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
  double* partial;  // [nmass * nmix][nbc] chi2 per bin chunk (k_scan_expand2, nbc > 1)
};

// stage B splits the bins into chunks of kScanBinChunk (even) when the grid alone gives too few
// blocks (the fit's 9 x 9 stencil: 27 blocks for 10^4 bins); chi^2 is then summed from
// per-chunk partials in chunk order (k_scan_chi2_fold)
#ifndef GNA_SCAN_BIN_CHUNK
#define GNA_SCAN_BIN_CHUNK 512
#endif
#ifndef GNA_SCAN_CHUNK_BPSM
#define GNA_SCAN_CHUNK_BPSM 4  // chunk the bins when the grid has fewer blocks per SM than this
#endif
constexpr int64_t kScanBinChunk = GNA_SCAN_BIN_CHUNK;
__host__ __device__ inline int64_t scan_nbc(int64_t nbins) {
  return (nbins + kScanBinChunk - 1) / kScanBinChunk;
}

size_t scan_ws_bytes(int64_t nmix, int64_t nmass, int64_t nbins) {
  size_t b = align32((size_t)nmass * 3 * nbins * sizeof(double));
  b += 2 * align32((size_t)nbins * sizeof(double));
  b += align32((size_t)nmix * 4 * sizeof(double));
  b += align32((size_t)nmass * nmix * scan_nbc(nbins) * sizeof(double));
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
  c += align32((size_t)nmix * 4 * sizeof(double));
  w.partial = (double*)c;
  return w;
}

// stage A: thread per (mass point c, bin k): the three pairs share each node's
// reciprocal and run as three independent sin^2 chains (two nodes per iteration:
// six chains) -> G[c][*][k]; threads with c == 0 also write H[k] and 1/D[k]; extra
// threads compute the mixing weights of each mixing point.
#ifndef GNA_SCAN_G_DEFAULT
#define GNA_SCAN_G_DEFAULT 4
#endif
// Nodes are taken kG at a time: the kG reciprocals and the 3 x kG sin^2 terms of a group are
// independent chains (ILP 3 kG; round 1's scalar loop ran ~2 chains and was latency-bound:
// 9.5 us for ~2.3 us of FP64 work, profiles/r02_ncu_scan_summary.txt); each term is then
// folded over the group's nodes in ascending order with the same FMAs, so G is unchanged.
// G[ij] of one (mass point, bin): sum_b omega_b h sum_i w_i sin^2 Delta_ij, nodes in groups of
// kG (the kG reciprocals and 3 kG sin^2 terms independent chains), each term folded over the
// nodes in ascending order.
// kOrd > 0: the order as a compile-time constant (GNA_SCAN_ORD10: GL10), node loop unrolled
// and the GL nodes / weights constant-bank operands; the same operations in the same order.
// s_ij(b) = sum_i w_i (-1)^q v of one baseline b (the three pairs share each node's reciprocal)
template <int kG, int kOrd = 0>
__device__ __forceinline__ void scan_base_s(const ScanArgs& a, int b, double m21, double m31,
                                            double m32, double ctr, double h, double& s0,
                                            double& s1, double& s2) {
  const int order = kOrd > 0 ? kOrd : a.order;
  const int off = GNA_GL_OFF(order);
  const double k0 = phase_slope(m21, a.L[b]);
  const double k1 = phase_slope(m31, a.L[b]);
  const double k2 = phase_slope(m32, a.L[b]);
  s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int i0 = 0; i0 < order; i0 += kG) {
    const int n = order - i0 < kG ? order - i0 : kG;
    double v0[kG], v1[kG], v2[kG];
#pragma unroll
    for (int i = 0; i < kG; ++i) {
      const double invE = gna::rcp(fma(h, c_gl_t[off + i0 + (i < n ? i : 0)], ctr));
      v0[i] = gna::sin2c(k0, invE);
      v1[i] = gna::sin2c(k1, invE);
      v2[i] = gna::sin2c(k2, invE);
    }
#pragma unroll
    for (int i = 0; i < kG; ++i) {
      if (i < n) {
        const double wi = c_gl_w[off + i0 + i];
        s0 = fma(wi, v0[i], s0);
        s1 = fma(wi, v1[i], s1);
        s2 = fma(wi, v2[i], s2);
      }
    }
  }
}

template <int kG, int kOrd = 0>
__device__ __forceinline__ void scan_bin_G(const ScanArgs& a, double m21, double m31,
                                           double ctr, double h, double wsum, double& G0,
                                           double& G1, double& G2) {
  const double m32 = m31 - m21;
  G0 = 0.0, G1 = 0.0, G2 = 0.0;
  for (int b = 0; b < a.nbase; ++b) {
    double s0, s1, s2;
    scan_base_s<kG, kOrd>(a, b, m21, m31, m32, ctr, h, s0, s1, s2);
    // h sum_i w_i sin^2 = h (W/2 + sum_i w_i (-1)^q v)
    const double ob = a.omega[b] * h;
    G0 = fma(ob, fma(0.5, wsum, s0), G0);
    G1 = fma(ob, fma(0.5, wsum, s1), G1);
    G2 = fma(ob, fma(0.5, wsum, s2), G2);
  }
}

__device__ __forceinline__ double gl_wsum(int order) {
  const int off = GNA_GL_OFF(order);
  double wsum = 0.0;
#pragma unroll
  for (int i = 0; i < order; ++i) wsum += c_gl_w[off + i];
  return wsum;
}

__device__ __forceinline__ void scan_wmix(double th12, double th13, double* wm) {
  double s12, c12, s13, c13;
  sincos(th12, &s12, &c12);
  sincos(th13, &s13, &c13);
  mixing_weights(s12, c12, s13, c13, &wm[0], &wm[1], &wm[2]);
  wm[3] = 0.0;
}

#ifndef GNA_SCAN_ORD10
#define GNA_SCAN_ORD10 1
#endif
#ifndef GNA_SCAN_SETUP_MINB
#define GNA_SCAN_SETUP_MINB 3
#endif
template <int kG, int kOrd = 0>
__global__ void __launch_bounds__(128, GNA_SCAN_SETUP_MINB) k_scan_setup(ScanArgs a, const double* __restrict__ th12,
                                                    const double* __restrict__ th13,
                                                    const double* __restrict__ d21,
                                                    const double* __restrict__ d31,
                                                    const double* __restrict__ edges,
                                                    const double* __restrict__ data, ScanWs w) {
  // PDL (GNA_PDL_SCAN): stage B may be scheduled now; nothing is read or written before the
  // predecessor (the fit's grid update, or the previous call) has completed
  pdl_launch_dependents();
  pdl_wait();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n1 = a.nmass * a.nbins;
  if (t < n1) {
    const int64_t c = t / a.nbins;
    const int64_t k = t - c * a.nbins;
    const double e0 = edges[k], e1 = edges[k + 1];
    const double ctr = 0.5 * (e0 + e1);
    const double h = 0.5 * (e1 - e0);
    const double wsum = gl_wsum(kOrd > 0 ? kOrd : a.order);
    double G0, G1, G2;
    scan_bin_G<kG, kOrd>(a, d21[c], d31[c], ctr, h, wsum, G0, G1, G2);
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
    scan_wmix(th12[mm], th13[mm], w.wmix + 4 * mm);
  }
}

// stage B: block = (mass point c, chunk of kScanA (4) mixing points).  Each thread loads
// G[c][*][k], H[k], D[k], 1/D[k] of its bins once and writes T for all kScanA points
// (coalesced rows), so G is read once per chunk instead of once per point; chi2 of each
// point is reduced in the block (fixed shuffle tree + warps in order) and written directly.
// spectra stored with the evict-first hint (st.global.cs): the 80 MB written once stream through
// L2 without displacing G, H, D, 1/D (cfg4grid 26.96 -> 26.72 us mean over 3 x 200 steps,
// profiles/variants_r02/scan3/summary.txt); the same values
#ifndef GNA_SCAN_STREAMING_STORES
#define GNA_SCAN_STREAMING_STORES 1
#endif
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
  pdl_launch_dependents();
  pdl_wait();  // stage A's G, H, 1/D and mixing weights are complete and visible
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
#if GNA_SCAN_STREAMING_STORES
        if (out) __stcs(out + (int64_t)j * nbins + k, T);
#else
        if (out) out[(int64_t)j * nbins + k] = T;
#endif
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

// Stage B for even nbins and 16-byte aligned outputs (GNA_SCAN_EXPAND2, default):
// k_scan_expand with each thread on two adjacent bins (16-byte loads and stores: half the
// memory instructions and loop trips, twice the bytes in flight per load; cfg4grid
// 30.7 -> 28.6 us per step, expand 23 -> 20 us under ncu).  T is the same expression per bin,
// so the spectra are bitwise unchanged; a lane's chi^2 terms are accumulated pair by pair.
#ifndef GNA_SCAN_EXPAND2
#define GNA_SCAN_EXPAND2 1
#endif
// kChunked: the bins are split into chunks of kScanBinChunk across blocks (chi^2 partials);
// otherwise one block walks all bins (the round-1 shape, kept for large grids: the chunk
// bookkeeping alone cost cfg4grid 1.2 us)
template <bool kChunked>
__global__ void __launch_bounds__(kScanThreads) k_scan_expand2(int64_t nmix, int64_t nbins,
                                                               int64_t nchunk, ScanWs w,
                                                               double* __restrict__ spectra,
                                                               const double* __restrict__ data,
                                                               double* __restrict__ chi2) {
  __shared__ double s_x2[kScanA][kScanThreads / 32];
  pdl_launch_dependents();
  pdl_wait();  // stage A's G, H, 1/D and mixing weights are complete and visible
  const int64_t nbc = kChunked ? scan_nbc(nbins) : 1;
  const int64_t cb = kChunked ? blockIdx.x / nbc : blockIdx.x;  // (mass point, mixing chunk)
  const int64_t bc = kChunked ? blockIdx.x - cb * nbc : 0;      // bin chunk
  const int64_t c = cb / nchunk;
  const int64_t a0 = (cb - c * nchunk) * kScanA;
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
  const int64_t np = nbins >> 1;
  const double2* __restrict__ g0 = reinterpret_cast<const double2*>(w.G + (c * 3) * nbins);
  const double2* __restrict__ g1 = g0 + np;
  const double2* __restrict__ g2 = g1 + np;
  const double2* __restrict__ Hv = reinterpret_cast<const double2*>(w.H);
  const double2* __restrict__ Dv = reinterpret_cast<const double2*>(data);
  const double2* __restrict__ iDv = reinterpret_cast<const double2*>(w.invD);
  double2* __restrict__ out =
      spectra ? reinterpret_cast<double2*>(spectra + (c * nmix + a0) * nbins) : nullptr;
  const int64_t qend = kChunked ? min(np, (bc + 1) * (kScanBinChunk / 2)) : np;
  int64_t q = (kChunked ? bc * (kScanBinChunk / 2) : 0) + threadIdx.x;
  double2 G0 = {0, 0}, G1 = {0, 0}, G2 = {0, 0}, H = {0, 0}, D = {0, 0}, iD = {0, 0};
  if (q < qend) {
    G0 = g0[q], G1 = g1[q], G2 = g2[q], H = Hv[q];
    if (chi2) D = Dv[q], iD = iDv[q];
  }
  for (; q < qend; q += kScanThreads) {
    const int64_t qn = q + kScanThreads;
    double2 nG0 = {0, 0}, nG1 = {0, 0}, nG2 = {0, 0}, nH = {0, 0}, nD = {0, 0}, niD = {0, 0};
    if (qn < qend) {
      nG0 = g0[qn], nG1 = g1[qn], nG2 = g2[qn], nH = Hv[qn];
      if (chi2) nD = Dv[qn], niD = iDv[qn];
    }
#pragma unroll
    for (int j = 0; j < kScanA; ++j) {
      if (j < na) {
        double2 T;
        T.x = H.x - fma(w0[j], G0.x, fma(w1[j], G1.x, w2[j] * G2.x));
        T.y = H.y - fma(w0[j], G0.y, fma(w1[j], G1.y, w2[j] * G2.y));
#if GNA_SCAN_STREAMING_STORES
        if (out) __stcs(out + j * np + q, T);
#else
        if (out) out[j * np + q] = T;
#endif
        const double dx = T.x - D.x, dy = T.y - D.y;
        x2[j] = fma(dx * dx, iD.x, x2[j]);
        x2[j] = fma(dy * dy, iD.y, x2[j]);
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
      if (!kChunked)
        chi2[c * nmix + a0 + threadIdx.x] = t;
      else
        w.partial[(c * nmix + a0 + threadIdx.x) * nbc + bc] = t;
    }
  }
}

// chi2[p] = sum of the point's bin-chunk partials in chunk order (k_scan_expand2, nbc > 1)
__global__ void __launch_bounds__(128) k_scan_chi2_fold(const double* __restrict__ partial,
                                                        int64_t npoints, int64_t nbc,
                                                        double* __restrict__ chi2) {
  pdl_launch_dependents();
  pdl_wait();  // every chunk partial of stage B is written
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npoints) return;
  double t = 0.0;
  for (int64_t j = 0; j < nbc; ++j) t += partial[p * nbc + j];
  chi2[p] = t;
}

}  // namespace

/*
 * gna_b200.h — C ABI of the B200-native GNA hot path (libgna_b200.so).
 *
 * Source method: arXiv:1804.07682, "GNA: GPU support for the Global Neutrino
 * Analysis framework".  Citations: P:NNN = reference PAPER.md line NNN (§ given),
 * S:NNN = reference SPEC.md line NNN, BJ = BASELINE.json north_star, DESIGN.md Rn =
 * reading n in DESIGN.md.
 *
 * What the library computes (all fp64, IEEE binary64, round-to-nearest):
 *   P_ee(E) — the reactor electron-antineutrino survival probability, the
 *     alpha = beta = e case of the general vacuum formula P:631-639 (§4.1), with
 *     Delta_ij = 1.26693268 * dm2_ij[eV^2] * L[km] / (E[MeV] / 1000) (S:265,
 *     S:317; R1) and dm2_32 = dm2_31 - dm2_21.  For alpha =
 *     beta = e the formula reduces exactly to
 *       P_ee = 1 - w21 sin^2 D21 - w31 sin^2 D31 - w32 sin^2 D32,
 *       w21 = cos^4(t13) sin^2(2 t12), w31 = sin^2(2 t13) cos^2(t12),
 *       w32 = sin^2(2 t13) sin^2(t12)        (R2),
 *     so theta23, delta_cp and the antineutrino flag do not change the result.
 *   Per-bin Gauss-Legendre integrals of P_ee (BJ north_star; R5/R6):
 *       S_k = h_k * sum_i w_i P_ee(c_k + h_k t_i),
 *       c_k = (e_k + e_{k+1})/2, h_k = (e_{k+1} - e_k)/2, (t_i, w_i) the n-point
 *       GL rule on [-1, 1].
 *   Batched spectra over parameter points and baselines (BJ; the one-energy-
 *   node / several-OscProb topology of P:596-603 and S:431-439):
 *       T[p][k] = sum_b omega_b S_{p,b,k},  chi2[p] = sum_k (T[p][k] - D_k)^2 / D_k
 *       (R8).
 *
 * Conventions shared by every entry point
 *   Ownership: arrays are owned by the caller.  The
 *     device entry points never allocate, free or synchronise; inputs are read
 *     only; outputs are fully overwritten.  Input and output ranges must not
 *     overlap.  The *_host entry points stage through library-owned device
 *     buffers (grown on first use, released by gna_release()).
 *   Memory kind: "d_" arrays are DEVICE pointers (cudaMalloc / torch CUDA
 *     tensors) of the current device; "h_" arrays are HOST pointers (pinned
 *     memory gives overlapped copies; pageable memory works, slower).  Scalars
 *     and small per-call arrays (L_km, omega) are host values.
 *   Streams: work is enqueued on `stream` (a cudaStream_t; NULL = legacy default
 *     stream).  Device entry points return after enqueueing: the return code
 *     covers validation and launch; execution faults surface at the caller's
 *     next stream synchronisation (adapting P:798-800).  *_host entry points
 *     return after the results are in host memory.
 *   Errors: GNA_EINVAL is returned before any CUDA call for bad arguments;
 *     GNA_ENODEV if the current device is not compute capability 10.0
 *     (sm_100a); GNA_ECUDA if a CUDA call or launch failed (the cudaError_t is
 *     then available from gna_last_cuda_error(), thread-local); GNA_ENOMEM if
 *     staging allocation failed.  Preconditions NOT checked on the device
 *     (violations give unspecified values, never a fault): E > 0,
 *     edges strictly increasing, data > 0.
 *   Domain: phases with |y| = |2 Delta / pi| < 2^51, i.e. |Delta| < pi * 2^50
 *     (about 3.5e15 rad), are reduced exactly (the magic-number rint of y is an
 *     exact integer there); the result is accurate to the rounding of Delta
 *     itself (R7, R9, R10).
 *   Thread safety: stateless and re-entrant for the device entry points;
 *     concurrent calls on disjoint outputs are allowed.  The *_host
 *     entry points serialise on an internal lock per device (calls on different
 *     devices run concurrently).
 */
#ifndef GNA_B200_H
#define GNA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GNA_ABI_VERSION 1
#define GNA_MAX_ORDER 32  /* largest Gauss-Legendre order in the table        */
#define GNA_MAX_NBASE 64  /* largest number of baselines per batch call         */

enum gna_status {
  GNA_OK = 0,
  GNA_EINVAL = -1, /* invalid argument (returned before any CUDA call)        */
  GNA_ECUDA = -2,  /* a CUDA call or kernel launch failed                     */
  GNA_ENODEV = -3, /* current device is not sm_100 (B200)                     */
  GNA_ENOMEM = -4  /* library staging allocation failed (*_host only)         */
};

/* Oscillation parameters — SPEC OscParams.  Angles in radians,
 * dm2 in eV^2; a negative dm2_31 selects the inverted ordering.
 * theta23, delta_cp and antineutrino are accepted for interface parity with
 * the general formula; they do not change P_ee (R2).              */
typedef struct gna_osc_params {
  double theta12, theta13, theta23;
  double delta_cp;
  double dm2_21, dm2_31;
  int32_t antineutrino;
} gna_osc_params;

/* A batch of parameter points, structure of arrays, each [npoints] fp64.
 * Device pointers for gna_oscprob_batch, host pointers for
 * gna_oscprob_batch_host.                                                    */
typedef struct gna_param_batch {
  const double* theta12;
  const double* theta13;
  const double* dm2_21;
  const double* dm2_31;
  int64_t npoints;
} gna_param_batch;

/* ---------------------------------------------------------------------------
 * gna_oscprob_eval — the OscProb transformation (§4.1, Table 1):
 *   d_P[i] = P_ee(d_E[i]; L_km, *p)   for 0 <= i < n.
 * p: host struct (all fields finite).  L_km >= 0, finite.  d_E: device [n]
 * energies in MeV (> 0).  d_P: device [n] output.  n >= 1.
 * EINVAL: p/d_E/d_P NULL, n < 1, non-finite scalar, L_km < 0, d_E and d_P
 * ranges overlap, or a pointer that is not device memory.
 * ------------------------------------------------------------------------- */
int gna_oscprob_eval(const gna_osc_params* p, double L_km, const double* d_E, int64_t n,
                     double* d_P, void* stream);

/* ---------------------------------------------------------------------------
 * gna_oscprob_eval_ab — NEXT-2: the general vacuum formula of P:631-639 for any
 * channel alpha -> beta (0 = e, 1 = mu, 2 = tau):
 *   d_P[i] = delta_ab - 4 sum_{i>j} Re(X_ij) sin^2(Delta_ij) + 2 sum_{i>j} Im(X_ij) sin(2 Delta_ij),
 *   X_ij = V*_ai V_bi V_aj V*_bj,  V = R23 U13 R12, conj(V) for antineutrinos.
 * Here theta23, delta_cp and the antineutrino flag matter.  Same arguments, layout
 * and errors as gna_oscprob_eval, plus EINVAL for alpha or beta outside [0, 2].
 * ------------------------------------------------------------------------- */
int gna_oscprob_eval_ab(int32_t alpha, int32_t beta, const gna_osc_params* p, double L_km,
                        const double* d_E, int64_t n, double* d_P, void* stream);

/* ---------------------------------------------------------------------------
 * gna_gl_integrate — fused P_ee + per-bin Gauss-Legendre quadrature (BJ):
 *   d_bins[k] = h_k * sum_{i<order} w_i P_ee(c_k + h_k t_i),  0 <= k < nbins.
 * d_edges: device [nbins + 1] bin edges in MeV (strictly increasing, > 0).
 * order in [1, GNA_MAX_ORDER].  d_bins: device [nbins] output.
 * EINVAL as for gna_oscprob_eval, plus nbins < 1 or order out of range.
 * A bin's value depends only on its two edges (bitwise: the same for any nbins and
 * any split of the edges between calls).
 * ------------------------------------------------------------------------- */
int gna_gl_integrate(const gna_osc_params* p, double L_km, const double* d_edges, int64_t nbins,
                     int32_t order, double* d_bins, void* stream);

/* gna_gl_integrate_ab — NEXT-2 in binned form: per-bin Gauss-Legendre integrals of
 * P(nu_alpha -> nu_beta) (the general formula of gna_oscprob_eval_ab).  Arguments and
 * errors as gna_gl_integrate, plus EINVAL for alpha or beta outside [0, 2].          */
int gna_gl_integrate_ab(int32_t alpha, int32_t beta, const gna_osc_params* p, double L_km,
                        const double* d_edges, int64_t nbins, int32_t order, double* d_bins,
                        void* stream);

/* ---------------------------------------------------------------------------
 * gna_oscprob_batch — batch over parameter points x baselines (BJ north_star):
 *   T[p][k]  = sum_{b<nbase} omega[b] * S_{p,b,k}       -> d_spectra[p*nbins+k]
 *   chi2[p]  = sum_k (T[p][k] - d_data[k])^2 / d_data[k] -> d_chi2[p]
 * pts: host struct of DEVICE arrays [npoints] (npoints >= 1).
 * L_km, omega: HOST arrays [nbase], 1 <= nbase <= GNA_MAX_NBASE, L >= 0.
 * d_edges: device [nbins + 1].  order in [1, GNA_MAX_ORDER].
 * d_spectra: device [npoints][nbins] row-major output, or NULL.
 * d_data: device [nbins] (> 0), required iff d_chi2 != NULL.
 * d_chi2: device [npoints] output, or NULL (not both outputs NULL).
 * d_workspace: device scratch, 16-byte aligned, of at least
 *   gna_oscprob_batch_workspace_size(npoints, nbase, nbins, order) bytes (always
 *   required: it holds the per-point coefficients, the per-node 1/E and h*w
 *   tables and the chi2 partials); contents need no initialisation and are
 *   overwritten; it must not overlap any other argument.
 * Results are bitwise deterministic and independent of how the points are
 * split between calls (one point's arithmetic never depends on the others).
 * ------------------------------------------------------------------------- */
size_t gna_oscprob_batch_workspace_size(int64_t npoints, int32_t nbase, int64_t nbins,
                                        int32_t order);  /* 0 for invalid sizes */

int gna_oscprob_batch(const gna_param_batch* pts, const double* L_km, const double* omega,
                      int32_t nbase, const double* d_edges, int64_t nbins, int32_t order,
                      double* d_spectra, const double* d_data, double* d_chi2,
                      void* d_workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * gna_oscprob_batch_ex — gna_oscprob_batch with the gather fused into the kernel
 * epilogue: d_spectra / d_chi2 may point into another GPU's
 * memory (a symmetric-memory window over NVLink) instead of this GPU's, so that
 * each rank writes its rows of the gathered result directly, with no separate
 * collective.
 *   flags = 0                  same as gna_oscprob_batch;
 *   flags = GNA_OUT_PEER       outputs are peer-mapped unicast addresses (e.g. the
 *                              root's buffer): plain stores + a system-scope fence;
 *   flags = GNA_OUT_MULTICAST  outputs are NVLS multicast addresses: multimem.st
 *                              writes every participating GPU's copy (all-gather);
 *   | GNA_PREC_MIXED           the mixed-precision tier below (with flags = GNA_PREC_MIXED
 *                              alone the outputs are local device memory, validated as
 *                              in gna_oscprob_batch);
 *   | GNA_WS_TABLES_VALID      reuse the node tables already in the workspace (below).
 * The caller synchronises the ranks after the call (e.g. a symmetric-memory or
 * NCCL barrier on the stream) before reading the gathered result.  Inputs and the
 * workspace must be this GPU's memory; output pointers are not type-checked.
 * Other arguments and errors as gna_oscprob_batch; EINVAL for unknown or
 * conflicting flags.
 * ------------------------------------------------------------------------- */
#define GNA_OUT_PEER 1u
#define GNA_OUT_MULTICAST 2u
/* Mixed-precision tier (the paper's single-precision remark,
 * P:691-694), combinable with either output flag: the phases y = kq/E and their
 * reduction modulo 2 (y = 2m + 2h, |h| <= 1/2) stay fp64; h is rounded to fp32,
 * -cos(pi y)/2 = -cos(2 pi h)/2 is an fp32 degree-6 minimax evaluated two chains
 * at a time (packed FFMA2), and the terms of one node are summed in fp32 (weights
 * rounded to fp32); node, bin and chi^2 sums stay fp64.  Error per sin^2 term
 * <= 2.3e-7; spectra are tested against the oracle at 1e-5 relative (tier
 * tolerance; measured <= 8.2e-7 on cfg4/cfg5) — not the
 * 1e-12 / 1e-11 of the default path.                                            */
#define GNA_PREC_MIXED 4u
/* GNA_WS_TABLES_VALID: the per-node tables at the front of d_workspace (1/E and h*w of
 * every GL node, 2 * align16(order * nbins * 8) bytes; their offset does not depend on
 * npoints) were built by an earlier gna_oscprob_batch / _ex call on this workspace with
 * the same edge values, nbins and order, and that call is complete in stream order.
 * The call then forms only the per-point coefficients (a2) before the main pass, instead
 * of re-deriving 1/E for every node ((a1): the energy grid is set up once).
 * For callers that split one batch over several calls (chunked gathers, fit loops).
 * Outputs are bitwise identical to a call without the flag.  Validation is unchanged;
 * a workspace that does not hold such tables gives unspecified results (never a fault). */
#define GNA_WS_TABLES_VALID 8u

int gna_oscprob_batch_ex(const gna_param_batch* pts, const double* L_km, const double* omega,
                         int32_t nbase, const double* d_edges, int64_t nbins, int32_t order,
                         double* d_spectra, const double* d_data, double* d_chi2,
                         void* d_workspace, size_t workspace_bytes, uint32_t flags,
                         void* stream);

/* ---------------------------------------------------------------------------
 * gna_oscprob_eval_ex / gna_gl_integrate_ex — gna_oscprob_eval / gna_gl_integrate
 * with flags: 0 = the same call; GNA_PREC_MIXED = the mixed-precision tier above
 * (fp64 phase and modulo-2 reduction, fp32 polynomial and term sum, two energies or
 * GL nodes per packed FP32 FMA).  Tier tolerance: 1e-6 absolute on P, 1e-5
 * relative on bin integrals.  Any other flag bit: GNA_EINVAL.
 * Arguments, layouts and other errors as the fp64 calls.
 * ------------------------------------------------------------------------- */
int gna_oscprob_eval_ex(const gna_osc_params* p, double L_km, const double* d_E, int64_t n,
                        double* d_P, uint32_t flags, void* stream);

int gna_gl_integrate_ex(const gna_osc_params* p, double L_km, const double* d_edges,
                        int64_t nbins, int32_t order, double* d_bins, uint32_t flags,
                        void* stream);

/* ---------------------------------------------------------------------------
 * gna_fit_pattern_search — NEXT-4 (second part): a chi^2 minimiser that stays on the
 * GPU (the minimisation of P:446-451).  Deterministic compass search over
 * x = (theta12, theta13, dm2_21, dm2_31): each iteration evaluates chi^2 of the 81
 * points x_c + s * {-1, 0, +1}^4 (baselines, bins, order and data as in
 * gna_oscprob_batch) — a 9 x 9 product of (theta12, theta13) and (dm2_21, dm2_31)
 * values, evaluated with the separable scan of gna_oscprob_scan — moves x_c to the
 * argmin (lowest index on ties) or halves s when x_c is already best.  Everything is stream-ordered (no host
 * synchronisation), so the niter iterations can be captured in one CUDA graph.
 * d_state: device [8] = x_c[4] followed by s[4], updated in place.
 * d_hist: device [niter] best chi^2 after each iteration, or NULL.
 * d_workspace: >= gna_fit_workspace_size(nbase, nbins, order) bytes, 16-byte aligned.
 * ------------------------------------------------------------------------- */
size_t gna_fit_workspace_size(int32_t nbase, int64_t nbins, int32_t order);

int gna_fit_pattern_search(const double* L_km, const double* omega, int32_t nbase,
                           const double* d_edges, int64_t nbins, int32_t order,
                           const double* d_data, double* d_state, int32_t niter, double* d_hist,
                           void* d_workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * gna_oscprob_scan — separable grid scan (the paper's
 * "computed only once ... re-computed only if any of the variables or inputs it
 * depends on were modified", and one transformation per formula item,
 * P:641-642).  The parameter points are the grid {mixing point a} x {mass point c}:
 *   point p = c * nmix + a  <->  (theta12[a], theta13[a], dm2_21[c], dm2_31[c]).
 * The result is the same quantity as gna_oscprob_batch on that expanded list of
 * points (same tolerance, different association): with
 *   G[c][ij][k] = sum_b omega_b h_k sum_i w_i sin^2 Delta_ij(c, b, E_ki),
 *   H[k] = (sum_b omega_b) h_k sum_i w_i,
 *   T[p][k] = H[k] - sum_ij w_ij(a) G[c][ij][k],  chi2[p] as for the batch,
 * the sin^2 work scales with nmass instead of nmass * nmix; the rest is a rank-3
 * update per point, bound by writing the spectra.
 * g: host struct of DEVICE arrays theta12/theta13 [nmix], dm2_21/dm2_31 [nmass].
 * d_spectra: device [nmass][nmix][nbins] or NULL; d_chi2: device [nmass][nmix] or
 * NULL (not both); d_data as for the batch.  d_workspace: device, 32-byte aligned,
 * >= gna_oscprob_scan_workspace_size(nmix, nmass, nbins) bytes.  L_km/omega/nbase/
 * d_edges/nbins/order and errors as for gna_oscprob_batch.
 * ------------------------------------------------------------------------- */
typedef struct gna_scan_grid {
  const double* theta12;
  const double* theta13;
  int64_t nmix;
  const double* dm2_21;
  const double* dm2_31;
  int64_t nmass;
} gna_scan_grid;

size_t gna_oscprob_scan_workspace_size(int64_t nmix, int64_t nmass, int64_t nbins);

int gna_oscprob_scan(const gna_scan_grid* g, const double* L_km, const double* omega,
                     int32_t nbase, const double* d_edges, int64_t nbins, int32_t order,
                     double* d_spectra, const double* d_data, double* d_chi2, void* d_workspace,
                     size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Host-buffer variants (the end-to-end path; §4.1 "CUDA Streams,
 * datasets are divided into smaller sizes to organize overlapped execution,
 * asynchronous memory copying").  Same arithmetic as the device entry points
 * (bitwise identical results); inputs are copied host->device and results
 * device->host in chunks on three library-owned streams (H2D, compute, D2H; a
 * ring of three chunk slots ordered by events), so chunk c's D2H and chunk c+2's
 * H2D overlap chunk c+1's kernel while every kernel has the whole GPU.  chunk = 0
 * picks a default (eval: 4 Mi energies, GL: 1 Mi bins, batch: ~8 MiB of spectra
 * per chunk, or a single chunk when only chi^2 is requested; the batch uploads all
 * points and builds the node tables once per call).  Pinned (page-locked) host
 * arrays give full PCIe speed; pageable ones work but copy synchronously.  Batch
 * spectra in page-locked memory (and chunk_points = 0) are stored by the kernel
 * straight into host memory over PCIe during the one launch over all points — unless
 * the points-across-lanes kernel runs (<= 2 baselines and >= 256 points), whose
 * scattered stores are staged instead.
 * Returns after the results are in host memory (also on error).
 * ------------------------------------------------------------------------- */
int gna_oscprob_eval_host(const gna_osc_params* p, double L_km, const double* h_E, int64_t n,
                          double* h_P, int64_t chunk, void* stream);

int gna_gl_integrate_host(const gna_osc_params* p, double L_km, const double* h_edges,
                          int64_t nbins, int32_t order, double* h_bins, int64_t chunk,
                          void* stream);

int gna_oscprob_batch_host(const gna_param_batch* h_pts, const double* L_km, const double* omega,
                           int32_t nbase, const double* h_edges, int64_t nbins, int32_t order,
                           double* h_spectra, const double* h_data, double* h_chi2,
                           int64_t chunk_points, void* stream);

/* Frees the library-owned staging buffers of the *_host entry points. */
void gna_release(void);

/* Copies the library's Gauss-Legendre rule of the given order (nodes ascending
 * on [-1, 1]) into host arrays t[order], w[order].  EINVAL for a bad order.   */
int gna_gl_rule(int32_t order, double* t, double* w);

/* Human-readable text for a gna_status code (static storage). */
const char* gna_strerror(int code);

/* cudaError_t behind the last GNA_ECUDA returned on this thread (0 if none). */
int gna_last_cuda_error(void);

/* GNA_ABI_VERSION of the loaded library. */
int gna_abi_version(void);

/* Number of kernels launched through the library (all threads) since load
 * (diagnostics for the bench's gpu_launches count).                          */
int64_t gna_launch_count(void);

/* Degree in u = f^2 of the minimax v(u) = -cos(pi sqrt u)/2 compiled into the sin^2
 * kernels (7: max error 1.1e-15 per term; 8: 1.1e-16).  Each sin^2 term costs
 * degree + 5 FP64 instructions; the bench's roofline uses it.  */
int gna_sin2_poly_degree(void);

#ifdef __cplusplus
}
#endif
#endif /* GNA_B200_H */

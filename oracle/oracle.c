/*
 * oracle.c — plain, slow, obviously-correct CPU oracle for the GNA hot path
 * (arXiv:1804.07682, "GNA: GPU support for the Global Neutrino Analysis framework").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load or call this library.  The product
 * path (paper_1804_07682_b200/) never imports, links or executes anything here,
 * and this file shares no code, header, table or constant generator with it.
 *
 * Citations: P:NNN = PAPER.md line NNN, S:NNN = SPEC.md line NNN,
 * DESIGN.md Rn = reading n in DESIGN.md section "Readings of the paper".
 *
 * Precision: IEEE-754 binary64 throughout, compiled with -O2 -ffp-contract=off
 * (no FMA contraction, no fast-math), glibc sin/cos.  Sums run left to right in
 * the order the cited passage writes them.
 *
 * Parity pins (tests/test_oracle_pins.py): every function below is pinned to
 * something other than itself — closed forms, textbook special cases, mpmath
 * at 40 digits, numpy.polynomial.legendre.leggauss, the sine-integral closed
 * form of the bin integral, brute-force quadrature.  No function here is
 * "parity unpinned".
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* S:265, S:317 (Design decision "Phase/units convention"): the literal used for
 * Delta_ij = 1.26693268 * dm2[eV^2] * L[km] / E[GeV].  DESIGN.md R1.           */
#define ORACLE_PHASE_K 1.26693268

#define PI_ORACLE 3.14159265358979323846

/* ---------------------------------------------------------------------------
 * PMNS matrix V (§4.1 "complex unitary matrix called a PMNS matrix";
 * factorisation S:253-256 and S:316: V = R23(theta23) . U13(theta13, delta) .
 * R12(theta12); antineutrino -> elementwise complex conjugate).
 * V is row-major [alpha][i], alpha = e, mu, tau; i = 1, 2, 3 (0-based here).
 * ------------------------------------------------------------------------- */
void oracle_pmns(double theta12, double theta13, double theta23, double delta_cp,
                 int antineutrino, double complex V[9]) {
  double c12 = cos(theta12), s12 = sin(theta12);
  double c13 = cos(theta13), s13 = sin(theta13);
  double c23 = cos(theta23), s23 = sin(theta23);
  double complex eid = cexp(I * delta_cp); /* e^{+i delta} */

  double complex R23[9] = {1, 0, 0,
                           0, c23, s23,
                           0, -s23, c23};
  double complex U13[9] = {c13, 0, s13 * conj(eid),
                           0, 1, 0,
                           -s13 * eid, 0, c13};
  double complex R12[9] = {c12, s12, 0,
                           -s12, c12, 0,
                           0, 0, 1};
  double complex T[9];
  /* T = R23 . U13 */
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double complex acc = 0;
      for (int k = 0; k < 3; ++k) acc += R23[3 * r + k] * U13[3 * k + c];
      T[3 * r + c] = acc;
    }
  /* V = T . R12 */
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double complex acc = 0;
      for (int k = 0; k < 3; ++k) acc += T[3 * r + k] * R12[3 * k + c];
      V[3 * r + c] = acc;
    }
  if (antineutrino)
    for (int k = 0; k < 9; ++k) V[k] = conj(V[k]);
}

/* ---------------------------------------------------------------------------
 * Oscillation phase:
 *   Delta = 1.26693268 * dm2 * L / (E / 1000),  E in MeV, L in km, dm2 in eV^2.
 * Evaluated left to right exactly as S:265 writes it.
 * ------------------------------------------------------------------------- */
double oracle_phase(double dm2, double L_km, double E_MeV) {
  return ORACLE_PHASE_K * dm2 * L_km / (E_MeV / 1000.0);
}

/* ---------------------------------------------------------------------------
 * General vacuum oscillation probability, §4.1 (displayed multline):
 *   P(a->b) = delta_ab - 4 sum_{i>j} Re(X_ij) sin^2(Delta_ij)
 *                      + 2 sum_{i>j} Im(X_ij) sin(2 Delta_ij),
 *   X_ij = V*_{a i} V_{b i} V_{a j} V*_{b j},
 * with Delta_ij = dm2_ij L / 4E (S:265 units; the paper's sin(dm2 L / 2E) is
 * sin(2 Delta_ij), "Design decisions"), pairs in the order (2,1), (3,1),
 * (3,2), summed left to right, and dm2_32 = dm2_31 - dm2_21
 * (S:237).  alpha, beta in {0,1,2} = {e, mu, tau}.
 * ------------------------------------------------------------------------- */
double oracle_prob(int alpha, int beta, const double complex V[9], double dm2_21,
                   double dm2_31, double L_km, double E_MeV) {
  const int pi_[3] = {1, 2, 2}; /* i of the pair, 0-based: (2,1),(3,1),(3,2) */
  const int pj_[3] = {0, 0, 1}; /* j of the pair                              */
  double dm2[3];
  dm2[0] = dm2_21;
  dm2[1] = dm2_31;
  dm2[2] = dm2_31 - dm2_21;

  double re_sum = 0.0, im_sum = 0.0;
  for (int p = 0; p < 3; ++p) {
    int i = pi_[p], j = pj_[p];
    double complex X = conj(V[3 * alpha + i]) * V[3 * beta + i] * V[3 * alpha + j] *
                       conj(V[3 * beta + j]);
    double D = oracle_phase(dm2[p], L_km, E_MeV);
    double s = sin(D);
    re_sum += creal(X) * (s * s);
    im_sum += cimag(X) * sin(2.0 * D);
  }
  double kron = (alpha == beta) ? 1.0 : 0.0;
  return kron - 4.0 * re_sum + 2.0 * im_sum;
}

/* ---------------------------------------------------------------------------
 * Independent amplitude form ("oscprob_amplitude_oracle"):
 *   P(a->b) = | sum_i V*_{a i} V_{b i} exp(-i 2 Delta_{i1}) |^2,
 * Delta_{11} = 0, Delta_{21} from dm2_21, Delta_{31} from dm2_31.
 * Shares no arithmetic with oracle_prob other than oracle_phase.
 * ------------------------------------------------------------------------- */
double oracle_prob_amplitude(int alpha, int beta, const double complex V[9],
                             double dm2_21, double dm2_31, double L_km, double E_MeV) {
  double D[3];
  D[0] = 0.0;
  D[1] = oracle_phase(dm2_21, L_km, E_MeV);
  D[2] = oracle_phase(dm2_31, L_km, E_MeV);
  double complex A = 0;
  for (int i = 0; i < 3; ++i)
    A += conj(V[3 * alpha + i]) * V[3 * beta + i] * cexp(-I * 2.0 * D[i]);
  double a = cabs(A);
  return a * a;
}

/* Two-flavour survival probability: 1 - sin^2(2 theta) sin^2(Delta). */
double oracle_two_flavor(double theta, double dm2, double L_km, double E_MeV) {
  double s2t = sin(2.0 * theta);
  double sD = sin(oracle_phase(dm2, L_km, E_MeV));
  return 1.0 - (s2t * s2t) * (sD * sD);
}

static int set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
  return nthreads;
#else
  (void)nthreads;
  return 1;
#endif
}

/* ---------------------------------------------------------------------------
 * Elementwise P(a->b) over an energy vector (the OscProb transformation of
 * P:641-647 §4.1; Table 1 times it).  alpha = beta = e is the hot
 * path's P_ee.  Returns the number of threads used.
 * ------------------------------------------------------------------------- */
int oracle_prob_array(int alpha, int beta, double theta12, double theta13, double theta23,
                      double delta_cp, int antineutrino, double dm2_21, double dm2_31,
                      double L_km, const double* E, int64_t n, double* P, int nthreads) {
  double complex V[9];
  oracle_pmns(theta12, theta13, theta23, delta_cp, antineutrino, V);
  int nt = set_threads(nthreads);
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int64_t k = 0; k < n; ++k)
    P[k] = oracle_prob(alpha, beta, V, dm2_21, dm2_31, L_km, E[k]);
  return nt;
}

/* ---------------------------------------------------------------------------
 * Gauss-Legendre nodes and weights on [-1, 1] (textbook Newton iteration on the
 * Legendre polynomial P_n via its three-term recurrence; R5: GL is
 * not in the paper, it comes from BASELINE.json north_star).
 *   start z0 = cos(pi (i + 3/4) / (n + 1/2)); Newton until |dz| <= 4e-16 or
 *   100 iterations; w = 2 / ((1 - z^2) P_n'(z)^2); nodes ascending; the
 *   middle node of odd n is +0.0.
 * ------------------------------------------------------------------------- */
static void legendre_pn(int n, double z, double* pn, double* dpn) {
  double p1 = 1.0, p2 = 0.0;
  for (int j = 1; j <= n; ++j) {
    double p3 = p2;
    p2 = p1;
    p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
  }
  *pn = p1;                                  /* P_n(z)     */
  *dpn = n * (z * p1 - p2) / (z * z - 1.0);  /* P_n'(z)    */
}

int oracle_gauleg(int n, double* t, double* w) {
  if (n < 1) return -1;
  int m = (n + 1) / 2;
  for (int i = 0; i < m; ++i) {
    double z = cos(PI_ORACLE * (i + 0.75) / (n + 0.5));
    double pn, dpn;
    for (int it = 0; it < 100; ++it) {
      legendre_pn(n, z, &pn, &dpn);
      double z1 = z;
      z = z1 - pn / dpn;
      if (fabs(z - z1) <= 4e-16) break;
    }
    if ((n & 1) && i == m - 1) z = 0.0; /* middle node of odd n */
    legendre_pn(n, z, &pn, &dpn);
    double wi = 2.0 / ((1.0 - z * z) * dpn * dpn);
    t[i] = -z;            /* ascending: negative root first */
    t[n - 1 - i] = z;
    w[i] = wi;
    w[n - 1 - i] = wi;
  }
  if (n & 1) t[m - 1] = 0.0;
  return 0;
}

/* ---------------------------------------------------------------------------
 * Per-bin Gauss-Legendre integral of P_ee (north_star; R5, R6):
 *   c_k = (e_k + e_{k+1}) / 2,  h_k = (e_{k+1} - e_k) / 2,
 *   S_k = h_k * sum_{i=0}^{n-1} w_i * P_ee(c_k + h_k t_i),  i ascending.
 * ------------------------------------------------------------------------- */
int oracle_gl_integrate(double theta12, double theta13, double theta23, double delta_cp,
                        int antineutrino, double dm2_21, double dm2_31, double L_km,
                        const double* edges, int64_t nbins, int order, double* bins,
                        int nthreads) {
  double t[64], w[64];
  if (order < 1 || order > 64) return -1;
  oracle_gauleg(order, t, w);
  double complex V[9];
  oracle_pmns(theta12, theta13, theta23, delta_cp, antineutrino, V);
  int nt = set_threads(nthreads);
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int64_t k = 0; k < nbins; ++k) {
    double c = (edges[k] + edges[k + 1]) / 2.0;
    double h = (edges[k + 1] - edges[k]) / 2.0;
    double s = 0.0;
    for (int i = 0; i < order; ++i)
      s += w[i] * oracle_prob(0, 0, V, dm2_21, dm2_31, L_km, c + h * t[i]);
    bins[k] = h * s;
  }
  return nt;
}

/* ---------------------------------------------------------------------------
 * Per-bin Gauss-Legendre integral of P(alpha -> beta) for any channel (the general
 * formula of oracle_prob; binned as in oracle_gl_integrate):
 *   S_k = h_k * sum_{i=0}^{n-1} w_i * P_ab(c_k + h_k t_i),  i ascending.
 * ------------------------------------------------------------------------- */
int oracle_gl_integrate_ab(int alpha, int beta, double theta12, double theta13, double theta23,
                           double delta_cp, int antineutrino, double dm2_21, double dm2_31,
                           double L_km, const double* edges, int64_t nbins, int order,
                           double* bins, int nthreads) {
  double t[64], w[64];
  if (order < 1 || order > 64) return -1;
  oracle_gauleg(order, t, w);
  double complex V[9];
  oracle_pmns(theta12, theta13, theta23, delta_cp, antineutrino, V);
  int nt = set_threads(nthreads);
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int64_t k = 0; k < nbins; ++k) {
    double c = (edges[k] + edges[k + 1]) / 2.0;
    double h = (edges[k + 1] - edges[k]) / 2.0;
    double s = 0.0;
    for (int i = 0; i < order; ++i)
      s += w[i] * oracle_prob(alpha, beta, V, dm2_21, dm2_31, L_km, c + h * t[i]);
    bins[k] = h * s;
  }
  return nt;
}

/* ---------------------------------------------------------------------------
 * Batch over parameter points and baselines (north_star "batched over
 * parameter points"; baseline merge = SPEC weighted_sum S:299-307 over the
 * one-E-node / m-OscProb topology S:431-439):
 *   T[p][k]  = sum_b omega[b] * S_{p,b,k}          (b ascending)
 *   chi2[p]  = sum_k (T[p][k] - D[k])^2 / D[k]     (k ascending; R8)
 * Points are SoA arrays theta12[P], theta13[P], dm2_21[P], dm2_31[P]; theta23,
 * delta_cp and the antineutrino flag are shared scalars (they do not change
 * P_ee, R2, but the general formula takes them).
 * spectra (P*nbins) and chi2 (P) may be NULL independently; chi2 needs data.
 * ------------------------------------------------------------------------- */
int oracle_batch(const double* theta12, const double* theta13, const double* dm2_21,
                 const double* dm2_31, int64_t npoints, double theta23, double delta_cp,
                 int antineutrino, const double* L_km, const double* omega, int nbase,
                 const double* edges, int64_t nbins, int order, double* spectra,
                 const double* data, double* chi2, int nthreads) {
  double t[64], w[64];
  if (order < 1 || order > 64) return -1;
  oracle_gauleg(order, t, w);
  int nt = set_threads(nthreads);
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int64_t p = 0; p < npoints; ++p) {
    double complex V[9];
    oracle_pmns(theta12[p], theta13[p], theta23, delta_cp, antineutrino, V);
    double x2 = 0.0;
    for (int64_t k = 0; k < nbins; ++k) {
      double c = (edges[k] + edges[k + 1]) / 2.0;
      double h = (edges[k + 1] - edges[k]) / 2.0;
      double T = 0.0;
      for (int b = 0; b < nbase; ++b) {
        double s = 0.0;
        for (int i = 0; i < order; ++i)
          s += w[i] * oracle_prob(0, 0, V, dm2_21[p], dm2_31[p], L_km[b], c + h * t[i]);
        T += omega[b] * (h * s);
      }
      if (spectra) spectra[p * nbins + k] = T;
      if (chi2 && data) {
        double d = T - data[k];
        x2 += d * d / data[k];
      }
    }
    if (chi2 && data) chi2[p] = x2;
  }
  return nt;
}

int oracle_max_threads(void) { return set_threads(0); }

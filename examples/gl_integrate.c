/* examples/gl_integrate.c — the C ABI used from plain C11 (no Python, no torch).
 *
 * Computes the per-bin Gauss-Legendre integrals of P_ee (gna_gl_integrate,
 * include/gna_b200.h) for the SPEC canonical point at L = 52.5 km over
 * 1-10 MeV, and checks two properties that hold exactly or nearly so:
 *   zero mixing  -> every bin equals its width (P_ee = 1);
 *   canonical    -> 0 < S_k < width_k, and the host-buffer entry point gives the same bits.
 * Device memory comes from the CUDA runtime's C API; the library never allocates.
 *
 * Build (tests/test_abi_cpu.py does this):
 *   gcc -std=c11 -O2 -Iinclude -I/usr/local/cuda/include examples/gl_integrate.c \
 *       -Lpaper_1804_07682_b200 -lgna_b200 -L/usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,$PWD/paper_1804_07682_b200 -o build/gl_integrate_c
 * Exit status 0 = all checks passed.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "gna_b200.h"

#define NBINS 1000
#define ORDER 10

static int check(int rc, const char* what) {
  if (rc != GNA_OK) fprintf(stderr, "%s: %s\n", what, gna_strerror(rc));
  return rc != GNA_OK;
}

int main(void) {
  static double edges[NBINS + 1], bins[NBINS], bins_host[NBINS];
  for (int k = 0; k <= NBINS; ++k) edges[k] = 1.0 + 9.0 * k / NBINS;

  double *d_edges = NULL, *d_bins = NULL;
  if (cudaMalloc((void**)&d_edges, sizeof edges) != cudaSuccess ||
      cudaMalloc((void**)&d_bins, sizeof bins) != cudaSuccess) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 2;
  }
  cudaMemcpy(d_edges, edges, sizeof edges, cudaMemcpyHostToDevice);

  gna_osc_params zero = {0.0, 0.0, 0.0, 0.0, 7.53e-5, 2.52e-3, 0};
  gna_osc_params canon = {0.5838, 0.1496, 0.0, 0.0, 7.53e-5, 2.52e-3, 0};
  int bad = 0;

  bad |= check(gna_gl_integrate(&zero, 52.5, d_edges, NBINS, ORDER, d_bins, NULL),
               "gna_gl_integrate(zero mixing)");
  cudaMemcpy(bins, d_bins, sizeof bins, cudaMemcpyDeviceToHost);  /* syncs the stream */
  double worst = 0.0;
  for (int k = 0; k < NBINS; ++k) {
    const double w = edges[k + 1] - edges[k];
    worst = fmax(worst, fabs(bins[k] / w - 1.0));
  }
  printf("zero mixing: max |S_k / width - 1| = %.3g\n", worst);
  bad |= worst > 1e-15;

  bad |= check(gna_gl_integrate(&canon, 52.5, d_edges, NBINS, ORDER, d_bins, NULL),
               "gna_gl_integrate(canonical)");
  cudaMemcpy(bins, d_bins, sizeof bins, cudaMemcpyDeviceToHost);
  for (int k = 0; k < NBINS; ++k) {
    const double w = edges[k + 1] - edges[k];
    if (!(bins[k] > 0.0 && bins[k] < w)) bad = 1;
  }
  bad |= check(gna_gl_integrate_host(&canon, 52.5, edges, NBINS, ORDER, bins_host, 0, NULL),
               "gna_gl_integrate_host");
  bad |= memcmp(bins, bins_host, sizeof bins) != 0;
  printf("canonical: S_0 = %.17g, S_%d = %.17g, host path bitwise equal: %s\n", bins[0],
         NBINS - 1, bins[NBINS - 1], memcmp(bins, bins_host, sizeof bins) ? "no" : "yes");

  /* argument validation happens before any launch */
  bad |= gna_gl_integrate(&canon, 52.5, d_edges, NBINS, 0, d_bins, NULL) != GNA_EINVAL;
  bad |= gna_gl_integrate(&canon, -1.0, d_edges, NBINS, ORDER, d_bins, NULL) != GNA_EINVAL;

  cudaFree(d_edges);
  cudaFree(d_bins);
  printf("%s\n", bad ? "FAILED" : "ok");
  return bad;
}

// Accuracy probe of rcp.approx.ftz.f64 (MUFU.RCP64H seed) and of one cubic Newton step,
// over 2^24 inputs spanning [1, 2) and the energy range 1-10 MeV.  Decides how many
// Newton steps the kernels need.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void k(double* err_seed, double* err_cubic, double* err_quad2, int n, double lo, double hi) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = lo + (hi - lo) * ((double)i + 0.5) / n;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double exact = 1.0 / x;  // IEEE correctly rounded
  err_seed[i] = fabs(r - exact) / exact;
  double e = fma(-x, r, 1.0);
  double e2 = fma(e, e, e);
  double rc = fma(r, e2, r);
  err_cubic[i] = fabs(rc - exact) / exact;
  double rq = fma(r, e, r);
  e = fma(-x, rq, 1.0);
  rq = fma(rq, e, rq);
  err_quad2[i] = fabs(rq - exact) / exact;
}

int main() {
  const int n = 1 << 24;
  double *a, *b, *c;
  cudaMallocManaged(&a, n * 8); cudaMallocManaged(&b, n * 8); cudaMallocManaged(&c, n * 8);
  const double ranges[2][2] = {{1.0, 2.0}, {1.0, 10.0}};
  for (auto& rg : ranges) {
    k<<<(n + 255) / 256, 256>>>(a, b, c, n, rg[0], rg[1]);
    cudaDeviceSynchronize();
    double ms = 0, mc = 0, mq = 0;
    for (int i = 0; i < n; ++i) { ms = fmax(ms, a[i]); mc = fmax(mc, b[i]); mq = fmax(mq, c[i]); }
    printf("{\"range\": [%g, %g], \"seed_max_rel\": %.3e, \"seed_bits\": %.1f, \"cubic_max_rel\": %.3e, "
           "\"two_quadratic_max_rel\": %.3e, \"ulp_rel\": %.3e}\n", rg[0], rg[1], ms, -log2(ms), mc, mq,
           ldexp(1.0, -52));
  }
  return 0;
}

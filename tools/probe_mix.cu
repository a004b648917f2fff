// probe_mix.cu — FP64-pipe ceiling of the exact sin^2 instruction mix of the batch kernel
// (gna_device.cuh sin2c: 3 reduction ops, DMUL, degree-7 Horner, sign flip, accumulate),
// with no memory traffic: coefficients from the constant bank, 1/E from the thread id.
// Prints the FP64 instruction rate as a fraction of 148 x 64 x clock, per chain count N
// and warps per SM.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_mix probe_mix.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

__constant__ double c_p[8];
__constant__ double2 c_coef[24];

__device__ __forceinline__ double s2(double kq, double iE) {
  const double M = 6755399441055744.0;
  const double t = fma(kq, iE, M);
  const double q = t - M;
  const double f = fma(kq, iE, -q);
  const double u = f * f;
  double p = fma(u, c_p[7], c_p[6]);
  p = fma(p, u, c_p[5]);
  p = fma(p, u, c_p[4]);
  p = fma(p, u, c_p[3]);
  p = fma(p, u, c_p[2]);
  p = fma(p, u, c_p[1]);
  p = fma(p, u, c_p[0]);
  const int odd = __double2loint(t) << 31;
  return __hiloint2double(__double2hiint(p) ^ odd, __double2loint(p));
}

template <int N>
__global__ void k_mix(double* out, int reps) {
  double iE[N], a[N];
#pragma unroll
  for (int n = 0; n < N; ++n) {
    iE[n] = 0.1 + 1e-6 * (threadIdx.x + 37 * n + blockIdx.x);
    a[n] = 0.0;
  }
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int n = 0; n < N; ++n) iE[n] += 1e-9;  // not loop-invariant (1 DADD per 288 ops)
#pragma unroll 2
    for (int j = 0; j < 24; ++j) {
      const double2 cw = c_coef[j];
#pragma unroll
      for (int n = 0; n < N; ++n) a[n] = fma(cw.y, s2(cw.x, iE[n]), a[n]);
    }
  }
  double s = 0;
#pragma unroll
  for (int n = 0; n < N; ++n) s += a[n];
  if (s == 1234.5) out[0] = s;
}

template <int N>
int run(int warps_per_sm, int sms, double clk_ghz) {
  const int reps = 200;
  const int blocks = sms * warps_per_sm;
  double* d;
  CK(cudaMalloc(&d, 8));
  k_mix<N><<<blocks, 32>>>(d, reps);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_mix<N><<<blocks, 32>>>(d, reps);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = (double)blocks * 32 * reps * 24 * N * 12;  // 12 FP64 per term
  const double rate = ops / (ms * 1e-3);
  const double peak = (double)sms * 64 * clk_ghz * 1e9;
  printf("{\"N\": %d, \"warps_per_sm\": %d, \"ms\": %.4f, \"T_fp64_per_s\": %.3f, \"frac\": %.4f}\n",
         N, warps_per_sm, ms, rate / 1e12, rate / peak);
  cudaFree(d);
  return 0;
}

int main() {
  double p[8] = {-0.5, 1.2337005501361697, -0.2536695079010480, 0.0208634807633529,
                 -0.0009192602748394, 0.0000252020423806, -0.0000004710874779, 0.0000000063866030};
  double2 cf[24];
  for (int j = 0; j < 24; ++j) cf[j] = make_double2(1000.0 + 37.0 * j, 0.01 * (j + 1));
  CK(cudaMemcpyToSymbol(c_p, p, sizeof(p)));
  CK(cudaMemcpyToSymbol(c_coef, cf, sizeof(cf)));
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const double ghz = clk / 1e6;
  printf("{\"sms\": %d, \"clock_ghz\": %.3f}\n", sms, ghz);
  for (int w : {4, 8, 12, 16, 20, 24, 32}) {
    run<5>(w, sms, ghz);
    run<10>(w, sms, ghz);
  }
  return 0;
}

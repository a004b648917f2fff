// FP64-pipe microbenchmark for B200 (sm_100a): measures the per-chip issue rate
// of DFMA / DMUL / DADD, FRND.F64 (cvt.rni.f64.f64), MUFU.RCP64H
// (rcp.approx.ftz.f64) and DFMA interleaved with integer ALU work.
// Used to fix the FP64 roofline denominator in DESIGN.md (the B200 guide states
// no FP64 number). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 probe_fp64.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

constexpr int CH = 8;  // independent chains per thread

__global__ void k_dfma(double* out, double a, double b, int iters) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dadd(double* out, double a, double b, int iters) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = x[c] + a;
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

// alternating FRND + DADD per chain: rate compared with 2x DADD
__global__ void k_frnd(double* out, double a, double b, int iters) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      double r;
      asm volatile("cvt.rni.f64.f64 %0, %1;" : "=d"(r) : "d"(x[c]));
      x[c] = r + a;
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

// alternating MUFU.RCP64H + DADD
__global__ void k_rcp(double* out, double a, double b, int iters) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = 1.5 + threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      double r;
      asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[c]));
      x[c] = r + a;
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

// DFMA with one integer op (on the hi word of a side value) per DFMA
__global__ void k_dfma_int(double* out, double a, double b, int iters) {
  double x[CH];
  uint32_t m[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x * 1e-3 + c; m[c] = threadIdx.x + c; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      x[c] = fma(x[c], a, b);
      m[c] = (m[c] ^ (uint32_t)i) + 0x9e3779b9u;
    }
  }
  double s = 0;
  uint32_t t = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) { s += x[c]; t ^= m[c]; }
  if (s == 12345.678 || t == 0x12345u) out[0] = s + t;
}

// F2F.F32.F64 (double -> float, round to nearest) alternating with a DADD: rate of the
// conversion relative to the FP64 pipe (mixed-precision tier, NEXT-3)
__global__ void k_f2f(double* out, double a, double b, int iters) {
  double x[CH];
  float y[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = 1.5 + threadIdx.x * 1e-3 + c; y[c] = 0.f; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const float f = __double2float_rn(x[c]);
      y[c] = fmaf(y[c], 0.999f, f);
      x[c] = x[c] + a;
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c] + y[c];
  if (s == 12345.678) out[0] = s;
}

// FP32 FFMA chains (FP32 pipe rate)
__global__ void k_ffma(double* out, double a, double b, int iters) {
  float x[CH];
  const float fa = (float)a, fb = (float)b;
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], fa, fb);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678f) out[0] = s;
}

typedef void (*kfn)(double*, double, double, int);

static int run(const char* name, kfn f, double ops_per_inner, int blocks, int threads, int iters,
               double* d_out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  f<<<blocks, threads>>>(d_out, 0.999999, 1e-7, iters);  // warm
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    f<<<blocks, threads>>>(d_out, 0.999999, 1e-7, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  double ops = (double)blocks * threads * iters * CH * ops_per_inner;
  printf("{\"probe\": \"%s\", \"blocks\": %d, \"threads\": %d, \"ms\": %.4f, \"Gops_per_s\": %.1f}\n",
         name, blocks, threads, best, ops / (best * 1e-3) / 1e9);
  return 0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sm\": %d, \"cc\": \"%d.%d\", \"clock_khz\": %d}\n", p.name,
         p.multiProcessorCount, p.major, p.minor, clk);
  double* d_out; CK(cudaMalloc(&d_out, 64));
  int sms = p.multiProcessorCount;
  if (getenv("PROBE_DFMA_ONLY")) {  // bench.py: the live FP64 denominator, ~10 ms of GPU time
    run("dfma", k_dfma, 1.0, sms * 8, 256, 20000, d_out);
    return 0;
  }
  for (int occ : {4, 8}) {
    run("dfma", k_dfma, 1.0, sms * occ, 256, 20000, d_out);
    run("dadd", k_dadd, 1.0, sms * occ, 256, 20000, d_out);
    run("frnd+dadd(count=pairs)", k_frnd, 1.0, sms * occ, 256, 10000, d_out);
    run("rcp64h+dadd(count=pairs)", k_rcp, 1.0, sms * occ, 256, 10000, d_out);
    run("dfma+int(count=dfma)", k_dfma_int, 1.0, sms * occ, 256, 20000, d_out);
    run("f2f+ffma+dadd(count=triples)", k_f2f, 1.0, sms * occ, 256, 10000, d_out);
    run("ffma", k_ffma, 1.0, sms * occ, 256, 40000, d_out);
  }
  if (getenv("PROBE_SUSTAINED")) run("dfma_sustained", k_dfma, 1.0, sms * 8, 256, 800000, d_out);
  return 0;
}

// probe_lat.cu — dependent-issue latency (cycles) of DFMA / DADD / DMUL / IMAD+LOP3 sign flip on
// one warp of one SM, and DFMA throughput of one warp with K independent chains.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_lat probe_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP, int K>
__global__ void k_lat(double* out, long long* cyc, double a, double b, int iters) {
  double x[K];
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = threadIdx.x * 1e-3 + k;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (OP == 0) x[k] = fma(x[k], a, b);
      if (OP == 1) x[k] = x[k] + a;
      if (OP == 2) x[k] = x[k] * a;
      if (OP == 3) {  // DFMA then sign flip of the hi word (the sin2c tail)
        const double y = fma(x[k], a, b);
        x[k] = __hiloint2double(__double2hiint(y) ^ (__double2loint(y) << 31), __double2loint(y));
      }
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k];
  if (s == 1234.5) out[0] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int OP, int K>
void run(const char* name, double* d, long long* c) {
  const int iters = 4096;
  k_lat<OP, K><<<1, 32>>>(d, c, 1.0000001, 1e-7, iters);
  cudaDeviceSynchronize();
  k_lat<OP, K><<<1, 32>>>(d, c, 1.0000001, 1e-7, iters);
  long long h = 0;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("{\"op\": \"%s\", \"chains\": %d, \"cycles_per_iter_per_chain_step\": %.2f, "
         "\"cycles_per_op\": %.2f}\n", name, K, (double)h / iters, (double)h / iters / K);
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 8);
  cudaMalloc(&c, 8);
  run<0, 1>("dfma", d, c);
  run<1, 1>("dadd", d, c);
  run<2, 1>("dmul", d, c);
  run<3, 1>("dfma+signflip", d, c);
  run<0, 2>("dfma", d, c);
  run<0, 4>("dfma", d, c);
  run<0, 8>("dfma", d, c);
  run<0, 16>("dfma", d, c);
  run<0, 32>("dfma", d, c);
  return 0;
}

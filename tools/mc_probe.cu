// Can this GPU create an NVLS multicast object on its own (one device)?  Driver API, printed
// step by step.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o build/mc_probe
//                        tools/mc_probe.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#define P(x) do { CUresult r_ = (x); const char* s_ = nullptr; cuGetErrorName(r_, &s_); \
  printf("%-60s -> %s\n", #x, s_ ? s_ : "?"); if (r_ != CUDA_SUCCESS) return 1; } while (0)

__global__ void k_mc_store(double* mc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(mc + i), "d"(1.0 + i) : "memory");
}

int main() {
  cudaFree(0);
  CUdevice dev;
  P(cuDeviceGet(&dev, 0));
  int mcs = 0;
  cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  printf("multicast supported: %d\n", mcs);
  for (int ht = 0; ht < 3; ++ht) {
    CUmulticastObjectProp prop = {};
    prop.numDevices = 1;
    prop.handleTypes = ht == 0 ? CU_MEM_HANDLE_TYPE_NONE
                       : ht == 1 ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_FABRIC;
    prop.size = 2 << 20;
    size_t gran = 0;
    cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    CUmemGenericAllocationHandle mc;
    CUresult r = cuMulticastCreate(&mc, &prop);
    const char* s = nullptr;
    cuGetErrorName(r, &s);
    printf("handleTypes %d gran %zu create -> %s\n", ht, gran, s);
    if (r != CUDA_SUCCESS) continue;
    P(cuMulticastAddDevice(mc, dev));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    ap.requestedHandleTypes = (CUmemAllocationHandleType)prop.handleTypes;
    CUmemGenericAllocationHandle mem;
    P(cuMemCreate(&mem, prop.size, &ap, 0));
    P(cuMulticastBindMem(mc, 0, mem, 0, prop.size, 0));
    CUdeviceptr uc, mv;
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = 0;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    P(cuMemAddressReserve(&uc, prop.size, prop.size, 0, 0));
    P(cuMemMap(uc, prop.size, 0, mem, 0));
    P(cuMemSetAccess(uc, prop.size, &acc, 1));
    P(cuMemAddressReserve(&mv, prop.size, prop.size, 0, 0));
    P(cuMemMap(mv, prop.size, 0, mc, 0));
    P(cuMemSetAccess(mv, prop.size, &acc, 1));
    k_mc_store<<<4, 256>>>((double*)mv, 1024);
    cudaError_t e = cudaDeviceSynchronize();
    printf("multimem.st kernel: %s\n", cudaGetErrorString(e));
    double h[4];
    cuMemcpyDtoH(h, uc + 8 * 1000, sizeof(h));
    printf("readback via unicast: %g %g %g %g (expect 1001 1002 1003 1004)\n", h[0], h[1], h[2], h[3]);
    return 0;
  }
  return 2;
}

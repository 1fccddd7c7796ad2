// NVSwitch multicast (NVLS) feasibility + bandwidth on B200 (NEXT-2): one multicast object bound to
// a buffer on each of N GPUs; a kernel on GPU 0 streams a local source buffer into the multicast
// address with multimem.st (the switch replicates every store to all N buffers).  Single process.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mc_bench mc_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s: %s\n", #x, s); exit(1); } } while (0)
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int U>
__global__ void __launch_bounds__(256) k_mc_store(const uint4* __restrict__ src, uint4* mc, size_t n) {
  for (size_t i0 = (size_t)blockIdx.x * 256 * U + threadIdx.x; i0 < n; i0 += (size_t)gridDim.x * 256 * U) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (i0 + k * 256 < n)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(src + i0 + k * 256));
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (i0 + k * 256 < n)
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + i0 + k * 256),
                     "r"(v[k].x), "r"(v[k].y), "r"(v[k].z), "r"(v[k].w)
                     : "memory");
  }
}

int main() {
  CU(cuInit(0));
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  for (int d = 0; d < ndev; ++d) {
    CUdevice dev;
    CU(cuDeviceGet(&dev, d));
    int mc = 0;
    CU(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    printf("device %d multicast supported: %d\n", d, mc);
  }
  if (ndev < 2) return 0;
  const size_t bytes = (size_t)2 << 30;
  for (int n : {2, 4}) {
    if (n > ndev) break;
    CUmulticastObjectProp mp = {};
    mp.numDevices = n;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = bytes;
    size_t gran = 0;
    CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    mp.size = (bytes + gran - 1) / gran * gran;
    CUmemGenericAllocationHandle mc;
    CU(cuMulticastCreate(&mc, &mp));
    for (int d = 0; d < n; ++d) {
      CUdevice dev;
      CU(cuDeviceGet(&dev, d));
      CU(cuMulticastAddDevice(mc, dev));
    }
    std::vector<CUmemGenericAllocationHandle> mem(n);
    std::vector<CUdeviceptr> va(n);
    for (int d = 0; d < n; ++d) {
      CK(cudaSetDevice(d));
      CUmemAllocationProp ap = {};
      ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
      ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      ap.location.id = d;
      ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
      size_t g2 = 0;
      CU(cuMemGetAllocationGranularity(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
      CU(cuMemCreate(&mem[d], mp.size, &ap, 0));
      CU(cuMulticastBindMem(mc, 0, mem[d], 0, mp.size, 0));
      CU(cuMemAddressReserve(&va[d], mp.size, 0, 0, 0));
      CU(cuMemMap(va[d], mp.size, 0, mem[d], 0));
      CUmemAccessDesc acc = {};
      acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      acc.location.id = d;
      acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
      CU(cuMemSetAccess(va[d], mp.size, &acc, 1));
      CK(cudaMemset((void*)va[d], 0, mp.size));
    }
    CK(cudaSetDevice(0));
    CUdeviceptr mcva;
    CU(cuMemAddressReserve(&mcva, mp.size, 0, 0, 0));
    CU(cuMemMap(mcva, mp.size, 0, mc, 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = 0;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemSetAccess(mcva, mp.size, &acc, 1));
    char* src;
    CK(cudaMalloc(&src, bytes));
    CK(cudaMemset(src, 0x5A, bytes));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int ctas : {32, 64, 148, 296}) {
      float best = 1e9;
      for (int r = 0; r < 4; ++r) {
        CK(cudaEventRecord(e0));
        k_mc_store<4><<<ctas, 256>>>((const uint4*)src, (uint4*)mcva, bytes / 16);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
      }
      CK(cudaGetLastError());
      printf("multicast to %d GPUs, %3d CTAs: %.1f GB/s per receiver (%.2f ms for %.1f GB)\n", n, ctas,
             bytes / (best / 1e3) / 1e9, best, bytes / 1e9);
    }
    for (int d = 0; d < n; ++d) {  // every receiver got the bytes
      unsigned char h[4] = {};
      CK(cudaSetDevice(d));
      CK(cudaMemcpy(h, (void*)(va[d] + bytes - 4), 4, cudaMemcpyDefault));
      printf("  device %d last bytes %02x %02x %02x %02x\n", d, h[0], h[1], h[2], h[3]);
    }
    CK(cudaSetDevice(0));
    for (int ctas : {148, 296}) {
      float best = 1e9;
      for (int r = 0; r < 4; ++r) {
        CK(cudaEventRecord(e0));
        k_mc_store<8><<<ctas, 256>>>((const uint4*)src, (uint4*)mcva, bytes / 16);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
      }
      printf("multicast to %d GPUs, %3d CTAs, unroll 8: %.1f GB/s per receiver\n", n, ctas, bytes / (best / 1e3) / 1e9);
    }
    CK(cudaFree(src));
  }
  return 0;
}

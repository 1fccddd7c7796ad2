// P2P copy design-space microbenchmark (B200, NVLink 5): which SM-driven copy style reaches the
// NVLink ceiling with how many CTAs.  Modes (GPU a -> GPU b, `bytes` per copy):
//   pull    kernel on b: 16-B loads from a's memory, stores to b's      (receiver-driven)
//   push    kernel on a: 16-B loads local, stores to b's memory          (sender-driven)
//   tma     kernel on b: cp.async.bulk global(a) -> smem -> cp.async.bulk smem -> global(b)
//   ce      cudaMemcpyPeerAsync (copy engines, zero SMs)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_bench p2p_bench.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int U>
__global__ void __launch_bounds__(512) k_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t i0 = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; i0 < n; i0 += stride) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      size_t i = i0 + (size_t)k * blockDim.x;
      if (i < n) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                              : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(src + i));
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      size_t i = i0 + (size_t)k * blockDim.x;
      if (i < n) dst[i] = v[k];
    }
  }
}

// TMA bulk pipeline: one elected thread per CTA; STAGES x SB bytes of smem
template <int STAGES, int SB>
__global__ void __launch_bounds__(128) k_tma(const char* __restrict__ src, char* __restrict__ dst, size_t bytes) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) unsigned long long bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
  }
  asm volatile("fence.mbarrier_init.release.cluster;");
  size_t nblk = bytes / SB;
  unsigned phase[STAGES] = {0};
  size_t first = blockIdx.x, step = gridDim.x;
  // prologue
  int s = 0;
  size_t issued = first, done = first;
  for (s = 0; s < STAGES && issued < nblk; ++s, issued += step) {
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    unsigned d = (unsigned)__cvta_generic_to_shared(smem + s * SB);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(SB));
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d), "l"(src + issued * SB), "r"(SB), "r"(b) : "memory");
  }
  s = 0;
  while (done < nblk) {
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    unsigned d = (unsigned)__cvta_generic_to_shared(smem + s * SB);
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                 ::"r"(b), "r"(phase[s]));
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + done * SB), "r"(d), "r"(SB) : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    done += step;
    if (issued < nblk) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(SB));
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(d), "l"(src + issued * SB), "r"(SB), "r"(b) : "memory");
      issued += step;
    }
    s = (s + 1) % STAGES;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  int a = 0, b = 1;
  size_t bytes = (size_t)2 << 30;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
  char *pa, *pb, *pb2;
  CK(cudaSetDevice(a)); CK(cudaMalloc(&pa, bytes)); CK(cudaMemset(pa, 1, bytes)); CK(cudaDeviceEnablePeerAccess(b, 0));
  CK(cudaSetDevice(b)); CK(cudaMalloc(&pb, bytes)); CK(cudaMalloc(&pb2, bytes)); CK(cudaDeviceEnablePeerAccess(a, 0));
  auto timeit = [&](int dev, auto fn) {
    CK(cudaSetDevice(dev));
    cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    fn(); CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0)); fn(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
    }
    CK(cudaGetLastError());
    return bytes / (best / 1e3) / 1e9;
  };
  size_t n = bytes / 16;
  int ctas[] = {16, 32, 48, 64, 96, 148, 296};
  printf("mode      ctas  unroll  GB/s\n");
  for (int c : ctas) {
    printf("pull  %6d  %6d  %7.1f\n", c, 8, timeit(b, [&] { k_copy<8><<<c, 512>>>((const uint4*)pa, (uint4*)pb, n); }));
    printf("pull  %6d  %6d  %7.1f\n", c, 16, timeit(b, [&] { k_copy<16><<<c, 512>>>((const uint4*)pa, (uint4*)pb, n); }));
    printf("push  %6d  %6d  %7.1f\n", c, 4, timeit(a, [&] { k_copy<4><<<c, 512>>>((const uint4*)pa, (uint4*)pb, n); }));
    printf("push  %6d  %6d  %7.1f\n", c, 8, timeit(a, [&] { k_copy<8><<<c, 512>>>((const uint4*)pa, (uint4*)pb, n); }));
  }
  CK(cudaSetDevice(b));
  constexpr int ST = 6, SB = 32768;
  CK(cudaFuncSetAttribute(k_tma<ST, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * SB));
  for (int c : ctas)
    printf("tma   %6d  %6d  %7.1f\n", c, ST, timeit(b, [&] { k_tma<ST, SB><<<c, 128, ST * SB>>>(pa, pb, bytes); }));
  printf("ce (memcpyPeer)      %7.1f\n", timeit(b, [&] { CK(cudaMemcpyPeerAsync(pb, b, pa, a, bytes, 0)); }));
  printf("local copy (HBM r+w) %7.1f (x2 for r+w)\n", timeit(b, [&] { k_copy<8><<<148 * 4, 512>>>((const uint4*)pb2, (uint4*)pb, n); }));
  // bidirectional: a pulls from b while b pulls from a (chain middle node sees both directions)
  return 0;
}

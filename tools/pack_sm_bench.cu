// How much cast-pack (fp32 -> bf16, 6 B of HBM traffic per element) can k SMs move?  The actor-step
// inflation of a concurrent publish is ~ (SMs the pack holds) x (its duration) / 148 (bench.py
// actor_stall sweep), so an SM-light pack needs a high per-SM rate.  Compares, for k SMs:
//   ldg   the k_pack access pattern: 256-thread CTAs, all resident CTAs of k SMs, 4 x 32-B loads in
//         flight per thread, 16-B streaming stores
//   tma   one CTA per SM: a producer lane issues cp.async.bulk global->smem loads into a ring of
//         STAGES x 32 KiB (fp32) with mbarrier completion; 16 consumer warps cast from smem and
//         write 16-B streaming stores
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pack_sm_bench tools/pack_sm_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t rne(uint32_t u) {
  uint32_t r = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
  return ((u & 0x7FFFFFFFu) > 0x7F800000u) ? 0x7FC0u : r;
}
__device__ __forceinline__ uint32_t p2(uint32_t a, uint32_t b) { return rne(a) | (rne(b) << 16); }
__device__ __forceinline__ uint4 ldg(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void stcs(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint32_t smid() { uint32_t s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); return s; }
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// 128 KiB fp32 units handed out by a counter; CTAs on SMs >= k leave at once
__global__ void __launch_bounds__(256) k_ldg(const float* __restrict__ src, uint8_t* __restrict__ dst, uint32_t n_units,
                                             uint32_t* work, uint32_t k) {
  __shared__ uint32_t s_u;
  if (smid() >= k) return;
  for (;;) {
    if (threadIdx.x == 0) s_u = atomicAdd(work, 1u);
    __syncthreads();
    const uint32_t u = s_u;
    __syncthreads();
    if (u >= n_units) return;
    const float* s = src + (size_t)u * 32768;
    uint8_t* d = dst + (size_t)u * 65536;
    for (uint32_t v = threadIdx.x; v < 4096; v += 4 * 256) {
      uint4 a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { a[q] = ldg(s + 8 * (v + q * 256)); b[q] = ldg(s + 8 * (v + q * 256) + 4); }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        stcs(d + 16 * (v + q * 256), make_uint4(p2(a[q].x, a[q].y), p2(a[q].z, a[q].w), p2(b[q].x, b[q].y), p2(b[q].z, b[q].w)));
    }
  }
}

constexpr int kSt = 6, kSb = 32768, kCons = 512;
__global__ void __launch_bounds__(kCons + 32, 1) k_tma(const float* __restrict__ src, uint8_t* __restrict__ dst,
                                                      uint32_t n_blocks, uint32_t k) {
  extern __shared__ __align__(1024) uint8_t buf[];
  __shared__ __align__(8) uint64_t full[kSt], empty[kSt];
  if (smid() >= k) return;
  // blocks of 32 KiB fp32 (8192 elements); CTA c of the k working ones takes blocks c, c+k, ...
  const uint32_t me = smid();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSt; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(kCons / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == kCons / 32) {
    if (lane) return;
    uint32_t j = 0;
    for (uint32_t b = me; b < n_blocks; b += k, ++j) {
      const uint32_t s = j % kSt;
      if (j >= kSt)
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(
                         sa(&empty[s])), "r"(((j / kSt) + 1) & 1u));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(kSb));
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(buf + s * kSb)), "l"((const uint8_t*)src + (size_t)b * kSb), "r"(kSb), "r"(sa(&full[s]))
                   : "memory");
    }
    return;
  }
  uint32_t j = 0;
  for (uint32_t b = me; b < n_blocks; b += k, ++j) {
    const uint32_t s = j % kSt;
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(
                     sa(&full[s])), "r"((j / kSt) & 1u) : "memory");
    const uint8_t* sb = buf + s * kSb;
    uint8_t* d = dst + (size_t)b * (kSb / 2);
    for (uint32_t v = threadIdx.x; v < kSb / 32; v += kCons) {   // 32 B in -> 16 B out
      uint4 a, c;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "r"(sa(sb + 32 * v)));
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "r"(sa(sb + 32 * v + 16)));
      stcs(d + 16 * v, make_uint4(p2(a.x, a.y), p2(a.z, a.w), p2(c.x, c.y), p2(c.z, c.w)));
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
  }
}

int main() {
  const size_t n = (size_t)2 << 30;   // 2 Gi fp32 = 8 GiB in, 4 GiB out (>> L2)
  float* src;
  uint8_t* dst;
  uint32_t* work;
  CK(cudaMalloc(&src, n * 4));
  CK(cudaMalloc(&dst, n * 2));
  CK(cudaMalloc(&work, 4));
  CK(cudaMemset(src, 0x3f, n * 4));
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kSt * kSb));
  int per = 0, sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_ldg, 256, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double bytes = 6.0 * n;
  for (uint32_t k : {8u, 16u, 24u, 32u, 48u, 64u, 96u, 148u}) {
    float best[2] = {1e9f, 1e9f};
    for (int rep = 0; rep < 4; ++rep) {
      float ms;
      CK(cudaMemset(work, 0, 4));
      CK(cudaEventRecord(e0));
      k_ldg<<<sms * per, 256>>>(src, dst, (uint32_t)(n / 32768), work, k);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep && ms < best[0]) best[0] = ms;
      CK(cudaEventRecord(e0));
      k_tma<<<sms, kCons + 32, kSt * kSb>>>(src, dst, (uint32_t)(n * 4 / kSb), k);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep && ms < best[1]) best[1] = ms;
    }
    CK(cudaGetLastError());
    printf("k=%3u SMs  ldg %7.1f GB/s (%5.1f GB/s/SM, %6.2f ms)   tma %7.1f GB/s (%5.1f GB/s/SM, %6.2f ms)\n", k,
           bytes / best[0] / 1e6, bytes / best[0] / 1e6 / k, best[0], bytes / best[1] / 1e6, bytes / best[1] / 1e6 / k,
           best[1]);
  }
  return 0;
}

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
#include <vector>

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

// TMA push: local global -> smem -> peer global
template <int STAGES, int SB>
__global__ void __launch_bounds__(128) k_tma_push(const char* __restrict__ src, char* __restrict__ dst, size_t bytes) {
  k_tma<STAGES, SB>(src, dst, bytes);
}

struct Bufs { char* a[8]; };

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
  const size_t bytes = (size_t)2 << 30;
  // per GPU: src buffer (own data) and dst buffer (received data)
  char *src[8], *dst[8];
  for (int d = 0; d < ndev; ++d) {
    CK(cudaSetDevice(d)); CK(cudaMalloc(&src[d], bytes)); CK(cudaMalloc(&dst[d], bytes)); CK(cudaMemset(src[d], d + 1, bytes));
    for (int e = 0; e < ndev; ++e) if (e != d) { cudaError_t r = cudaDeviceEnablePeerAccess(e, 0); if (r != cudaSuccess) cudaGetLastError(); }
  }
  constexpr int ST = 6, SB = 32768;
  for (int d = 0; d < ndev; ++d) { CK(cudaSetDevice(d)); CK(cudaFuncSetAttribute(k_tma<ST, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * SB)); }
  cudaStream_t st[8]; cudaEvent_t e0[8], e1[8];
  for (int d = 0; d < ndev; ++d) { CK(cudaSetDevice(d)); CK(cudaStreamCreate(&st[d])); CK(cudaEventCreate(&e0[d])); CK(cudaEventCreate(&e1[d])); }
  // run a set of concurrent copies; each copy = (device running it, src ptr, dst ptr, kind)
  struct Copy { int dev; const char* s; char* d; int kind; };  // kind 0 = TMA kernel, 1 = copy engine, 2 = 16-B push
  auto run = [&](const char* name, std::vector<Copy> cs, int ctas) {
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      for (int d = 0; d < ndev; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      for (auto& c : cs) { CK(cudaSetDevice(c.dev)); CK(cudaEventRecord(e0[c.dev], st[c.dev])); }
      for (auto& c : cs) {
        CK(cudaSetDevice(c.dev));
        if (c.kind == 0) k_tma<ST, SB><<<ctas, 128, ST * SB, st[c.dev]>>>(c.s, c.d, bytes);
        else if (c.kind == 1) CK(cudaMemcpyAsync(c.d, c.s, bytes, cudaMemcpyDefault, st[c.dev]));
        else k_copy<8><<<ctas, 512, 0, st[c.dev]>>>((const uint4*)c.s, (uint4*)c.d, bytes / 16);
      }
      float worst = 0;
      for (auto& c : cs) { CK(cudaSetDevice(c.dev)); CK(cudaEventRecord(e1[c.dev], st[c.dev])); }
      for (auto& c : cs) { CK(cudaSetDevice(c.dev)); CK(cudaEventSynchronize(e1[c.dev])); float ms; CK(cudaEventElapsedTime(&ms, e0[c.dev], e1[c.dev])); if (ms > worst) worst = ms; }
      CK(cudaGetLastError());
      if (worst < best) best = worst;
    }
    printf("%-44s ctas=%3d  per-copy %6.1f GB/s\n", name, ctas, bytes / (best / 1e3) / 1e9);
  };
  auto run_tma = [&](const char* name, std::vector<Copy> cs, int ctas, auto kern, int smem) {
    for (int d = 0; d < ndev; ++d) { CK(cudaSetDevice(d)); CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); }
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      for (int d = 0; d < ndev; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      for (auto& c : cs) { CK(cudaSetDevice(c.dev)); CK(cudaEventRecord(e0[c.dev], st[c.dev])); }
      for (auto& c : cs) { CK(cudaSetDevice(c.dev)); kern<<<ctas, 128, smem, st[c.dev]>>>(c.s, c.d, bytes); }
      float worst = 0;
      for (auto& c : cs) { CK(cudaSetDevice(c.dev)); CK(cudaEventRecord(e1[c.dev], st[c.dev])); }
      for (auto& c : cs) { CK(cudaSetDevice(c.dev)); CK(cudaEventSynchronize(e1[c.dev])); float ms; CK(cudaEventElapsedTime(&ms, e0[c.dev], e1[c.dev])); if (ms > worst) worst = ms; }
      CK(cudaGetLastError());
      if (worst < best) best = worst;
    }
    printf("%-44s ctas=%3d  per-copy %6.1f GB/s\n", name, ctas, bytes / (best / 1e3) / 1e9);
  };
  std::vector<Copy> chain3 = {{1, src[0], dst[1], 0}, {2, src[1], dst[2], 0}, {3, src[2], dst[3], 0}};
  std::vector<Copy> push3 = {{0, src[0], dst[1], 0}, {1, src[1], dst[2], 0}, {2, src[2], dst[3], 0}};
  for (int ctas : {16, 24, 32, 48}) {
    run_tma("chain3 pull SB=16K x12", chain3, ctas, k_tma<12, 16384>, 12 * 16384);
    run_tma("chain3 pull SB=32K x6", chain3, ctas, k_tma<6, 32768>, 6 * 32768);
    run_tma("chain3 pull SB=64K x3", chain3, ctas, k_tma<3, 65536>, 3 * 65536);
    run_tma("chain3 pull SB=96K x2", chain3, ctas, k_tma<2, 98304>, 2 * 98304);
    run_tma("chain3 push SB=32K x6", push3, ctas, k_tma<6, 32768>, 6 * 32768);
    run_tma("chain3 push SB=64K x3", push3, ctas, k_tma<3, 65536>, 3 * 65536);
  }
  run("CE 1<-0", {{1, src[0], dst[1], 1}}, 0);
  if (ndev >= 4) run("CE chain 1<-0, 2<-1, 3<-2", {{1, src[0], dst[1], 1}, {2, src[1], dst[2], 1}, {3, src[2], dst[3], 1}}, 0);
  return 0;
}

// Chain-broadcast transport microbenchmark (B200, NVLink 5 through NVSwitch): which copy style keeps a
// MIDDLE relay (receiving from its predecessor while its successor receives from it) closest to the
// one-way NVLink ceiling.  Single process, peer access; chain 0 -> 1 -> ... -> n-1 with every hop
// moving `bytes` concurrently (steady state of the pipelined chain).
//   pull-tma   kernel on the receiver: cp.async.bulk peer global -> smem -> cp.async.bulk smem -> local
//   push-tma   kernel on the sender:   cp.async.bulk local global -> smem -> cp.async.bulk smem -> peer
//   push-reg   kernel on the sender:   16-B loads local, 16-B stores to the peer (posted writes)
//   pull-reg   kernel on the receiver: 16-B loads from the peer, 16-B stores local
//   split      each hop half pulled by the receiver (TMA) and half pushed by the sender (TMA)
//   ce         cudaMemcpyAsync on the receiver's stream (copy engines, zero SMs)
// Reported: per-hop GB/s of the slowest hop (= what the chain sustains).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/chain_bench tools/chain_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// TMA bulk copy src -> smem -> dst; one elected thread per CTA, STAGES x SB bytes of smem in flight.
// Blocks of SB are distributed round-robin over CTAs.
template <int STAGES, int SB>
__global__ void __launch_bounds__(32) k_tma(const char* __restrict__ src, char* __restrict__ dst, size_t bytes) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) unsigned long long bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const size_t nblk = bytes / SB, step = gridDim.x;
  size_t issued = blockIdx.x, done = blockIdx.x;
  for (int s = 0; s < STAGES && issued < nblk; ++s, issued += step) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(SB));
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(smem + s * SB)), "l"(src + issued * SB), "r"(SB), "r"(sa(&bar[s])) : "memory");
  }
  unsigned phase = 0;
  for (int s = 0; done < nblk;) {
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                 ::"r"(sa(&bar[s])), "r"(phase));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + done * SB),
                 "r"(sa(smem + s * SB)), "r"(SB) : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    done += step;
    if (issued < nblk) {
      // the stage is reused only once its store has read it
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(SB));
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(smem + s * SB)), "l"(src + issued * SB), "r"(SB), "r"(sa(&bar[s])) : "memory");
      issued += step;
    }
    if (++s == STAGES) { s = 0; phase ^= 1; }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int U>
__global__ void __launch_bounds__(512) k_reg(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t i0 = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; i0 < n; i0 += stride) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const size_t i = i0 + (size_t)k * blockDim.x;
      if (i < n) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                              : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(src + i));
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const size_t i = i0 + (size_t)k * blockDim.x;
      if (i < n) asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst + i), "r"(v[k].x), "r"(v[k].y),
                              "r"(v[k].z), "r"(v[k].w) : "memory");
    }
  }
}

constexpr int ST = 6, SB = 32768;

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("need >= 2 GPUs\n"); return 0; }
  const size_t bytes = (size_t)1 << 30;
  std::vector<char*> src(ndev), dst(ndev);
  for (int d = 0; d < ndev; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMalloc(&src[d], bytes));
    CK(cudaMalloc(&dst[d], bytes));
    CK(cudaMemset(src[d], d + 1, bytes));
    for (int e = 0; e < ndev; ++e)
      if (e != d && cudaDeviceEnablePeerAccess(e, 0) != cudaSuccess) cudaGetLastError();
    CK(cudaFuncSetAttribute(k_tma<ST, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * SB));
  }
  std::vector<cudaStream_t> st(2 * ndev);
  std::vector<cudaEvent_t> e0(2 * ndev), e1(2 * ndev);
  for (int d = 0; d < ndev; ++d) {
    CK(cudaSetDevice(d));
    for (int k = 0; k < 2; ++k) {
      CK(cudaStreamCreateWithFlags(&st[2 * d + k], cudaStreamNonBlocking));
      CK(cudaEventCreate(&e0[2 * d + k]));
      CK(cudaEventCreate(&e1[2 * d + k]));
    }
  }
  // one hop a -> b of `len` bytes at byte offset `off`, run by `dev` (stream slot k) in style `kind`
  struct Op { int dev, k; const char* s; char* d; size_t len; int kind; };   // 0 tma, 1 reg, 2 ce
  auto launch = [&](const Op& o, int ctas) {
    CK(cudaSetDevice(o.dev));
    cudaStream_t s = st[2 * o.dev + o.k];
    if (o.kind == 0) k_tma<ST, SB><<<ctas, 32, ST * SB, s>>>(o.s, o.d, o.len);
    else if (o.kind == 1) k_reg<8><<<ctas, 512, 0, s>>>((const uint4*)o.s, (uint4*)o.d, o.len / 16);
    else CK(cudaMemcpyAsync(o.d, o.s, o.len, cudaMemcpyDefault, s));
  };
  auto run = [&](const char* name, int n, int ctas, auto make) {
    std::vector<Op> ops;
    for (int h = 0; h + 1 < n; ++h) make(h, h + 1, ops);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      for (int d = 0; d < ndev; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      for (auto& o : ops) { CK(cudaSetDevice(o.dev)); CK(cudaEventRecord(e0[2 * o.dev + o.k], st[2 * o.dev + o.k])); }
      for (auto& o : ops) launch(o, ctas);
      for (auto& o : ops) { CK(cudaSetDevice(o.dev)); CK(cudaEventRecord(e1[2 * o.dev + o.k], st[2 * o.dev + o.k])); }
      float worst = 0;
      for (auto& o : ops) {
        CK(cudaSetDevice(o.dev));
        CK(cudaEventSynchronize(e1[2 * o.dev + o.k]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[2 * o.dev + o.k], e1[2 * o.dev + o.k]));
        worst = ms > worst ? ms : worst;
      }
      CK(cudaGetLastError());
      if (rep && worst < best) best = worst;    // rep 0 = warm-up
    }
    printf("%-10s chain of %d  ctas=%3d  per hop %6.1f GB/s\n", name, n, ctas, bytes / (best / 1e3) / 1e9);
    fflush(stdout);
  };
  auto pull_tma = [&](int a, int b, std::vector<Op>& ops) { ops.push_back({b, 0, src[a], dst[b], bytes, 0}); };
  auto push_tma = [&](int a, int b, std::vector<Op>& ops) { ops.push_back({a, 0, src[a], dst[b], bytes, 0}); };
  auto push_reg = [&](int a, int b, std::vector<Op>& ops) { ops.push_back({a, 0, src[a], dst[b], bytes, 1}); };
  auto pull_reg = [&](int a, int b, std::vector<Op>& ops) { ops.push_back({b, 0, src[a], dst[b], bytes, 1}); };
  auto split = [&](int a, int b, std::vector<Op>& ops) {
    ops.push_back({b, 0, src[a], dst[b], bytes / 2, 0});
    ops.push_back({a, 1, src[a] + bytes / 2, dst[b] + bytes / 2, bytes / 2, 0});
  };
  auto ce = [&](int a, int b, std::vector<Op>& ops) { ops.push_back({b, 0, src[a], dst[b], bytes, 2}); };
  for (int n = 2; n <= ndev; n = (n == 4 ? ndev : n + 1)) {
    if (n != 2 && n != 3 && n != 4 && n != ndev) continue;
    for (int ctas : {32, 64, 148}) {
      run("pull-tma", n, ctas, pull_tma);
      run("push-tma", n, ctas, push_tma);
      run("split", n, ctas / 2, split);
    }
    for (int ctas : {64, 148, 296}) {
      run("push-reg", n, ctas, push_reg);
      run("pull-reg", n, ctas, pull_reg);
    }
    run("ce", n, 0, ce);
  }
  return 0;
}

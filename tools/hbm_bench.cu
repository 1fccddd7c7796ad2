// HBM streaming microbenchmark (B200): practical ceilings for the two local shapes of this path.
//   copy  1:1  (k_pull):  read 16 B, write 16 B
//   pack  2:1  (k_pack):  read 32 B fp32, write 16 B bf16 (integer RNE, like the product kernel)
// Variants: CTAs per SM, vectors in flight per thread, store cache hint (default / .cs / L2::evict_first).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_bench hbm_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint4 ldnc(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
template <int HINT>
__device__ __forceinline__ void st(void* p, uint4 v) {
  if (HINT == 0) asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else if (HINT == 1) asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint32_t rne(uint32_t u) {
  uint32_t r = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
  return ((u & 0x7FFFFFFFu) > 0x7F800000u) ? 0x7FC0u : r;
}

template <int U, int HINT>
__global__ void __launch_bounds__(256) k_copy(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
  for (size_t i0 = (size_t)blockIdx.x * 256 * U + threadIdx.x; i0 < n; i0 += (size_t)gridDim.x * 256 * U) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) if (i0 + k * 256 < n) v[k] = ldnc(s + i0 + k * 256);
#pragma unroll
    for (int k = 0; k < U; ++k) if (i0 + k * 256 < n) st<HINT>(d + i0 + k * 256, v[k]);
  }
}

template <int U, int HINT>
__global__ void __launch_bounds__(256) k_pack(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n_out) {
  for (size_t i0 = (size_t)blockIdx.x * 256 * U + threadIdx.x; i0 < n_out; i0 += (size_t)gridDim.x * 256 * U) {
    uint4 a[U], b[U];
#pragma unroll
    for (int k = 0; k < U; ++k) if (i0 + k * 256 < n_out) { a[k] = ldnc(s + 2 * (i0 + k * 256)); b[k] = ldnc(s + 2 * (i0 + k * 256) + 1); }
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (i0 + k * 256 < n_out)
        st<HINT>(d + i0 + k * 256, make_uint4(rne(a[k].x) | rne(a[k].y) << 16, rne(a[k].z) | rne(a[k].w) << 16,
                                              rne(b[k].x) | rne(b[k].y) << 16, rne(b[k].z) | rne(b[k].w) << 16));
  }
}

int main() {
  const size_t out_bytes = (size_t)8 << 30;  // 8 GiB written; pack reads 16 GiB
  char *src, *dst;
  CK(cudaMalloc(&src, 2 * out_bytes));
  CK(cudaMalloc(&dst, out_bytes));
  CK(cudaMemset(src, 1, 2 * out_bytes));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  auto t = [&](auto fn) {
    fn(); CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) { CK(cudaEventRecord(e0)); fn(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); best = ms < best ? ms : best; }
    CK(cudaGetLastError());
    return best;
  };
  size_t n = out_bytes / 16;
  printf("shape  ctas/SM  unroll  hint   TB/s (read+write)\n");
#define RUN(SHAPE, K, U, H, BYTES)                                                                      \
  for (int cps : {4, 6, 8}) {                                                                          \
    float ms = t([&] { K<U, H><<<sms * cps, 256>>>((const uint4*)src, (uint4*)dst, n); });            \
    printf("%-6s %7d  %6d  %4d  %6.3f\n", SHAPE, cps, U, H, (BYTES) / (ms / 1e3) / 1e12);              \
  }
  RUN("copy", k_copy, 1, 0, 2.0 * out_bytes) RUN("copy", k_copy, 2, 0, 2.0 * out_bytes) RUN("copy", k_copy, 4, 0, 2.0 * out_bytes)
  RUN("copy", k_copy, 2, 1, 2.0 * out_bytes) RUN("copy", k_copy, 4, 1, 2.0 * out_bytes) RUN("copy", k_copy, 4, 2, 2.0 * out_bytes)
  RUN("pack", k_pack, 1, 0, 3.0 * out_bytes) RUN("pack", k_pack, 2, 0, 3.0 * out_bytes) RUN("pack", k_pack, 4, 0, 3.0 * out_bytes)
  RUN("pack", k_pack, 2, 1, 3.0 * out_bytes) RUN("pack", k_pack, 4, 1, 3.0 * out_bytes) RUN("pack", k_pack, 2, 2, 3.0 * out_bytes)
  float ms = t([&] { CK(cudaMemcpyAsync(dst, src, out_bytes, cudaMemcpyDeviceToDevice)); });
  printf("cudaMemcpy D2D       %6.3f\n", 2.0 * out_bytes / (ms / 1e3) / 1e12);
  return 0;
}

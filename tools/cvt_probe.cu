// Does the hardware conversion cvt.rn.bf16x2.f32 equal the pack's integer round-to-nearest-even
// (reading R1: subnormals kept, overflow to inf, every NaN -> 0x7FC0) on all 2^32 fp32
// patterns?  Counts mismatches among non-NaN inputs and lists the distinct bf16 results NaN inputs get.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cvt_probe tools/cvt_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t rne(uint32_t u) {
  uint32_t r = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
  return ((u & 0x7FFFFFFFu) > 0x7F800000u) ? 0x7FC0u : r;
}

__global__ void probe(uint64_t* bad_finite, uint32_t* nan_out, uint32_t* first_bad) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (1ull << 32); i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = (uint32_t)i;
    uint32_t d;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(__uint_as_float(u)), "f"(__uint_as_float(u)));
    const uint32_t hw = d & 0xFFFFu;
    if ((u & 0x7FFFFFFFu) > 0x7F800000u) {
      atomicOr(&nan_out[hw >> 5], 1u << (hw & 31));     // set of NaN results
    } else if (hw != rne(u)) {
      if (atomicAdd((unsigned long long*)bad_finite, 1ull) == 0) *first_bad = u;
    }
  }
}

int main() {
  uint64_t* bad;
  uint32_t *nan, *first;
  cudaMalloc(&bad, 8);
  cudaMalloc(&nan, 65536 / 8);
  cudaMalloc(&first, 4);
  cudaMemset(bad, 0, 8);
  cudaMemset(nan, 0, 65536 / 8);
  cudaMemset(first, 0, 4);
  probe<<<148 * 8, 256>>>(bad, nan, first);
  cudaError_t e = cudaDeviceSynchronize();
  uint64_t hb = 0;
  uint32_t hf = 0, hn[2048];
  cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&hf, first, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hn, nan, sizeof hn, cudaMemcpyDeviceToHost);
  printf("status %s; non-NaN mismatches vs integer RNE: %llu (first input 0x%08x)\nNaN inputs -> bf16:", cudaGetErrorString(e),
         (unsigned long long)hb, hf);
  int shown = 0;
  for (uint32_t h = 0; h < 65536 && shown < 16; ++h)
    if (hn[h >> 5] >> (h & 31) & 1u) { printf(" 0x%04x", h); ++shown; }
  printf("\n");
  return 0;
}

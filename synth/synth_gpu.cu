// Harness kernel: fill an fp32 device (or host-mapped) buffer with the synthetic master weights
// of synth/synth.cuh.  Used by tests and bench.py to create the actor's fp32 shards in HBM.
// C ABI:  int synth_fill_f32(float* dst, uint64_t count, uint64_t seed, uint64_t version,
//                            uint32_t tensor_id, uint64_t idx0, int specials, void* stream)
// Element i of dst gets the value of flat element (idx0 + i) of tensor `tensor_id` at `version`.
// Returns 0 or the cudaError_t of the launch.
#include <cuda_runtime.h>
#include "synth.cuh"

__global__ void __launch_bounds__(256) k_gen(float* __restrict__ dst, uint64_t count, uint64_t base,
                                             uint64_t idx0, int specials) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
  for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < count; i += stride) {
    if (i + 4 <= count && (((uintptr_t)(dst + i)) & 15) == 0) {
      uint4 v;
      v.x = synth_bits(base, idx0 + i + 0, specials);
      v.y = synth_bits(base, idx0 + i + 1, specials);
      v.z = synth_bits(base, idx0 + i + 2, specials);
      v.w = synth_bits(base, idx0 + i + 3, specials);
      *reinterpret_cast<uint4*>(dst + i) = v;
    } else {
      for (uint64_t j = i; j < i + 4 && j < count; ++j)
        reinterpret_cast<uint32_t*>(dst)[j] = synth_bits(base, idx0 + j, specials);
    }
  }
}

extern "C" int synth_fill_f32(float* dst, uint64_t count, uint64_t seed, uint64_t version,
                              uint32_t tensor_id, uint64_t idx0, int specials, void* stream) {
  if (count == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t want = (count + 1023) / 1024;
  unsigned grid = (unsigned)(want < (uint64_t)sms * 8 ? (want ? want : 1) : (uint64_t)sms * 8);
  k_gen<<<grid, 256, 0, (cudaStream_t)stream>>>(dst, count, synth_base(seed, version, tensor_id), idx0,
                                                  specials);
  return (int)cudaGetLastError();
}

// Seeded synthetic fp32 master weights — CUDA/C twin of synth/synth.py (same definition,
// written again).  Input generator only: no arithmetic of the method lives here.
// Definition:
//   key = seed ^ (v * 0x9E3779B97F4A7C15) ^ (tensor_id << 44) ^ idx
//   x   = splitmix64(key);  m = (x >> 40) - 2^23;  w = m * 2^-30
//   specials: if ((x & 0xFFF) == 0x5A5) bits = SPECIALS[(x >> 12) % 19]
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define SYNTH_HD __host__ __device__ __forceinline__
#else
#define SYNTH_HD static inline
#endif

#define SYNTH_N_SPECIALS 19

SYNTH_HD uint32_t synth_special(uint32_t i) {
  switch (i) {
    case 0: return 0x3F808000u;  case 1: return 0x3F818000u;  case 2: return 0xBF808000u;
    case 3: return 0x7F7F7FFFu;  case 4: return 0x7F7F8000u;  case 5: return 0x7F7FFFFFu;
    case 6: return 0xFF7F8000u;  case 7: return 0x00008000u;  case 8: return 0x00018000u;
    case 9: return 0x00000001u;  case 10: return 0x80000001u; case 11: return 0x007FFFFFu;
    case 12: return 0x80000000u; case 13: return 0x7F800000u; case 14: return 0xFF800000u;
    case 15: return 0x7FC00000u; case 16: return 0x7F800001u; case 17: return 0xFFFFFFFFu;
    default: return 0x00000000u;
  }
}

SYNTH_HD uint64_t synth_splitmix64(uint64_t state) {
  uint64_t z = state + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

SYNTH_HD uint64_t synth_base(uint64_t seed, uint64_t version, uint32_t tensor_id) {
  return seed ^ (version * 0x9E3779B97F4A7C15ull) ^ ((uint64_t)tensor_id << 44);
}

// fp32 bit pattern of element idx given base = synth_base(seed, v, tensor_id)
SYNTH_HD uint32_t synth_bits(uint64_t base, uint64_t idx, int specials) {
  uint64_t x = synth_splitmix64(base ^ idx);
  int32_t m = (int32_t)(x >> 40) - (1 << 23);
  float w = (float)m * 9.313225746154785e-10f;  // 2^-30, exact
  uint32_t bits;
#ifdef __CUDA_ARCH__
  bits = __float_as_uint(w);
#else
  union { float f; uint32_t u; } cv; cv.f = w; bits = cv.u;
#endif
  if (specials && (x & 0xFFFull) == 0x5A5ull) bits = synth_special((uint32_t)((x >> 12) % SYNTH_N_SPECIALS));
  return bits;
}

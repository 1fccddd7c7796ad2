// sm_100a kernels of the relay-tier weight synchronization path.
//
//   k_pack  — publish: fp32 master shard -> bf16 RNE (integer
//             arithmetic, NaN -> 0x7FC0) -> 16-B stores into the version's bucket image, per-chunk
//             checksum (S1, S2) by warp shuffles + one u64 atomic pair per unit; the CTA finishing a
//             chunk publishes its header and flag (st.release.sys) so the next relay, on another
//             GPU, can start pulling that chunk while later chunks are still being packed.
//   k_hop   — chain-pipelined broadcast hop (A3/A4), hop.cuh: receiver-driven
//             TMA bulk pipeline.  Per chunk, the node waits (ld.acquire.sys on the predecessor flag,
//             over NVLink), bulk-copies the chunk from the predecessor slot through shared memory into
//             local HBM, recomputes the checksum on the way, and releases its own flag only if it
//             matches the predecessor's header.  Few CTAs (SM-light).
//   k_pull  — pull-time TP reshard (A6): copy-plan driven 2-D block copy from
//             the pinned relay slot (local HBM or peer GPU) into the rollout's TP buffers.
#include <cuda_runtime.h>
#include <stdlib.h>

#include <algorithm>

#include "lam_internal.h"

namespace lam {

// ------------------------------------------------------------------------------- primitives
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
// streaming store (evict-first): every output of this path is written once and is far larger than
// L2 (tools/hbm_bench.cu: +5-7 % on the pack's 2:1 read:write stream)
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// NVSwitch multicast stores (LAM_HOP_MULTICAST, mcast.cpp): one store through the multicast VA lands
// at the same offset in every team GPU's member (the switch replicates it).
__device__ __forceinline__ void mc_st_v4(void* p, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void mc_st_b32(void* p, uint32_t v) {
  asm volatile("multimem.st.relaxed.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void mc_st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("multimem.st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Release a chunk flag (device memory, read by the next relay over NVLink) and mirror it to host
// shared memory, where lam_relay_step of any process sees it and drives streaming pulls.  Multicast
// mode: the flag also goes through the switch to every relay GPU's member (after the chunk's data,
// which took the same path), where that relay polls it in local HBM.
__device__ __forceinline__ void publish_flag(const ChunkMeta& meta, uint32_t chunk, uint64_t value) {
  if (meta.mc_flags) mc_st_release_u64(meta.mc_flags + chunk, value);
  st_release_sys(meta.flags + chunk, value);
  if (meta.mirror) st_release_sys(meta.mirror + chunk, value);
}

// 16 bytes to an address that may be only 2-B aligned (colocated subscriber of an odd FSDP split)
__device__ __forceinline__ void st_v4_any(uint8_t* p, uint4 v) {
  if ((((uintptr_t)p) & 15) == 0) {
    st_v4(p, v);
  } else if ((((uintptr_t)p) & 3) == 0) {
    uint32_t* q = reinterpret_cast<uint32_t*>(p);
    q[0] = v.x; q[1] = v.y; q[2] = v.z; q[3] = v.w;
  } else {
    uint16_t* q = reinterpret_cast<uint16_t*>(p);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) { q[2 * i] = (uint16_t)w[i]; q[2 * i + 1] = (uint16_t)(w[i] >> 16); }
  }
}

// fp32 bits -> bf16 bits, round to nearest even; every NaN -> 0x7FC0 (reading R1).
__device__ __forceinline__ uint32_t rne_bf16(uint32_t u) {
  uint32_t r = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
  return ((u & 0x7FFFFFFFu) > 0x7F800000u) ? 0x7FC0u : r;
}
// Two elements at once on the conversion unit: cvt.rn.bf16x2.f32 (F2FP) rounds to nearest even, keeps
// subnormals and overflows to inf exactly like rne_bf16 (tools/cvt_probe.cu on the box: 0 mismatches over
// all 2^32 non-NaN patterns); its NaN result (0x7FFF) is replaced by 0x7FC0 (HSET2 NaN mask + LOP3).
// 3 instructions per 2 elements instead of ~16.
__device__ __forceinline__ uint32_t pack2(uint32_t lo, uint32_t hi) {
  uint32_t d, m;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(__uint_as_float(hi)), "f"(__uint_as_float(lo)));
  asm("set.nan.u32.bf16x2 %0, %1, %1;" : "=r"(m) : "r"(d));
  return (d & ~m) | (0x7FC07FC0u & m);
}

// checksum contribution of 4 consecutive words starting at word index i0:
//   S1 += sum w, S2 += sum (i+1) w = (i0+1)*sum + w1 + 2 w2 + 3 w3      (mod 2^64)
__device__ __forceinline__ void cks4(uint64_t i0, uint4 w, uint64_t& s1, uint64_t& s2) {
  uint64_t sum = (uint64_t)w.x + w.y + w.z + w.w;
  s1 += sum;
  s2 += (i0 + 1) * sum + (uint64_t)w.y + 2ull * w.z + 3ull * w.w;
}

template <int THREADS>
__device__ __forceinline__ void block_reduce2(uint64_t& a, uint64_t& b, uint64_t (*sh)[THREADS / 32]) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sh[0][w] = a; sh[1][w] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = 0; b = 0;
#pragma unroll
    for (int i = 0; i < THREADS / 32; ++i) { a += sh[0][i]; b += sh[1][i]; }
  }
}

// Persistent grids: exactly one wave of resident CTAs (SMs x CTAs/SM the occupancy calculator
// allows for this kernel's registers) — a partial second wave made k_pack 20 % slower.
template <typename K>
int resident_ctas(K kernel, int threads, size_t smem = 0) {
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem);
  return sms * (per > 0 ? per : 1);
}

// ------------------------------------------------------------------------------------ k_pack
constexpr int kPackThreads = 256;
constexpr int kPackGroups = 4;

// Add a CTA's share of chunk `g` (n units, checksum partial sums) into the header; the CTA that
// completes the chunk publishes the header fields and releases the flag for the next relay.
__device__ void pack_flush(ChunkMeta meta, const uint32_t* units_per_chunk, const uint64_t* chunk_len, uint32_t g,
                           uint64_t s1, uint64_t s2, uint32_t n, uint64_t version, uint64_t n_total) {
  lam_chunk_header* h = meta.hdr + g;
  atomicAdd((unsigned long long*)&h->s1, (unsigned long long)s1);
  atomicAdd((unsigned long long*)&h->s2, (unsigned long long)s2);
  __threadfence_system();
  const uint32_t prev = atomicAdd(meta.cnt + g, n);
  if (prev + n == units_per_chunk[g]) {
    __threadfence_system();
    h->version = version;
    h->idx = g;
    h->n = n_total;
    h->bytes = chunk_len[g];
    __threadfence_system();
    publish_flag(meta, g, version);
  }
}

// SUB: compiled with the colocated-subscriber stores (separate instantiation: the plain pack keeps
// its register budget and occupancy).  MC: `mc_dst` is the multicast VA of node 0's slot (NEXT-2): every
// 16-B store is a multimem.st, so the bf16 bytes land in the actor GPU's slot and in every relay GPU's
// replica in the same pass.
template <bool SUB, bool MC>
__global__ void __launch_bounds__(kPackThreads) k_pack(const PackUnit* __restrict__ units, uint32_t n_units,
                                                       const float* const* __restrict__ shard_ptrs,
                                                       uint8_t* __restrict__ dst, uint8_t* mc_dst, ChunkMeta meta,
                                                       const uint32_t* __restrict__ units_per_chunk,
                                                       uint64_t version, uint64_t n_total,
                                                       const uint64_t* __restrict__ chunk_len,
                                                       uint8_t* const* __restrict__ sub_dst,
                                                       uint32_t* __restrict__ work, uint32_t sms) {
  __shared__ uint64_t red[2][kPackThreads / 32];
  __shared__ uint32_t s_next;
  // SM confinement (lam_config.pack_sms): the grid is one full wave over every SM; CTAs that landed on
  // an SM outside [0, sms) leave at once, so the pack holds only `sms` SMs (fully occupied) and the
  // trainer's kernels keep the rest.  Every unit then comes from the work counter.
  uint32_t first = blockIdx.x;
  if (sms) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (smid >= sms) return;
    if (threadIdx.x == 0) s_next = atomicAdd(work, 1u);
    __syncthreads();
    first = s_next;
    __syncthreads();
  }
  // Dynamic unit distribution: a CTA's first unit is blockIdx.x, every further one comes from a work
  // counter (zeroed before the launch), fetched at the start of the current unit so its latency is
  // hidden.  The static round-robin left ncu's per-SM active cycles at min 14.4 M / avg 17.9 M / max
  // 21.5 M of 21.0 M elapsed (r1d): early SMs idled while late ones finished the wave.  Each CTA still
  // sees increasing unit indices, so its chunks change monotonically and the per-chunk flush holds.
  // Per-CTA accumulation: the CTA's checksum and unit count for its current chunk are flushed once
  // when it moves on to another chunk (units are chunk-ordered), not per unit — the per-unit atomics
  // on a handful of hot header addresses serialised in L2.
  uint32_t cur = 0xFFFFFFFFu, acc_n = 0;
  uint64_t acc1 = 0, acc2 = 0;
  const uint32_t base = sms ? 0u : gridDim.x;   // unconfined: units [0, grid) are the CTAs' first ones
  for (uint32_t ui = first; ui < n_units;) {
    if (threadIdx.x == 0) s_next = base + atomicAdd(work, 1u);   // read after the barriers below
    const PackUnit u = units[ui];
    if (u.chunk != cur) {                                   // uniform: every thread read the same unit
      if (cur != 0xFFFFFFFFu) {
        __threadfence_system();                             // this thread's stores of the finished chunk
        __syncthreads();
        if (threadIdx.x == 0) pack_flush(meta, units_per_chunk, chunk_len, cur, acc1, acc2, acc_n, version, n_total);
      }
      cur = u.chunk;
      acc1 = acc2 = 0;
      acc_n = 0;
    }
    const float* src = shard_ptrs[u.shard] + u.src_elem;
    const bool mcs = MC;
    uint8_t* out = (mcs ? mc_dst : dst) + u.dst_off;
    // colocated subscriber (lam_subscribe): the same bf16 bytes also go to its TP=1 buffer
    uint8_t* out2 = SUB ? sub_dst[ui] : nullptr;
    uint64_t s1 = 0, s2 = 0;
    const uint32_t nvec = u.n >> 3;  // groups of 8 elements = 32 B in, 16 B out
    if ((((uintptr_t)src) & 15) == 0) {
      uint32_t v = threadIdx.x;
      constexpr int G = kPackGroups;  // groups of 8 elements in flight per thread (G x 32 B of loads)
      for (; v + (G - 1) * kPackThreads < nvec; v += G * kPackThreads) {
        uint4 a[G], b[G];
#pragma unroll
        for (int k = 0; k < G; ++k) {
          a[k] = ld_stream_v4(src + 8 * (size_t)(v + k * kPackThreads));
          b[k] = ld_stream_v4(src + 8 * (size_t)(v + k * kPackThreads) + 4);
        }
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const uint32_t vk = v + k * kPackThreads;
          const uint4 w = make_uint4(pack2(a[k].x, a[k].y), pack2(a[k].z, a[k].w), pack2(b[k].x, b[k].y),
                                     pack2(b[k].z, b[k].w));
          if (mcs) mc_st_v4(out + 16 * (size_t)vk, w); else st_v4(out + 16 * (size_t)vk, w);
          if (out2) st_v4_any(out2 + 16 * (size_t)vk, w);
          cks4((uint64_t)u.word0 + 4ull * vk, w, s1, s2);
        }
      }
      for (; v < nvec; v += kPackThreads) {
        const uint4 a = ld_stream_v4(src + 8 * (size_t)v), b = ld_stream_v4(src + 8 * (size_t)v + 4);
        const uint4 w = make_uint4(pack2(a.x, a.y), pack2(a.z, a.w), pack2(b.x, b.y), pack2(b.z, b.w));
        if (mcs) mc_st_v4(out + 16 * (size_t)v, w); else st_v4(out + 16 * (size_t)v, w);
        if (out2) st_v4_any(out2 + 16 * (size_t)v, w);
        cks4((uint64_t)u.word0 + 4ull * v, w, s1, s2);
      }
    } else {  // caller's shard pointer not 16-B aligned: scalar loads, same 16-B stores
      const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);
      for (uint32_t v = threadIdx.x; v < nvec; v += kPackThreads) {
        const uint32_t* q = s32 + 8 * (size_t)v;
        const uint4 w = make_uint4(pack2(q[0], q[1]), pack2(q[2], q[3]), pack2(q[4], q[5]), pack2(q[6], q[7]));
        if (mcs) mc_st_v4(out + 16 * (size_t)v, w); else st_v4(out + 16 * (size_t)v, w);
        if (out2) st_v4_any(out2 + 16 * (size_t)v, w);
        cks4((uint64_t)u.word0 + 4ull * v, w, s1, s2);
      }
    }
    // ragged tail (< 8 elements, only at a segment end): element pairs -> words, zero high half
    {
      const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);
      uint16_t* o16 = reinterpret_cast<uint16_t*>(out);
      for (uint32_t e = nvec * 8 + 2 * threadIdx.x; e < u.n; e += 2 * kPackThreads) {
        const uint32_t lo = rne_bf16(s32[e]);
        const uint32_t hi = (e + 1 < u.n) ? rne_bf16(s32[e + 1]) : 0u;
        if (mcs) {  // one word (e even, out 16-B aligned); the half past the segment is zero pad anyway
          mc_st_b32(o16 + e, lo | (hi << 16));
        } else {
          o16[e] = (uint16_t)lo;
          if (e + 1 < u.n) o16[e + 1] = (uint16_t)hi;
        }
        if (out2) {
          reinterpret_cast<uint16_t*>(out2)[e] = (uint16_t)lo;
          if (e + 1 < u.n) reinterpret_cast<uint16_t*>(out2)[e + 1] = (uint16_t)hi;
        }
        const uint64_t w = lo | (hi << 16);
        s1 += w;
        s2 += ((uint64_t)u.word0 + e / 2 + 1) * w;
      }
    }
    block_reduce2<kPackThreads>(s1, s2, red);
    if (threadIdx.x == 0) { acc1 += s1; acc2 += s2; ++acc_n; }
    ui = s_next;      // written by thread 0 before block_reduce2's barrier
    __syncthreads();  // red[] and s_next reuse
  }
  if (cur != 0xFFFFFFFFu) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) pack_flush(meta, units_per_chunk, chunk_len, cur, acc1, acc2, acc_n, version, n_total);
  }
}

int launch_pack(const PackUnit* units, uint32_t n_units, const float* const* shard_ptrs, uint8_t* dst, uint8_t* mc_dst,
                ChunkMeta meta, const uint32_t* units_per_chunk, uint64_t version, uint64_t n_total,
                const uint64_t* chunk_len, int ctas, void* stream, uint8_t* const* sub_dst, uint32_t* work,
                int sms) {
  if (n_units == 0) return 0;
  cudaError_t e = cudaMemsetAsync(work, 0, sizeof(uint32_t), (cudaStream_t)stream);
  if (e != cudaSuccess) return (int)e;
  const bool mc = meta.mc_flags != nullptr;
  auto kern = sub_dst ? (mc ? k_pack<true, true> : k_pack<true, false>) : (mc ? k_pack<false, true> : k_pack<false, false>);
  if (ctas <= 0 || sms > 0) ctas = resident_ctas(kern, kPackThreads);
  // confined: the full wave must land everywhere (the CTAs on SMs >= sms leave), not n_units of it
  unsigned grid = (unsigned)(sms > 0 || n_units >= (uint32_t)ctas ? (uint32_t)ctas : n_units);
  kern<<<grid, kPackThreads, 0, (cudaStream_t)stream>>>(units, n_units, shard_ptrs, dst, mc_dst, meta, units_per_chunk, version,
                                                        n_total, chunk_len, sub_dst, work, (uint32_t)(sms > 0 ? sms : 0));
  return (int)cudaGetLastError();
}

#include "hop.cuh"  // k_hop: TMA bulk pipeline

// ------------------------------------------------------------------------------------ k_pull
constexpr int kPullThreads = 512;
constexpr int kPullUnroll = 4;

// 8x8 transpose of bf16 in registers: in[j] = 8 consecutive elements of source row j; column i of
// the micro-tile (word m = (in[2m].e_i, in[2m+1].e_i)) is assembled by byte permutes only.
__device__ __forceinline__ uint32_t word_of(const uint4& v, int q) {
  return q == 0 ? v.x : (q == 1 ? v.y : (q == 2 ? v.z : v.w));
}
__device__ __forceinline__ uint4 transpose_col(const uint4 (&in)[8], int i) {
  const uint32_t sel = (i & 1) ? 0x7632u : 0x5410u;
  uint4 o;
  o.x = __byte_perm(word_of(in[0], i >> 1), word_of(in[1], i >> 1), sel);
  o.y = __byte_perm(word_of(in[2], i >> 1), word_of(in[3], i >> 1), sel);
  o.z = __byte_perm(word_of(in[4], i >> 1), word_of(in[5], i >> 1), sel);
  o.w = __byte_perm(word_of(in[6], i >> 1), word_of(in[7], i >> 1), sel);
  return o;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Element-wise K-major copy of rows [ra, rb) x columns [ka, kb) of a tile (edges / unaligned tiles).
__device__ __forceinline__ void pull_t_scalar(const uint8_t* src, uint8_t* dst, uint32_t sp, uint32_t dp,
                                              uint32_t ra, uint32_t rb, uint32_t ka, uint32_t kb) {
  const uint32_t nk = kb - ka, total = (rb - ra) * nk;
  for (uint32_t v = threadIdx.x; v < total; v += kPullThreads) {
    const uint32_t r = ra + v / nk, k = ka + v % nk;
    *reinterpret_cast<uint16_t*>(dst + (size_t)k * dp + 2 * (size_t)r) =
        *reinterpret_cast<const uint16_t*>(src + (size_t)r * sp + 2 * (size_t)k);
  }
}

// K-major tile (R16): element k of source row r -> dst + k*dst_pitch + 2r.
// The kernel is bound by L2 requests (ncu: time tracks lts__t_requests, ~10 ps each, for every variant
// tried), so both sides must move whole 128-B lines.  Each warp owns 8 KiB of shared memory and walks
// the tile in 64-row x 64-column blocks:
//   load   16 x cp.async 16 B per thread, all in flight (no register staging): an instruction reads 4
//          source rows x one full line into smem row r, 16-B chunk c at chunk position c ^ ((r >> 3) & 7)
//          (conflict-free on both sides)
//   store  per thread two 8x8 micro-tiles (source rows 8*(lane%8).., columns 8*(lane/8 + 4h)..):
//          8 x LDS.128, transpose in registers by byte permutes, 8 x STG.128: an instruction writes
//          4 destination rows x one full line.
// Edges (rows or columns not a multiple of 8, unaligned tiles) go element by element.
constexpr int kTBlk = 64;                                   // block rows = block columns
constexpr int kTWarpSmem = kTBlk * kTBlk * 2;               // 8 KiB per warp
constexpr int kPullSmem = kTWarpSmem * (kPullThreads / 32); // 128 KiB per CTA

__device__ __forceinline__ void pull_transposed(const CopyTile& T, const uint8_t* src, uint8_t* dst,
                                                uint8_t* smem) {
  const uint32_t R = T.rows, K = T.row_bytes >> 1, sp = T.src_pitch, dp = T.dst_pitch;
  if ((T.align & 0xFFu) != 16) {
    pull_t_scalar(src, dst, sp, dp, 0, R, 0, K);
    return;
  }
  const uint32_t RG = R >> 3, KG = K >> 3;                  // whole 8-row / 8-column groups
  const uint32_t BR = (RG + 7) >> 3, BK = (KG + 7) >> 3;    // 64 x 64 blocks
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ws = smem + warp * kTWarpSmem;
  for (uint32_t blk = warp; blk < BR * BK; blk += kPullThreads / 32) {
    const uint32_t br = blk % BR, bk = blk / BR;            // walk down the rows first
    const uint32_t row0 = br * kTBlk, col0 = bk * kTBlk;
    // ---- load: row = 4k + lane/8, chunk = lane%8
    const uint32_t lc = lane & 7, lr = lane >> 3;
    // loads k < kn are in the tile (rows row0 + 4k + lr < 8*RG, column group inside)
    const int32_t left = (int32_t)(RG * 8 - row0) - (int32_t)lr;
    const int kn = bk * 8 + lc < KG ? (left > 0 ? min(16, (left + 3) >> 2) : 0) : 0;
    const uint8_t* p = src + (size_t)(row0 + lr) * sp + 2 * (size_t)(col0 + 8 * lc);
    const size_t step = 4 * (size_t)sp;
#pragma unroll
    for (int k = 0; k < 16; ++k) {   // asynchronous global -> smem copies: all 16 in flight
      const uint32_t r = 4 * k + lr;
      if (k < kn) cp_async16(ws + r * 128 + 16 * (lc ^ ((r >> 3) & 7)), p + k * step);
    }
    cp_async_wait_all();
    __syncwarp();
    // ---- store: micro-tile (rows 8*rb.., columns 8*cc..), rb = lane%8, cc = lane/8 + 4h
    const uint32_t rb = lane & 7;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t cc = (lane >> 3) + 4 * h;
      if (br * 8 + rb < RG && bk * 8 + cc < KG) {
        uint4 in[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t r = 8 * rb + j;
          in[j] = *reinterpret_cast<const uint4*>(ws + r * 128 + 16 * (cc ^ rb));
        }
        uint8_t* d0 = dst + (size_t)(col0 + 8 * cc) * dp + 2 * (size_t)(row0 + 8 * rb);
#pragma unroll
        for (int i = 0; i < 8; ++i) st_v4(d0 + (size_t)i * dp, transpose_col(in, i));
      }
    }
    __syncwarp();
  }
  if (RG * 8 < R) pull_t_scalar(src, dst, sp, dp, RG * 8, R, 0, K);
  if (KG * 8 < K) pull_t_scalar(src, dst, sp, dp, 0, RG * 8, KG * 8, K);
}

// Zero-filled block (vocabulary padding rows, R15).
__device__ __forceinline__ void pull_zero(const CopyTile& T, uint8_t* dst) {
  const uint32_t a = T.align & 0xFFu;
  const uint32_t per = T.row_bytes / a, total = per * T.rows;
  for (uint32_t v = threadIdx.x; v < total; v += kPullThreads) {
    uint8_t* p = dst + (size_t)(v / per) * T.dst_pitch + (size_t)(v % per) * a;
    if (a == 16) st_v4(p, make_uint4(0, 0, 0, 0));
    else if (a == 4) *reinterpret_cast<uint32_t*>(p) = 0;
    else *reinterpret_cast<uint16_t*>(p) = 0;
  }
}

// K-major tiles only (one CTA per SM: 128 KiB of staging smem); other tiles are skipped.
__global__ void __launch_bounds__(kPullThreads, 1) k_pull_t(const CopyTile* __restrict__ tiles, uint32_t n_tiles,
                                                         const uint8_t* const* __restrict__ rank_base,
                                                         uint32_t* __restrict__ work) {
  extern __shared__ __align__(128) uint8_t pull_smem[];
  __shared__ uint32_t s_next[2];
  uint32_t it = 0;
  for (uint32_t ti = blockIdx.x; ti < n_tiles; ++it) {
    if (threadIdx.x == 0) s_next[it & 1] = gridDim.x + atomicAdd(work, 1u);   // next tile, fetched ahead
    const CopyTile T = tiles[ti];
    if (T.src_rank != LAM_TILE_ZERO && (T.align & LAM_TILE_TRANSPOSE))
      pull_transposed(T, rank_base[T.src_rank] + T.src_off, reinterpret_cast<uint8_t*>(T.dst), pull_smem);
    __syncthreads();
    ti = s_next[it & 1];   // double-buffered: rewritten only after the next barrier
  }
}

__device__ __forceinline__ void pull_tile(const CopyTile& T, const uint8_t* const* __restrict__ rank_base) {
  {
    uint8_t* dst = reinterpret_cast<uint8_t*>(T.dst);
    if (T.src_rank == LAM_TILE_ZERO) {
      pull_zero(T, dst);
      return;
    }
    if (T.align & LAM_TILE_TRANSPOSE) return;
    const uint8_t* src = rank_base[T.src_rank] + T.src_off;
    if (T.align == 16) {
      const uint32_t vpr = T.row_bytes >> 4, total = vpr * T.rows;
      if (T.rows == 1) {
        for (uint32_t v0 = threadIdx.x; v0 < total; v0 += kPullThreads * kPullUnroll) {
          uint4 w[kPullUnroll];
#pragma unroll
          for (int k = 0; k < kPullUnroll; ++k) {
            const uint32_t v = v0 + k * kPullThreads;
            if (v < total) w[k] = ld_stream_v4(src + 16 * (size_t)v);
          }
#pragma unroll
          for (int k = 0; k < kPullUnroll; ++k) {
            const uint32_t v = v0 + k * kPullThreads;
            if (v < total) st_v4(dst + 16 * (size_t)v, w[k]);
          }
        }
      } else {
        for (uint32_t v0 = threadIdx.x; v0 < total; v0 += kPullThreads * kPullUnroll) {
          uint4 w[kPullUnroll];
#pragma unroll
          for (int k = 0; k < kPullUnroll; ++k) {
            const uint32_t v = v0 + k * kPullThreads;
            if (v < total) {
              const uint32_t r = v / vpr, c = v - r * vpr;
              w[k] = ld_stream_v4(src + (size_t)r * T.src_pitch + 16 * (size_t)c);
            }
          }
#pragma unroll
          for (int k = 0; k < kPullUnroll; ++k) {
            const uint32_t v = v0 + k * kPullThreads;
            if (v < total) {
              const uint32_t r = v / vpr, c = v - r * vpr;
              st_v4(dst + (size_t)r * T.dst_pitch + 16 * (size_t)c, w[k]);
            }
          }
        }
      }
    } else if (T.align == 4) {
      const uint32_t wpr = T.row_bytes >> 2, total = wpr * T.rows;
      for (uint32_t v = threadIdx.x; v < total; v += kPullThreads) {
        const uint32_t r = v / wpr, c = v - r * wpr;
        *reinterpret_cast<uint32_t*>(dst + (size_t)r * T.dst_pitch + 4 * (size_t)c) =
            *reinterpret_cast<const uint32_t*>(src + (size_t)r * T.src_pitch + 4 * (size_t)c);
      }
    } else {
      const uint32_t hpr = T.row_bytes >> 1, total = hpr * T.rows;
      for (uint32_t v = threadIdx.x; v < total; v += kPullThreads) {
        const uint32_t r = v / hpr, c = v - r * hpr;
        *reinterpret_cast<uint16_t*>(dst + (size_t)r * T.dst_pitch + 2 * (size_t)c) =
            *reinterpret_cast<const uint16_t*>(src + (size_t)r * T.src_pitch + 2 * (size_t)c);
      }
    }
  }
}

// Row-major and zero tiles (no shared memory: co-resides with k_hop); K-major tiles are skipped.
// Tiles are distributed dynamically (first tile = blockIdx.x, then a per-launch work counter zeroed
// on the launch stream, fetched one tile ahead): the static round-robin left ncu's per-SM active cycles
// at min 3.45 M / avg 4.36 M / max 4.96 M of 4.96 M elapsed (r1d, 7B TP=2) — the same imbalance the
// pack had.
__global__ void __launch_bounds__(kPullThreads) k_pull(const CopyTile* __restrict__ tiles, uint32_t n_tiles,
                                                       const uint8_t* const* __restrict__ rank_base,
                                                       uint32_t* __restrict__ work) {
  __shared__ uint32_t s_next[2];
  uint32_t it = 0;
  for (uint32_t ti = blockIdx.x; ti < n_tiles; ++it) {
    if (threadIdx.x == 0) s_next[it & 1] = gridDim.x + atomicAdd(work, 1u);   // next tile, fetched ahead
    pull_tile(tiles[ti], rank_base);
    __syncthreads();
    ti = s_next[it & 1];   // double-buffered: rewritten only after the next barrier
  }
}


int launch_pull(const CopyTile* tiles, uint32_t n_tiles, const uint8_t* const* rank_base, int ctas, void* stream,
                uint32_t kinds, uint32_t* work) {
  if (n_tiles == 0) return 0;
  // work[0]: k_pull_t's tile counter, work[1]: k_pull's (both kernels run in order on `stream`)
  cudaError_t me = cudaMemsetAsync(work, 0, 2 * sizeof(uint32_t), (cudaStream_t)stream);
  if (me != cudaSuccess) return (int)me;
  int dev = 0;
  cudaGetDevice(&dev);
  if (kinds & kPullKMajor) {
    static uint32_t attr_set = 0;   // per device: k_pull_t's dynamic shared memory limit
    if (!(attr_set & (1u << dev))) {
      cudaError_t e = cudaFuncSetAttribute(k_pull_t, cudaFuncAttributeMaxDynamicSharedMemorySize, kPullSmem);
      if (e != cudaSuccess) return (int)e;
      attr_set |= 1u << dev;
    }
    const int n = ctas > 0 ? ctas : resident_ctas(k_pull_t, kPullThreads, kPullSmem);
    const unsigned grid = (unsigned)std::min<uint32_t>(n_tiles, (uint32_t)n);
    k_pull_t<<<grid, kPullThreads, kPullSmem, (cudaStream_t)stream>>>(tiles, n_tiles, rank_base, work);
  }
  if (kinds & kPullRowMajor) {
    const int n = ctas > 0 ? ctas : resident_ctas(k_pull, kPullThreads);
    const unsigned grid = (unsigned)std::min<uint32_t>(n_tiles, (uint32_t)n);
    k_pull<<<grid, kPullThreads, 0, (cudaStream_t)stream>>>(tiles, n_tiles, rank_base, work + 1);
  }
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------------- k_verify
// Copy-engine hop, receiver side: the chunk was copied by a copy engine; recompute its
// checksum from local HBM, compare with the predecessor's header, and release (or poison) the flag.
constexpr int kVerifyThreads = 512;

__global__ void __launch_bounds__(kVerifyThreads) k_verify(const uint8_t* __restrict__ data, uint32_t chunk,
                                                           uint64_t len, uint64_t* pred_flags,
                                                           const lam_chunk_header* pred_hdr, ChunkMeta meta,
                                                           uint64_t version, uint32_t* err_word,
                                                           const uint32_t* __restrict__ my_chunks, uint32_t pos,
                                                           uint32_t n_my) {
  __shared__ uint64_t red[2][kVerifyThreads / 32];
  const uint64_t nvec = len / 16;
  const uint64_t per = (nvec + gridDim.x - 1) / gridDim.x;
  const uint64_t v0 = per * blockIdx.x, v1 = min(nvec, v0 + per);
  uint64_t s1 = 0, s2 = 0;
  for (uint64_t v = v0 + threadIdx.x; v < v1; v += 4 * kVerifyThreads) {
    uint4 w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (v + k * kVerifyThreads < v1) w[k] = ld_stream_v4(data + 16 * (v + k * kVerifyThreads));
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (v + k * kVerifyThreads < v1) cks4(4 * (v + k * kVerifyThreads), w[k], s1, s2);
  }
  block_reduce2<kVerifyThreads>(s1, s2, red);
  if (threadIdx.x != 0) return;
  lam_chunk_header* h = meta.hdr + chunk;
  atomicAdd((unsigned long long*)&h->s1, (unsigned long long)s1);
  atomicAdd((unsigned long long*)&h->s2, (unsigned long long)s2);
  __threadfence();
  if (atomicAdd(meta.cnt + chunk, 1u) + 1 != gridDim.x) return;
  __threadfence();
  const uint64_t got1 = atomicAdd((unsigned long long*)&h->s1, 0ull);
  const uint64_t got2 = atomicAdd((unsigned long long*)&h->s2, 0ull);
  const lam_chunk_header* ph = pred_hdr + chunk;
  const bool ok = ld_acquire_sys(pred_flags + chunk) == version && got1 == ld_relaxed_sys(&ph->s1) &&
                  got2 == ld_relaxed_sys(&ph->s2);
  if (ok) {
    h->version = ld_relaxed_sys(&ph->version);
    h->idx = ld_relaxed_sys(&ph->idx);
    h->n = ld_relaxed_sys(&ph->n);
    h->bytes = ld_relaxed_sys(&ph->bytes);
    __threadfence_system();
    publish_flag(meta, chunk, version);
  } else {
    // failure stays local: poison our own flag (the successor aborts) and raise our abort flag, which
    // the flag waits queued for this part's later chunks poll (k_wait_flag) — never write into the
    // predecessor's flags (its state is its own)
    atomicCAS(err_word, 0u, (uint32_t)(-LAM_ECHECKSUM));
    atomicExch(meta.abort_flag, 1);
    publish_flag(meta, chunk, version | kPoison);
    __threadfence_system();
  }
}

__global__ void k_wait_flag(const uint64_t* flag, uint64_t v, uint64_t timeout_ns, const int32_t* abort_flag) {
  const uint64_t deadline = globaltimer() + timeout_ns;
  for (uint32_t spin = 0;; ++spin) {
    if ((int64_t)(ld_acquire_sys(flag) - v) >= 0) return;
    if (abort_flag && *(volatile const int32_t*)abort_flag) return;   // this part failed / was superseded
    if ((spin & 63) == 63 && globaltimer() > deadline) return;  // k_verify then reports the failure
    __nanosleep(200);
  }
}

int launch_wait_flag(const uint64_t* flag, uint64_t v, uint64_t timeout_ns, const int32_t* abort_flag, void* stream) {
  k_wait_flag<<<1, 1, 0, (cudaStream_t)stream>>>(flag, v, timeout_ns, abort_flag);
  return (int)cudaGetLastError();
}

int launch_verify(const uint8_t* data, uint32_t chunk, uint64_t len, uint64_t* pred_flags,
                  const lam_chunk_header* pred_hdr, ChunkMeta meta, uint64_t version, uint32_t* err_word,
                  const uint32_t* my_chunks, uint32_t pos, uint32_t n_my, int ctas, void* stream) {
  uint64_t nvec = len / 16;
  unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)ctas, std::max<uint64_t>(1, nvec / 2048));
  k_verify<<<grid, kVerifyThreads, 0, (cudaStream_t)stream>>>(data, chunk, len, pred_flags, pred_hdr, meta, version,
                                                             err_word, my_chunks, pos, n_my);
  return (int)cudaGetLastError();
}

}  // namespace lam

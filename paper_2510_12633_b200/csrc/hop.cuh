// k_hop — one hop of the chain-pipelined broadcast ("pipelines model chunk transfers
// along a chain of relays, overlapping communication among different hops"; L693).
// Included by kernels.cu (shares its primitives).
//
// Receiver-driven, TMA bulk pipeline (measured on B200 NVLink 5: 16 CTAs of bulk copies reach
// ~760 GB/s and 32 reach ~785 GB/s, where 16-B peer loads need ~148 CTAs — tools/p2p_bench.cu).
// Each CTA walks a fixed job list (its tiles cut into 32 KiB sub-blocks); stage ring of 6 x 32 KiB:
//   producer (thread 0): before the first sub-block of a new chunk, check the predecessor's chunk
//     flag (ld.acquire.sys over NVLink); cp.async.bulk peer global -> smem stage, completion on an
//     mbarrier (expect_tx).  Refills are non-blocking, so a chunk's completion is never held
//     behind the wait for the next chunk; only an empty pipeline makes it spin.
//   all 128 threads: checksum (S1, S2) of the stage from shared memory (conflict-free 16-B reads);
//     one __syncthreads per stage.
//   thread 0: cp.async.bulk smem -> local HBM (one bulk group per stage).  A stage is refilled one
//     iteration later (wait_group.read 1), so the store just issued is never waited on.
//   tile end: block-reduce the checksum; the tile's completion (atomics into the chunk header,
//     counter, flag) is deferred until two more store groups were issued (wait_group 2), so the
//     drain of its stores overlaps the next tile.  The CTA completing a chunk compares with the
//     predecessor's header and releases the flag (st.release.sys) — or poisons it on mismatch so
//     the successor aborts too.

constexpr int kHopThreads = 128;
constexpr int kHopStages = 6;
constexpr uint32_t kHopSub = 32768;  // bytes per pipeline stage
constexpr size_t kHopSmem = (size_t)kHopStages * kHopSub;

enum : int { kHopOk = 0, kHopPoison = 1, kHopAbort = 2, kHopTimeout = 3 };

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{ .reg .pred p; WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra WAIT_%=; }" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");  // async-proxy writes before generic release
}

__device__ void hop_fail(ChunkMeta meta, uint32_t* err_word, uint32_t chunk, uint64_t version, int why) {
  atomicExch(meta.abort_flag, 1);
  const uint32_t code = (why == kHopTimeout) ? (uint32_t)(-LAM_ETIMEOUT) : (uint32_t)(-LAM_ECHECKSUM);
  atomicCAS(err_word, 0u, code);
  st_release_sys(meta.flags + chunk, version | kPoison);  // tell our successor
  __threadfence_system();
}

// Tile finished and its stores complete: fold its checksum into the chunk header; the CTA that
// completes the chunk verifies it against the predecessor and publishes (or poisons) the flag.
__device__ void hop_complete_tile(ChunkMeta meta, const RankLink& L, const uint32_t* tiles_per_chunk, uint32_t chunk,
                                  uint64_t s1, uint64_t s2, uint64_t version, uint32_t* err_word) {
  __threadfence_system();
  lam_chunk_header* h = meta.hdr + chunk;
  atomicAdd((unsigned long long*)&h->s1, (unsigned long long)s1);
  atomicAdd((unsigned long long*)&h->s2, (unsigned long long)s2);
  __threadfence();
  const uint32_t prev = atomicAdd(meta.cnt + chunk, 1u);
  if (prev + 1 != tiles_per_chunk[chunk]) return;
  __threadfence();
  const uint64_t got1 = atomicAdd((unsigned long long*)&h->s1, 0ull);
  const uint64_t got2 = atomicAdd((unsigned long long*)&h->s2, 0ull);
  const lam_chunk_header* ph = L.src_hdr + chunk;
  if (got1 == ld_relaxed_sys(&ph->s1) && got2 == ld_relaxed_sys(&ph->s2)) {
    h->version = ld_relaxed_sys(&ph->version);
    h->idx = ld_relaxed_sys(&ph->idx);
    h->n = ld_relaxed_sys(&ph->n);
    h->bytes = ld_relaxed_sys(&ph->bytes);
    __threadfence_system();
    st_release_sys(meta.flags + chunk, version);
  } else {
    hop_fail(meta, err_word, chunk, version, kHopPoison);
  }
}

__global__ void __launch_bounds__(kHopThreads, 1)
    k_hop(const HopTile* __restrict__ tiles, uint32_t n_tiles, const RankLink* __restrict__ links, ChunkMeta meta,
          const uint32_t* __restrict__ tiles_per_chunk, uint64_t version, uint32_t* err_word, uint64_t timeout_ns) {
  extern __shared__ __align__(1024) uint8_t stage_buf[];
  __shared__ __align__(8) uint64_t bar[kHopStages];
  __shared__ uint64_t red[2][kHopThreads / 32];
  __shared__ int s_status;
  __shared__ uint32_t s_fail_chunk;

  const uint32_t my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  uint32_t total = 0;  // jobs of this CTA (every thread knows the job list)
  for (uint32_t m = 0; m < my_tiles; ++m) total += (tiles[blockIdx.x + m * gridDim.x].bytes + kHopSub - 1) / kHopSub;

  // producer cursor (thread 0 only)
  uint32_t p_tile = 0, p_sub = 0, waited = 0xFFFFFFFFu, issued = 0;
  const uint64_t deadline = globaltimer() + timeout_ns;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kHopStages; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_status = kHopOk;
  }
  __syncthreads();

  // thread 0: issue the next job if its chunk is available; block=true spins until it is.
  auto try_issue = [&](bool block) -> bool {
    if (issued >= total || s_status != kHopOk) return false;
    const HopTile T = tiles[blockIdx.x + p_tile * gridDim.x];
    const RankLink& L = links[T.rank];
    if (T.chunk != waited) {
      for (uint32_t spin = 0;; ++spin) {
        const uint64_t f = ld_acquire_sys(L.src_flags + T.chunk);
        if (f == version) break;
        if (f == (version | kPoison)) { s_fail_chunk = T.chunk; s_status = kHopPoison; return false; }
        if (!block) return false;
        if (*(volatile int32_t*)meta.abort_flag) { s_fail_chunk = T.chunk; s_status = kHopAbort; return false; }
        if ((spin & 63) == 63 && globaltimer() > deadline) { s_fail_chunk = T.chunk; s_status = kHopTimeout; return false; }
        __nanosleep(spin < 64 ? 100 : 1000);
      }
      waited = T.chunk;
    }
    const uint32_t st = issued % kHopStages;
    const uint32_t off = p_sub * kHopSub;
    const uint32_t bytes = min(kHopSub, T.bytes - off);
    mbar_expect_tx(&bar[st], bytes);
    bulk_g2s(stage_buf + (size_t)st * kHopSub, L.src + T.region_off + off, bytes, &bar[st]);
    if (off + bytes >= T.bytes) { p_sub = 0; ++p_tile; } else { ++p_sub; }
    ++issued;
    return true;
  };

  if (threadIdx.x == 0 && total > 0) {
    try_issue(true);
    while (issued < kHopStages - 1 && try_issue(false)) {}
  }

  // consumer cursor (all threads); deferred tile completion (thread 0)
  uint32_t c_tile = 0, c_sub = 0, phases = 0, k = 0;
  uint64_t s1 = 0, s2 = 0;
  bool pend = false;
  uint32_t pend_chunk = 0, pend_rank = 0, groups_after = 0;
  uint64_t pend_s1 = 0, pend_s2 = 0;
  for (; k < total; ++k) {
    const uint32_t st = k % kHopStages;
    if (threadIdx.x == 0 && issued <= k) {        // pipeline empty: wait for the predecessor
      if (!try_issue(true)) mbar_arrive(&bar[st]);  // failure: release the waiters, exit below
    }
    mbar_wait(&bar[st], (phases >> st) & 1u);
    phases ^= 1u << st;
    const HopTile T = tiles[blockIdx.x + c_tile * gridDim.x];
    const uint32_t off = c_sub * kHopSub;
    const uint32_t bytes = min(kHopSub, T.bytes - off);
    const uint8_t* sb = stage_buf + (size_t)st * kHopSub;
    const uint64_t w0 = (uint64_t)T.word0 + off / 4;
    for (uint32_t v = threadIdx.x; v < bytes / 16; v += kHopThreads)
      cks4(w0 + 4ull * v, *reinterpret_cast<const uint4*>(sb + 16 * v), s1, s2);
    __syncthreads();                               // stage fully read; s_status uniform from here
    if (s_status != kHopOk) break;
    const RankLink& L = links[T.rank];
    if (threadIdx.x == 0) {
      bulk_s2g(L.dst + T.region_off + off, sb, bytes);
      if (pend) ++groups_after;
    }
    if (off + bytes >= T.bytes) {                  // tile end
      block_reduce2<kHopThreads>(s1, s2, red);
      if (threadIdx.x == 0) {
        if (pend) {                                // previous tile still pending: finish it now
          bulk_wait<1>();
          hop_complete_tile(meta, links[pend_rank], tiles_per_chunk, pend_chunk, pend_s1, pend_s2, version, err_word);
        }
        pend = true;
        pend_chunk = T.chunk;
        pend_rank = T.rank;
        pend_s1 = s1;
        pend_s2 = s2;
        groups_after = 0;
      }
      s1 = s2 = 0;
      c_sub = 0;
      ++c_tile;
    } else {
      ++c_sub;
    }
    if (threadIdx.x == 0) {
      if (pend && groups_after >= 2) {
        bulk_wait<2>();
        hop_complete_tile(meta, links[pend_rank], tiles_per_chunk, pend_chunk, pend_s1, pend_s2, version, err_word);
        pend = false;
      }
      bulk_wait_read<1>();                         // store k-1 has read its stage: refill it
      while (issued < k + kHopStages && try_issue(false)) {}
    }
  }
  if (threadIdx.x == 0) {
    bulk_wait<0>();
    if (pend && s_status == kHopOk)
      hop_complete_tile(meta, links[pend_rank], tiles_per_chunk, pend_chunk, pend_s1, pend_s2, version, err_word);
    if (s_status != kHopOk) {
      for (uint32_t j = k + 1; j < issued; ++j) {  // drain loads still landing in shared memory
        const uint32_t st = j % kHopStages;
        mbar_wait(&bar[st], (phases >> st) & 1u);
        phases ^= 1u << st;
      }
      // abort flag 2 = superseded by a chain rebuild (runtime restarts the fill): exit quietly,
      // keep the verified chunks and do not poison the successor
      if (!(s_status == kHopAbort && *(volatile int32_t*)meta.abort_flag == 2))
        hop_fail(meta, err_word, s_fail_chunk, version, s_status == kHopTimeout ? kHopTimeout : kHopPoison);
    }
  }
}

int launch_hop(const HopTile* tiles, uint32_t n_tiles, const RankLink* links, ChunkMeta meta,
               const uint32_t* tiles_per_chunk, uint64_t version, uint32_t* err_word, uint64_t timeout_ns,
               int ctas, void* stream) {
  if (n_tiles == 0) return 0;
  static bool attr[64] = {};  // the attribute is per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr[dev]) {
    cudaFuncSetAttribute(k_hop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHopSmem);
    attr[dev] = true;
  }
  unsigned grid = (unsigned)(n_tiles < (uint32_t)ctas ? n_tiles : (uint32_t)ctas);
  k_hop<<<grid, kHopThreads, kHopSmem, (cudaStream_t)stream>>>(tiles, n_tiles, links, meta, tiles_per_chunk, version,
                                                              err_word, timeout_ns);
  return (int)cudaGetLastError();
}

// k_hop — one hop of the chain-pipelined broadcast ("pipelines model chunk transfers
// along a chain of relays, overlapping communication among different hops"; L693).
// Included by kernels.cu (shares its primitives).
//
// Receiver-driven.  The NVLink pull is the latency-bound part, so it goes to TMA (bulk copies reach
// ~785 GB/s with 32 CTAs where 16-B peer loads need ~148 — tools/p2p_bench.cu); the local part is
// done by the threads that read the stage anyway:
//   producer (thread 0): before the first sub-block of a new chunk, check the predecessor's chunk
//     flag (ld.acquire.sys over NVLink); cp.async.bulk peer global -> smem stage, completion on an
//     mbarrier (expect_tx).  Refills are non-blocking, so the chunk in hand is never held behind the
//     wait for the next one; only an empty pipeline makes it spin.
//   all 512 threads, per 32 KiB stage: 16-B shared loads -> streaming 16-B stores to local HBM +
//     checksum (S1, S2); one __syncthreads, after which the stage is refilled immediately.
//   A CTA folds its share of a chunk into the chunk header once, after its last tile of that chunk
//     (fence, 3 atomics); the CTA completing the chunk compares with the predecessor's header and
//     releases the flag (st.release.sys) — or poisons it on mismatch so the successor aborts too
//     (SPEC L643).
// Cycle accounting of the previous design (128 threads, TMA store per stage; LAM_HOP_PROF): thread 0
// spent only 11-23 % waiting for data and ~80 % in the checksum pass and in waiting for its store to
// release the stage.

// Optional per-CTA cycle accounting of thread 0 (LAM_HOP_PROF=1; diagnostics only):
// [0] data wait, [1] copy + checksum, [2] barrier, [3] chunk flush, [4] refill, [5] empty-pipeline spin, [6] total
__device__ unsigned long long* g_hop_prof = nullptr;

constexpr int kHopThreads = 512;
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
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(smem_u32(p)));
  return v;
}

__device__ void hop_fail(ChunkMeta meta, uint32_t* err_word, uint32_t chunk, uint64_t version, int why) {
  atomicExch(meta.abort_flag, 1);
  const uint32_t code = (why == kHopTimeout) ? (uint32_t)(-LAM_ETIMEOUT) : (uint32_t)(-LAM_ECHECKSUM);
  atomicCAS(err_word, 0u, code);
  publish_flag(meta, chunk, version | kPoison);  // tell our successor
  __threadfence_system();
}

// A CTA's share of chunk `chunk` (n tiles) is in local HBM: fold it into the header; the CTA that
// completes the chunk verifies it against the predecessor and publishes (or poisons) the flag.
__device__ void hop_flush(ChunkMeta meta, const RankLink& L, const uint32_t* tiles_per_chunk, uint32_t chunk,
                          uint32_t n, uint64_t s1, uint64_t s2, uint64_t version, uint32_t* err_word) {
  lam_chunk_header* h = meta.hdr + chunk;
  atomicAdd((unsigned long long*)&h->s1, (unsigned long long)s1);
  atomicAdd((unsigned long long*)&h->s2, (unsigned long long)s2);
  __threadfence_system();
  const uint32_t prev = atomicAdd(meta.cnt + chunk, n);
  if (prev + n != tiles_per_chunk[chunk]) return;
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
    publish_flag(meta, chunk, version);
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
    while (issued < kHopStages && try_issue(false)) {}
  }

  unsigned long long* prof = g_hop_prof;
  unsigned long long pc[7] = {}, t_a = clock64(), t_b;
  const unsigned long long t_start = t_a;
#define HOP_LAP(i)                            \
  if (prof && threadIdx.x == 0) {             \
    t_b = clock64();                          \
    pc[i] += t_b - t_a;                       \
    t_a = t_b;                                \
  }
  // consumer cursor (all threads); per-chunk accumulation of this CTA's checksum share
  uint32_t c_tile = 0, c_sub = 0, phases = 0, k = 0, n_in_chunk = 0;
  uint64_t s1 = 0, s2 = 0;
  for (; k < total; ++k) {
    const uint32_t st = k % kHopStages;
    if (threadIdx.x == 0 && issued <= k) {        // pipeline empty: wait for the predecessor
      if (!try_issue(true)) mbar_arrive(&bar[st]);  // failure: release the waiters, exit below
    }
    HOP_LAP(5)
    mbar_wait(&bar[st], (phases >> st) & 1u);
    phases ^= 1u << st;
    HOP_LAP(0)
    const HopTile T = tiles[blockIdx.x + c_tile * gridDim.x];
    const uint32_t off = c_sub * kHopSub;
    const uint32_t bytes = min(kHopSub, T.bytes - off);
    const uint8_t* sb = stage_buf + (size_t)st * kHopSub;
    const RankLink& L = links[T.rank];
    uint8_t* dst = L.dst + T.region_off + off;
    const uint64_t w0 = (uint64_t)T.word0 + off / 4;
    if (s_status == kHopOk) {                      // (on failure the stage holds nothing valid)
      for (uint32_t v = threadIdx.x; v < bytes / 16; v += kHopThreads) {
        const uint4 w = lds128(sb + 16 * v);
        st_v4(dst + 16 * (size_t)v, w);
        cks4(w0 + 4ull * v, w, s1, s2);
      }
    }
    HOP_LAP(1)
    __syncthreads();                               // stage fully read; s_status uniform from here
    HOP_LAP(2)
    if (s_status != kHopOk) break;
    if (threadIdx.x == 0)                          // refill: every stage but the ones in flight is free
      while (issued < k + 1 + kHopStages && try_issue(false)) {}
    HOP_LAP(4)
    if (off + bytes >= T.bytes) {                  // tile end
      ++n_in_chunk;
      ++c_tile;
      c_sub = 0;
      const bool chunk_end = c_tile >= my_tiles || tiles[blockIdx.x + c_tile * gridDim.x].chunk != T.chunk;
      if (chunk_end) {                             // this CTA's last tile of the chunk: flush its share
        __threadfence_system();                    // this thread's stores before the header / flag
        block_reduce2<kHopThreads>(s1, s2, red);
        if (threadIdx.x == 0) hop_flush(meta, L, tiles_per_chunk, T.chunk, n_in_chunk, s1, s2, version, err_word);
        __syncthreads();                           // red[] reuse
        s1 = s2 = 0;
        n_in_chunk = 0;
      }
      HOP_LAP(3)
    } else {
      ++c_sub;
    }
  }
  if (prof && threadIdx.x == 0) {
    pc[6] = clock64() - t_start;
    for (int i = 0; i < 7; ++i) atomicAdd(prof + i, pc[i]);
  }
#undef HOP_LAP
  if (threadIdx.x == 0 && s_status != kHopOk) {
    for (uint32_t j = k + 1; j < issued; ++j) {    // drain loads still landing in shared memory
      const uint32_t st = j % kHopStages;
      mbar_wait(&bar[st], (phases >> st) & 1u);
      phases ^= 1u << st;
    }
    // abort flag 2 = superseded by a chain rebuild (runtime restarts the fill): exit quietly, keep
    // the verified chunks and do not poison the successor
    if (!(s_status == kHopAbort && *(volatile int32_t*)meta.abort_flag == 2))
      hop_fail(meta, err_word, s_fail_chunk, version, s_status == kHopTimeout ? kHopTimeout : kHopPoison);
  }
}

// LAM_HOP_PROF diagnostics: point g_hop_prof of the current device at a 7-counter buffer (or null).
int hop_set_profile(unsigned long long* buf) {
  return (int)cudaMemcpyToSymbol(g_hop_prof, &buf, sizeof buf);
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

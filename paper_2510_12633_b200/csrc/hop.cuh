// k_hop — one hop of the chain-pipelined broadcast ("pipelines model chunk transfers
// along a chain of relays, overlapping communication among different hops"; L693).
// Included by kernels.cu (shares its primitives).
//
// Receiver-driven.  The NVLink pull is the latency-bound part, so it goes to TMA (bulk copies reach
// ~785 GB/s with 32 CTAs where 16-B peer loads need ~148 — tools/p2p_bench.cu); the local part is
// done by the threads that read the stage anyway.  Warp-specialised (v4):
//   producer warp (lane 0): walks the CTA's tiles; before the first sub-block of a new chunk, checks
//     the predecessor's chunk flag (ld.acquire.sys over NVLink); waits for the stage to be empty
//     (mbarrier, one arrival per consumer warp) and issues cp.async.bulk peer global -> smem with
//     completion on the stage's full mbarrier (expect_tx).  It runs up to kHopStages ahead and never
//     waits on the consumers' per-stage work.
//   16 consumer warps, per 32 KiB stage: wait full -> 16-B shared loads -> streaming 16-B stores to
//     local HBM (or a host-memory relay) + checksum (S1, S2) -> __syncwarp, lane 0 arrives on empty.
//     No CTA-wide barrier per stage: v3 (one __syncthreads per stage, thread 0 both producer and
//     consumer) left thread 0 ~50 % in the copy, ~21 % in dependent tile/link loads of the refill and
//     only 11-16 % waiting for data (LAM_HOP_PROF, chain N=4), i.e. the refill latency sat on every
//     stage's critical path.
//   flusher warp (lane 0): a CTA folds its share of a chunk into the chunk header once, after its
//     last tile of that chunk: each consumer warp fences its stores, reduces its sums by shuffles and
//     lane 0 deposits them (double-buffered) and arrives on the chunk's flush mbarrier; the flusher
//     sums the 16 partials and does the 3 atomics; the CTA completing the chunk compares with the
//     predecessor's header (and re-reads the predecessor's flag: a chunk the predecessor poisoned
//     carries the sums of its own corrupt bytes) and releases the flag (st.release.sys) — or poisons
//     it on mismatch so the successor aborts too.  Multicast modes read the chunk from
//     this GPU's replica of node 0's slot instead of the predecessor's memory (links[].src).  v4 did this on consumer thread 0 between two CTA-wide
//     named barriers: ~10 % of the consumers' time (remote header loads, system fences).
//   Failure (predecessor poisoned, abort, timeout): the producer records the job index it stopped
//     at and arrives (without bytes) on that stage's full barrier; consumers finish every earlier
//     stage (all of them real, in-flight TMA) and stop there, so no copy is left landing in smem.

// Optional per-CTA cycle accounting (LAM_HOP_PROF=1; diagnostics only):
// [0] consumer data wait, [1] consumer copy + checksum, [2] producer empty-stage wait, [3] chunk
// flush, [4] producer issue (tile/link loads + TMA), [5] producer flag spin, [6] consumer total
__device__ unsigned long long* g_hop_prof = nullptr;

constexpr int kHopConsumers = 512;                 // 16 consumer warps
constexpr int kHopThreads = kHopConsumers + 64;    // + producer warp + flusher warp
// Pipeline geometry: kHopStages x kHopSub bytes of staging = 224 KiB of the 227 KiB.  Two instantiations:
// 7 x 32 KiB (default) and 14 x 16 KiB (LAM_HOP_STAGE_KB=16: finer-grained hand-off, same bytes in flight).
constexpr size_t kHopSmem = (size_t)7 * 32768;

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
  // the pred's own verdict too: a chunk it poisoned carries the sums of its (corrupt) bytes
  if (ld_acquire_sys(L.pred_flags + chunk) == version && got1 == ld_relaxed_sys(&ph->s1) &&
      got2 == ld_relaxed_sys(&ph->s2)) {
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

template <int kHopStages, uint32_t kHopSub>
__global__ void __launch_bounds__(kHopThreads, 1)
    k_hop(const HopTile* __restrict__ tiles, uint32_t n_tiles, const RankLink* __restrict__ links, ChunkMeta meta,
          const uint32_t* __restrict__ tiles_per_chunk, uint64_t version, uint32_t* err_word, uint64_t timeout_ns) {
  extern __shared__ __align__(1024) uint8_t stage_buf[];
  __shared__ __align__(8) uint64_t full[kHopStages], empty[kHopStages];
  __shared__ __align__(8) uint64_t fl_full[2], fl_free[2];   // flush hand-off, double-buffered
  __shared__ uint64_t red[2][2][kHopConsumers / 32];         // [buffer][s1|s2][consumer warp]
  __shared__ uint32_t s_fail_job;
  __shared__ int s_consumers_failed;

  const uint32_t my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* prof = g_hop_prof;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kHopStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kHopConsumers / 32);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&fl_full[b], kHopConsumers / 32);
      mbar_init(&fl_free[b], 1);
    }
    s_consumers_failed = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_fail_job = 0xFFFFFFFFu;
  }
  __syncthreads();

  if (warp == kHopConsumers / 32) {
    // ------------------------------------------------------------------ producer (one lane)
    if (lane != 0) return;
    unsigned long long pc[3] = {}, t_a = clock64(), t_b;
    const uint64_t deadline = globaltimer() + timeout_ns;
    uint32_t job = 0, waited = 0xFFFFFFFFu, fail_chunk = 0;
    int status = kHopOk;
    for (uint32_t m = 0; m < my_tiles && status == kHopOk; ++m) {
      const HopTile T = tiles[blockIdx.x + m * gridDim.x];
      const uint8_t* src = links[T.rank].src + T.region_off;
      const uint64_t* tf = links[T.rank].tile_flags;
      if (tf) {                                    // two-level broadcast, peer source: this tile only
        if (prof) { t_b = clock64(); pc[1] += t_b - t_a; t_a = t_b; }
        for (uint32_t spin = 0;; ++spin) {
          const uint64_t f = ld_acquire_sys(tf + T.tile);
          if (f == version) break;
          if (*(volatile int32_t*)meta.abort_flag) { status = kHopAbort; break; }
          if ((spin & 63) == 63 && globaltimer() > deadline) { status = kHopTimeout; break; }
          __nanosleep(spin < 64 ? 64 : 512);
        }
        if (prof) { t_b = clock64(); pc[2] += t_b - t_a; t_a = t_b; }
        if (status != kHopOk) { fail_chunk = T.chunk; break; }
        asm volatile("fence.proxy.async.global;" ::: "memory");
        waited = 0xFFFFFFFFu;                      // a later node-0 tile re-checks its chunk flag
      } else if (T.chunk != waited) {
        const uint64_t* flag = links[T.rank].src_flags + T.chunk;
        if (prof) { t_b = clock64(); pc[1] += t_b - t_a; t_a = t_b; }
        for (uint32_t spin = 0;; ++spin) {
          const uint64_t f = ld_acquire_sys(flag);
          if (f == version) break;
          if (f == (version | kPoison)) { status = kHopPoison; break; }
          if (*(volatile int32_t*)meta.abort_flag) { status = kHopAbort; break; }
          if ((spin & 63) == 63 && globaltimer() > deadline) { status = kHopTimeout; break; }
          __nanosleep(spin < 64 ? 100 : 1000);
        }
        if (prof) { t_b = clock64(); pc[2] += t_b - t_a; t_a = t_b; }
        if (status != kHopOk) { fail_chunk = T.chunk; break; }
        // the flag was acquired by a generic-proxy load; the chunk's bytes are read by the async
        // proxy (cp.async.bulk): order those reads after the acquire
        asm volatile("fence.proxy.async.global;" ::: "memory");
        waited = T.chunk;
      }
      for (uint32_t off = 0; off < T.bytes; off += kHopSub, ++job) {
        const uint32_t st = job % kHopStages;
        if (job >= (uint32_t)kHopStages) {
          if (prof) { t_b = clock64(); pc[1] += t_b - t_a; t_a = t_b; }
          mbar_wait(&empty[st], ((job / kHopStages) + 1) & 1u);
          if (prof) { t_b = clock64(); pc[0] += t_b - t_a; t_a = t_b; }
        }
        const uint32_t bytes = min(kHopSub, T.bytes - off);
        mbar_expect_tx(&full[st], bytes);
        bulk_g2s(stage_buf + (size_t)st * kHopSub, src + off, bytes, &full[st]);
      }
    }
    if (status != kHopOk) {
      // release the consumers at the stage this job would have used; every earlier stage is a real
      // copy they will wait for, so nothing is still landing in shared memory when they stop
      const uint32_t st = job % kHopStages;
      if (job >= (uint32_t)kHopStages) mbar_wait(&empty[st], ((job / kHopStages) + 1) & 1u);
      *(volatile uint32_t*)&s_fail_job = job;
      mbar_arrive(&full[st]);
      // abort flag 2 = superseded by a chain rebuild (the runtime restarts the fill): exit quietly,
      // keep the verified chunks and do not poison the successor
      if (!(status == kHopAbort && *(volatile int32_t*)meta.abort_flag == 2))
        hop_fail(meta, err_word, fail_chunk, version, status == kHopTimeout ? kHopTimeout : kHopPoison);
    }
    if (prof) {
      t_b = clock64();
      pc[1] += t_b - t_a;
      atomicAdd(prof + 2, pc[0]);
      atomicAdd(prof + 4, pc[1]);
      atomicAdd(prof + 5, pc[2]);
    }
    return;
  }

  if (warp == kHopConsumers / 32 + 1) {
    // ------------------------------------------------------------------- flusher (one lane)
    if (lane != 0) return;
    unsigned long long t_f = 0, t0;
    uint32_t q = 0, n_in_chunk = 0;
    for (uint32_t m = 0; m < my_tiles; ++m) {
      const HopTile T = tiles[blockIdx.x + m * gridDim.x];
      ++n_in_chunk;
      if (!(m + 1 >= my_tiles || tiles[blockIdx.x + (m + 1) * gridDim.x].chunk != T.chunk)) continue;
      const uint32_t b = q & 1u;
      mbar_wait(&fl_full[b], (q >> 1) & 1u);
      if (*(volatile int*)&s_consumers_failed) break;
      t0 = prof ? clock64() : 0;
      uint64_t a = 0, c = 0;
#pragma unroll
      for (int i = 0; i < kHopConsumers / 32; ++i) { a += red[b][0][i]; c += red[b][1][i]; }
      mbar_arrive(&fl_free[b]);
      hop_flush(meta, links[T.rank], tiles_per_chunk, T.chunk, n_in_chunk, a, c, version, err_word);
      if (prof) t_f += clock64() - t0;
      n_in_chunk = 0;
      ++q;
    }
    if (prof) atomicAdd(prof + 3, t_f);
    return;
  }

  // -------------------------------------------------------------------- consumers (16 warps)
  unsigned long long pc[3] = {}, t_a = clock64(), t_b;
  const unsigned long long t_start = t_a;
#define HOP_LAP(i)                            \
  if (prof && threadIdx.x == 0) {             \
    t_b = clock64();                          \
    pc[i] += t_b - t_a;                       \
    t_a = t_b;                                \
  }
  uint32_t job = 0, q = 0;   // q: this CTA's chunk-end count (flush buffer q & 1)
  uint64_t s1 = 0, s2 = 0;
  bool failed = false;
  for (uint32_t m = 0; m < my_tiles && !failed; ++m) {
    const HopTile T = tiles[blockIdx.x + m * gridDim.x];
    uint8_t* dst = links[T.rank].dst + T.region_off;
    for (uint32_t off = 0; off < T.bytes; off += kHopSub, ++job) {
      const uint32_t st = job % kHopStages;
      mbar_wait(&full[st], (job / kHopStages) & 1u);
      HOP_LAP(0)
      if (*(volatile uint32_t*)&s_fail_job == job) { failed = true; break; }
      const uint32_t bytes = min(kHopSub, T.bytes - off);
      const uint8_t* sb = stage_buf + (size_t)st * kHopSub;
      const uint64_t w0 = (uint64_t)T.word0 + off / 4;
      for (uint32_t v = threadIdx.x; v < bytes / 16; v += kHopConsumers) {
        const uint4 w = lds128(sb + 16 * v);
        st_v4(dst + off + 16 * (size_t)v, w);
        cks4(w0 + 4ull * v, w, s1, s2);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      HOP_LAP(1)
    }
    if (failed) break;
    if (meta.tile_flags) {                         // two-level broadcast: the tile is in our HBM — release it
      __threadfence_system();                      // to the peers that pull it (before our chunk verdict)
      asm volatile("bar.sync 1, %0;" ::"r"(kHopConsumers) : "memory");
      if (threadIdx.x == 0) st_release_sys(meta.tile_flags + T.tile, version);
    }
    const bool chunk_end = m + 1 >= my_tiles || tiles[blockIdx.x + (m + 1) * gridDim.x].chunk != T.chunk;
    if (chunk_end) {                               // this CTA's last tile of the chunk: hand its share over
      __threadfence_system();                      // this thread's stores before the header / flag
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      if (lane == 0) {
        const uint32_t b = q & 1u;
        if (q >= 2) mbar_wait(&fl_free[b], ((q >> 1) + 1) & 1u);   // the flusher took chunk q-2's sums
        red[b][0][warp] = s1;
        red[b][1][warp] = s2;
        mbar_arrive(&fl_full[b]);
      }
      ++q;
      s1 = s2 = 0;
      HOP_LAP(2)
    }
  }
  if (failed && lane == 0) {                       // wake the flusher at the chunk that never ended
    if (threadIdx.x == 0) *(volatile int*)&s_consumers_failed = 1;   // before warp 0's arrival below
    const uint32_t b = q & 1u;
    if (q >= 2) mbar_wait(&fl_free[b], ((q >> 1) + 1) & 1u);
    mbar_arrive(&fl_full[b]);
  }
  if (prof && threadIdx.x == 0) {
    atomicAdd(prof + 0, pc[0]);
    atomicAdd(prof + 1, pc[1]);
    atomicAdd(prof + 3, pc[2]);
    atomicAdd(prof + 6, clock64() - t_start);
  }
#undef HOP_LAP
}

// LAM_HOP_PROF diagnostics: point g_hop_prof of the current device at a 7-counter buffer (or null).
int hop_set_profile(unsigned long long* buf) {
  return (int)cudaMemcpyToSymbol(g_hop_prof, &buf, sizeof buf);
}

int launch_hop(const HopTile* tiles, uint32_t n_tiles, const RankLink* links, ChunkMeta meta,
               const uint32_t* tiles_per_chunk, uint64_t version, uint32_t* err_word, uint64_t timeout_ns,
               int ctas, void* stream) {
  if (n_tiles == 0) return 0;
  static const bool fine = [] {
    const char* e = getenv("LAM_HOP_STAGE_KB");
    return e && atoi(e) == 16;
  }();
  static bool attr[64] = {};  // the attribute is per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr[dev]) {
    cudaFuncSetAttribute(k_hop<7, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHopSmem);
    cudaFuncSetAttribute(k_hop<14, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHopSmem);
    attr[dev] = true;
  }
  unsigned grid = (unsigned)(n_tiles < (uint32_t)ctas ? n_tiles : (uint32_t)ctas);
  if (fine)
    k_hop<14, 16384><<<grid, kHopThreads, kHopSmem, (cudaStream_t)stream>>>(
        tiles, n_tiles, links, meta, tiles_per_chunk, version, err_word, timeout_ns);
  else
    k_hop<7, 32768><<<grid, kHopThreads, kHopSmem, (cudaStream_t)stream>>>(
        tiles, n_tiles, links, meta, tiles_per_chunk, version, err_word, timeout_ns);
  return (int)cudaGetLastError();
}

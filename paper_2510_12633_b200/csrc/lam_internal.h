// Internal types of liblam (not part of the ABI).  Host planning structures and the device
// work-descriptor formats the kernels consume.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/lam.h"

namespace lam {

constexpr uint64_t kSegAlign = 256;      // segment start alignment in a rank region
constexpr uint64_t kChunkAlign = 4096;   // chunk size granularity
constexpr uint64_t kSlotAlign = 2u << 20;
constexpr uint32_t kPackUnitElems = 32768;     // fp32 elements per pack work unit (128 KiB read)
constexpr uint32_t kHopTileBytes = 1u << 20;   // bytes per chain-hop tile
constexpr uint32_t kPullTileBytes = 256u << 10;
constexpr uint32_t kPullTRows = 256;     // K-major pull tile: source rows ...
constexpr uint32_t kPullTCols = 512;     // ... x columns (<= 256 KiB per tile)
// flag = version | kPoison marks a failed chunk.  Bit 62 (not 63) so that a stream memory op waiting
// for "(int64)(flag - version) >= 0" is released by a poisoned flag as well.
constexpr uint64_t kPoison = 1ull << 62;

inline uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
inline uint64_t align_up(uint64_t a, uint64_t b) { return cdiv(a, b) * b; }

// ------------------------------------------------------------------------------- model table
struct Tensor {
  std::string name;
  int64_t d0, d1;   // d1 = 1 for 1-D tensors
  int ndim;
  int64_t heads = 0;   // attention heads stacked along dim 0 (q/k/v weights and biases), else 0
  uint64_t numel() const { return (uint64_t)d0 * (uint64_t)d1; }
};
std::vector<Tensor> model_tensors(const lam_model_dims& d);
bool model_valid(const lam_model_dims& d);

struct DstPart { uint32_t tensor; int rule; };
struct VllmDst { std::string name; int64_t rows, cols; std::vector<DstPart> parts; };
// vLLM Qwen2 destination list for tp; returns false if the dims are not divisible.
bool vllm_layout(const lam_model_dims& d, int tp, std::vector<VllmDst>* out);
// Source slice of a part for rank `rank`: rows [r0, r1) x cols [c0, c1) (1-D: cols [0, 1)),
// followed in the destination by `pad` zero rows (vocabulary padding, LAM_VOCAB_DIM0 only).
constexpr int64_t kVocabPad = 64;   // vLLM DEFAULT_VOCAB_PADDING_SIZE (R15)
bool part_slice(const Tensor& t, int rule, int tp, int rank, int64_t* r0, int64_t* r1, int64_t* c0,
                int64_t* c1, int64_t* pad);

// ------------------------------------------------------------------------------- image plan
struct Segment {
  uint32_t tensor, rank;
  uint64_t elem0, count;
  uint64_t off;      // byte offset in the rank region
};

struct ImagePlan {
  uint64_t C = 0;
  int N = 0;
  std::vector<Segment> segs;                  // rank order, tensor order
  std::vector<std::vector<uint32_t>> by_tensor;  // segment indices per tensor
  std::vector<uint64_t> region_len, n_chunks, chunk_base;  // per rank
  uint64_t total_chunks = 0;
  std::vector<uint32_t> chunk_rank;           // per global chunk
  uint64_t chunk_len(uint64_t g) const;
};
bool build_image_plan(const std::vector<Tensor>& ts, int N, int layout, uint64_t C, ImagePlan* out);

// ------------------------------------------------------------------------- device work units
struct __attribute__((aligned(16))) PackUnit {   // fp32 shard range -> bf16 image range
  uint64_t src_elem;   // element offset inside the shard
  uint64_t dst_off;    // byte offset inside the node part's slot data (16-B aligned)
  uint32_t shard;      // index into the per-publish shard pointer table
  uint32_t n;          // elements
  uint32_t chunk;      // global chunk index
  uint32_t word0;      // u32 word index inside the chunk of the unit's first output word
};

struct __attribute__((aligned(16))) HopTile {    // one tile of a chunk moved pred -> this node
  uint64_t region_off; // byte offset inside the rank region (same in pred and here)
  uint32_t chunk;      // global chunk index
  uint32_t rank;       // actor rank whose region holds the chunk
  uint32_t bytes;      // multiple of 16
  uint32_t word0;      // u32 word index inside the chunk
  uint32_t tile;       // index in the part's tile list (tile flags of the two-level broadcast)
};

struct __attribute__((aligned(16))) RankLink {   // per actor rank, for the hop kernel
  const uint8_t* src;         // pred node: rank region base in the pinned pred slot
  const uint64_t* src_flags;  // chunk j's bytes may be read from src once src_flags[j] == version (the
                              // pred's flags, or its multicast replica's)
  const lam_chunk_header* src_hdr;   // pred's headers (the checksum the chunk must reproduce)
  uint8_t* dst;               // this node part: rank region base in the filling slot
  const uint64_t* pred_flags; // pred's flags: a chunk is committed only if the pred committed it
  const uint64_t* tile_flags; // two-level broadcast, peer source: wait per tile on these, not per chunk
};

struct __attribute__((aligned(16))) CopyTile {   // one 2-D block of a pull (reshard)
  uint64_t src_off;    // byte offset inside rank region of src_rank
  uint64_t dst;        // absolute destination address of the first row
  uint32_t src_pitch, dst_pitch;  // bytes
  uint32_t rows, row_bytes;
  uint32_t src_rank, align;       // align: 16, 4 or 2 — widest access all addresses allow;
                                  // | LAM_TILE_TRANSPOSE: element k of row r -> dst + k*dst_pitch + 2r;
                                  // src_rank == LAM_TILE_ZERO: zero-fill, no source
  bool transposed() const { return (align & LAM_TILE_TRANSPOSE) != 0; }
  bool zero() const { return src_rank == LAM_TILE_ZERO; }
};

// Build pack units for actor rank r from the caller's shards; returns false if uncovered.
bool build_pack_units(const ImagePlan& p, const std::vector<Tensor>& ts, int rank,
                      const std::vector<lam_shard>& shards, uint64_t region_base_in_part,
                      std::vector<PackUnit>* units, std::vector<uint32_t>* units_per_chunk,
                      std::string* err);
void build_hop_tiles(const ImagePlan& p, const std::vector<int>& ranks, std::vector<HopTile>* tiles,
                     std::vector<uint32_t>* tiles_per_chunk);
// LAM_HOP_TREE: relay `node`'s walk of `tiles` (hop order) — chunk runs in groups of R, the j-th run of
// a group owned by relay j + 1, rotated so the node's own run comes first; each tile's links index =
// source * N + rank, source = the run's owner when it is another relay in `peer_mask`, else node 0.
std::vector<HopTile> tree_hop_tiles(const std::vector<HopTile>& tiles, int R, int node, uint64_t peer_mask, int N);
// dst_base[k] = device address of destination k; src rank alignment assumed >= 256 B.
bool build_copy_tiles(const ImagePlan& p, const std::vector<Tensor>& ts, const lam_tp_layout& L,
                      std::vector<CopyTile>* tiles, uint64_t* bytes, std::string* err);
// Source chunk of a tile; cut tiles at source-chunk boundaries and order them by chunk.
uint32_t chunk_of(const ImagePlan& p, const CopyTile& t);
uint64_t chunk_order(const ImagePlan& p, uint32_t g, int rot);
std::vector<CopyTile> split_by_chunk(const ImagePlan& p, const std::vector<CopyTile>& in, int rot);
// Rank rotation of a TP rank's pull: spreads the TP ranks over the source rank regions.
inline int pull_rotation(const ImagePlan& p, const lam_tp_layout& L) {
  return L.tp_size > 0 ? (int)((int64_t)L.tp_rank * p.N / L.tp_size) : 0;
}

// ------------------------------------------------------------------------------ kernel entry
struct ChunkMeta {          // device view of one slot's metadata in a node part
  uint64_t* flags;          // [total_chunks]
  lam_chunk_header* hdr;    // [total_chunks]
  uint32_t* cnt;            // [total_chunks]
  int32_t* abort_flag;      // [1]
  uint64_t* mirror;         // [total_chunks] host-visible copy of flags (shared memory) or null
  uint64_t* mc_flags;       // LAM_HOP_MULTICAST pack: multicast VA of the slot's flag array, else null
  uint64_t* tile_flags;     // LAM_HOP_TREE hop: per-tile flags released as each tile lands, else null
};
constexpr uint32_t kMirrorChunks = 2048;  // chunks per slot mirrored to the host (streaming pulls)

// mc_dst: multicast VA of the same slot (LAM_HOP_MULTICAST, with meta.mc_flags), else null
int launch_pack(const PackUnit* units, uint32_t n_units, const float* const* shard_ptrs, uint8_t* dst, uint8_t* mc_dst,
                ChunkMeta meta, const uint32_t* units_per_chunk, uint64_t version, uint64_t n_total,
                const uint64_t* chunk_len, int ctas, void* stream, uint8_t* const* sub_dst, uint32_t* work,
                int sms = 0);   // sms > 0: only CTAs on SMs [0, sms) work (the rest exit at once)
int launch_hop(const HopTile* tiles, uint32_t n_tiles, const RankLink* links, ChunkMeta meta,
               const uint32_t* tiles_per_chunk, uint64_t version, uint32_t* err_word,
               uint64_t timeout_ns, int ctas, void* stream);
constexpr uint32_t kPullRowMajor = 1, kPullKMajor = 2;   // tile kinds present in a pull (launch_pull)
int launch_pull(const CopyTile* tiles, uint32_t n_tiles, const uint8_t* const* rank_base, int ctas,
                void* stream, uint32_t kinds, uint32_t* work);  // work: 2 counters, zeroed on `stream` here
// Diagnostics (LAM_HOP_PROF=1): 7 per-device cycle counters accumulated by k_hop's thread 0.
int hop_set_profile(unsigned long long* buf);
// One-thread kernel: spin until (int64)(*flag - v) >= 0, *abort_flag != 0 or timeout (fallback for
// stream memory ops).
int launch_wait_flag(const uint64_t* flag, uint64_t v, uint64_t timeout_ns, const int32_t* abort_flag,
                     void* stream);
// Copy-engine hop: verify chunk `chunk` (len bytes at `data`, already copied from the predecessor)
// against the predecessor's header; publish the header and flag — or poison our own flag and raise our
// abort flag, so that the part's remaining flag waits fall through (the runtime also stops enqueuing).
int launch_verify(const uint8_t* data, uint32_t chunk, uint64_t len, uint64_t* pred_flags,
                  const lam_chunk_header* pred_hdr, ChunkMeta meta, uint64_t version, uint32_t* err_word,
                  const uint32_t* my_chunks, uint32_t pos, uint32_t n_my, int ctas, void* stream);

}  // namespace lam

// liblam runtime: relay rings + version tables, publish, progress engine, pull, IPC.
//
// Control plane (PAPER L526-529 relays; L548-550 steps 5-7; SPEC L527-663 relay semantics):
//   * node 0 = the master: the actor's publish slots on the actor GPUs (the chain head);
//     nodes 1..R = relays in chain order.  Every node has S ring slots ("retain 2").
//   * slot states FREE -> FILLING(v) -> COMPLETE(v); `latest` only moves up and only
//     to COMPLETE versions (SPEC L633 complete-only serving).
//   * a node starts receiving the NEWEST version its predecessor holds (FILLING or COMPLETE) into a
//     FREE slot or a COMPLETE slot with no readers that is not its latest (latest-wins),
//     pinning the predecessor's slot until its hop kernels finish.
//   * a pull pins the latest slot (readers++) until its reshard kernel completes.
// The block lives in POSIX shared memory when there is one process per GPU (torchrun), guarded by
// a robust process-shared mutex; peer slots are mapped with CUDA IPC handles.
#include <cuda_runtime.h>
#include <errno.h>
#include <fcntl.h>
#include <pthread.h>
#include <stdio.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "control.h"
#include "lam_internal.h"
#include "mcast.h"

namespace lam {

using ctl::acquire_slot;
using ctl::find_slot;
using ctl::newest_held;

struct SlotMeta {   // byte offsets inside a slot's metadata block
  uint64_t flags, hdr, cnt, abort, tflags, bytes;   // tflags: LAM_HOP_TREE per-tile flags
};

struct Part {
  int node = 0, device = 0, index = 0, pos = 0;  // pos: index within its node (launch-mask bit)
  std::vector<int> ranks;            // actor ranks whose regions this part stores
  std::vector<int64_t> rank_off;     // [N] offset of rank r's region in slot data, -1 if not here
  uint64_t slot_data = 0, slot_stride = 0, meta_base = 0, meta_stride = 0, alloc_bytes = 0;
  bool local = false;
  uint8_t* base = nullptr;           // valid in this process (own allocation or IPC mapping)
  bool ipc_opened = false;
  uint8_t* data = nullptr;           // slot 0's data (HBM: base; host tier: pinned host mapping)
  uint8_t* meta = nullptr;           // slot 0's metadata block (always HBM of `device`)
  // host-memory tier (lam_node_desc.host_memory, NEXT-3): slot data in a memfd mapping
  bool host = false;
  int host_fd = -1;                  // memfd (owner) or /proc/<pid>/fd reopen (other processes)
  size_t host_bytes = 0;
  bool host_registered = false;
  // LAM_HOP_MULTICAST: node 0's slot data is the actor GPU's member of the multicast team (mcast.h);
  // the metadata block is a separate allocation (exported by IPC like a host part's)
  bool mc = false;
  // local-only
  cudaStream_t stream = nullptr;
  cudaEvent_t done_ev[LAM_MAX_SLOTS] = {};
  uint64_t inflight_version[LAM_MAX_SLOTS] = {};   // version of the kernel in flight (0 none)
  uint32_t* err_host = nullptr;      // [S] host-mapped error words
  uint32_t* err_dev = nullptr;
  HopTile* d_tiles = nullptr;
  uint32_t n_tiles = 0;
  uint32_t* d_tiles_per_chunk = nullptr;
  RankLink* d_links = nullptr;       // [S][S][N] (my slot, pred slot, rank)
  // copy-engine hop mode
  cudaStream_t vstream = nullptr;    // verify stream
  std::vector<uint32_t> my_chunks;   // this part's chunks in processing order
  uint32_t* d_my_chunks = nullptr;
  std::vector<cudaEvent_t> chunk_ev; // [n_my + 1]: per-chunk copy done, last = verify stream done
  uint32_t ce_next = 0;              // next chunk to enqueue (bounded window, see ce_topup)
  int ce_slot = -1, ce_ps = -1;
  uint64_t ce_version = 0;           // non-zero while chunks remain to be enqueued
  cudaEvent_t ce_t0 = nullptr;
  // chain repair (NEXT-1): what this part last launched into each slot, resume tables
  uint64_t launched_version[LAM_MAX_SLOTS] = {};
  uint32_t launched_epoch[LAM_MAX_SLOTS] = {};
  std::vector<HopTile> h_tiles;      // host copy of the full tile list
  HopTile* d_resume = nullptr;       // tiles of the chunks still missing after a rebuild
  RankLink* d_links_dyn = nullptr;   // links to a predecessor other than node - 1
  // tree: per-launch tiles (staggered, links index = source node * N + rank) and links [(R+1) N]
  HopTile* d_tiles_tree = nullptr;
  RankLink* d_links_tree = nullptr;
  const RankLink* last_links[LAM_MAX_SLOTS] = {};   // link table of the slot's last launch
  int mc_retry[LAM_MAX_SLOTS] = {};  // multicast modes: verification retries of the slot's fill
  unsigned long long* prof_host = nullptr;  // LAM_HOP_PROF counters (host-mapped)
};

struct RankPub {   // per local actor rank (node 0)
  cudaEvent_t ev[LAM_MAX_SLOTS] = {};
  uint64_t inflight_version[LAM_MAX_SLOTS] = {};
  std::vector<lam_shard> key;        // cached shard list of the last unit build
  PackUnit* d_units = nullptr;
  uint32_t n_units = 0, cap_units = 0;
  uint32_t* d_units_per_chunk = nullptr;
  const float** d_ptrs = nullptr;
  uint32_t cap_ptrs = 0;
  const float** h_ptrs = nullptr;    // pinned staging of the shard pointer table
  std::vector<PackUnit> h_units;     // host copy of the units (colocated subscriptions)
  uint64_t units_gen = 0;            // bumped whenever the units are rebuilt
  // colocated subscription (lam_subscribe): per-unit destination in the subscriber's buffers
  int32_t sub_rid = -1;              // pending subscriber (-1: none)
  std::vector<uint64_t> sub_tensor_dst;  // [n_tensors] dst address of element 0 of each tensor
  uint64_t sub_gen = ~0ull;          // units_gen the table was built for
  uint8_t** d_sub = nullptr;
  uint32_t cap_sub = 0;
};

struct PullPlan {
  CopyTile* d_tiles = nullptr;        // ordered by source chunk
  uint32_t n_tiles = 0;
  uint64_t bytes = 0, local_bytes = 0, remote_bytes = 0;
  uint32_t kinds = 0;                 // kPullRowMajor (row-major / zero tiles) | kPullKMajor
  std::vector<uint32_t> chunk_ids;    // source chunks in order
  std::vector<uint32_t> chunk_begin;  // [chunk_ids.size() + 1] tile ranges per chunk
  int device = 0;
  uint64_t last_use = 0;              // LRU stamp (bounded cache, kMaxPlans)
  cudaEvent_t last_ev = nullptr;      // recorded after the latest launch reading d_tiles
};

constexpr size_t kMaxPlans = 64;   // pull-plan cache bound (LRU)

struct PendingPull {
  cudaEvent_t ev;
  int node, slot, device;
};

struct DevLocal {
  uint64_t* d_chunk_len = nullptr;   // per device: [total_chunks]
  uint32_t* d_pack_work = nullptr;   // k_pack's dynamic unit counter (packs are serialised on `side`)
  cudaStream_t side = nullptr;
};

}  // namespace lam

using namespace lam;

struct lam_ctx {
  lam_config cfg;
  std::vector<Tensor> ts;
  ImagePlan plan;
  uint64_t params = 0;
  int S = 2, n_nodes = 1;
  SlotMeta sm;
  std::vector<std::vector<int>> node_parts;   // node -> part indices
  std::vector<std::vector<int>> node_rank_part;  // node -> [N] part index holding rank r
  std::vector<Part> parts;
  std::vector<RankPub> pubs;                  // [N]; local ranks only used
  std::map<int, DevLocal> dev;                // devices owned by this process
  bool star = false;                          // LAM_HOP_MULTICAST: every relay is fed by node 0
  bool mcast = false;                         // a multicast team exists (LAM_HOP_MULTICAST)
  bool tree = false;                          // LAM_HOP_TREE: two-level broadcast
  McTeam mc;                                  // the multicast team (NEXT-2)
  std::map<std::string, PullPlan> plans;
  uint64_t plan_clock = 0;
  struct PullRing { uint32_t* d = nullptr; uint32_t next = 0; std::vector<cudaEvent_t> ev; };
  std::map<int, PullRing> pull_work;  // per device: ring of k_pull tile-counter pairs
  std::map<std::pair<int, int>, const uint8_t**> d_rank_base;  // (node*S+slot, device) -> device array
  std::vector<PendingPull> pending;
  std::map<int, std::vector<cudaEvent_t>> ev_pool;  // per device
  Shm* shm = nullptr;
  bool shm_owner = false, shm_mapped = false;
  bool connected = false;
  lam_status pending_error = LAM_OK;
  uint64_t timeout_ns = 60ull * 1000000000ull;
  int pack_ctas = 0, hop_ctas = 0, pull_ctas = 0, pack_sms = 0;
  uint64_t* mirror_dev = nullptr;     // device view of shm->chunk_done (null: no streaming pulls)
  bool shm_registered = false;
  struct StreamPull {                 // lam_pull_stream in progress (per rollout)
    bool active = false;
    bool subscription = false;        // lam_subscribe: completed by the pack, not by chunk progress
    int node = 0, slot = 0, device = 0;
    uint64_t v = 0;
    lam_status status = LAM_OK;
    PullPlan* plan = nullptr;
    uint32_t next = 0;                // next chunk (index into plan->chunk_ids) to launch
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
    cudaEvent_t last = nullptr;       // recorded after the latest reshard launch (on the rollout's device)
  };
  std::vector<StreamPull> streams;    // [n_rollouts]
  // kernel timing (lam_set_profiling)
  bool profiling = false;
  struct Timed { int kind, dev; cudaEvent_t a, b; };
  std::vector<Timed> timed;
  std::map<int, std::vector<cudaEvent_t>> tev_pool;  // timing-enabled events per device
  std::map<int, cudaStream_t> util;   // per device: stream-ordered allocations while hops run
};

namespace {

using Lock = ShmLock;

bool owns(const lam_ctx* c, int device) {
  return device >= 0 && device < LAM_MAX_DEVICES && c->cfg.proc_of_device[device] == c->cfg.proc_rank;
}

int node_part_device(const lam_ctx* c, int node, int rank) {
  return node == 0 ? c->cfg.actor_device[rank] : c->cfg.relay[node - 1].part_device[rank];
}

// The predecessor a relay node has while nobody failed: node - 1 (chain), or node 0 (multicast star).
int base_pred(const lam_ctx* c, int node) { return c->star || c->tree ? 0 : node - 1; }

#define CK(x)                                             \
  do {                                                    \
    cudaError_t e_ = (x);                                 \
    if (e_ != cudaSuccess) {                              \
      fprintf(stderr, "liblam: %s failed: %s (%s:%d)\n", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return LAM_ECUDA;                                   \
    }                                                     \
  } while (0)

// events belong to the device current at creation: pool them per device (caller set the device)
cudaEvent_t get_event(lam_ctx* c, int dev) {
  auto& pool = c->ev_pool[dev];
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  return e;
}

cudaEvent_t prof_begin(lam_ctx* c, int dev, cudaStream_t st) {
  if (!c->profiling) return nullptr;
  auto& pool = c->tev_pool[dev];
  cudaEvent_t e = nullptr;
  if (!pool.empty()) { e = pool.back(); pool.pop_back(); } else { cudaEventCreate(&e); }
  cudaEventRecord(e, st);
  return e;
}

void prof_end(lam_ctx* c, int kind, int dev, cudaStream_t st, cudaEvent_t a) {
  if (!a) return;
  auto& pool = c->tev_pool[dev];
  cudaEvent_t e = nullptr;
  if (!pool.empty()) { e = pool.back(); pool.pop_back(); } else { cudaEventCreate(&e); }
  cudaEventRecord(e, st);
  c->timed.push_back({kind, dev, a, e});
}

ChunkMeta meta_of(const lam_ctx* c, const Part& p, int slot) {
  uint8_t* m = p.meta + (uint64_t)slot * p.meta_stride;
  ChunkMeta cm;
  cm.flags = reinterpret_cast<uint64_t*>(m + c->sm.flags);
  cm.hdr = reinterpret_cast<lam_chunk_header*>(m + c->sm.hdr);
  cm.cnt = reinterpret_cast<uint32_t*>(m + c->sm.cnt);
  cm.abort_flag = reinterpret_cast<int32_t*>(m + c->sm.abort);
  cm.mirror = c->mirror_dev ? c->mirror_dev + ((uint64_t)p.node * LAM_MAX_SLOTS + slot) * kShmMirrorChunks : nullptr;
  cm.mc_flags = nullptr;
  cm.tile_flags = c->tree && p.node > 0 ? reinterpret_cast<uint64_t*>(m + c->sm.tflags) : nullptr;
  return cm;
}

uint8_t* slot_data(const Part& p, int slot) { return p.data + (uint64_t)slot * p.slot_stride; }

// Device memory allocated (or freed) while hops may be running: cudaMalloc / cudaFree are implicit
// synchronisation points, so the first pull of a layout (its copy plan) would hold the caller until
// every hop kernel of the GPU ended.  Stream-ordered allocation on a per-device utility stream has no
// such wait.  The caller set the device.
cudaStream_t util_stream(lam_ctx* c, int dev) {
  cudaStream_t& s = c->util[dev];
  if (!s && cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) s = nullptr;
  return s;
}
cudaError_t dev_alloc(lam_ctx* c, int dev, void** p, size_t bytes) {
  cudaStream_t s = util_stream(c, dev);
  if (!s) return cudaErrorUnknown;
  cudaError_t e = cudaMallocAsync(p, bytes, s);
  return e != cudaSuccess ? e : cudaStreamSynchronize(s);
}
cudaError_t dev_upload(lam_ctx* c, int dev, void* dst, const void* src, size_t bytes) {
  cudaStream_t s = util_stream(c, dev);
  if (!s) return cudaErrorUnknown;
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  return e != cudaSuccess ? e : cudaStreamSynchronize(s);
}
void dev_free(lam_ctx* c, int dev, void* p) {
  cudaStream_t s = util_stream(c, dev);
  if (s) cudaFreeAsync(p, s);
}

// Host-memory tier: map `bytes` of the memfd `fd` and pin it for every device (mapped, portable).
lam_status map_host_part(Part& p, int fd, size_t bytes) {
  void* h = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  if (h == MAP_FAILED) {
    fprintf(stderr, "liblam: mmap of the host relay part (%.2f GB) failed: %s\n", bytes / 1e9, strerror(errno));
    return LAM_ENOMEM;
  }
  p.host_fd = fd;
  p.host_bytes = bytes;
  cudaError_t e = cudaHostRegister(h, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    fprintf(stderr, "liblam: cudaHostRegister(%.2f GB) failed: %s\n", bytes / 1e9, cudaGetErrorString(e));
    munmap(h, bytes);
    return LAM_ENOMEM;
  }
  p.host_registered = true;
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, h, 0) != cudaSuccess) return LAM_ECUDA;
  p.data = (uint8_t*)d;
  p.base = (uint8_t*)h;   // host address (munmap / unregister)
  return LAM_OK;
}

// Tile counters of the pull kernels' dynamic distribution: every launch takes the next pair of a
// per-device ring (zeroed by launch_pull on the launch's own stream), so launches in flight on
// different streams never share a counter.  Each entry carries the event recorded after its last
// launch; an entry whose launch has not completed is waited for before reuse (only possible with
// kPullRing launches queued at once).  The caller records *ev after its launch.
constexpr uint32_t kPullRing = 1024;
uint32_t* pull_counter(lam_ctx* c, int dev, cudaEvent_t* ev) {
  lam_ctx::PullRing& r = c->pull_work[dev];
  if (!r.d) {
    if (dev_alloc(c, dev, (void**)&r.d, 2 * sizeof(uint32_t) * kPullRing) != cudaSuccess) {
      r.d = nullptr;
      return nullptr;
    }
    r.ev.assign(kPullRing, nullptr);
  }
  const uint32_t i = r.next++ % kPullRing;
  if (!r.ev[i]) {
    if (cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming) != cudaSuccess) return nullptr;
  } else if (cudaEventSynchronize(r.ev[i]) != cudaSuccess) {   // normally long complete: returns at once
    return nullptr;
  }
  *ev = r.ev[i];
  return r.d + 2 * i;
}

lam_status validate(const lam_config& c, std::string* why) {
  auto bad = [&](const std::string& s) { *why = s; return LAM_EINVAL; };
  if (!model_valid(c.model)) return bad("model dims");
  if (c.actor_layout != LAM_FSDP2_DIM0 && c.actor_layout != LAM_FSDP1_FLAT) return bad("actor_layout");
  if (c.fsdp_size < 1 || c.fsdp_size > LAM_MAX_RANKS) return bad("fsdp_size");
  if (c.n_relays < 0 || c.n_relays > LAM_MAX_NODES) return bad("n_relays");
  if (c.slots < 2 || c.slots > LAM_MAX_SLOTS) return bad("slots");
  if (c.chunk_bytes % kChunkAlign) return bad("chunk_bytes must be a multiple of 4096");
  if (c.n_procs < 1 || c.proc_rank < 0 || c.proc_rank >= c.n_procs) return bad("proc_rank/n_procs");
  auto dev_ok = [&](int d) { return d >= 0 && d < LAM_MAX_DEVICES && c.proc_of_device[d] >= 0 && c.proc_of_device[d] < c.n_procs; };
  for (int r = 0; r < c.fsdp_size; ++r)
    if (!dev_ok(c.actor_device[r])) return bad("actor_device[" + std::to_string(r) + "]");
  for (int i = 0; i < c.n_relays; ++i)
    for (int r = 0; r < c.fsdp_size; ++r)
      if (!dev_ok(c.relay[i].part_device[r])) return bad("relay part_device");
  if (c.n_rollouts < 0 || c.n_rollouts > LAM_MAX_ROLLOUTS) return bad("n_rollouts");
  for (int i = 0; i < c.n_rollouts; ++i)
    if (c.rollout[i].node < 0 || c.rollout[i].node > c.n_relays || !dev_ok(c.rollout[i].device))
      return bad("rollout " + std::to_string(i));
  if (c.n_procs > 1 && c.shm_name[0] == 0) return bad("shm_name required with n_procs > 1");
  if (c.hop_mode != LAM_HOP_KERNEL && c.hop_mode != LAM_HOP_COPY_ENGINE && c.hop_mode != LAM_HOP_MULTICAST &&
      c.hop_mode != LAM_HOP_TREE)
    return bad("hop_mode");
  if (c.hop_mode == LAM_HOP_TREE) {   // relays read each other's slots: whole, in HBM, one per GPU, off the actors
    std::set<int> used(c.actor_device, c.actor_device + c.fsdp_size);
    for (int i = 0; i < c.n_relays; ++i) {
      const int d = c.relay[i].part_device[0];
      for (int r = 1; r < c.fsdp_size; ++r)
        if (c.relay[i].part_device[r] != d) return bad("tree hops: a relay node split over GPUs");
      if (c.relay[i].host_memory) return bad("tree hops need HBM relay nodes");
      if (!used.insert(d).second) return bad("tree hops: relays must sit on distinct non-actor GPUs");
    }
  }
  if (c.hop_mode == LAM_HOP_MULTICAST) {
    // one source GPU (the multicast writer), HBM relays, node-0 readers on the source GPU
    for (int r = 1; r < c.fsdp_size; ++r)
      if (c.actor_device[r] != c.actor_device[0]) return bad("multicast hops need every actor rank on one GPU");
    for (int i = 0; i < c.n_relays; ++i)
      if (c.relay[i].host_memory) return bad("multicast hops need HBM relay nodes");
    for (int i = 0; i < c.n_rollouts; ++i)
      if (c.rollout[i].node == 0 && c.rollout[i].device != c.actor_device[0])
        return bad("multicast hops: a rollout of node 0 must be on the actor GPU");
  }
  return LAM_OK;
}

lam_status setup_shm(lam_ctx* c) {
  if (c->cfg.n_procs == 1) {
    c->shm = shm_heap();
    return c->shm ? LAM_OK : LAM_ENOMEM;
  }
  c->shm_owner = c->cfg.proc_rank == 0;
  c->shm = c->shm_owner ? shm_create(c->cfg.shm_name) : shm_attach(c->cfg.shm_name);
  c->shm_mapped = c->shm != nullptr;
  return c->shm ? LAM_OK : LAM_EIPC;
}

lam_status alloc_parts(lam_ctx* c) {
  const int N = c->cfg.fsdp_size, S = c->S;
  const uint64_t total = c->plan.total_chunks;
  c->sm.flags = 0;
  c->sm.hdr = align_up(c->sm.flags + 8 * total, 64);
  c->sm.cnt = align_up(c->sm.hdr + sizeof(lam_chunk_header) * total, 64);
  c->sm.abort = align_up(c->sm.cnt + 4 * total, 64);
  c->sm.tflags = align_up(c->sm.abort + 64, 64);
  uint64_t ntiles = 0;
  if (c->cfg.hop_mode == LAM_HOP_TREE) {   // a whole node's tile list (every relay of the tree is whole)
    std::vector<int> all(N);
    for (int r = 0; r < N; ++r) all[r] = r;
    std::vector<HopTile> tl;
    std::vector<uint32_t> tpc;
    build_hop_tiles(c->plan, all, &tl, &tpc);
    ntiles = tl.size();
  }
  c->sm.bytes = align_up(c->sm.tflags + 8 * ntiles, 4096);
  c->node_parts.assign(c->n_nodes, {});
  c->node_rank_part.assign(c->n_nodes, std::vector<int>(N, -1));
  for (int node = 0; node < c->n_nodes; ++node) {
    std::map<int, int> by_dev;
    for (int r = 0; r < N; ++r) {
      int d = node_part_device(c, node, r);
      auto it = by_dev.find(d);
      if (it == by_dev.end()) {
        Part p;
        p.node = node;
        p.device = d;
        p.index = (int)c->parts.size();
        p.pos = (int)c->node_parts[node].size();
        p.rank_off.assign(N, -1);
        p.local = owns(c, d);
        p.host = node > 0 && c->cfg.relay[node - 1].host_memory != 0;
        by_dev[d] = p.index;
        c->node_parts[node].push_back(p.index);
        c->parts.push_back(p);
        it = by_dev.find(d);
      }
      Part& p = c->parts[it->second];
      p.rank_off[r] = (int64_t)p.slot_data;
      p.slot_data += c->plan.n_chunks[r] * c->plan.C;
      p.ranks.push_back(r);
      c->node_rank_part[node][r] = it->second;
    }
  }
  for (Part& p : c->parts) {
    p.slot_stride = align_up(std::max<uint64_t>(p.slot_data, 1), kSlotAlign);
    p.meta_base = p.slot_stride * S;
    p.meta_stride = c->sm.bytes;
    p.alloc_bytes = p.meta_base + p.meta_stride * S;
  }
  if (c->mcast) {
    // multicast team members (NEXT-2): node 0's S slots followed by S flag arrays, on the actor GPU
    // and every relay GPU this process owns
    const Part& p0 = c->parts[c->node_parts[0][0]];
    c->mc.flag_stride = align_up(8 * std::max<uint64_t>(total, 1), 4096);
    c->mc.flags_off = p0.slot_stride * S;
    std::vector<int> local;
    for (int d : c->mc.devices)
      if (owns(c, d)) local.push_back(d);
    if (!local.empty()) {
      lam_status ms = mc_alloc_members(c->mc, local, c->mc.flags_off + c->mc.flag_stride * S);
      if (ms != LAM_OK) return ms;
    }
  }
  for (Part& p : c->parts) {
    if (!p.local) continue;
    CK(cudaSetDevice(p.device));
    if (p.node == 0 && c->mcast) {
      // slot data = the actor GPU's member of the multicast team (zero-filled); metadata separate
      p.mc = true;
      p.data = c->mc.va.at(p.device);
      if (cudaMalloc(&p.meta, (size_t)p.meta_stride * S) != cudaSuccess) return LAM_ENOMEM;
      CK(cudaMemset(p.meta, 0, (size_t)p.meta_stride * S));
    } else if (p.host) {
      // slot data in pinned host memory (zero-filled by the kernel), metadata in HBM
      const size_t hb = (size_t)p.slot_stride * S;
      int fd = (int)memfd_create("lam_host_relay", 0);
      if (fd < 0 || ftruncate(fd, (off_t)hb) != 0) {
        fprintf(stderr, "liblam: memfd for the host relay part (%.2f GB) failed: %s\n", hb / 1e9, strerror(errno));
        if (fd >= 0) close(fd);
        return LAM_ENOMEM;
      }
      lam_status hs = map_host_part(p, fd, hb);
      if (hs != LAM_OK) return hs;
      if (cudaMalloc(&p.meta, (size_t)p.meta_stride * S) != cudaSuccess) return LAM_ENOMEM;
      CK(cudaMemset(p.meta, 0, (size_t)p.meta_stride * S));
    } else {
      if (cudaMalloc(&p.base, p.alloc_bytes) != cudaSuccess) {
        fprintf(stderr, "liblam: cudaMalloc(%.2f GB) failed on device %d\n", p.alloc_bytes / 1e9, p.device);
        return LAM_ENOMEM;
      }
      CK(cudaMemset(p.base, 0, p.alloc_bytes));
      p.data = p.base;
      p.meta = p.base + p.meta_base;
    }
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // relay hops at the greatest priority: a hop (32 SM-light CTAs) launched while a rollout's reshard
    // fills the GPU gets the first SMs that free up instead of queueing behind the rest of the pull
    CK(cudaStreamCreateWithPriority(&p.stream, cudaStreamNonBlocking, p.node > 0 ? hi : lo));
    for (int s = 0; s < S; ++s) CK(cudaEventCreateWithFlags(&p.done_ev[s], cudaEventDisableTiming));
    CK(cudaHostAlloc(&p.err_host, sizeof(uint32_t) * LAM_MAX_SLOTS, cudaHostAllocMapped | cudaHostAllocPortable));
    memset(p.err_host, 0, sizeof(uint32_t) * LAM_MAX_SLOTS);
    CK(cudaHostGetDevicePointer((void**)&p.err_dev, p.err_host, 0));
    if (!c->dev.count(p.device)) {
      DevLocal dl;
      std::vector<uint64_t> len(total);
      for (uint64_t g = 0; g < total; ++g) len[g] = c->plan.chunk_len(g);
      CK(cudaMalloc(&dl.d_chunk_len, 8 * std::max<uint64_t>(total, 1)));
      if (total) CK(cudaMemcpy(dl.d_chunk_len, len.data(), 8 * total, cudaMemcpyHostToDevice));
      CK(cudaStreamCreateWithPriority(&dl.side, cudaStreamNonBlocking, lo));
      CK(cudaMalloc(&dl.d_pack_work, sizeof(uint32_t)));
      c->dev[p.device] = dl;
    }
    if (p.node > 0) {
      std::vector<HopTile> tiles;
      std::vector<uint32_t> tpc;
      build_hop_tiles(c->plan, p.ranks, &tiles, &tpc);
      p.n_tiles = (uint32_t)tiles.size();
      CK(cudaMalloc(&p.d_tiles, sizeof(HopTile) * std::max<size_t>(tiles.size(), 1)));
      if (!tiles.empty()) CK(cudaMemcpy(p.d_tiles, tiles.data(), sizeof(HopTile) * tiles.size(), cudaMemcpyHostToDevice));
      if (getenv("LAM_HOP_PROF")) {
        unsigned long long* dptr = nullptr;
        CK(cudaHostAlloc(&p.prof_host, 8 * 8, cudaHostAllocMapped | cudaHostAllocPortable));
        memset(p.prof_host, 0, 64);
        CK(cudaHostGetDevicePointer((void**)&dptr, p.prof_host, 0));
        if (hop_set_profile(dptr)) return LAM_ECUDA;
      }
      CK(cudaMalloc(&p.d_resume, sizeof(HopTile) * std::max<size_t>(tiles.size(), 1)));
      CK(cudaMalloc(&p.d_links_dyn, sizeof(RankLink) * N));
      if (c->tree) {
        CK(cudaMalloc(&p.d_tiles_tree, sizeof(HopTile) * std::max<size_t>(tiles.size(), 1)));
        CK(cudaMalloc(&p.d_links_tree, sizeof(RankLink) * N * c->n_nodes));
      }
      p.h_tiles = tiles;
      CK(cudaMalloc(&p.d_tiles_per_chunk, 4 * std::max<uint64_t>(total, 1)));
      if (total) CK(cudaMemcpy(p.d_tiles_per_chunk, tpc.data(), 4 * total, cudaMemcpyHostToDevice));
      // copy-engine mode: chunk order, verify stream, per-chunk events
      for (const HopTile& t : tiles)
        if (p.my_chunks.empty() || p.my_chunks.back() != t.chunk) p.my_chunks.push_back(t.chunk);
      CK(cudaMalloc(&p.d_my_chunks, 4 * std::max<size_t>(p.my_chunks.size(), 1)));
      if (!p.my_chunks.empty())
        CK(cudaMemcpy(p.d_my_chunks, p.my_chunks.data(), 4 * p.my_chunks.size(), cudaMemcpyHostToDevice));
      if (c->cfg.hop_mode == LAM_HOP_COPY_ENGINE) {
        CK(cudaStreamCreateWithPriority(&p.vstream, cudaStreamNonBlocking, lo));
        p.chunk_ev.resize(p.my_chunks.size() + 1);
        for (auto& e : p.chunk_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      }
    }
  }
  return LAM_OK;
}

// LAM_HOP_MULTICAST: create/import the multicast object, add and bind this process's team devices.
// Called outside the control-block lock (cuMulticastBindMem blocks until every process added its GPU).
lam_status mc_connect(lam_ctx* c) {
  if (!c->mcast || c->mc.mc) return LAM_OK;
  std::vector<int> local;
  std::set<int> procs;
  for (int d : c->mc.devices) {
    if (owns(c, d)) local.push_back(d);
    procs.insert(c->cfg.proc_of_device[d]);
  }
  if (local.empty()) return LAM_OK;
  const bool owner = owns(c, c->mc.owner_dev);
  const std::string sock = std::string("lam-mc-") + c->cfg.shm_name;
  lam_status st = mc_setup(c->mc, local, owner, owner ? (int)procs.size() - 1 : 0, sock.c_str());
  if (st != LAM_OK) return st;
  if (!owner)   // node 0's slot data as seen from this process: the owner's member, mapped over NVLink
    for (Part& p : c->parts)
      if (p.node == 0 && p.mc && !p.local) p.data = c->mc.owner_va;
  return LAM_OK;
}

lam_status connect_links(lam_ctx* c) {
  const int N = c->cfg.fsdp_size, S = c->S;
  // single process: enable peer access among every pair of used devices
  if (c->cfg.n_procs == 1) {
    std::set<int> devs;
    for (auto& p : c->parts) devs.insert(p.device);
    for (int i = 0; i < c->cfg.n_rollouts; ++i) devs.insert(c->cfg.rollout[i].device);
    for (int a : devs)
      for (int b : devs) {
        if (a == b) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, a, b);
        if (!can) continue;
        cudaSetDevice(a);
        cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return LAM_ECUDA;
        cudaGetLastError();
      }
  }
  for (auto& p : c->parts)
    if ((!p.data && !p.mc) || !p.meta) {
      fprintf(stderr, "liblam: part of node %d on device %d not mapped (missing lam_import_ipc?)\n", p.node, p.device);
      return LAM_EIPC;
    }
  // hop link tables: [my slot][pred slot][rank]
  for (Part& p : c->parts) {
    if (!p.local || p.node == 0) continue;
    std::vector<RankLink> links((size_t)S * S * N);
    for (int s = 0; s < S; ++s)
      for (int ps = 0; ps < S; ++ps)
        for (int r : p.ranks) {
          const Part& q = c->parts[c->node_rank_part[base_pred(c, p.node)][r]];
          ChunkMeta qm = meta_of(c, q, ps);
          RankLink& L = links[((size_t)s * S + ps) * N + r];
          L.src = slot_data(q, ps) + q.rank_off[r];
          L.src_flags = qm.flags;
          L.src_hdr = qm.hdr;
          L.pred_flags = qm.flags;
          if (c->star) {
            // the relay's replica of node 0's slot in its own GPU's team member, and the chunk flags
            // the pack multicast next to it: data and flags are read from local HBM
            uint8_t* mine = c->mc.va.at(p.device);
            L.src = mine + (uint64_t)ps * q.slot_stride + q.rank_off[r];
            L.src_flags = reinterpret_cast<const uint64_t*>(mine + c->mc.flags_off + (uint64_t)ps * c->mc.flag_stride);
          }
          L.dst = slot_data(p, s) + p.rank_off[r];
        }
    CK(cudaSetDevice(p.device));
    CK(cudaMalloc(&p.d_links, sizeof(RankLink) * links.size()));
    CK(cudaMemcpy(p.d_links, links.data(), sizeof(RankLink) * links.size(), cudaMemcpyHostToDevice));
  }
  // pull source tables: per (node, slot, rollout device)
  std::set<std::pair<int, int>> need;
  for (int i = 0; i < c->cfg.n_rollouts; ++i)
    if (owns(c, c->cfg.rollout[i].device)) need.insert({c->cfg.rollout[i].node, c->cfg.rollout[i].device});
  for (auto nd : need) {
    for (int s = 0; s < S; ++s) {
      std::vector<const uint8_t*> base(N);
      for (int r = 0; r < N; ++r) {
        const Part& q = c->parts[c->node_rank_part[nd.first][r]];
        base[r] = slot_data(q, s) + q.rank_off[r];
      }
      CK(cudaSetDevice(nd.second));
      const uint8_t** d = nullptr;
      CK(cudaMalloc(&d, sizeof(void*) * N));
      CK(cudaMemcpy(d, base.data(), sizeof(void*) * N, cudaMemcpyHostToDevice));
      c->d_rank_base[{nd.first * LAM_MAX_SLOTS + s, nd.second}] = d;
    }
  }
  c->connected = true;
  return LAM_OK;
}

// ------------------------------------------------------------------------ copy-engine hop mode
// cuStreamWaitValue64 through the runtime's driver entry point (no link dependency on libcuda).
typedef int (*WaitValue64Fn)(void* stream, unsigned long long addr, unsigned long long value, unsigned int flags);

WaitValue64Fn wait_value_fn() {
  static WaitValue64Fn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", (void**)&fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    cudaGetLastError();
  }
  return fn;
}

// Stream waits until (int64)(*flag - v) >= 0 (flag == v, or v | kPoison): a front-end stream memory
// operation when the driver supports it, else a one-thread polling kernel.
lam_status stream_wait_flag(lam_ctx* c, cudaStream_t st, const uint64_t* flag, uint64_t v, const int32_t* abort_flag) {
  // Stream memory ops on CUDA-IPC-mapped peer memory never released in multi-process runs on
  // B200 / driver 580 (observed hang); there, poll with a one-thread kernel instead.
  WaitValue64Fn fn = c->cfg.n_procs == 1 ? wait_value_fn() : nullptr;
  if (fn && fn((void*)st, (unsigned long long)(uintptr_t)flag, v, 0x0 /*CU_STREAM_WAIT_VALUE_GEQ*/) == 0)
    return LAM_OK;
  if (launch_wait_flag(flag, v, c->timeout_ns, abort_flag, st)) return LAM_ECUDA;
  c->shm->stats.kernel_launches++;
  return LAM_OK;
}

// Enqueue the next chunks of the part's copy-engine hop.  Gating, in order of preference:
//  * host mirror (the producers mirror every chunk flag into the shared control block): a chunk is
//    enqueued only once the predecessor verified it (or poisoned it: the copy is then made and
//    k_verify fails it, which propagates the failure down the chain), so the copy stream holds
//    nothing but copies — no wait kernel that a busy GPU (e.g. a streaming pull filling every SM)
//    could delay, and the copy engines run back to back while the chain is flowing;
//  * otherwise a device-side wait per chunk (stream memory op / one-thread polling kernel), at most
//    kCeWindow chunks ahead of the copies that completed: enqueueing hundreds of flag waits at once
//    can block the host thread (full push buffer) while it holds the cross-process lock.
// lam_relay_step tops the queue up.
constexpr uint32_t kCeWindow = 8;
constexpr uint32_t kCeMirrorWindow = 24;   // copies in flight when gated by the mirror

lam_status ce_topup(lam_ctx* c, Part& p) {
  if (!p.ce_version) return LAM_OK;
  const int s = p.ce_slot, ps = p.ce_ps;
  const uint64_t u = p.ce_version;
  ChunkMeta m = meta_of(c, p, s);
  const uint32_t n = (uint32_t)p.my_chunks.size();
  CK(cudaSetDevice(p.device));
  for (uint32_t i = p.ce_next; i < n; i = ++p.ce_next) {
    if (*(volatile uint32_t*)&p.err_host[s]) {   // a chunk failed verification: enqueue nothing more, close the hop
      p.ce_next = n;
      break;
    }
    const uint32_t g = p.my_chunks[i];
    const uint64_t* mir = c->mirror_dev ? c->shm->chunk_done[p.node - 1][ps] : nullptr;
    const uint32_t window = mir ? kCeMirrorWindow : kCeWindow;
    if (i >= window) {
      cudaError_t q = cudaEventQuery(p.chunk_ev[i - window]);
      if (q == cudaErrorNotReady) return LAM_OK;
      if (q != cudaSuccess) return LAM_ECUDA;
    }
    if (mir) {
      const uint64_t f = __atomic_load_n(mir + g, __ATOMIC_ACQUIRE);
      if (f != u && f != (u | kPoison)) return LAM_OK;   // not verified at the predecessor yet
    }
    const int r = (int)c->plan.chunk_rank[g];
    const Part& q = c->parts[c->node_rank_part[p.node - 1][r]];
    ChunkMeta qm = meta_of(c, q, ps);
    const uint64_t off = (g - c->plan.chunk_base[r]) * c->plan.C, len = c->plan.chunk_len(g);
    const uint8_t* src = slot_data(q, ps) + q.rank_off[r] + off;
    uint8_t* dst = slot_data(p, s) + p.rank_off[r] + off;
    cudaStream_t cs = p.stream;
    if (!mir) {
      lam_status st = stream_wait_flag(c, cs, qm.flags + g, u, m.abort_flag);
      if (st != LAM_OK) return st;
    }
    CK(cudaMemcpyAsync(dst, src, len, cudaMemcpyDefault, cs));
    CK(cudaEventRecord(p.chunk_ev[i], cs));
    CK(cudaStreamWaitEvent(p.vstream, p.chunk_ev[i], 0));
    if (launch_verify(dst, g, len, qm.flags, qm.hdr, m, u, p.err_dev + s, p.d_my_chunks, i, n, 32, p.vstream))
      return LAM_ECUDA;
    c->shm->stats.kernel_launches++;
  }
  // all chunks enqueued: join the verify stream, close the timing bracket, arm completion polling
  CK(cudaEventRecord(p.chunk_ev.back(), p.vstream));
  CK(cudaStreamWaitEvent(p.stream, p.chunk_ev.back(), 0));
  prof_end(c, 1, p.device, p.stream, p.ce_t0);
  CK(cudaEventRecord(p.done_ev[s], p.stream));
  p.inflight_version[s] = u;
  p.ce_version = 0;
  return LAM_OK;
}

// ---------------------------------------------------------------------- chain repair (NEXT-1)
// Ask the part's in-flight hop kernel for slot s to exit without poisoning anything (abort = 2).
cudaError_t abort_part_kernel(lam_ctx* c, Part& p, int s) {
  static const int32_t two = 2;
  ChunkMeta m = meta_of(c, p, s);
  // a separate stream: the write must not queue behind the kernel it stops
  cudaError_t e = cudaMemcpyAsync(m.abort_flag, &two, sizeof two, cudaMemcpyHostToDevice, c->dev[p.device].side);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(c->dev[p.device].side);
}

// Resume list after a rebuild: every tile of every chunk the slot has not verified yet, with the
// chunk's header sums and counter reset (chunks already verified keep their bytes and header).
lam_status build_resume(lam_ctx* c, Part& p, int s, uint64_t u, uint32_t* n_out) {
  ChunkMeta m = meta_of(c, p, s);
  const uint64_t total = c->plan.total_chunks;
  std::vector<uint64_t> flags(total);
  CK(cudaStreamSynchronize(p.stream));
  CK(cudaMemcpy(flags.data(), m.flags, 8 * total, cudaMemcpyDeviceToHost));
  std::vector<HopTile> res;
  std::vector<uint32_t> missing;
  for (const HopTile& t : p.h_tiles) {
    if (flags[t.chunk] == u) continue;
    if (missing.empty() || missing.back() != t.chunk) missing.push_back(t.chunk);
    res.push_back(t);
  }
  if (!res.empty()) CK(cudaMemcpy(p.d_resume, res.data(), sizeof(HopTile) * res.size(), cudaMemcpyHostToDevice));
  for (uint32_t g : missing) {
    CK(cudaMemsetAsync(m.hdr + g, 0, sizeof(lam_chunk_header), p.stream));
    CK(cudaMemsetAsync(m.cnt + g, 0, 4, p.stream));
  }
  CK(cudaMemsetAsync(m.abort_flag, 0, 4, p.stream));
  *n_out = (uint32_t)res.size();
  return LAM_OK;
}

// Hop links of part p (my slot s) to predecessor node `pred` (slot ps) — for rebuilt chains.
lam_status build_links(lam_ctx* c, Part& p, int s, int pred, int ps) {
  std::vector<RankLink> links(c->cfg.fsdp_size);
  for (int r : p.ranks) {
    const Part& q = c->parts[c->node_rank_part[pred][r]];
    ChunkMeta qm = meta_of(c, q, ps);
    links[r].src = slot_data(q, ps) + q.rank_off[r];
    links[r].src_flags = qm.flags;
    links[r].src_hdr = qm.hdr;
    links[r].dst = slot_data(p, s) + p.rank_off[r];
    links[r].pred_flags = qm.flags;
  }
  CK(cudaStreamSynchronize(p.stream));
  CK(cudaMemcpy(p.d_links_dyn, links.data(), sizeof(RankLink) * links.size(), cudaMemcpyHostToDevice));
  return LAM_OK;
}

uint64_t steady_ns() {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (uint64_t)ts.tv_sec * 1000000000ull + (uint64_t)ts.tv_nsec;
}

// Stop this process's kernels of a failed node (a simulated failure keeps its memory alive; nothing
// reads it after the rebuild).
lam_status abort_node_locked(lam_ctx* c, int node) {
  for (Part& p : c->parts) {
    if (!p.local || p.node != node) continue;
    CK(cudaSetDevice(p.device));
    for (int s = 0; s < c->S; ++s)
      if (p.inflight_version[s]) {
        CK(abort_part_kernel(c, p, s));
        p.inflight_version[s] = 0;
      }
    p.ce_version = 0;
  }
  return LAM_OK;
}

// A node failed: rebuild the chain (control plane), then stop this process's kernels of that node.
lam_status fail_node_locked(lam_ctx* c, int node) {
  if (!ctl::fail_node(c->shm, c->S, node, steady_ns())) return LAM_EINVAL;
  c->shm->stats.chain_rebuilds++;
  return abort_node_locked(c, node);
}

// Heartbeats ("detects the failure via heartbeat monitoring"): every lam_relay_step
// stamps this process; a process silent for longer than heartbeat_timeout_s is declared failed and
// every relay node with a part on its GPUs is removed from the chain (ctl::heartbeat, O(1) each).
lam_status heartbeat_locked(lam_ctx* c) {
  std::vector<uint64_t> node_procs(c->n_nodes, 0);
  for (const Part& p : c->parts) node_procs[p.node] |= 1ull << c->cfg.proc_of_device[p.device];
  const uint64_t limit = c->cfg.heartbeat_timeout_s > 0 ? (uint64_t)(c->cfg.heartbeat_timeout_s * 1e9) : 0;
  const uint64_t failed = ctl::heartbeat(c->shm, c->S, c->cfg.proc_rank, c->cfg.n_procs, steady_ns(), limit,
                                         node_procs.data(), c->n_nodes);
  for (int node = 1; node < c->n_nodes; ++node)
    if (failed >> node & 1ull) {
      lam_status st = abort_node_locked(c, node);
      if (st != LAM_OK) return st;
    }
  return LAM_OK;
}

// ----------------------------------------------------------------------------- progress engine
// Launch the hop kernel of local part p (node >= 1) for FILLING slot s.  Returns true if launched.
lam_status launch_hop_part(lam_ctx* c, Part& p, int s, bool* launched) {
  *launched = false;
  ShmNode& n = c->shm->node[p.node];
  ShmSlot& sl = n.slot[s];
  const int ps = sl.src_slot;
  const int pred = n.pred;
  const uint64_t u = sl.version;
  CK(cudaSetDevice(p.device));
  // Restart after a chain rebuild (same version, new epoch): resume from the lowest missing chunks.
  const bool resume = p.launched_version[s] == u && p.launched_epoch[s] != sl.epoch;
  if (resume && p.inflight_version[s] == u) {
    // the superseded kernel may be spinning on the failed predecessor: ask it to exit quietly
    CK(abort_part_kernel(c, p, s));
    CK(cudaStreamSynchronize(p.stream));
    p.inflight_version[s] = 0;
  }
  // predecessor parts on the same GPU must have finished (never spin on a kernel of the same GPU)
  std::set<int> waits;
  for (int r : p.ranks) {
    int qi = c->node_rank_part[pred][r];
    const Part& q = c->parts[qi];
    if (q.device != p.device) continue;
    if (!q.local) return LAM_EINVAL;  // one process per GPU: cannot happen
    if (pred == 0) {
      if (!(c->shm->node[0].slot[ps].launched_mask >> r & 1ull)) return LAM_OK;  // not yet published
      if (c->pubs[r].inflight_version[ps] == u) CK(cudaStreamWaitEvent(p.stream, c->pubs[r].ev[ps], 0));
    } else {
      waits.insert(qi);
    }
  }
  for (int qi : waits) {
    const Part& q = c->parts[qi];
    const ShmSlot& qs = c->shm->node[q.node].slot[ps];
    if (qs.state == S_FILLING && !(qs.launched_mask >> q.pos & 1ull)) return LAM_OK;  // wait
    if (q.inflight_version[ps] == u) CK(cudaStreamWaitEvent(p.stream, q.done_ev[ps], 0));
  }
  ChunkMeta m = meta_of(c, p, s);
  const HopTile* tiles = p.d_tiles;
  uint32_t n_tiles = p.n_tiles;
  if (resume) {
    // keep the chunks this slot already verified (own flag == u); redo every other chunk whole
    lam_status st = build_resume(c, p, s, u, &n_tiles);
    if (st != LAM_OK) return st;
    tiles = p.d_resume;
    c->shm->stats.chain_resumes++;
    if (c->shm->last_fail_ns) c->shm->stats.last_repair_ns = steady_ns() - c->shm->last_fail_ns;
  } else {
    CK(cudaMemsetAsync((uint8_t*)m.hdr, 0, c->sm.abort + 64 - c->sm.hdr, p.stream));  // hdr, cnt, abort
  }
  p.err_host[s] = 0;
  p.launched_version[s] = u;
  p.launched_epoch[s] = sl.epoch;
  cudaEvent_t t0 = prof_begin(c, p.device, p.stream);
  if (c->cfg.hop_mode == LAM_HOP_COPY_ENGINE && !resume && pred == p.node - 1) {
    p.ce_slot = s;
    p.ce_ps = ps;
    p.ce_next = 0;
    p.ce_version = u;
    p.ce_t0 = t0;
    sl.launched_mask |= 1ull << p.pos;
    c->shm->stats.hops_launched++;
    *launched = true;
    return ce_topup(c, p);
  } else {
    const int N = c->cfg.fsdp_size;
    const RankLink* links = p.d_links + (size_t)(s * c->S + ps) * N;
    if (pred != base_pred(c, p.node)) {  // rebuilt chain: links to the new predecessor
      lam_status st = build_links(c, p, s, pred, ps);
      if (st != LAM_OK) return st;
      links = p.d_links_dyn;
    } else if (c->tree && !resume) {
      // two-level broadcast: sources = node 0 (links [0, N)) and every relay this fill pinned (links
      // [o N, (o+1) N)); the tile order and each chunk's source come from tree_hop_tiles (plan.cpp)
      const int R = c->n_nodes - 1;
      std::vector<RankLink> tl((size_t)c->n_nodes * N);
      for (int src = 0; src < c->n_nodes; ++src) {
        if (src == p.node || (src > 0 && !(sl.peer_mask >> src & 1ull))) continue;
        const int qs = src == 0 ? ps : sl.peer_slot[src];
        for (int r : p.ranks) {
          const Part& q = c->parts[c->node_rank_part[src][r]];
          const Part& q0 = c->parts[c->node_rank_part[0][r]];
          ChunkMeta qm = meta_of(c, q, qs), q0m = meta_of(c, q0, ps);
          RankLink& L = tl[(size_t)src * N + r];
          L.src = slot_data(q, qs) + q.rank_off[r];
          L.src_flags = qm.flags;
          // a peer's tile is read as soon as it landed there (its tile flag), before the peer verified
          // the chunk: the chunk is checked against node 0's header and verdict, which every copy shares
          L.tile_flags = src > 0 ? qm.tile_flags : nullptr;
          L.src_hdr = q0m.hdr;
          L.pred_flags = q0m.flags;
          L.dst = slot_data(p, s) + p.rank_off[r];
        }
      }
      const std::vector<HopTile> tt = tree_hop_tiles(p.h_tiles, R, p.node, sl.peer_mask, N);
      CK(cudaStreamSynchronize(p.stream));   // the previous launch (another version) used these tables
      CK(cudaMemcpy(p.d_links_tree, tl.data(), sizeof(RankLink) * tl.size(), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(p.d_tiles_tree, tt.data(), sizeof(HopTile) * tt.size(), cudaMemcpyHostToDevice));
      links = p.d_links_tree;
      tiles = p.d_tiles_tree;
    }
    p.last_links[s] = links;
    p.mc_retry[s] = 0;
    int rc = launch_hop(tiles, n_tiles, links, m, p.d_tiles_per_chunk, u, p.err_dev + s, c->timeout_ns,
                        // host-tier destination: PCIe stores need more CTAs in flight (v6 box run:
                        // 32 CTAs 29 GB/s, 148 CTAs 47 GB/s but starved the concurrent pulls)
                        p.host && c->cfg.hop_ctas <= 0 ? 96 : c->hop_ctas, p.stream);
    if (rc) {
      fprintf(stderr, "liblam: hop launch failed: %s\n", cudaGetErrorString((cudaError_t)rc));
      return LAM_ECUDA;
    }
    if (n_tiles) c->shm->stats.kernel_launches++;
  }
  prof_end(c, 1, p.device, p.stream, t0);
  CK(cudaEventRecord(p.done_ev[s], p.stream));
  p.inflight_version[s] = u;
  sl.launched_mask |= 1ull << p.pos;
  c->shm->stats.hops_launched++;
  *launched = true;
  return LAM_OK;
}

// Multicast modes: relaunch slot s's fill for the chunks it has not committed (kept chunks keep their
// bytes, header and flag), with the link table of its last launch.
lam_status retry_part(lam_ctx* c, Part& p, int s) {
  ShmSlot& sl = c->shm->node[p.node].slot[s];
  const uint64_t u = p.inflight_version[s];
  CK(cudaSetDevice(p.device));
  uint32_t n = 0;
  lam_status st = build_resume(c, p, s, u, &n);
  if (st != LAM_OK) return st;
  p.err_host[s] = 0;
  p.mc_retry[s]++;
  fprintf(stderr, "liblam: node %d slot %d v%llu: re-verifying %u tiles from the multicast replica (retry %d)\n",
          p.node, s, (unsigned long long)u, n, p.mc_retry[s]);
  ChunkMeta m = meta_of(c, p, s);
  if (launch_hop(p.d_resume, n, p.last_links[s], m, p.d_tiles_per_chunk, u, p.err_dev + s, c->timeout_ns, c->hop_ctas,
                 p.stream))
    return LAM_ECUDA;
  if (n) c->shm->stats.kernel_launches++;
  CK(cudaEventRecord(p.done_ev[s], p.stream));
  (void)sl;
  return LAM_OK;
}

// Streaming pull progress (lam_pull_stream): launch the reshard of every newly verified chunk (the
// producers mirror chunk flags into the shared control block), then close with the done event.
constexpr uint32_t kStreamBatches = 8;
lam_status stream_progress(lam_ctx* c, int rid, int* transitions) {
  lam_ctx::StreamPull& sp = c->streams[rid];
  if (!sp.active) return LAM_OK;
  Shm* sh = c->shm;
  const ShmSlot& sl = sh->node[sp.node].slot[sp.slot];
  CK(cudaSetDevice(sp.device));
  const bool failed = sl.version != sp.v || (sl.state != S_FILLING && sl.state != S_COMPLETE) || sh->node[sp.node].dead;
  const uint32_t n = (uint32_t)sp.plan->chunk_ids.size();
  if (!failed) {
    const uint64_t* mir = sh->chunk_done[sp.node][sp.slot];
    const uint32_t first = sp.next;
    while (sp.next < n && (sl.state == S_COMPLETE ||
                           __atomic_load_n(mir + sp.plan->chunk_ids[sp.next], __ATOMIC_ACQUIRE) == sp.v))
      ++sp.next;
    // While the previous reshard launch is still running, wait for a batch of >= n/8 chunks (or the
    // rest): launches on one stream serialise and each pays a tail of straggling tiles, so hundreds of
    // one-chunk launches behind each other cost more than they overlap.  An idle stream (the usual
    // case behind a chain hop, where chunks arrive slower than they reshard) launches at once.
    const uint32_t min_batch = std::max<uint32_t>(1, (n + kStreamBatches - 1) / kStreamBatches);
    if (sp.next > first && sp.next - first < min_batch && sp.next < n && sl.state != S_COMPLETE && sp.last &&
        cudaEventQuery(sp.last) == cudaErrorNotReady)
      sp.next = first;
    if (sp.next > first) {
      auto rb = c->d_rank_base.find({sp.node * LAM_MAX_SLOTS + sp.slot, sp.device});
      const uint32_t b = sp.plan->chunk_begin[first], e = sp.plan->chunk_begin[sp.next];
      cudaEvent_t t0 = prof_begin(c, sp.device, sp.stream);
      cudaEvent_t wev = nullptr;
      uint32_t* work = pull_counter(c, sp.device, &wev);
      if (!work) return LAM_ENOMEM;
      if (launch_pull(sp.plan->d_tiles + b, e - b, rb->second, c->pull_ctas, sp.stream, sp.plan->kinds, work))
        return LAM_ECUDA;
      c->shm->stats.kernel_launches += __builtin_popcount(sp.plan->kinds);
      CK(cudaEventRecord(wev, sp.stream));
      CK(cudaEventRecord(sp.plan->last_ev, sp.stream));
      prof_end(c, 2, sp.device, sp.stream, t0);
      if (!sp.last) CK(cudaEventCreateWithFlags(&sp.last, cudaEventDisableTiming));
      CK(cudaEventRecord(sp.last, sp.stream));
      (*transitions)++;
    }
    if (sp.next < n) return LAM_OK;
  } else {
    sp.status = LAM_ECHECKSUM;
  }
  if (sp.done) CK(cudaEventRecord(sp.done, sp.stream));
  cudaEvent_t ev = get_event(c, sp.device);
  CK(cudaEventRecord(ev, sp.stream));
  c->pending.push_back({ev, sp.node, sp.slot, sp.device});  // unpin once the stream gets there
  sp.active = false;
  (*transitions)++;
  return LAM_OK;
}

lam_status step_locked(lam_ctx* c, int* transitions, bool* busy) {
  Shm* sh = c->shm;
  const int S = c->S;
  lam_status first_err = LAM_OK;
  *busy = false;
  lam_status hb = heartbeat_locked(c);
  if (hb != LAM_OK) return hb;
  // (1) completions of local packs (node 0)
  for (int r = 0; r < c->cfg.fsdp_size; ++r) {
    if (!owns(c, c->cfg.actor_device[r])) continue;
    RankPub& rp = c->pubs[r];
    for (int s = 0; s < S; ++s) {
      if (!rp.inflight_version[s]) continue;
      cudaError_t q = cudaEventQuery(rp.ev[s]);
      if (q == cudaErrorNotReady) { *busy = true; continue; }
      if (q != cudaSuccess) return LAM_ECUDA;
      if (ctl::pack_done(sh, c->cfg.fsdp_size, s, rp.inflight_version[s])) (*transitions)++;
      rp.inflight_version[s] = 0;
    }
  }
  // (2) copy-engine hops: top up the enqueue window; completions of local hops
  for (Part& p : c->parts) {
    if (!p.local || p.node == 0) continue;
    if (p.ce_version) {
      *busy = true;
      lam_status st = ce_topup(c, p);
      if (st != LAM_OK) return st;
    }
    for (int s = 0; s < S; ++s) {
      if (!p.inflight_version[s]) continue;
      cudaError_t q = cudaEventQuery(p.done_ev[s]);
      if (q == cudaErrorNotReady) { *busy = true; continue; }
      if (q != cudaSuccess) return LAM_ECUDA;
      if (p.prof_host) {
        const unsigned long long* q = p.prof_host;
        const double tot = (double)(q[6] ? q[6] : 1);
        fprintf(stderr, "k_hop node %d dev %d: consumer wait %.1f%% copy+cks %.1f%% flush %.1f%% | producer empty-wait %.1f%% issue %.1f%% flag-spin %.1f%% (%.2f Gcyc)\n",
                p.node, p.device, 100 * q[0] / tot, 100 * q[1] / tot, 100 * q[3] / tot, 100 * q[2] / tot,
                100 * q[4] / tot, 100 * q[5] / tot, tot / 1e9);
        memset(p.prof_host, 0, 64);
      }
      const lam_status e = p.err_host[s] ? -(lam_status)p.err_host[s] : LAM_OK;
      if (e == LAM_ECHECKSUM && c->mcast && p.mc_retry[s] < 2) {
        // multicast modes: bytes stored through the switch may land at a replica after the chunk's flag
        // (a rare mismatch under load, seen with a withdrawn multicast + chain mode): verify the failed chunks again from the
        // replica before giving the version up.  A chunk whose bytes are really wrong fails again.
        lam_status rs = retry_part(c, p, s);
        if (rs != LAM_OK) return rs;
        *busy = true;
        continue;
      }
      if (e != LAM_OK && getenv("LAM_DEBUG_FAIL")) {   // diagnostics: which chunk failed first
        std::vector<uint64_t> f(c->plan.total_chunks);
        ChunkMeta fm = meta_of(c, p, s);
        if (cudaMemcpy(f.data(), fm.flags, 8 * f.size(), cudaMemcpyDeviceToHost) == cudaSuccess)
          for (size_t g = 0; g < f.size(); ++g)
            if (f[g] & kPoison) {
              fprintf(stderr, "liblam: node %d dev %d slot %d v%llu: chunk %zu of %zu failed (%s)\n", p.node, p.device,
                      s, (unsigned long long)p.inflight_version[s], g, f.size(), lam_strerror(e));
              break;
            }
      }
      if (ctl::part_done(sh, p.node, s, p.inflight_version[s], (int)c->node_parts[p.node].size(), e,
                         p.launched_epoch[s])) {
        (*transitions)++;
        if (e != LAM_OK && first_err == LAM_OK) first_err = e;
      }
      p.inflight_version[s] = 0;
    }
  }
  // (2b) streaming pulls of this process's rollouts
  for (int rid = 0; rid < (int)c->streams.size(); ++rid) {
    if (!c->streams[rid].active) continue;
    if (c->streams[rid].subscription) {
      *busy = true;
      continue;
    }
    lam_status st = stream_progress(c, rid, transitions);
    if (st != LAM_OK) return st;
    if (c->streams[rid].active) *busy = true;
  }
  // (3) pull pins
  for (size_t i = 0; i < c->pending.size();) {
    cudaError_t q = cudaEventQuery(c->pending[i].ev);
    if (q == cudaErrorNotReady) { *busy = true; ++i; continue; }
    if (q != cudaSuccess) return LAM_ECUDA;
    ctl::unpin(sh, c->pending[i].node, c->pending[i].slot);
    c->ev_pool[c->pending[i].device].push_back(c->pending[i].ev);
    c->pending[i] = c->pending.back();
    c->pending.pop_back();
    (*transitions)++;
  }
  // (4) start new versions (latest-wins) and launch local parts
  for (int node = 1; node < c->n_nodes; ++node) {
    ShmNode& n = sh->node[node];
    bool opened = false;
    const int fill = ctl::start(sh, S, node, &opened);
    if (opened) (*transitions)++;
    if (fill >= 0) {
      for (int pi : c->node_parts[node]) {
        Part& p = c->parts[pi];
        if (!p.local || (n.slot[fill].launched_mask >> p.pos & 1ull)) continue;
        bool launched = false;
        lam_status st = launch_hop_part(c, p, fill, &launched);
        if (st != LAM_OK) return st;
        if (launched) (*transitions)++;
      }
    }
  }
  // (5) anything still moving anywhere?
  if (!*busy) *busy = ctl::busy(sh, S, c->n_nodes);
  return first_err;
}

std::string layout_key(int node, const lam_tp_layout& L);

// Cached copy plan of (node, layout); build on miss (caller holds the lock, device = rollout's).
lam_status get_plan(lam_ctx* c, const lam_rollout_desc& ro, const lam_tp_layout& L, const std::string& key,
                    PullPlan** out) {
  auto it = c->plans.find(key);
  if (it != c->plans.end()) {
    c->shm->stats.plan_cache_hits++;
    it->second.last_use = ++c->plan_clock;
    *out = &it->second;
    return LAM_OK;
  }
  // bounded cache (keys hold destination addresses, which callers may reallocate): evict the least
  // recently used plan no streaming pull is using, once its last launch has completed
  if (c->plans.size() >= kMaxPlans) {
    auto victim = c->plans.end();
    for (auto jt = c->plans.begin(); jt != c->plans.end(); ++jt) {
      bool busy = false;
      for (const auto& sp : c->streams) busy |= sp.active && sp.plan == &jt->second;
      if (!busy && (victim == c->plans.end() || jt->second.last_use < victim->second.last_use)) victim = jt;
    }
    if (victim != c->plans.end()) {
      PullPlan& v = victim->second;
      CK(cudaSetDevice(v.device));
      if (v.last_ev) {
        CK(cudaEventSynchronize(v.last_ev));
        cudaEventDestroy(v.last_ev);
      }
      dev_free(c, v.device, v.d_tiles);
      c->plans.erase(victim);
      CK(cudaSetDevice(ro.device));
    }
  }
  std::vector<CopyTile> tiles;
  uint64_t bytes = 0;
  std::string err;
  if (!build_copy_tiles(c->plan, c->ts, L, &tiles, &bytes, &err)) {
    fprintf(stderr, "liblam: lam_pull: %s\n", err.c_str());
    return LAM_EINVAL;
  }
  // start with the rank region stored on the rollout's own GPU (colocated FSDP shards): pullers then
  // walk the source GPUs as a permutation at every step instead of queueing on the same peer
  int rot = pull_rotation(c->plan, L);
  for (int r = 0; r < c->cfg.fsdp_size; ++r)
    if (c->parts[c->node_rank_part[ro.node][r]].device == ro.device) { rot = r; break; }
  tiles = split_by_chunk(c->plan, tiles, rot);
  PullPlan pp;
  pp.n_tiles = (uint32_t)tiles.size();
  pp.bytes = bytes;
  for (uint32_t i = 0; i < tiles.size(); ++i) {
    const uint32_t g = chunk_of(c->plan, tiles[i]);
    if (pp.chunk_ids.empty() || pp.chunk_ids.back() != g) {
      pp.chunk_ids.push_back(g);
      pp.chunk_begin.push_back(i);
    }
  }
  pp.chunk_begin.push_back((uint32_t)tiles.size());
  for (const CopyTile& t : tiles) {
    pp.kinds |= t.transposed() ? kPullKMajor : kPullRowMajor;
    if (t.zero()) continue;   // padding rows: written, nothing read
    const Part& q = c->parts[c->node_rank_part[ro.node][t.src_rank]];
    // local = this GPU's HBM; remote = a peer's HBM over NVLink, or the host tier over PCIe
    (q.device == ro.device && !q.host ? pp.local_bytes : pp.remote_bytes) += (uint64_t)t.rows * t.row_bytes;
  }
  CK(dev_alloc(c, ro.device, (void**)&pp.d_tiles, sizeof(CopyTile) * std::max<size_t>(tiles.size(), 1)));
  if (!tiles.empty()) CK(dev_upload(c, ro.device, pp.d_tiles, tiles.data(), sizeof(CopyTile) * tiles.size()));
  CK(cudaEventCreateWithFlags(&pp.last_ev, cudaEventDisableTiming));
  pp.device = ro.device;
  pp.last_use = ++c->plan_clock;
  *out = &c->plans.emplace(key, pp).first->second;
  c->shm->stats.plan_cache_misses++;
  return LAM_OK;
}

std::string layout_key(int node, const lam_tp_layout& L) {
  std::string k = std::to_string(node) + ":" + std::to_string(L.tp_size) + ":" + std::to_string(L.tp_rank);
  for (int i = 0; i < L.n_dsts; ++i) {
    const lam_dst& d = L.dsts[i];
    char b[96];
    snprintf(b, sizeof b, "|%p,%lld,%d", d.dst, (long long)d.dst_row_pitch_bytes, d.transpose);
    k += b;
    for (int j = 0; j < d.n_parts; ++j) k += "," + std::to_string(d.parts[j].tensor_id) + "/" + std::to_string(d.parts[j].rule);
  }
  return k;
}

}  // namespace

// ===================================================================================== C ABI
extern "C" size_t lam_config_size(void) { return sizeof(lam_config); }

extern "C" const char* lam_strerror(lam_status s) {
  switch (s) {
    case LAM_OK: return "ok";
    case LAM_ENOVERSION: return "no complete version yet";
    case LAM_IDLE: return "idle";
    case LAM_EINVAL: return "invalid argument";
    case LAM_ESTALE: return "version not newer than the last published";
    case LAM_ECUDA: return "CUDA error";
    case LAM_ECHECKSUM: return "chunk checksum mismatch (version not committed)";
    case LAM_ENOMEM: return "out of memory";
    case LAM_ESHUTDOWN: return "shutting down";
    case LAM_EBUSY: return "publish slots busy";
    case LAM_ETIMEOUT: return "chain hop timed out waiting for its predecessor";
    case LAM_EIPC: return "shared memory / IPC setup failed";
    default: return "unknown status";
  }
}

extern "C" lam_status lam_init(const lam_config* cfg, lam_ctx** out) {
  if (!cfg || !out) return LAM_EINVAL;
  *out = nullptr;
  std::string why;
  lam_status st = validate(*cfg, &why);
  if (st != LAM_OK) {
    fprintf(stderr, "liblam: invalid config: %s\n", why.c_str());
    return st;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    fprintf(stderr, "liblam: no CUDA device (this library has no CPU fallback)\n");
    return LAM_ECUDA;
  }
  auto c = std::make_unique<lam_ctx>();
  c->cfg = *cfg;
  c->S = cfg->slots;
  c->n_nodes = cfg->n_relays + 1;
  c->ts = model_tensors(cfg->model);
  for (auto& t : c->ts) c->params += t.numel();
  uint64_t C = cfg->chunk_bytes;
  if (C == 0) {
    double tb = cfg->t_byte_s > 0 ? cfg->t_byte_s : 1.0 / 750e9;
    // T_start calibrated on B200: per-chunk flag propagation + pipeline refill.  k_hop v3 (bench
    // --chunk-mb sweep at N=4: 64 MB 38.0 ms, 138 MB 34.2 ms, 256 MB 33.1 ms) implied ~20 us; with the
    // flusher warp (v5) 128 MB beats 256 MB at N=4 (25.5 vs 25.9 ms): ~10 us
    double tsu = cfg->t_start_s > 0 ? cfg->t_start_s : 10e-6;
    // the pack is one more pipeline stage ahead of the chain (reading R12); the star
    // (multicast pack, then each relay's verify) and the two-level tree (node 0 -> owner -> peer) have
    // fixed depths of 3 and 4 nodes whatever the relay count
    const int depth = cfg->hop_mode == LAM_HOP_MULTICAST ? 3 : cfg->hop_mode == LAM_HOP_TREE ? 4 : c->n_nodes + 1;
    int64_t k = lam_optimal_chunks(depth, 2.0 * (double)c->params, tb, tsu, 1024);
    C = align_up(cdiv(2 * c->params, (uint64_t)k), kChunkAlign);
    // practical cap: the chunk is also the checksum / completion-signal unit
    C = std::min<uint64_t>(C, 128ull << 20);
  }
  if (!build_image_plan(c->ts, cfg->fsdp_size, cfg->actor_layout, C, &c->plan)) return LAM_EINVAL;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  c->pack_ctas = cfg->pack_ctas > 0 ? cfg->pack_ctas : 0;  // 0: one resident wave (occupancy API)
  c->pack_sms = cfg->pack_sms > 0 && cfg->pack_sms < sms ? cfg->pack_sms : 0;
  c->hop_ctas = cfg->hop_ctas > 0 ? cfg->hop_ctas : 32;  // TMA hop: ~785 GB/s at 32 CTAs
  c->pull_ctas = cfg->pull_ctas > 0 ? cfg->pull_ctas : 0;
  if (cfg->spin_timeout_s > 0) c->timeout_ns = (uint64_t)(cfg->spin_timeout_s * 1e9);
  c->pubs.resize(cfg->fsdp_size);
  if (cfg->hop_mode == LAM_HOP_MULTICAST) {
    c->star = true;
    c->mcast = true;
    std::set<int> team{cfg->actor_device[0]};
    for (int i = 0; i < cfg->n_relays; ++i)
      for (int r = 0; r < cfg->fsdp_size; ++r) team.insert(cfg->relay[i].part_device[r]);
    c->mc.devices.assign(team.begin(), team.end());
    c->mc.owner_dev = cfg->actor_device[0];
    for (int d : c->mc.devices)
      if (owns(c.get(), d) && !mc_supported(d, &why)) {
        fprintf(stderr, "liblam: LAM_HOP_MULTICAST: %s\n", why.c_str());
        return LAM_EINVAL;
      }
  }
  st = setup_shm(c.get());
  if (st != LAM_OK) return st;
  c->tree = cfg->hop_mode == LAM_HOP_TREE;
  if (cfg->n_procs == 1 || cfg->proc_rank == 0) ctl::init(c->shm, c->n_nodes, c->star, c->tree);
  c->streams.resize(cfg->n_rollouts);
  // map the control block for the producer kernels' chunk-flag mirror (streaming pulls)
  for (int d = 0; d < LAM_MAX_DEVICES; ++d)
    if (owns(c.get(), d)) {
      cudaSetDevice(d);
      break;
    }
  if (c->plan.total_chunks <= kShmMirrorChunks &&
      cudaHostRegister(c->shm, sizeof(Shm), cudaHostRegisterMapped | cudaHostRegisterPortable) == cudaSuccess) {
    c->shm_registered = true;
    void* dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, c->shm, 0) == cudaSuccess)
      c->mirror_dev = reinterpret_cast<Shm*>(dp)->chunk_done[0][0];
  }
  cudaGetLastError();
  st = alloc_parts(c.get());
  if (st != LAM_OK) {
    lam_destroy(c.release());
    return st;
  }
  for (int r = 0; r < cfg->fsdp_size; ++r) {
    if (!owns(c.get(), cfg->actor_device[r])) continue;
    cudaSetDevice(cfg->actor_device[r]);
    for (int s = 0; s < c->S; ++s) cudaEventCreateWithFlags(&c->pubs[r].ev[s], cudaEventDisableTiming);
  }
  if (cfg->n_procs == 1) {
    st = mc_connect(c.get());
    if (st == LAM_OK) st = connect_links(c.get());
    if (st != LAM_OK) {
      lam_destroy(c.release());
      return st;
    }
  }
  *out = c.release();
  return LAM_OK;
}

struct IpcEntry {
  int32_t part, device;
  cudaIpcMemHandle_t h;          // HBM part: the whole allocation; host part: the metadata block
  int32_t host, pid, fd, mc;     // host part: memfd of the slot data, reopened via /proc/<pid>/fd/<fd>;
                                 // mc: node 0 of LAM_HOP_MULTICAST (metadata block only, data = own member)
  uint64_t host_bytes;
};

extern "C" lam_status lam_export_ipc(lam_ctx* c, void* buf, size_t cap, size_t* len) {
  if (!c || !len) return LAM_EINVAL;
  std::vector<IpcEntry> v;
  for (Part& p : c->parts)
    if (p.local) {
      IpcEntry e{p.index, p.device, {}, p.host ? 1 : 0, (int32_t)getpid(), p.host_fd, p.mc ? 1 : 0, p.host_bytes};
      cudaSetDevice(p.device);
      CK(cudaIpcGetMemHandle(&e.h, (p.host || p.mc) ? p.meta : p.base));
      v.push_back(e);
    }
  size_t need = sizeof(int32_t) + v.size() * sizeof(IpcEntry);
  *len = need;
  if (!buf || cap < need) return buf ? LAM_EINVAL : LAM_OK;
  int32_t n = (int32_t)v.size();
  memcpy(buf, &n, sizeof n);
  if (!v.empty()) memcpy((char*)buf + sizeof n, v.data(), v.size() * sizeof(IpcEntry));
  return LAM_OK;
}

extern "C" lam_status lam_import_ipc(lam_ctx* c, int32_t proc, const void* buf, size_t len) {
  if (!c || !buf || len < sizeof(int32_t)) return LAM_EINVAL;
  if (proc == c->cfg.proc_rank) return LAM_OK;
  int32_t n = 0;
  memcpy(&n, buf, sizeof n);
  if (len < sizeof n + (size_t)n * sizeof(IpcEntry)) return LAM_EINVAL;
  int my_dev = -1;
  for (int d = 0; d < LAM_MAX_DEVICES; ++d)
    if (owns(c, d)) { my_dev = d; break; }
  if (my_dev < 0) return LAM_OK;  // this process owns no GPU work
  CK(cudaSetDevice(my_dev));
  for (int i = 0; i < n; ++i) {
    IpcEntry e;
    memcpy(&e, (const char*)buf + sizeof n + (size_t)i * sizeof(IpcEntry), sizeof e);
    if (e.part < 0 || e.part >= (int)c->parts.size()) return LAM_EINVAL;
    Part& p = c->parts[e.part];
    if (p.local || p.meta) continue;
    void* ptr = nullptr;
    cudaError_t err = cudaIpcOpenMemHandle(&ptr, e.h, cudaIpcMemLazyEnablePeerAccess);
    if (err != cudaSuccess) {
      fprintf(stderr, "liblam: cudaIpcOpenMemHandle(part %d, dev %d): %s\n", e.part, e.device, cudaGetErrorString(err));
      return LAM_EIPC;
    }
    p.ipc_opened = true;
    if (e.mc) {
      p.mc = true;
      p.meta = (uint8_t*)ptr;
      p.data = nullptr;   // set by lam_connect: the actor GPU's member, imported with the multicast object
    } else if (e.host) {
      p.meta = (uint8_t*)ptr;
      char path[64];
      snprintf(path, sizeof path, "/proc/%d/fd/%d", e.pid, e.fd);
      int fd = open(path, O_RDWR);
      if (fd < 0) {
        fprintf(stderr, "liblam: open(%s) for the host relay part failed: %s\n", path, strerror(errno));
        return LAM_EIPC;
      }
      lam_status hs = map_host_part(p, fd, e.host_bytes);
      if (hs != LAM_OK) return hs;
    } else {
      p.base = (uint8_t*)ptr;
      p.data = p.base;
      p.meta = p.base + p.meta_base;
    }
  }
  return LAM_OK;
}

extern "C" lam_status lam_connect(lam_ctx* c) {
  if (!c) return LAM_EINVAL;
  if (c->connected) return LAM_OK;
  lam_status st = mc_connect(c);   // before the lock: binding waits for the other processes
  if (st != LAM_OK) return st;
  Lock l(c->shm);
  return connect_links(c);
}

static lam_status publish_impl(lam_ctx* c, uint64_t v, int32_t rank, const lam_shard* shards, int32_t n,
                               void* actor_stream, void* reads_done);

extern "C" lam_status lam_publish(lam_ctx* c, uint64_t v, int32_t rank, const lam_shard* shards, int32_t n,
                                  void* actor_stream, void* reads_done) {
  const uint64_t t0 = steady_ns();
  const lam_status st = publish_impl(c, v, rank, shards, n, actor_stream, reads_done);
  if (st == LAM_OK) {
    const uint64_t dt = steady_ns() - t0;
    Lock l(c->shm);
    c->shm->stats.publish_ns_total += dt;
    if (dt > c->shm->stats.publish_ns_max) c->shm->stats.publish_ns_max = dt;
  }
  return st;
}

static lam_status publish_impl(lam_ctx* c, uint64_t v, int32_t rank, const lam_shard* shards, int32_t n,
                               void* actor_stream, void* reads_done) {
  if (!c || !c->connected || rank < 0 || rank >= c->cfg.fsdp_size || n < 0 || (n && !shards) || v == 0)
    return LAM_EINVAL;
  if (!owns(c, c->cfg.actor_device[rank])) return LAM_EINVAL;
  const int dev = c->cfg.actor_device[rank];
  RankPub& rp = c->pubs[rank];
  Part& p = c->parts[c->node_rank_part[0][rank]];
  CK(cudaSetDevice(dev));
  // (re)build the pack units when the shard list changed (outside the lock: host-only work)
  std::vector<lam_shard> key(shards, shards + n);
  bool same = key.size() == rp.key.size() &&
              (key.empty() || memcmp(key.data(), rp.key.data(), sizeof(lam_shard) * key.size()) == 0);
  if (!same) {
    std::vector<PackUnit> units;
    std::vector<uint32_t> upc;
    std::string err;
    if (!build_pack_units(c->plan, c->ts, rank, key, (uint64_t)p.rank_off[rank], &units, &upc, &err)) {
      fprintf(stderr, "liblam: lam_publish: %s\n", err.c_str());
      return LAM_EINVAL;
    }
    CK(cudaStreamSynchronize(c->dev[dev].side));  // tables may be in use by an earlier pack
    if (units.size() > rp.cap_units) {
      if (rp.d_units) cudaFree(rp.d_units);
      CK(cudaMalloc(&rp.d_units, sizeof(PackUnit) * units.size()));
      rp.cap_units = (uint32_t)units.size();
    }
    if (!units.empty()) CK(cudaMemcpy(rp.d_units, units.data(), sizeof(PackUnit) * units.size(), cudaMemcpyHostToDevice));
    rp.n_units = (uint32_t)units.size();
    if (!rp.d_units_per_chunk) CK(cudaMalloc(&rp.d_units_per_chunk, 4 * std::max<uint64_t>(c->plan.total_chunks, 1)));
    if (c->plan.total_chunks) CK(cudaMemcpy(rp.d_units_per_chunk, upc.data(), 4 * c->plan.total_chunks, cudaMemcpyHostToDevice));
    if ((uint32_t)n > rp.cap_ptrs) {
      if (rp.d_ptrs) cudaFree(rp.d_ptrs);
      CK(cudaMalloc((void**)&rp.d_ptrs, sizeof(float*) * std::max(n, 1)));
      rp.cap_ptrs = (uint32_t)std::max(n, 1);
    }
    std::vector<const float*> ptrs(n);
    for (int i = 0; i < n; ++i) ptrs[i] = shards[i].ptr;
    if (n) CK(cudaMemcpy((void*)rp.d_ptrs, ptrs.data(), sizeof(float*) * n, cudaMemcpyHostToDevice));
    rp.key = key;
    rp.h_units = units;
    rp.units_gen++;
  }
  Lock l(c->shm);
  Shm* sh = c->shm;
  int s = -1;
  lam_status pst = ctl::publish(sh, c->S, c->cfg.fsdp_size, v, rank, &s);
  if (pst != LAM_OK) return pst;
  // enqueue: side stream waits for the work already on the actor stream, then packs
  cudaStream_t side = c->dev[dev].side;
  cudaEvent_t fork = get_event(c, dev);
  CK(cudaEventRecord(fork, (cudaStream_t)actor_stream));
  CK(cudaStreamWaitEvent(side, fork, 0));
  c->ev_pool[dev].push_back(fork);  // reuse is safe: a later record only affects later waits
  ChunkMeta m = meta_of(c, p, s);
  const uint64_t g0 = c->plan.chunk_base[rank], ng = c->plan.n_chunks[rank];
  if (ng) {
    CK(cudaMemsetAsync(m.hdr + g0, 0, sizeof(lam_chunk_header) * ng, side));
    CK(cudaMemsetAsync(m.cnt + g0, 0, 4 * ng, side));
  }
  cudaEvent_t t0 = prof_begin(c, dev, side);
  uint8_t* const* sub = nullptr;
  const int sub_rid = rp.sub_rid;
  if (sub_rid >= 0) {  // colocated subscriber: per-unit destinations (rebuilt only when units change)
    if (rp.sub_gen != rp.units_gen) {
      std::vector<uint8_t*> tab(rp.n_units);
      for (uint32_t i = 0; i < rp.n_units; ++i) {
        const PackUnit& u = rp.h_units[i];
        const lam_shard& sh = rp.key[u.shard];
        tab[i] = (uint8_t*)(uintptr_t)(rp.sub_tensor_dst[sh.tensor_id] + 2 * (sh.elem_offset + u.src_elem));
        if ((uintptr_t)tab[i] % 2) {  // k_pack narrows its stores to whatever alignment remains
          fprintf(stderr, "liblam: lam_subscribe: destination not 2-B aligned\n");
          return LAM_EINVAL;
        }
      }
      if (rp.n_units > rp.cap_sub) {
        if (rp.d_sub) cudaFree(rp.d_sub);
        CK(cudaMalloc(&rp.d_sub, sizeof(uint8_t*) * std::max<uint32_t>(rp.n_units, 1)));
        rp.cap_sub = rp.n_units;
      }
      CK(cudaStreamSynchronize(side));
      if (rp.n_units) CK(cudaMemcpy(rp.d_sub, tab.data(), sizeof(uint8_t*) * rp.n_units, cudaMemcpyHostToDevice));
      rp.sub_gen = rp.units_gen;
    }
    sub = rp.d_sub;
  }
  uint8_t* dst = slot_data(p, s);
  uint8_t* mc_dst = nullptr;
  if (p.mc) {   // NEXT-2: store through the multicast VA (the switch replicates into every relay GPU)
    if (!c->mc.mc_va) return LAM_ECUDA;
    mc_dst = c->mc.mc_va + (uint64_t)s * p.slot_stride;
    m.mc_flags = reinterpret_cast<uint64_t*>(c->mc.mc_va + c->mc.flags_off + (uint64_t)s * c->mc.flag_stride);
  }
  int rc = launch_pack(rp.d_units, rp.n_units, rp.d_ptrs, dst, mc_dst, m, rp.d_units_per_chunk, v,
                       c->plan.total_chunks, c->dev[dev].d_chunk_len, c->pack_ctas, side, sub,
                       c->dev[dev].d_pack_work, c->pack_sms);
  if (rc) {
    fprintf(stderr, "liblam: pack launch failed: %s\n", cudaGetErrorString((cudaError_t)rc));
    return LAM_ECUDA;
  }
  if (rp.n_units) c->shm->stats.kernel_launches++;
  prof_end(c, 0, dev, side, t0);
  if (reads_done) CK(cudaEventRecord((cudaEvent_t)reads_done, side));
  CK(cudaEventRecord(rp.ev[s], side));
  rp.inflight_version[s] = v;
  if (sub_rid >= 0) {  // one-shot: complete the subscription once every local rank packed v
    rp.sub_rid = -1;
    lam_ctx::StreamPull& sp = c->streams[sub_rid];
    bool all = true;
    for (int r = 0; r < c->cfg.fsdp_size; ++r)
      if (c->cfg.actor_device[r] == dev && c->pubs[r].sub_rid == sub_rid) all = false;
    if (all) {
      if (sp.done) CK(cudaEventRecord(sp.done, side));
      sp.active = false;
      sp.subscription = false;
      sp.v = v;
      sp.status = LAM_OK;
      c->shm->stats.pulls++;
    }
  }
  return LAM_OK;
}

extern "C" lam_status lam_subscribe(lam_ctx* c, int32_t rid, const lam_tp_layout* L, void* done) {
  if (!c || !c->connected || !L || rid < 0 || rid >= c->cfg.n_rollouts) return LAM_EINVAL;
  const lam_rollout_desc ro = c->cfg.rollout[rid];
  if (ro.node != 0 || !owns(c, ro.device) || L->tp_size != 1) return LAM_EINVAL;
  // the layout must put every tensor, whole and dense, somewhere in the rollout's buffers
  std::vector<uint64_t> tdst(c->ts.size(), 0);
  for (int k = 0; k < L->n_dsts; ++k) {
    const lam_dst& d = L->dsts[k];
    if (d.transpose || !d.dst) return LAM_EINVAL;
    uint64_t off = 0;
    for (int q = 0; q < d.n_parts; ++q) {
      const uint32_t t = d.parts[q].tensor_id;
      if (t >= c->ts.size() || tdst[t]) return LAM_EINVAL;
      // vocabulary padding rows would have to be zero-filled: not a plain image of the tensor
      if (d.parts[q].rule == LAM_VOCAB_DIM0 && c->ts[t].d0 % kVocabPad) return LAM_EINVAL;
      if (d.dst_row_pitch_bytes && (uint64_t)d.dst_row_pitch_bytes != 2 * (uint64_t)c->ts[t].d1) return LAM_EINVAL;
      tdst[t] = (uint64_t)(uintptr_t)d.dst + off;
      off += 2 * c->ts[t].numel();
    }
  }
  for (uint64_t a : tdst)
    if (!a) return LAM_EINVAL;
  // the pack writes only the shards packed on the rollout's own GPU: every actor rank must be there,
  // otherwise the rollout would see a partial version (pull the others with lam_pull instead)
  for (int r = 0; r < c->cfg.fsdp_size; ++r)
    if (c->cfg.actor_device[r] != ro.device) return LAM_EINVAL;
  Lock l(c->shm);
  lam_ctx::StreamPull& sp = c->streams[rid];
  if (sp.active) return LAM_EBUSY;
  bool any = false;
  for (int r = 0; r < c->cfg.fsdp_size; ++r) {
    RankPub& rp = c->pubs[r];
    if (rp.sub_tensor_dst != tdst) {
      rp.sub_tensor_dst = tdst;
      rp.sub_gen = ~0ull;
    }
    rp.sub_rid = rid;
    any = true;
  }
  if (!any) return LAM_EINVAL;
  sp.active = true;      // until the pack of the next version is enqueued
  sp.subscription = true;
  sp.node = 0;
  sp.device = ro.device;
  sp.v = 0;
  sp.status = LAM_OK;
  sp.plan = nullptr;
  sp.done = (cudaEvent_t)done;
  return LAM_OK;
}

extern "C" lam_status lam_relay_step(lam_ctx* c, int32_t* n_transitions) {
  if (!c || !c->connected) return LAM_EINVAL;
  Lock l(c->shm);
  int t = 0;
  bool busy = false;
  lam_status st = step_locked(c, &t, &busy);
  if (n_transitions) *n_transitions = t;
  if (st != LAM_OK) return st;
  return busy ? LAM_OK : LAM_IDLE;
}

extern "C" lam_status lam_pull(lam_ctx* c, int32_t rid, const lam_tp_layout* L, void* stream, uint64_t* vout) {
  if (vout) *vout = 0;
  if (!c || !c->connected || !L || rid < 0 || rid >= c->cfg.n_rollouts) return LAM_EINVAL;
  const lam_rollout_desc ro = c->cfg.rollout[rid];
  if (!owns(c, ro.device)) return LAM_EINVAL;
  CK(cudaSetDevice(ro.device));
  std::string key = layout_key(ro.node, *L);
  Lock l(c->shm);
  PullPlan* pp = nullptr;
  lam_status pst = get_plan(c, ro, *L, key, &pp);
  if (pst != LAM_OK) return pst;
  int s = -1;
  const uint64_t u = ctl::pin_latest(c->shm, c->S, ro.node, &s);
  if (u == 0) return LAM_ENOVERSION;
  auto rb = c->d_rank_base.find({ro.node * LAM_MAX_SLOTS + s, ro.device});
  if (rb == c->d_rank_base.end()) {
    ctl::unpin(c->shm, ro.node, s);
    return LAM_EINVAL;
  }
  cudaEvent_t t0 = prof_begin(c, ro.device, (cudaStream_t)stream);
  cudaEvent_t wev = nullptr;
  uint32_t* work = pull_counter(c, ro.device, &wev);
  int rc = work ? launch_pull(pp->d_tiles, pp->n_tiles, rb->second, c->pull_ctas, stream, pp->kinds, work)
                : (int)cudaErrorMemoryAllocation;
  if (rc) {
    ctl::unpin(c->shm, ro.node, s);
    fprintf(stderr, "liblam: pull launch failed: %s\n", cudaGetErrorString((cudaError_t)rc));
    return LAM_ECUDA;
  }
  CK(cudaEventRecord(wev, (cudaStream_t)stream));
  CK(cudaEventRecord(pp->last_ev, (cudaStream_t)stream));
  if (pp->n_tiles) c->shm->stats.kernel_launches += __builtin_popcount(pp->kinds);
  prof_end(c, 2, ro.device, (cudaStream_t)stream, t0);
  cudaEvent_t ev = get_event(c, ro.device);
  CK(cudaEventRecord(ev, (cudaStream_t)stream));
  c->pending.push_back({ev, ro.node, s, ro.device});
  c->shm->stats.pulls++;
  if (vout) *vout = u;
  return LAM_OK;
}

extern "C" lam_status lam_pull_stream(lam_ctx* c, int32_t rid, const lam_tp_layout* L, void* stream, void* done,
                                      uint64_t min_version, uint64_t* vout) {
  if (vout) *vout = 0;
  if (!c || !c->connected || !L || rid < 0 || rid >= c->cfg.n_rollouts) return LAM_EINVAL;
  const lam_rollout_desc ro = c->cfg.rollout[rid];
  if (!owns(c, ro.device)) return LAM_EINVAL;
  CK(cudaSetDevice(ro.device));
  std::string key = layout_key(ro.node, *L);
  Lock l(c->shm);
  lam_ctx::StreamPull& sp = c->streams[rid];
  if (sp.active) return LAM_EBUSY;
  ShmNode& n = c->shm->node[ro.node];
  if (n.dead) return LAM_ENOVERSION;
  if (n.latest && n.latest >= min_version) {         // already complete: an ordinary pull
    lam_status st = lam_pull(c, rid, L, stream, vout);
    if (st == LAM_OK && done) CK(cudaEventRecord((cudaEvent_t)done, (cudaStream_t)stream));
    sp.v = vout ? *vout : 0;
    sp.status = LAM_OK;
    return st;
  }
  int s = -1;
  for (int i = 0; i < c->S; ++i)
    if (n.slot[i].state == S_FILLING && n.slot[i].version >= min_version) s = i;
  if (s < 0 || !c->mirror_dev || !c->d_rank_base.count({ro.node * LAM_MAX_SLOTS + s, ro.device}))
    return LAM_ENOVERSION;
  PullPlan* pp = nullptr;
  lam_status pst = get_plan(c, ro, *L, key, &pp);
  if (pst != LAM_OK) return pst;
  n.slot[s].readers++;                                 // pin the version being received
  sp.active = true;
  sp.subscription = false;
  sp.node = ro.node;
  sp.slot = s;
  sp.device = ro.device;
  sp.v = n.slot[s].version;
  sp.status = LAM_OK;
  sp.plan = pp;
  sp.next = 0;
  sp.stream = (cudaStream_t)stream;
  sp.done = (cudaEvent_t)done;
  c->shm->stats.pulls++;
  if (vout) *vout = sp.v;
  int t = 0;
  return stream_progress(c, rid, &t);
}

extern "C" lam_status lam_pull_state(lam_ctx* c, int32_t rid, uint64_t* vout, int32_t* state) {
  if (!c || rid < 0 || rid >= c->cfg.n_rollouts || !state) return LAM_EINVAL;
  Lock l(c->shm);
  const lam_ctx::StreamPull& sp = c->streams[rid];
  if (vout) *vout = sp.v;
  *state = sp.active ? 1 : (sp.status < 0 ? sp.status : 0);
  return LAM_OK;
}

extern "C" lam_status lam_fail_node(lam_ctx* c, int32_t node) {
  if (!c || !c->connected || node <= 0 || node >= c->n_nodes) return LAM_EINVAL;
  Lock l(c->shm);
  return fail_node_locked(c, node);
}

extern "C" lam_status lam_latest(lam_ctx* c, int32_t node, uint64_t* vout) {
  if (!c || !vout || node < 0 || node >= c->n_nodes) return LAM_EINVAL;
  Lock l(c->shm);
  *vout = c->shm->node[node].latest;
  return *vout ? LAM_OK : LAM_ENOVERSION;
}

extern "C" lam_status lam_get_plan_info(lam_ctx* c, lam_plan_info* o) {
  if (!c || !o) return LAM_EINVAL;
  o->image_bytes = c->plan.C * c->plan.total_chunks;
  o->chunk_bytes = c->plan.C;
  o->total_chunks = c->plan.total_chunks;
  o->snapshot_bytes = 2 * c->params;
  o->params = c->params;
  o->n_tensors = (int32_t)c->ts.size();
  o->n_nodes = c->n_nodes;
  return LAM_OK;
}

extern "C" lam_status lam_get_stats(lam_ctx* c, lam_stats* o) {
  if (!c || !o) return LAM_EINVAL;
  Lock l(c->shm);
  *o = c->shm->stats;
  return LAM_OK;
}

static lam_status locate(lam_ctx* c, int node, uint64_t v, int* slot) {
  if (!c || node < 0 || node >= c->n_nodes) return LAM_EINVAL;
  *slot = find_slot(c->shm->node[node], c->S, v, S_COMPLETE);
  return *slot < 0 ? LAM_ENOVERSION : LAM_OK;
}

extern "C" lam_status lam_read_image(lam_ctx* c, int32_t node, uint64_t v, uint64_t off, uint64_t nbytes, void* host) {
  if (!c || !host) return LAM_EINVAL;
  Lock l(c->shm);
  int s;
  lam_status st = locate(c, node, v, &s);
  if (st != LAM_OK) return st;
  const uint64_t C = c->plan.C, end = off + nbytes;
  if (end > C * c->plan.total_chunks) return LAM_EINVAL;
  uint8_t* h = (uint8_t*)host;
  while (off < end) {
    uint64_t g = off / C;
    int r = (int)c->plan.chunk_rank[g];
    uint64_t rend = (c->plan.chunk_base[r] + c->plan.n_chunks[r]) * C;
    uint64_t n = std::min(end, rend) - off;
    const Part& p = c->parts[c->node_rank_part[node][r]];
    const uint8_t* src = slot_data(p, s) + p.rank_off[r] + (off - c->plan.chunk_base[r] * C);
    // own parts: copy from their device (a multicast member is mapped for its own GPU only)
    if (p.local) CK(cudaSetDevice(p.device));
    CK(cudaMemcpy(h, src, n, cudaMemcpyDefault));
    h += n;
    off += n;
  }
  return LAM_OK;
}

extern "C" lam_status lam_read_headers(lam_ctx* c, int32_t node, uint64_t v, lam_chunk_header* host,
                                       uint64_t first, uint64_t count) {
  if (!c || !host) return LAM_EINVAL;
  Lock l(c->shm);
  int s;
  lam_status st = locate(c, node, v, &s);
  if (st != LAM_OK) return st;
  if (first + count > c->plan.total_chunks) return LAM_EINVAL;
  for (uint64_t g = first; g < first + count; ++g) {
    const Part& p = c->parts[c->node_rank_part[node][c->plan.chunk_rank[g]]];
    ChunkMeta m = meta_of(c, p, s);
    CK(cudaMemcpy(host + (g - first), m.hdr + g, sizeof(lam_chunk_header), cudaMemcpyDefault));
  }
  return LAM_OK;
}

extern "C" lam_status lam_pull_bytes(lam_ctx* c, int32_t rid, const lam_tp_layout* L, uint64_t* local,
                                     uint64_t* remote) {
  if (!c || !c->connected || !L || rid < 0 || rid >= c->cfg.n_rollouts || !local || !remote) return LAM_EINVAL;
  const lam_rollout_desc ro = c->cfg.rollout[rid];
  if (!owns(c, ro.device)) return LAM_EINVAL;
  CK(cudaSetDevice(ro.device));
  Lock l(c->shm);
  PullPlan* pp = nullptr;
  lam_status st = get_plan(c, ro, *L, layout_key(ro.node, *L), &pp);
  if (st != LAM_OK) return st;
  *local = pp->local_bytes;
  *remote = pp->remote_bytes;
  return LAM_OK;
}

extern "C" lam_status lam_set_pack_sms(lam_ctx* c, int32_t sms) {
  if (!c || sms < 0) return LAM_EINVAL;
  Lock l(c->shm);
  c->pack_sms = sms;
  return LAM_OK;
}

extern "C" lam_status lam_set_profiling(lam_ctx* c, int32_t on) {
  if (!c) return LAM_EINVAL;
  Lock l(c->shm);
  c->profiling = on != 0;
  return LAM_OK;
}

extern "C" lam_status lam_kernel_times(lam_ctx* c, double ms[3], uint64_t cnt[3]) {
  if (!c || !ms || !cnt) return LAM_EINVAL;
  Lock l(c->shm);
  for (int k = 0; k < 3; ++k) { ms[k] = 0; cnt[k] = 0; }
  std::vector<lam_ctx::Timed> keep;
  for (auto& t : c->timed) {
    if (cudaEventQuery(t.b) != cudaSuccess) { cudaGetLastError(); keep.push_back(t); continue; }
    float x = 0;
    CK(cudaEventElapsedTime(&x, t.a, t.b));
    ms[t.kind] += x;
    cnt[t.kind]++;
    c->tev_pool[t.dev].push_back(t.a);
    c->tev_pool[t.dev].push_back(t.b);
  }
  c->timed.swap(keep);
  return LAM_OK;
}

extern "C" lam_status lam_debug_region(lam_ctx* c, int32_t node, uint64_t v, int32_t rank, void** ptr) {
  if (!c || !ptr || node < 0 || node >= c->n_nodes || rank < 0 || rank >= c->cfg.fsdp_size) return LAM_EINVAL;
  Lock l(c->shm);
  const ShmNode& n = c->shm->node[node];
  int s = find_slot(n, c->S, v, S_COMPLETE);
  if (s < 0) s = find_slot(n, c->S, v, S_FILLING);
  if (s < 0) return LAM_ENOVERSION;
  const Part& p = c->parts[c->node_rank_part[node][rank]];
  if (!p.data) return LAM_EINVAL;
  *ptr = slot_data(p, s) + p.rank_off[rank];
  return LAM_OK;
}

extern "C" lam_status lam_debug_replica(lam_ctx* c, int32_t device, uint64_t v, int32_t rank, void** ptr) {
  if (!c || !ptr || rank < 0 || rank >= c->cfg.fsdp_size || !c->mcast) return LAM_EINVAL;
  Lock l(c->shm);
  auto it = c->mc.va.find(device);
  if (it == c->mc.va.end()) return LAM_EINVAL;
  const ShmNode& n = c->shm->node[0];
  int s = find_slot(n, c->S, v, S_COMPLETE);
  if (s < 0) s = find_slot(n, c->S, v, S_FILLING);
  if (s < 0) return LAM_ENOVERSION;
  const Part& p0 = c->parts[c->node_rank_part[0][rank]];
  *ptr = it->second + (uint64_t)s * p0.slot_stride + p0.rank_off[rank];
  return LAM_OK;
}

extern "C" void lam_destroy(lam_ctx* c) {
  if (!c) return;
  for (Part& p : c->parts) {
    if (p.local && p.meta) {
      cudaSetDevice(p.device);
      cudaDeviceSynchronize();
    }
  }
  for (auto& kv : c->dev) {
    cudaSetDevice(kv.first);
    cudaDeviceSynchronize();
    if (kv.second.d_chunk_len) cudaFree(kv.second.d_chunk_len);
    if (kv.second.d_pack_work) cudaFree(kv.second.d_pack_work);
    if (kv.second.side) cudaStreamDestroy(kv.second.side);
  }
  for (auto& kv : c->plans) {
    cudaSetDevice(kv.second.device);
    cudaFreeAsync(kv.second.d_tiles, util_stream(c, kv.second.device));
    if (kv.second.last_ev) cudaEventDestroy(kv.second.last_ev);
  }
  for (auto& kv : c->pull_work) {
    cudaSetDevice(kv.first);
    if (kv.second.d) cudaFreeAsync(kv.second.d, util_stream(c, kv.first));
    for (cudaEvent_t e : kv.second.ev)
      if (e) cudaEventDestroy(e);
  }
  for (auto& kv : c->d_rank_base) {
    cudaSetDevice(kv.first.second);
    cudaFree((void*)kv.second);
  }
  for (RankPub& rp : c->pubs) {
    if (rp.d_units) cudaFree(rp.d_units);
    if (rp.d_units_per_chunk) cudaFree(rp.d_units_per_chunk);
    if (rp.d_ptrs) cudaFree((void*)rp.d_ptrs);
    if (rp.d_sub) cudaFree(rp.d_sub);
    for (int s = 0; s < LAM_MAX_SLOTS; ++s)
      if (rp.ev[s]) cudaEventDestroy(rp.ev[s]);
  }
  for (Part& p : c->parts) {
    if (p.host) {
      if (p.host_registered) cudaHostUnregister(p.base);
      if (p.base) munmap(p.base, p.host_bytes);
      if (p.host_fd >= 0) close(p.host_fd);
      if (p.ipc_opened) cudaIpcCloseMemHandle(p.meta);
      else if (p.local && p.meta) { cudaSetDevice(p.device); cudaFree(p.meta); }
      p.base = nullptr;
    } else if (p.mc) {
      if (p.ipc_opened) cudaIpcCloseMemHandle(p.meta);
      else if (p.local && p.meta) { cudaSetDevice(p.device); cudaFree(p.meta); }
    } else if (p.ipc_opened && p.base) {
      cudaIpcCloseMemHandle(p.base);
    }
    if (!p.local) continue;
    cudaSetDevice(p.device);
    if (p.d_tiles) cudaFree(p.d_tiles);
    if (p.d_tiles_per_chunk) cudaFree(p.d_tiles_per_chunk);
    if (p.d_links) cudaFree(p.d_links);
    if (p.d_tiles_tree) cudaFree(p.d_tiles_tree);
    if (p.d_links_tree) cudaFree(p.d_links_tree);
    if (p.d_my_chunks) cudaFree(p.d_my_chunks);
    for (cudaEvent_t e : p.chunk_ev) cudaEventDestroy(e);
    if (p.vstream) cudaStreamDestroy(p.vstream);
    if (p.base) cudaFree(p.base);
    if (p.err_host) cudaFreeHost(p.err_host);
    for (int s = 0; s < LAM_MAX_SLOTS; ++s)
      if (p.done_ev[s]) cudaEventDestroy(p.done_ev[s]);
    if (p.stream) cudaStreamDestroy(p.stream);
  }
  for (auto& pp : c->pending) cudaEventDestroy(pp.ev);
  for (auto& kv : c->ev_pool)
    for (cudaEvent_t e : kv.second) cudaEventDestroy(e);
  for (auto& kv : c->tev_pool)
    for (cudaEvent_t e : kv.second) cudaEventDestroy(e);
  for (auto& t : c->timed) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
  for (auto& kv : c->util) {
    cudaSetDevice(kv.first);
    cudaStreamSynchronize(kv.second);
    cudaStreamDestroy(kv.second);
  }
  mc_release(c->mc);
  if (c->shm_registered) cudaHostUnregister(c->shm);
  shm_release(c->shm, c->cfg.shm_name, c->shm_mapped, c->shm_owner);
  delete c;
}

/*
 * lam.h — C ABI of liblam.so: B200-native relay-tier weight synchronization
 * (arxiv 2510.12633, "Asynchronous Weight Synchronization Using Relay Workers", §4).
 *
 * The path (§3.2 steps 5-7; L652-670, §4.2):
 *   lam_publish     step 5  "the trainer pushes the new actor weights to the master relay and
 *                           immediately resumes its next training iteration" (L548): casts the
 *                           actor's fp32 master shard to bf16 (RNE) and packs it into the
 *                           version's chunked bucket image in the master node's ring slot.
 *   lam_relay_step  step 6  "the master relay then broadcasts the new weights directly to all
 *                           other relays" (L549) as "a chain-based pipelined broadcast" (L661-665):
 *                           non-blocking progress engine; launches chain-hop kernels that pull
 *                           chunk j from the predecessor over NVLink while it receives j+1.
 *   lam_pull        step 7  "A rollout can fetch the latest weights from its colocated relay at
 *                           any time" (L550), "without waiting for the resharding and broadcast to
 *                           complete" (L670); the reshard to the rollout's TP layout (L654) runs
 *                           here, at pull time, in one copy-plan-driven kernel.
 *
 * Conventions:
 *   - Versions are uint64, strictly increasing per publish, starting at 1; 0 means "none".
 *   - Ownership: the caller owns the fp32 shards (unmodified until `reads_done` fires) and the
 *     pull destination buffers (valid once `stream` reaches the enqueued work).  The library owns
 *     the relay rings, flags, headers and plans.
 *   - lam_publish never blocks on a relay: it enqueues and returns.  A pull never
 *     waits on a broadcast: it serves the newest COMPLETE version at call time.
 *   - Nothing is partially applied on error.  A corrupt chunk means the version is never marked
 *     complete at that relay, which keeps serving its previous version.
 *   - All calls are thread-safe (one mutex per context, process-shared across ranks).
 *   - No CPU fallback: every byte of the snapshot is moved by kernels in this library; calls
 *     return LAM_ECUDA when no CUDA device is usable.
 *   - Streams and events are passed as `void*` (cudaStream_t / cudaEvent_t) so this header does
 *     not depend on cuda_runtime.h.
 */
#ifndef LAM_H
#define LAM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lam_ctx lam_ctx;  /* opaque; owns relay rings, publish slots, flags, plans */
typedef int32_t lam_status;      /* 0 LAM_OK; >0 informational; <0 error */

enum {
  LAM_OK = 0,
  LAM_ENOVERSION = 1,   /* pull/latest: nothing complete yet (version_out = 0) */
  LAM_IDLE = 2,         /* relay_step: quiescent, nothing in flight */
  LAM_EINVAL = -1,      /* bad argument / configuration */
  LAM_ESTALE = -2,      /* publish: version <= last published */
  LAM_ECUDA = -3,       /* CUDA error (or no device) */
  LAM_ECHECKSUM = -4,   /* a relay received a corrupt chunk: version not committed there */
  LAM_ENOMEM = -5,      /* device or host allocation failed */
  LAM_ESHUTDOWN = -6,   /* context is being destroyed */
  LAM_EBUSY = -7,       /* publish: both master slots are in use (one is latest, the other is
                           still being read by the chain); nothing was enqueued, retry later */
  LAM_ETIMEOUT = -8,    /* a chain hop waited longer than spin_timeout_s for its predecessor */
  LAM_EIPC = -9         /* shared-memory / IPC setup between rank processes failed */
};

/* Actor partition layouts ("FSDP"). */
enum { LAM_FSDP2_DIM0 = 0, LAM_FSDP1_FLAT = 1 };

/* TP rules of a destination part (vLLM convention; "reshards them
 * according to the rollout sharding strategy", L1357 TP 1/4/8).  For rank r of tp, a part of source
 * tensor A (d0 x d1) contributes:
 *   LAM_REPLICATE   all of A
 *   LAM_SHARD_DIM0  rows [r*d0/tp, (r+1)*d0/tp)                     (d0 % tp == 0)
 *   LAM_SHARD_DIM1  columns [r*d1/tp, (r+1)*d1/tp) of every row      (2-D, d1 % tp == 0)
 *   LAM_VOCAB_DIM0  the vocabulary padded to Vp = 64*ceil(d0/64) rows; rank r owns padded rows
 *                   [r*Vp/tp, (r+1)*Vp/tp): its real rows, then zero rows for the padding (written
 *                   by the pull) — vLLM's VocabParallelEmbedding (R15)
 *   LAM_HEAD_DIM0   whole attention heads of head_dim rows (q/k/v weights and biases only; heads =
 *                   d0 / head_dim): tp <= heads: heads [r*heads/tp, (r+1)*heads/tp); tp > heads
 *                   (tp % heads == 0): head r / (tp/heads), i.e. KV heads replicated — vLLM's
 *                   QKVParallelLinear (R14) */
enum { LAM_REPLICATE = 0, LAM_SHARD_DIM0 = 1, LAM_SHARD_DIM1 = 2, LAM_VOCAB_DIM0 = 3, LAM_HEAD_DIM0 = 4 };

#define LAM_MAX_RANKS 64
#define LAM_MAX_NODES 32
#define LAM_MAX_ROLLOUTS 64
#define LAM_MAX_DEVICES 16
#define LAM_MAX_SLOTS 4

/* Qwen2-family model dimensions ("Qwen2.5").  Tensor table = HF state-dict order:
 * embed, per layer {q,q_b,k,k_b,v,v_b,o,gate,up,down,ln1,ln2}, final norm, lm_head (untied). */
typedef struct {
  int64_t hidden, intermediate, layers, heads, kv_heads, head_dim, vocab;
} lam_model_dims;

/* A relay node ("one relay per rollout machine"): for each actor rank r, the CUDA
 * device that stores rank r's region of the bucket image in this node.  All entries equal = the
 * node holds the full image on one GPU; different entries = range-sharded over several GPUs.
 * host_memory = 1 (the paper's own relay tier: "relay workers … store the
 * latest model weights in CPU memory"): the node's ring slots
 * live in pinned, device-mapped host memory (shared between rank processes through a memfd) instead
 * of HBM; part_device[r] is then the GPU whose SMs receive rank r's region into it over PCIe and
 * whose pulls read it from there.  Chunk headers, flags and counters stay in that GPU's HBM.  Zero
 * extra GPU memory; bandwidth is PCIe's.  Node 0 (the actor's slots) is always HBM. */
typedef struct {
  int32_t part_device[LAM_MAX_RANKS];
  int32_t host_memory;
} lam_node_desc;

/* A rollout: the node it pulls from (0 = the master/publish node) and the GPU its pull runs on. */
typedef struct {
  int32_t node;
  int32_t device;
} lam_rollout_desc;

typedef struct {
  lam_model_dims model;
  int32_t actor_layout;                    /* LAM_FSDP2_DIM0 | LAM_FSDP1_FLAT */
  int32_t fsdp_size;                       /* N actor ranks, 1..LAM_MAX_RANKS */
  int32_t actor_device[LAM_MAX_RANKS];     /* device of actor rank r (= node 0's part devices) */
  int32_t n_relays;                        /* relay nodes 1..n_relays, chain order 0->1->... */
  lam_node_desc relay[LAM_MAX_NODES];      /* relay[i-1] describes node i */
  int32_t slots;                           /* ring slots per node, 2..LAM_MAX_SLOTS */
  uint64_t chunk_bytes;                    /* C, multiple of 4096; 0 => Appendix D k* (below) with p =
                                              n_relays + 2 (chain + pack), 3 (multicast) or 4 (tree),
                                              capped at 128 MiB */
  double t_start_s, t_byte_s;              /* Appendix D parameters used when chunk_bytes == 0 */
  int32_t n_rollouts;
  lam_rollout_desc rollout[LAM_MAX_ROLLOUTS];
  /* processes: one per GPU (torchrun) or one for all (single-process mode: n_procs = 1) */
  int32_t proc_rank, n_procs;
  int32_t proc_of_device[LAM_MAX_DEVICES]; /* owning process of each device; -1 = unused */
  char shm_name[64];                       /* POSIX shm name for the control block (n_procs > 1) */
  /* tuning (0 => default) */
  int32_t pack_ctas, hop_ctas, pull_ctas;
  double spin_timeout_s;                   /* chain-hop wait limit (default 60 s) */
  int32_t hop_mode;                        /* LAM_HOP_KERNEL (default) | LAM_HOP_COPY_ENGINE */
  double heartbeat_timeout_s;              /* n_procs > 1: a process silent this long is declared
                                              failed and its relay nodes leave the chain (0 = off) */
  int32_t pack_sms;                        /* > 0: the pack runs on SMs 0..pack_sms-1 only (every SM
                                              fully occupied), leaving the others to the trainer's
                                              kernels (actor stall); 0 = all SMs */
} lam_config;

/* How a relay moves a chunk from its predecessor (all chunk-pipelined and verified):
 *  LAM_HOP_KERNEL       k_hop: TMA bulk copies through shared memory by ~32 SMs, checksum on the fly
 *  LAM_HOP_COPY_ENGINE  copy engines (zero SMs for the transfer): lam_relay_step enqueues a chunk's
 *                       cudaMemcpyAsync once the host mirror shows the predecessor's flag (without the
 *                       mapped control block: behind a stream wait on the flag), then k_verify
 *                       checksums it in local HBM and releases the flag.  Slower than LAM_HOP_KERNEL in
 *                       multi-process runs.
 *  LAM_HOP_MULTICAST    NVSwitch multicast broadcast (the bandwidth
 *                       term M·T_byte is the floor): no chain — every relay's predecessor is node 0.  The
 *                       pack stores the bf16 image once through a multicast object (multimem.st) bound
 *                       to node 0's slots on the actor GPU and to a replica of them on every relay GPU,
 *                       followed by each chunk's flag; each relay's k_hop then verifies and commits the
 *                       chunk from its local replica (HBM -> HBM).  The source GPU sends M once, relays
 *                       forward nothing.  Requires every actor rank on one GPU, HBM relay nodes, node-0
 *                       rollouts on that GPU, and multicast-capable devices (NVSwitch, >= 2 GPUs); costs
 *                       each relay GPU S extra image-sized replicas.  LAM_EINVAL otherwise.  A chunk that
 *                       fails verification from the replica is re-verified (twice) before the version
 *                       is given up: switch-stored bytes may land after the chunk's flag. */
/*  LAM_HOP_TREE         two-level broadcast over the same TMA hop kernel: relay k owns the j-th chunk of
 *                       the hop order with j mod R == k-1 (R relays; the hop order interleaves the FSDP
 *                       ranks' regions, see lam_plan_tree_tiles) and pulls it from node 0; every other chunk it pulls
 *                       from the relay that owns it, in an order staggered by k so the R-1 pullers of a
 *                       moment read from different owners; a peer's 1 MiB tile is read as soon as it
 *                       landed there (per-tile flags) and every chunk is verified against node 0's
 *                       header and verdict.  Every relay receives M and forwards
 *                       (R-1)/R of it, pipeline depth 2 (the chain: forwards M, depth R).  Control plane:
 *                       every relay's predecessor is node 0; the first relay to start v opens v at every
 *                       idle relay (gang start) and each fill pins the slot of v at the relays it reads
 *                       from; a chunk whose owner is not filling v comes from node 0.  Requires relay
 *                       nodes stored whole on distinct GPUs that are not actor GPUs, in HBM. */
enum { LAM_HOP_KERNEL = 0, LAM_HOP_COPY_ENGINE = 1, LAM_HOP_MULTICAST = 2, LAM_HOP_TREE = 4 };  /* 3: withdrawn */

/* One fp32 master shard piece owned by the caller: elements [elem_offset, elem_offset+elem_count)
 * of the flattened tensor `tensor_id`, at `ptr` (device memory of the actor rank's GPU). */
typedef struct {
  uint32_t tensor_id;
  uint32_t _pad;
  uint64_t elem_offset, elem_count;
  const float* ptr;
} lam_shard;

/* A destination buffer of a rollout TP rank: the parts' TP slices concatenated along dim 0
 * (e.g. qkv = [q_r; k_r; v_r]) into a (rows x cols) bf16 matrix A.
 *   transpose = 0: row-major, A[i][c] at dst + i*pitch + 2c; dst_row_pitch_bytes = 0 means 2*cols.
 *   transpose = 1: K-major (R16), A[i][c] at dst + c*pitch + 2i; dst_row_pitch_bytes =
 *                  0 means 2*rows, else >= 2*rows.  1-D destinations ignore the flag. */
typedef struct {
  uint32_t tensor_id;
  int32_t rule;
} lam_part;

typedef struct {
  const lam_part* parts;
  int32_t n_parts;
  int32_t transpose;                       /* 0 row-major, 1 K-major (transposed) */
  void* dst;                               /* device pointer on the rollout's GPU */
  int64_t dst_row_pitch_bytes;
} lam_dst;

typedef struct {
  int32_t tp_size, tp_rank;
  const lam_dst* dsts;
  int32_t n_dsts;
} lam_tp_layout;

/* Per-chunk header carried with every chunk: checksum (S1, S2) of C3. */
typedef struct {
  uint64_t version, idx, n, bytes, s1, s2, _pad[2];
} lam_chunk_header;

typedef struct {
  uint64_t image_bytes;       /* C * total_chunks */
  uint64_t chunk_bytes;       /* C */
  uint64_t total_chunks;
  uint64_t snapshot_bytes;    /* 2 * parameter count (the paper's M) */
  uint64_t params;
  int32_t n_tensors, n_nodes;
} lam_plan_info;

typedef struct {
  uint64_t publishes, publish_busy, hops_launched, versions_skipped, pulls, checksum_errors,
      timeouts, plan_cache_hits, plan_cache_misses;
  uint64_t chain_rebuilds;   /* relay failures handled (lam_fail_node or heartbeat timeout) */
  uint64_t chain_resumes;    /* hops restarted from a new predecessor, from the lowest missing chunk */
  uint64_t last_repair_ns;   /* failure declared -> successor's resumed hop launched (steady clock) */
  uint64_t kernel_launches;  /* every kernel this library launched (pack, hop, verify, flag wait, pull) */
  uint64_t publish_ns_total, publish_ns_max;  /* host time inside lam_publish (entry -> return, steady
                                                 clock), summed / largest over successful calls: the
                                                 actor's own stall per publish */
} lam_stats;

/* ---- lifecycle ------------------------------------------------------------------------- */
/* sizeof(lam_config) as this library was compiled: bindings compare it with their own struct
 * layout before the first call (a stale build fails loudly instead of misreading the config). */
size_t lam_config_size(void);
/* Validates cfg, builds the image plan, allocates this process's ring slots (S per node part on
 * its devices, zero-filled) and the control block.  n_procs > 1: rank 0 creates the shm block
 * `shm_name`, the others attach (waiting up to 60 s); then exchange handles with lam_export_ipc /
 * lam_import_ipc and call lam_connect.  n_procs == 1: connected on return. */
lam_status lam_init(const lam_config* cfg, lam_ctx** out);
/* Serialize this process's CUDA IPC handles into buf (cap bytes); *len = bytes written. */
lam_status lam_export_ipc(lam_ctx*, void* buf, size_t cap, size_t* len);
/* Import the blob another process exported (call once per other process, any order). */
lam_status lam_import_ipc(lam_ctx*, int32_t proc, const void* buf, size_t len);
/* Open peer mappings and build the per-slot link tables; required before publish/step/pull. */
lam_status lam_connect(lam_ctx*);
/* Waits for this process's in-flight work, unmaps and frees. */
void lam_destroy(lam_ctx*);
const char* lam_strerror(lam_status);

/* ---- the path -------------------------------------------------------------------------- */
/* Publish `version` for actor rank `actor_rank` (owned by this process).  `shards` must cover
 * every element the rank owns under cfg.actor_layout.  The pack runs on a library side stream
 * after the work already queued on `actor_stream`; `reads_done` (caller-created event on the
 * rank's device, may be NULL) is recorded when the shards have been read — the optimizer must
 * wait on it before overwriting the masters.  Returns immediately (host cost: microseconds).
 * With FSDP-N every rank calls lam_publish with the same version; the version becomes COMPLETE
 * at node 0 when all N packs finished.  Errors: LAM_ESTALE (version not newer), LAM_EBUSY. */
lam_status lam_publish(lam_ctx*, uint64_t version, int32_t actor_rank, const lam_shard* shards,
                       int32_t n_shards, void* actor_stream, void* reads_done);

/* Non-blocking progress: polls completions of this process's kernels, commits versions, starts
 * chain hops for relay nodes whose predecessor holds a newer version (latest-wins), releases
 * pins.  *n_transitions (may be NULL) = state changes made.  Returns LAM_IDLE when nothing is in
 * flight anywhere, LAM_OK otherwise, or the first error seen (LAM_ECHECKSUM / LAM_ETIMEOUT). */
lam_status lam_relay_step(lam_ctx*, int32_t* n_transitions);

/* Pull the newest COMPLETE version at rollout `rollout_id`'s node into `layout`'s destination
 * buffers, resharded to the TP rank, on `stream` (rollout's device).  *version_out = version
 * pulled, or 0 with LAM_ENOVERSION.  The slot is pinned until the kernel completes. */
lam_status lam_pull(lam_ctx*, int32_t rollout_id, const lam_tp_layout* layout, void* stream,
                    uint64_t* version_out);

/* Streaming pull — for a rollout that is waiting for new weights (a rollout
 * fetches on batch completion).  If the rollout's node holds a COMPLETE version >= min_version this is
 * lam_pull.  Otherwise, if the node is receiving one (FILLING), that version is pinned and resharded
 * chunk by chunk as its chunks arrive: every lam_relay_step of this process launches the reshard
 * of the newly verified chunks on `stream` (host-driven: no kernel waits on another kernel of the
 * same GPU); after the last chunk `done_event` (caller-created, rollout's device, may be NULL) is
 * recorded on `stream`.  The destination buffers are valid only once lam_pull_state reports 0 and
 * `stream` reached done_event.  *version_out = the version being pulled; 0 + LAM_ENOVERSION if none
 * >= min_version is complete or in flight; LAM_EBUSY if the rollout has a streaming pull running. */
lam_status lam_pull_stream(lam_ctx*, int32_t rollout_id, const lam_tp_layout* layout, void* stream,
                           void* done_event, uint64_t min_version, uint64_t* version_out);
/* Colocated subscription: rollout `rollout_id` sits on an actor GPU (node 0, same device) with a
 * TP=1 dense layout covering every tensor.  The next version published by the actor rank(s) on that
 * GPU is also written into the rollout's buffers by the pack kernel itself, in the same pass (the
 * bf16 bytes go to the master slot and to the rollout: 8 instead of 4 + 6 B/param of HBM traffic).
 * `done_event` (caller-created, may be NULL) is recorded after that pack; lam_pull_state then
 * reports (version, 0).  One-shot: subscribe again for the next version.  LAM_EINVAL if the rollout
 * or layout does not qualify (use lam_pull / lam_pull_stream instead) — in particular unless EVERY
 * actor rank is packed on the rollout's GPU (the pack only writes the shards it packs there). */
lam_status lam_subscribe(lam_ctx*, int32_t rollout_id, const lam_tp_layout* layout, void* done_event);

/* State of the rollout's streaming pull: 1 = chunks still arriving, 0 = all enqueued (or none),
 * < 0 = the version failed at the node (LAM_ECHECKSUM / LAM_ETIMEOUT): buffers hold no valid version. */
lam_status lam_pull_state(lam_ctx*, int32_t rollout_id, uint64_t* version_out, int32_t* state);

/* Newest COMPLETE version at a node (0 if none; node 0 = master). */
lam_status lam_latest(lam_ctx*, int32_t node, uint64_t* version_out);

/* Fault-tolerant broadcast (§4.3, "the scheduler … immediately reconstructs the
 * broadcast chain among the remaining rollout machines … a constant-time (O(1)) operation"):
 * declare relay `node` failed (as the rollout manager's heartbeat monitor would; with n_procs > 1
 * lam_relay_step also detects silent processes by itself, see heartbeat_timeout_s).  Its successor
 * is linked to its predecessor; a successor that was receiving from it resumes the same version
 * from the new predecessor, keeping every chunk it already verified.  Node 0 (the actor's slots)
 * cannot be failed: that is a trainer failure (checkpoint recovery, out of scope).  Pulls at a
 * failed node return LAM_ENOVERSION. */
lam_status lam_fail_node(lam_ctx*, int32_t node);

/* ---- introspection / helpers ----------------------------------------------------------- */
lam_status lam_get_plan_info(lam_ctx*, lam_plan_info* out);
lam_status lam_get_stats(lam_ctx*, lam_stats* out);
/* Copy nbytes of image bytes [offset, offset+nbytes) of node `node`'s COMPLETE `version` to host
 * memory (synchronous; debugging and parity tests).  LAM_ENOVERSION if not held complete. */
lam_status lam_read_image(lam_ctx*, int32_t node, uint64_t version, uint64_t offset, uint64_t nbytes,
                          void* host_dst);
lam_status lam_read_headers(lam_ctx*, int32_t node, uint64_t version, lam_chunk_header* host_dst,
                            uint64_t first_chunk, uint64_t n_chunks);

/* Kernel timing (for the roofline report): when enabled, every pack / hop / pull launch of this
 * process is bracketed by timing events on the stream it runs on.  lam_kernel_times returns, per
 * kind (0 = pack, 1 = hop, 2 = pull), the summed device milliseconds and launch count of launches
 * that completed since the last call, and resets them. */
lam_status lam_set_profiling(lam_ctx*, int32_t on);
/* Change lam_config.pack_sms for later publishes (0 = all SMs). */
lam_status lam_set_pack_sms(lam_ctx*, int32_t sms);
lam_status lam_kernel_times(lam_ctx*, double ms_out[3], uint64_t count_out[3]);

/* Bytes a pull of `layout` at rollout `rollout_id` reads from the rollout's own GPU's HBM (local) and
 * from elsewhere (remote: other GPUs over NVLink, or a host-memory relay node over PCIe); builds/caches
 * the copy plan.  For roofline accounting. */
lam_status lam_pull_bytes(lam_ctx*, int32_t rollout_id, const lam_tp_layout* layout, uint64_t* local_bytes,
                          uint64_t* remote_bytes);

/* Test hook: device pointer (valid in this process) of actor rank `rank`'s region of the slot
 * holding `version` (FILLING or COMPLETE) at `node`.  Used by fault-injection tests only. */
lam_status lam_debug_region(lam_ctx*, int32_t node, uint64_t version, int32_t rank, void** dev_ptr);
/* Test hook (LAM_HOP_MULTICAST): device pointer of actor rank `rank`'s region in device `device`'s
 * multicast replica of node 0's slot holding `version` (the device must be a team GPU of this
 * process).  LAM_EINVAL in the other hop modes.  Used by fault-injection tests only. */
lam_status lam_debug_replica(lam_ctx*, int32_t device, uint64_t version, int32_t rank, void** dev_ptr);

/* Model table of the library (independent of any caller-side copy). */
int32_t lam_model_n_tensors(const lam_model_dims*);
lam_status lam_model_tensor(const lam_model_dims*, int32_t tensor_id, char* name, int32_t name_cap,
                            int64_t shape[2], int32_t* ndim);
/* vLLM-convention destination list of one TP rank: fills up to cap_dsts dsts (dst = NULL,
 * pitch 0) and their parts (parts array of cap_parts, referenced by the dsts), names
 * (name_cap bytes each, in `names`), and each dst's (rows, cols) with cols = 1 for 1-D.
 * Returns the number of dsts, or <0 on error. */
int32_t lam_vllm_layout(const lam_model_dims*, int32_t tp_size, lam_dst* dsts, int32_t cap_dsts,
                        lam_part* parts, int32_t cap_parts, char* names, int32_t name_cap,
                        int64_t* rows, int64_t* cols);
/* Host-only plan introspection (no GPU needed; used by the CPU test-suite to check the planner).
 * Image layout: segments of cfg-equivalent (dims, layout, N, C); returns the count (or <0).  With
 * out == NULL only counts.  image_off = byte offset of the segment in IMG(v). */
typedef struct {
  uint32_t tensor_id, rank;
  uint64_t elem0, count, image_off;
} lam_segment_info;
int64_t lam_plan_segments(const lam_model_dims*, int32_t actor_layout, int32_t fsdp_size, uint64_t chunk_bytes,
                          lam_segment_info* out, int64_t cap);
/* The pull copy plan for a TP layout (destination pointers are taken as plain integers):
 * each tile copies `rows` rows of `row_bytes` from image rank region `src_rank` at byte
 * `src_off` (row stride src_pitch) to address `dst` (row stride dst_pitch).  Two variants, marked
 * in `align` (low byte = 16/4/2, the widest access every address allows):
 *   align & LAM_TILE_TRANSPOSE: element k of row r goes to dst + k*dst_pitch + 2r instead;
 *   src_rank == LAM_TILE_ZERO:  no source; the block is zero-filled (vocabulary padding rows). */
#define LAM_TILE_TRANSPOSE 0x100u
#define LAM_TILE_ZERO 0xFFFFFFFFu
typedef struct {
  uint64_t src_off, dst;
  uint32_t src_pitch, dst_pitch, rows, row_bytes, src_rank, align;
} lam_copy_tile_info;
int64_t lam_plan_copy_tiles(const lam_model_dims*, int32_t actor_layout, int32_t fsdp_size, uint64_t chunk_bytes,
                            const lam_tp_layout*, lam_copy_tile_info* out, int64_t cap);
/* LAM_HOP_TREE: the hop tiles relay `node` (1..n_relays) walks, in order, and the node each one is read
 * from (`source`: 0 = node 0, else the relay that owns the chunk, when it is in `peer_mask`). */
typedef struct {
  uint64_t region_off;
  uint32_t chunk, rank, bytes, source;
} lam_hop_tile_info;
int64_t lam_plan_tree_tiles(const lam_model_dims*, int32_t actor_layout, int32_t fsdp_size, uint64_t chunk_bytes,
                            int32_t n_relays, int32_t node, uint64_t peer_mask, lam_hop_tile_info* out, int64_t cap);

/* ---- control plane (host-only; no GPU) ------------------------------------------------- */
/* The version-table state machine the runtime runs under its cross-process lock, exposed so the
 * CPU test-suite can drive it from several processes.  `name` = POSIX shm name ("" = private heap
 * block); create = 1 for the creating process.  States: 0 FREE, 1 FILLING, 2 COMPLETE.
 * Semantics: PAPER L548-550, L652-670; SPEC L546-547, L633, L638, L643, L661 (see control.h). */
typedef struct lam_ctl lam_ctl;
lam_ctl* lam_ctl_open(const char* name, int32_t create, int32_t n_nodes, int32_t slots, int32_t fsdp_size);
/* Same, with the topology of a hop mode: LAM_HOP_MULTICAST = star (every relay's predecessor is node
 * 0), LAM_HOP_TREE = star + gang start + peer pins, others = chain. */
lam_ctl* lam_ctl_open_mode(const char* name, int32_t create, int32_t n_nodes, int32_t slots, int32_t fsdp_size,
                           int32_t hop_mode);
void lam_ctl_close(lam_ctl*);
lam_status lam_ctl_publish(lam_ctl*, uint64_t version, int32_t rank, int32_t* slot);  /* ESTALE, EBUSY */
int32_t lam_ctl_pack_done(lam_ctl*, int32_t slot, uint64_t version);                  /* 1 = changed */
int32_t lam_ctl_start(lam_ctl*, int32_t node, uint64_t* version, int32_t* started);   /* FILLING slot / -1 */
int32_t lam_ctl_part_done(lam_ctl*, int32_t node, int32_t slot, uint64_t version, int32_t n_parts,
                          lam_status err);
int32_t lam_ctl_fail(lam_ctl*, int32_t node);                                          /* 1 = rebuilt */
int32_t lam_ctl_pred(lam_ctl*, int32_t node);                                          /* -1 = dead */
uint64_t lam_ctl_pin(lam_ctl*, int32_t node, int32_t* slot);                           /* 0 = none */
void lam_ctl_unpin(lam_ctl*, int32_t node, int32_t slot);
uint64_t lam_ctl_latest(lam_ctl*, int32_t node);
int32_t lam_ctl_busy(lam_ctl*);
lam_status lam_ctl_slot(lam_ctl*, int32_t node, int32_t slot, uint64_t* version, int32_t* state, int32_t* readers);
/* Heartbeat: stamp process `proc` at now_ns (steady clock); declare dead every other process
 * whose stamp is older than limit_s and fail (O(1) rebuild) every live relay node with a part in a dead
 * process — node_procs[node] = bit mask of the processes holding a part of `node` (n_nodes entries).
 * Returns the bit mask of the nodes failed by this call.  The runtime runs the same function inside every
 * lam_relay_step (lam_config.heartbeat_timeout_s). */
uint64_t lam_ctl_heartbeat(lam_ctl*, int32_t proc, int32_t n_procs, uint64_t now_ns, double limit_s,
                           const uint64_t* node_procs);
uint64_t lam_ctl_dead_procs(lam_ctl*);                                                  /* bit mask */

/* Appendix D: chunk count k = clamp(round(sqrt((p-2) M T_byte / T_start)),
 * 1, k_cap); and T(p, k) = (p + k - 2)(M/k T_byte + T_start). */
int64_t lam_optimal_chunks(int32_t p, double M, double t_byte, double t_start, int64_t k_cap);
double lam_chain_latency(int32_t p, int64_t k, double M, double t_byte, double t_start);

#ifdef __cplusplus
}
#endif
#endif /* LAM_H */

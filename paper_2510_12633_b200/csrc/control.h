// Control plane of the relay tier: the version table and its state machine, with no CUDA in it.
//
// PAPER L548-550 (steps 5-7), L652-670 (§4.2); SPEC L527-663 (relay semantics):
//   * every node has S ring slots, FREE -> FILLING(v) -> COMPLETE(v);
//   * node 0 is the master (the actor's publish slots); a version is COMPLETE there when all FSDP
//     ranks packed it;
//   * a relay starts receiving the NEWEST version its predecessor holds (FILLING or COMPLETE; this is
//     what pipelines the chain) into a FREE slot or a COMPLETE slot with no readers that is not its
//     latest (latest-wins: versions may be skipped, never reordered), pinning the predecessor's slot;
//   * `latest` only moves up, and only to COMPLETE versions (SPEC L633 complete-only, L638 monotone);
//   * a corrupt chunk frees the slot without committing it.
// The block lives in POSIX shared memory when there is one process per GPU, behind a robust
// process-shared mutex.  The runtime (runtime.cpp) calls these functions under that mutex; the
// lam_ctl_* C entry points expose them to the CPU test-suite (multi-process, gloo).
#pragma once
#include <pthread.h>
#include <stdint.h>

#include "../../include/lam.h"

namespace lam {

enum : int32_t { S_FREE = 0, S_FILLING = 1, S_COMPLETE = 2 };

struct ShmSlot {
  uint64_t version;
  int32_t state, readers;
  int32_t parts_done, parts_finished;  // node 0: ranks packed; relays: parts completed ok / at all
  int32_t err, src_slot;               // first error; predecessor slot pinned while FILLING
  uint64_t launched_mask;              // node 0: ranks published; relays: parts launched
  uint32_t epoch;                      // bumped when the fill restarts from a new predecessor
  uint64_t peer_mask;                  // two-level broadcast: relays whose slot of `version` this fill
                                       // pinned (it pulls the chunks they own from them) ...
  int8_t peer_slot[LAM_MAX_NODES + 1]; // ... and which slot of each
};
struct ShmNode {
  ShmSlot slot[LAM_MAX_SLOTS];
  uint64_t latest, started, skipped;
  int32_t dead;                        // relay failed (heartbeat timeout or lam_fail_node)
  int32_t pred;                        // current predecessor in the chain (rebuilt on failures)
};
struct Shm {
  uint64_t magic;
  pthread_mutex_t mu;
  uint64_t last_published;
  int32_t n_nodes, ready_procs;
  lam_stats stats;
  uint64_t chain_epoch;                // chain rebuilds so far
  uint64_t fail_ns[LAM_MAX_NODES + 1]; // steady-clock time each node was declared failed
  uint64_t hb_ns[LAM_MAX_DEVICES];     // per process heartbeat (steady clock, ns)
  uint64_t dead_procs;                 // bit mask
  int32_t tree, _pad2;                 // LAM_HOP_TREE: two-level broadcast (gang start, peer pins)
  uint64_t last_fail_ns;               // most recent failure (repair-time accounting)
  ShmNode node[LAM_MAX_NODES + 1];
  // Host-visible mirror of every slot's chunk flags, written by the producer kernels through a
  // mapped (cudaHostRegister) view of this block: lets the rollout's process launch a streaming
  // pull's reshard chunk by chunk without any kernel waiting on another kernel of the same GPU.
  uint64_t chunk_done[LAM_MAX_NODES + 1][LAM_MAX_SLOTS][2048];
};
constexpr uint32_t kShmMirrorChunks = 2048;
constexpr uint64_t kMagic = 0x4c414d5f53484d35ull;  // "LAM_SHM5"

struct ShmLock {
  pthread_mutex_t* m;
  explicit ShmLock(Shm* s);
  ~ShmLock();
};

// Shared-memory block: create (owner), attach (waits up to ~60 s), or heap (single process).
Shm* shm_create(const char* name);
Shm* shm_attach(const char* name);
Shm* shm_heap();
void shm_release(Shm* s, const char* name, bool mapped, bool owner);

namespace ctl {
int find_slot(const ShmNode& n, int S, uint64_t v, int32_t state);
int acquire_slot(const ShmNode& n, int S);
uint64_t newest_held(const ShmNode& n, int S, int* slot);
// Actor rank `rank` publishes v at node 0 (joins v if another rank opened it).  *slot = its slot.
lam_status publish(Shm* sh, int S, int fsdp, uint64_t v, int rank, int* slot);
// One rank's pack of v in `slot` finished; returns true on a state change.
bool pack_done(Shm* sh, int fsdp, int slot, uint64_t v);
// Node `node` (>= 1): begin the newest version its predecessor holds if possible.  Returns the
// FILLING slot (new or already open) or -1; *started = true if this call opened it.
int start(Shm* sh, int S, int node, bool* started);
// One part of `node` finished v in `slot` (err = 0 or a LAM_E* code); returns true on a change.
// `epoch` = the slot epoch the finished kernel was launched for; results of superseded launches
// (the fill restarted after a chain rebuild) are ignored.
bool part_done(Shm* sh, int node, int slot, uint64_t v, int n_parts, lam_status err, uint32_t epoch);
// Pull side: pin the latest COMPLETE slot (0 if none) / release it.
uint64_t pin_latest(Shm* sh, int S, int node, int* slot);
void unpin(Shm* sh, int node, int slot);
// Anything FILLING, or a node behind its predecessor?
bool busy(Shm* sh, int S, int n_nodes);
// Chain of n_nodes (called once by the creator): every node alive, pred = node - 1; star (the
// LAM_HOP_MULTICAST broadcast, NEXT-2): every relay's predecessor is node 0.
// tree (LAM_HOP_TREE): star for the predecessor (node 0), plus a gang start — the first relay to start
// v opens v at every idle relay at once — and each fill pins the slot of v at every other relay that
// holds v (it pulls the chunks those relays own from them).
void init(Shm* sh, int n_nodes, bool star = false, bool tree = false);
// Relay failure: mark `node` dead and rebuild the chain in O(1): its successor is
// linked to its (live) predecessor.  A successor that was filling from it re-pins the same version
// at the new predecessor and restarts (slot epoch++, launch mask cleared: the runtime resumes from
// the lowest chunk it lacks); if the new predecessor does not hold that version the fill is
// abandoned and the successor starts over with the newest the new predecessor holds.
// Returns false if the node is node 0 (the actor's slots: trainer failure, out of scope) or dead.
bool fail_node(Shm* sh, int S, int node, uint64_t now_ns);
// Heartbeats ("detects the failure via heartbeat monitoring"): stamp process `proc` at
// now_ns; every other process whose last stamp is older than limit_ns is declared dead (once), and
// every live relay node with a part in a dead process (bit q of node_procs[node] = process q holds a
// part of it) fails through fail_node (O(1) rebuild each).  Processes that never stamped are not
// judged.  Returns the bit mask of the nodes this call failed.
uint64_t heartbeat(Shm* sh, int S, int proc, int n_procs, uint64_t now_ns, uint64_t limit_ns,
                   const uint64_t* node_procs, int n_nodes);
}  // namespace ctl

}  // namespace lam

// Control plane of the relay tier (see control.h): version table state machine + shared memory.
// Host-only C++ — no CUDA — so that the CPU test-suite can drive it from several processes.
#include "control.h"

#include <errno.h>
#include <fcntl.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <new>
#include <utility>
#include <vector>

namespace lam {

ShmLock::ShmLock(Shm* s) : m(&s->mu) {
  int rc = pthread_mutex_lock(m);
  if (rc == EOWNERDEAD) pthread_mutex_consistent(m);  // a rank died holding it: state is per-field valid
}
ShmLock::~ShmLock() { pthread_mutex_unlock(m); }

static void init_mutex(Shm* s, bool shared) {
  pthread_mutexattr_t a;
  pthread_mutexattr_init(&a);
  pthread_mutexattr_settype(&a, PTHREAD_MUTEX_RECURSIVE);
  if (shared) {
    pthread_mutexattr_setpshared(&a, PTHREAD_PROCESS_SHARED);
    pthread_mutexattr_setrobust(&a, PTHREAD_MUTEX_ROBUST);
  }
  pthread_mutex_init(&s->mu, &a);
  pthread_mutexattr_destroy(&a);
}

Shm* shm_heap() {
  void* mem = nullptr;  // page-aligned: the runtime cudaHostRegister()s the block
  if (posix_memalign(&mem, 4096, sizeof(Shm)) != 0) return nullptr;
  Shm* s = reinterpret_cast<Shm*>(mem);
  memset(s, 0, sizeof(Shm));
  init_mutex(s, false);
  s->magic = kMagic;
  return s;
}

Shm* shm_create(const char* name) {
  char path[96];
  snprintf(path, sizeof path, "/%s", name);
  shm_unlink(path);
  int fd = shm_open(path, O_CREAT | O_EXCL | O_RDWR, 0600);
  if (fd < 0) return nullptr;
  if (ftruncate(fd, sizeof(Shm)) != 0) {
    close(fd);
    return nullptr;
  }
  void* p = mmap(nullptr, sizeof(Shm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return nullptr;
  Shm* s = reinterpret_cast<Shm*>(p);
  init_mutex(s, true);
  __atomic_store_n(&s->magic, kMagic, __ATOMIC_RELEASE);  // attachers wait for this
  return s;
}

Shm* shm_attach(const char* name) {
  char path[96];
  snprintf(path, sizeof path, "/%s", name);
  int fd = -1;
  for (int i = 0; i < 6000 && fd < 0; ++i) {
    fd = shm_open(path, O_RDWR, 0600);
    if (fd < 0) usleep(10000);
  }
  if (fd < 0) return nullptr;
  struct stat st;
  for (int i = 0; i < 6000; ++i) {
    if (fstat(fd, &st) == 0 && (size_t)st.st_size >= sizeof(Shm)) break;
    usleep(10000);
  }
  void* p = mmap(nullptr, sizeof(Shm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return nullptr;
  Shm* s = reinterpret_cast<Shm*>(p);
  for (int i = 0; i < 6000 && __atomic_load_n(&s->magic, __ATOMIC_ACQUIRE) != kMagic; ++i) usleep(10000);
  if (__atomic_load_n(&s->magic, __ATOMIC_ACQUIRE) != kMagic) {
    munmap(p, sizeof(Shm));
    return nullptr;
  }
  return s;
}

void shm_release(Shm* s, const char* name, bool mapped, bool owner) {
  if (!s) return;
  if (mapped) {
    munmap(s, sizeof(Shm));
    if (owner) {
      char path[96];
      snprintf(path, sizeof path, "/%s", name);
      shm_unlink(path);
    }
  } else {
    pthread_mutex_destroy(&s->mu);
    free(s);
  }
}

namespace ctl {

int find_slot(const ShmNode& n, int S, uint64_t v, int32_t state) {
  for (int i = 0; i < S; ++i)
    if (n.slot[i].version == v && n.slot[i].state == state) return i;
  return -1;
}

int acquire_slot(const ShmNode& n, int S) {
  for (int i = 0; i < S; ++i)
    if (n.slot[i].state == S_FREE && n.slot[i].readers == 0) return i;
  for (int i = 0; i < S; ++i)
    if (n.slot[i].state == S_COMPLETE && n.slot[i].readers == 0 && n.slot[i].version != n.latest) return i;
  return -1;
}

uint64_t newest_held(const ShmNode& n, int S, int* slot) {
  uint64_t best = 0;
  *slot = -1;
  for (int i = 0; i < S; ++i)
    if ((n.slot[i].state == S_FILLING || n.slot[i].state == S_COMPLETE) && n.slot[i].version > best) {
      best = n.slot[i].version;
      *slot = i;
    }
  return best;
}

static void open_slot(ShmSlot& sl, uint64_t v, int src_slot) {
  sl.version = v;
  sl.state = S_FILLING;
  sl.readers = 0;
  sl.parts_done = sl.parts_finished = 0;
  sl.err = 0;
  sl.src_slot = src_slot;
  sl.peer_mask = 0;
  sl.launched_mask = 0;
  sl.epoch++;
}

void init(Shm* sh, int n_nodes, bool star, bool tree) {
  sh->n_nodes = n_nodes;
  sh->tree = tree ? 1 : 0;
  for (int i = 0; i <= LAM_MAX_NODES; ++i) {
    sh->node[i].dead = 0;
    sh->node[i].pred = (star || tree) && i > 0 ? 0 : i - 1;
  }
}

// A two-level fill's pins of its peers' slots of the same version end with the fill (or one peer's:
// the failed one, whose chunks the fill then takes from node 0).
static void unpin_peer(Shm* sh, ShmSlot& sl, int o) {
  if (!(sl.peer_mask >> o & 1ull)) return;
  ShmSlot& ps = sh->node[o].slot[sl.peer_slot[o]];
  if (ps.readers > 0) ps.readers--;
  sl.peer_mask &= ~(1ull << o);
}
static void unpin_peers(Shm* sh, ShmSlot& sl) {
  for (int o = 1; o <= LAM_MAX_NODES && sl.peer_mask; ++o) unpin_peer(sh, sl, o);
}

// Two-level fill of `node` in slot s: pin the slot of its version at every other live relay that holds
// it (FILLING or COMPLETE) — their chunks come from them, the rest from node 0.
static void pin_peers(Shm* sh, int S, int node, int s) {
  ShmSlot& sl = sh->node[node].slot[s];
  for (int o = 1; o < sh->n_nodes; ++o) {
    if (o == node || sh->node[o].dead) continue;
    int ps = find_slot(sh->node[o], S, sl.version, S_COMPLETE);
    if (ps < 0) ps = find_slot(sh->node[o], S, sl.version, S_FILLING);
    if (ps < 0) continue;
    sh->node[o].slot[ps].readers++;
    sl.peer_slot[o] = (int8_t)ps;
    sl.peer_mask |= 1ull << o;
  }
}

bool fail_node(Shm* sh, int S, int node, uint64_t now_ns) {
  if (node <= 0 || node >= sh->n_nodes || sh->node[node].dead) return false;
  ShmNode& d = sh->node[node];
  d.dead = 1;
  sh->fail_ns[node] = now_ns;
  sh->last_fail_ns = now_ns;
  sh->chain_epoch++;
  // the dead node's own fill no longer pins its predecessor
  for (int s = 0; s < S; ++s) {
    ShmSlot& sl = d.slot[s];
    if (sl.state == S_FILLING) {
      if (sl.src_slot >= 0 && sh->node[d.pred].slot[sl.src_slot].readers > 0) sh->node[d.pred].slot[sl.src_slot].readers--;
      unpin_peers(sh, sl);
      sl.state = S_FREE;
      sl.version = 0;
      sl.src_slot = -1;
    }
  }
  // two-level broadcast: fills that pull chunks from the dead relay restart (new epoch): their runtime
  // takes the missing chunks from node 0
  if (sh->tree)
    for (int j = 1; j < sh->n_nodes; ++j) {
      if (j == node || sh->node[j].dead) continue;
      for (int s = 0; s < S; ++s) {
        ShmSlot& sl = sh->node[j].slot[s];
        if (sl.state != S_FILLING || !(sl.peer_mask >> node & 1ull)) continue;
        unpin_peer(sh, sl, node);
        sl.launched_mask = 0;
        sl.parts_done = sl.parts_finished = 0;
        sl.epoch++;
      }
    }
  // O(1) rebuild: the (single) successor links to the failed node's predecessor
  for (int j = node + 1; j < sh->n_nodes; ++j) {
    ShmNode& n = sh->node[j];
    if (n.dead || n.pred != node) continue;
    n.pred = d.pred;
    ShmNode& np = sh->node[n.pred];
    for (int s = 0; s < S; ++s) {
      ShmSlot& sl = n.slot[s];
      if (sl.state != S_FILLING) continue;
      const int ps = find_slot(np, S, sl.version, S_COMPLETE) >= 0 ? find_slot(np, S, sl.version, S_COMPLETE)
                                                                 : find_slot(np, S, sl.version, S_FILLING);
      if (ps >= 0) {                       // resume the same version from the new predecessor
        np.slot[ps].readers++;
        sl.src_slot = ps;
        sl.launched_mask = 0;
        sl.parts_done = sl.parts_finished = 0;
        sl.epoch++;
      } else {                             // abandon: start over with what the new predecessor has
          sl.state = S_FREE;
        sl.version = 0;
        sl.src_slot = -1;
        n.started = n.latest;
      }
    }
  }
  return true;
}

lam_status publish(Shm* sh, int S, int fsdp, uint64_t v, int rank, int* slot) {
  ShmNode& n0 = sh->node[0];
  if (v == 0 || v < sh->last_published) return LAM_ESTALE;
  int s;
  if (v == sh->last_published) {             // another rank already opened v: join it
    s = find_slot(n0, S, v, S_FILLING);
    if (s < 0 || (n0.slot[s].launched_mask >> rank & 1ull)) return LAM_ESTALE;
  } else {
    const uint64_t all = fsdp == 64 ? ~0ull : ((1ull << fsdp) - 1);
    for (int i = 0; i < S; ++i)                // the previous version still waits for some ranks
      if (n0.slot[i].state == S_FILLING && n0.slot[i].launched_mask != all) return LAM_EBUSY;
    s = acquire_slot(n0, S);
    if (s < 0) {
      sh->stats.publish_busy++;
      return LAM_EBUSY;
    }
    open_slot(n0.slot[s], v, -1);
    sh->last_published = v;
    n0.started = v;
    sh->stats.publishes++;
  }
  n0.slot[s].launched_mask |= 1ull << rank;
  *slot = s;
  return LAM_OK;
}

bool pack_done(Shm* sh, int fsdp, int slot, uint64_t v) {
  ShmSlot& sl = sh->node[0].slot[slot];
  if (sl.version != v || sl.state != S_FILLING) return false;
  if (++sl.parts_done == fsdp) {
    sl.state = S_COMPLETE;
    if (v > sh->node[0].latest) sh->node[0].latest = v;
  }
  return true;
}

int start(Shm* sh, int S, int node, bool* started) {
  *started = false;
  ShmNode& n = sh->node[node];
  if (n.dead) return -1;
  ShmNode& pred = sh->node[n.pred];
  for (int s = 0; s < S; ++s)
    if (n.slot[s].state == S_FILLING) return s;
  int ps = -1;
  const uint64_t u = newest_held(pred, S, &ps);
  if (u <= n.started) return -1;
  const int s = acquire_slot(n, S);
  if (s < 0) return -1;
  if (!sh->tree && n.started && u > n.started + 1) {
    n.skipped += u - n.started - 1;
    sh->stats.versions_skipped += u - n.started - 1;
  }
  if (sh->tree) {
    // two-level broadcast: gang start — open u at every idle live relay that can take it (this one
    // included), then every newly opened fill pins the slot of u at each other relay holding it
    int mine = -1;
    std::vector<std::pair<int, int>> opened;
    for (int o = 1; o < sh->n_nodes; ++o) {
      ShmNode& no = sh->node[o];
      if (no.dead || u <= no.started) continue;
      bool filling = false;
      for (int k = 0; k < S; ++k) filling |= no.slot[k].state == S_FILLING;
      if (filling) continue;
      const int so = o == node ? s : acquire_slot(no, S);
      if (so < 0) continue;
      if (no.started && u > no.started + 1) {
        no.skipped += u - no.started - 1;
        sh->stats.versions_skipped += u - no.started - 1;
      }
      open_slot(no.slot[so], u, ps);
      sh->node[no.pred].slot[ps].readers++;
      no.started = u;
      opened.push_back({o, so});
      if (o == node) mine = so;
    }
    for (auto& os : opened) pin_peers(sh, S, os.first, os.second);
    *started = mine >= 0;
    return mine;
  }
  open_slot(n.slot[s], u, ps);
  pred.slot[ps].readers++;
  n.started = u;
  *started = true;
  return s;
}

bool part_done(Shm* sh, int node, int slot, uint64_t v, int n_parts, lam_status err, uint32_t epoch) {
  ShmNode& n = sh->node[node];
  ShmSlot& sl = n.slot[slot];
  if (sl.version != v || sl.state != S_FILLING || sl.epoch != epoch || n.dead) return false;
  sl.parts_finished++;
  if (err != LAM_OK) {
    if (!sl.err) sl.err = err;
    if (err == LAM_ETIMEOUT) sh->stats.timeouts++; else sh->stats.checksum_errors++;
  } else {
    sl.parts_done++;
  }
  if (sl.parts_finished == n_parts) {
    if (sl.src_slot >= 0) {
      ShmSlot& src = sh->node[n.pred].slot[sl.src_slot];
      if (src.readers > 0) src.readers--;
    }
    unpin_peers(sh, sl);
    if (sl.err == 0) {
      sl.state = S_COMPLETE;
      if (v > n.latest) n.latest = v;
    } else {
      sl.state = S_FREE;                       // never committed: keep serving the previous version
      sl.version = 0;
    }
    sl.src_slot = -1;
  }
  return true;
}

uint64_t pin_latest(Shm* sh, int S, int node, int* slot) {
  ShmNode& n = sh->node[node];
  *slot = -1;
  if (n.latest == 0 || n.dead) return 0;
  const int s = find_slot(n, S, n.latest, S_COMPLETE);
  if (s < 0) return 0;
  n.slot[s].readers++;
  *slot = s;
  return n.latest;
}

void unpin(Shm* sh, int node, int slot) {
  ShmSlot& sl = sh->node[node].slot[slot];
  if (sl.readers > 0) sl.readers--;
}

bool busy(Shm* sh, int S, int n_nodes) {
  for (int node = 0; node < n_nodes; ++node) {
    const ShmNode& n = sh->node[node];
    if (n.dead) continue;
    for (int s = 0; s < S; ++s)
      if (n.slot[s].state == S_FILLING) return true;
    int ps;
    if (node > 0 && newest_held(sh->node[n.pred], S, &ps) > n.started) return true;
  }
  return false;
}

uint64_t heartbeat(Shm* sh, int S, int proc, int n_procs, uint64_t now_ns, uint64_t limit_ns,
                   const uint64_t* node_procs, int n_nodes) {
  uint64_t failed = 0;
  if (proc >= 0 && proc < LAM_MAX_DEVICES) sh->hb_ns[proc] = now_ns;
  if (n_procs < 2 || limit_ns == 0) return 0;
  for (int q = 0; q < n_procs && q < LAM_MAX_DEVICES; ++q) {
    if (q == proc || (sh->dead_procs >> q & 1ull) || sh->hb_ns[q] == 0) continue;
    // a stamp newer than now_ns (taken by another process after the caller read its clock) is alive
    if (sh->hb_ns[q] >= now_ns || now_ns - sh->hb_ns[q] <= limit_ns) continue;
    sh->dead_procs |= 1ull << q;
    for (int node = 1; node < n_nodes; ++node)
      if ((node_procs[node] >> q & 1ull) && !sh->node[node].dead && fail_node(sh, S, node, now_ns)) {
        sh->stats.chain_rebuilds++;
        failed |= 1ull << node;
      }
  }
  return failed;
}

}  // namespace ctl
}  // namespace lam

// ------------------------------------------------------------------ C entry points (CPU tests)
using namespace lam;

struct lam_ctl {
  Shm* sh;
  int S, fsdp, n_nodes;
  bool mapped, owner;
  char name[64];
};

extern "C" lam_ctl* lam_ctl_open_mode(const char* name, int32_t create, int32_t n_nodes, int32_t slots,
                                      int32_t fsdp, int32_t hop_mode) {
  if (n_nodes < 1 || n_nodes > LAM_MAX_NODES + 1 || slots < 2 || slots > LAM_MAX_SLOTS || fsdp < 1 ||
      fsdp > LAM_MAX_RANKS)
    return nullptr;
  lam_ctl* c = new (std::nothrow) lam_ctl();
  if (!c) return nullptr;
  c->S = slots;
  c->fsdp = fsdp;
  c->n_nodes = n_nodes;
  snprintf(c->name, sizeof c->name, "%s", name ? name : "");
  c->mapped = name && name[0];
  c->owner = create != 0;
  c->sh = !c->mapped ? shm_heap() : (create ? shm_create(name) : shm_attach(name));
  if (!c->sh) {
    delete c;
    return nullptr;
  }
  if (create || !c->mapped)
    ctl::init(c->sh, n_nodes, hop_mode == LAM_HOP_MULTICAST, hop_mode == LAM_HOP_TREE);
  return c;
}

extern "C" lam_ctl* lam_ctl_open(const char* name, int32_t create, int32_t n_nodes, int32_t slots, int32_t fsdp) {
  return lam_ctl_open_mode(name, create, n_nodes, slots, fsdp, LAM_HOP_KERNEL);
}

extern "C" void lam_ctl_close(lam_ctl* c) {
  if (!c) return;
  shm_release(c->sh, c->name, c->mapped, c->owner);
  delete c;
}

extern "C" lam_status lam_ctl_publish(lam_ctl* c, uint64_t v, int32_t rank, int32_t* slot) {
  ShmLock l(c->sh);
  return ctl::publish(c->sh, c->S, c->fsdp, v, rank, slot);
}

extern "C" int32_t lam_ctl_pack_done(lam_ctl* c, int32_t slot, uint64_t v) {
  ShmLock l(c->sh);
  return ctl::pack_done(c->sh, c->fsdp, slot, v);
}

extern "C" int32_t lam_ctl_start(lam_ctl* c, int32_t node, uint64_t* version, int32_t* started) {
  ShmLock l(c->sh);
  bool st = false;
  int s = ctl::start(c->sh, c->S, node, &st);
  *version = s >= 0 ? c->sh->node[node].slot[s].version : 0;
  *started = st;
  return s;
}

extern "C" int32_t lam_ctl_part_done(lam_ctl* c, int32_t node, int32_t slot, uint64_t v, int32_t n_parts,
                                     lam_status err) {
  ShmLock l(c->sh);
  return ctl::part_done(c->sh, node, slot, v, n_parts, err, c->sh->node[node].slot[slot].epoch);
}

extern "C" int32_t lam_ctl_fail(lam_ctl* c, int32_t node) {
  ShmLock l(c->sh);
  return ctl::fail_node(c->sh, c->S, node, 0);
}

extern "C" int32_t lam_ctl_pred(lam_ctl* c, int32_t node) {
  ShmLock l(c->sh);
  return c->sh->node[node].dead ? -1 : c->sh->node[node].pred;
}

extern "C" uint64_t lam_ctl_pin(lam_ctl* c, int32_t node, int32_t* slot) {
  ShmLock l(c->sh);
  return ctl::pin_latest(c->sh, c->S, node, slot);
}

extern "C" void lam_ctl_unpin(lam_ctl* c, int32_t node, int32_t slot) {
  ShmLock l(c->sh);
  ctl::unpin(c->sh, node, slot);
}

extern "C" uint64_t lam_ctl_latest(lam_ctl* c, int32_t node) {
  ShmLock l(c->sh);
  return c->sh->node[node].latest;
}

extern "C" int32_t lam_ctl_busy(lam_ctl* c) {
  ShmLock l(c->sh);
  return ctl::busy(c->sh, c->S, c->n_nodes);
}

extern "C" lam_status lam_ctl_slot(lam_ctl* c, int32_t node, int32_t slot, uint64_t* version, int32_t* state,
                                   int32_t* readers) {
  ShmLock l(c->sh);
  const ShmSlot& s = c->sh->node[node].slot[slot];
  *version = s.version;
  *state = s.state;
  *readers = s.readers;
  return LAM_OK;
}

extern "C" uint64_t lam_ctl_heartbeat(lam_ctl* c, int32_t proc, int32_t n_procs, uint64_t now_ns, double limit_s,
                                      const uint64_t* node_procs) {
  ShmLock l(c->sh);
  return ctl::heartbeat(c->sh, c->S, proc, n_procs, now_ns, (uint64_t)(limit_s * 1e9), node_procs, c->n_nodes);
}

extern "C" uint64_t lam_ctl_dead_procs(lam_ctl* c) {
  ShmLock l(c->sh);
  return c->sh->dead_procs;
}

"""CPU tests of the relay control plane (liblam's lam_ctl_*: the version table the runtime drives).

* Differential: seeded random publish / relay-round / pin / unpin interleavings give the same
  per-node latest versions, skip counts and publish outcomes as the oracle's RelayChain model
  (oracle/relay.py, PAPER L661-665 with one chunk per version: a hop completes within its round).
* Multi-process (world_size 2, gloo): an actor process publishes while a relay process runs the
  chain and pins/unpins, on one POSIX shared-memory block — the N>1 host path of the library.
"""
import os
import random

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.relay import RelayChain
from paper_2510_12633_b200 import lam

FREE, FILLING, COMPLETE = 0, 1, 2


def _round(ctl: lam.Ctl, p: int):
    """One oracle round with k = 1: hops in tail-to-head order, each starts and completes a version."""
    for node in range(p - 1, 0, -1):
        s, v, opened = ctl.start(node)
        if s >= 0:
            assert ctl.part_done(node, s, v, 1, lam.LAM_OK)


def test_publish_rules():
    c = lam.Ctl("", True, n_nodes=2, slots=2)
    assert c.publish(0)[0] == lam.LAM_ESTALE
    st, s = c.publish(3)
    assert st == lam.LAM_OK
    assert c.publish(3)[0] == lam.LAM_ESTALE and c.publish(2)[0] == lam.LAM_ESTALE
    assert c.latest(0) == 0 and c.pin(0) == (0, -1)          # FILLING is never served
    assert c.pack_done(s, 3) and c.latest(0) == 3
    v, ps = c.pin(0)
    assert v == 3
    st4, s4 = c.publish(4)
    assert st4 == lam.LAM_OK and s4 != ps
    c.pack_done(s4, 4)
    assert c.publish(5)[0] == lam.LAM_EBUSY                  # 3 pinned, 4 latest
    c.unpin(0, ps)
    assert c.publish(5)[0] == lam.LAM_OK
    c.close()


def test_fsdp_ranks_join_one_version():
    c = lam.Ctl("", True, n_nodes=1, slots=2, fsdp=3)
    st, s = c.publish(1, rank=2)
    assert st == lam.LAM_OK
    assert c.publish(1, rank=2)[0] == lam.LAM_ESTALE          # same rank twice
    assert c.publish(2, rank=0)[0] == lam.LAM_EBUSY           # v1 still waits for ranks 0, 1
    for r in (0, 1):
        assert c.publish(1, rank=r) == (lam.LAM_OK, s)
    for _ in range(2):
        c.pack_done(s, 1)
        assert c.latest(0) == 0
    c.pack_done(s, 1)
    assert c.latest(0) == 1
    c.close()


def test_corrupt_version_is_not_committed():
    c = lam.Ctl("", True, n_nodes=2, slots=2)
    for v in (1, 2):
        st, s = c.publish(v)
        c.pack_done(s, v)
        s1, u, _ = c.start(1)
        c.part_done(1, s1, u, 2, lam.LAM_OK if v == 1 else lam.LAM_ECHECKSUM)
        c.part_done(1, s1, u, 2, lam.LAM_OK)
    assert c.latest(1) == 1 and c.latest(0) == 2
    assert not c.busy()                                      # node 1 does not retry the bad version
    c.close()


@pytest.mark.parametrize("seed", range(25))
def test_matches_oracle_relay_model(seed):
    rng = random.Random(seed)
    p, S = rng.randint(2, 5), rng.choice([2, 3])
    c = lam.Ctl("", True, n_nodes=p, slots=S)
    o = RelayChain(p, 1, slots=S)
    v, pins = 0, []
    for _ in range(300):
        a = rng.random()
        if a < 0.2:
            v += 1
            st, s = c.publish(v)
            want = o.publish(v)
            assert {"ok": lam.LAM_OK, "busy": lam.LAM_EBUSY, "stale": lam.LAM_ESTALE}[want] == st
            if st == lam.LAM_OK:
                c.pack_done(s, v)
        elif a < 0.4:
            node = rng.randrange(p)
            got, slot = c.pin(node)
            want, oslot = o.pin_latest(node)
            assert got == want
            if got:
                pins.append((node, slot, oslot))
        elif a < 0.55 and pins:
            node, slot, oslot = pins.pop(rng.randrange(len(pins)))
            c.unpin(node, slot)
            o.unpin(node, oslot)
        else:
            _round(c, p)
            o.step()
        assert [c.latest(n) for n in range(p)] == [n.latest for n in o.nodes]
    c.close()


# ---------------------------------------------------------------------- chain repair (NEXT-1)
def _publish_complete(c, v):
    st, s = c.publish(v)
    assert st == lam.LAM_OK
    c.pack_done(s, v)


def test_rebuild_chain_spec_example():
    """chain [m,a,b,c], fail b -> [m,a,c], a's successor is c (O(1) relink)."""
    c = lam.Ctl("", True, n_nodes=4, slots=2)
    assert [c.pred(n) for n in (1, 2, 3)] == [0, 1, 2]
    assert c.fail(2)
    assert [c.pred(n) for n in (1, 2, 3)] == [0, -1, 1]
    assert not c.fail(2) and not c.fail(0)                # already dead / the actor's slots
    _publish_complete(c, 1)
    for _ in range(4):
        _round(c, 4)
    assert [c.latest(n) for n in range(4)] == [1, 1, 0, 1]  # the dead node is skipped, never served
    assert c.pin(2) == (0, -1)
    assert not c.busy()
    c.close()


def test_fail_mid_broadcast_resumes_same_version():
    c = lam.Ctl("", True, n_nodes=4, slots=2)
    _publish_complete(c, 1)
    s1, v1, _ = c.start(1)
    c.part_done(1, s1, v1)                                # node 1 holds v1
    s2, v2, _ = c.start(2)                                # node 2 filling v1 from node 1
    s3, v3, _ = c.start(3)                                # node 3 filling v1 from node 2 (pipelined)
    assert (v2, v3) == (1, 1)
    assert c.fail(2)                                      # node 2 dies mid-broadcast
    assert c.pred(3) == 1
    ver, state, readers = c.slot(3, s3)
    assert (ver, state) == (1, FILLING)                   # same version, now pinned at node 1
    assert c.slot(1, s1)[2] == 1
    c.part_done(3, s3, 1)
    assert c.latest(3) == 1 and c.slot(1, s1)[2] == 0     # pin released at the new predecessor
    c.close()


def test_fail_abandons_version_the_new_predecessor_lacks():
    c = lam.Ctl("", True, n_nodes=4, slots=2)
    _publish_complete(c, 1)
    for _ in range(3):
        _round(c, 4)
    _publish_complete(c, 2)
    s1, v1, _ = c.start(1)                                # node 1 FILLING v2
    s2, v2, _ = c.start(2)                                # node 2 FILLING v2 from node 1
    assert c.fail(1)                                      # node 2 re-points to node 0, which has v2
    assert c.pred(2) == 0 and c.slot(2, s2)[:2] == (2, FILLING)
    assert c.fail(2)                                      # node 3 re-points to node 0 as well
    assert c.pred(3) == 0
    _publish_complete(c, 3)
    for _ in range(3):
        _round(c, 4)
    assert c.latest(3) == 3 and not c.busy()
    c.close()


# ------------------------------------------------------------------------------ two processes
def _worker(rank, world, port, name, versions, q, hop_mode=lam.LAM_HOP_KERNEL):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    errors = []
    try:
        c = lam.Ctl(name, rank == 0, n_nodes=3, slots=2, hop_mode=hop_mode)
        dist.barrier()
        rng = random.Random(rank)
        if rank == 0:                                        # the actor: publish as fast as it can
            published = []
            v = 0
            while v < versions:
                st, s = c.publish(v + 1)
                if st == lam.LAM_OK:
                    v += 1
                    c.pack_done(s, v)
                    published.append(v)
            q.put(("published", published))
        else:                                                # the relays + a rollout pulling
            seen = {1: 0, 2: 0}
            for _ in range(200000):
                for node in (1, 2):
                    s, u, opened = c.start(node)
                    if s >= 0 and rng.random() < 0.7:
                        c.part_done(node, s, u, 1, lam.LAM_OK)
                    lt = c.latest(node)
                    if lt < seen[node]:
                        errors.append(f"node {node} latest went back {seen[node]} -> {lt}")
                    seen[node] = lt
                node = rng.choice((1, 2))
                got, slot = c.pin(node)
                if got:
                    pv, pst, prd = c.slot(node, slot)
                    if (pv, pst) != (got, COMPLETE) or prd < 1:
                        errors.append(f"pinned slot not COMPLETE({got}): {(pv, pst, prd)}")
                    c.unpin(node, slot)
                if c.latest(1) == versions and c.latest(2) == versions:
                    break
        dist.barrier()
        if rank == 1:
            final = [c.latest(n) for n in range(3)]
            if final != [versions] * 3:
                errors.append(f"not quiescent at the newest version: {final}")
            pins = [c.slot(n, k)[2] for n in range(3) for k in range(2)]
            if any(pins):                                    # every pin (readers, fills, peers) released
                errors.append(f"readers left at quiescence: {pins}")
        dist.barrier()
        c.close()
    except Exception as e:  # pragma: no cover - reported to the parent
        errors.append(repr(e))
    q.put((rank, errors))
    dist.destroy_process_group()


@pytest.mark.parametrize("hop_mode", [lam.LAM_HOP_KERNEL, lam.LAM_HOP_MULTICAST, lam.LAM_HOP_TREE])
def test_two_processes_share_the_version_table(hop_mode):
    """Chain, star (multicast) and two-level (gang start + peer pins) control planes, across processes."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = f"lam_ctl_test_{os.getpid()}_{hop_mode}"
    versions = 60
    port = 29500 + (os.getpid() * 3 + hop_mode) % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, versions, q, hop_mode)) for r in range(2)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=120) for _ in range(3)]
    for pr in procs:
        pr.join(timeout=60)
    errs = [e for r in results if r[0] in (0, 1) for e in r[1]]
    assert errs == [], errs
    published = next(r[1] for r in results if r[0] == "published")
    assert published == list(range(1, versions + 1))


# ------------------------------------------------------------------ NEXT-1: a relay process dies
def _hb_worker(proc, n_procs, name, limit_s, node_procs, q, stop):
    """One rank process: stamps its heartbeat every 5 ms through lam_ctl_heartbeat (what every
    lam_relay_step does) and reports the nodes it saw failing and when (steady clock), until `stop`."""
    import time as _t
    c = lam.Ctl(name, False, len(node_procs), 2, 1)
    seen = 0
    c.heartbeat(proc, n_procs, _t.monotonic_ns(), limit_s, node_procs)
    q.put((proc, "ready"))
    while not stop.is_set():
        failed = c.heartbeat(proc, n_procs, _t.monotonic_ns(), limit_s, node_procs)
        if failed:
            seen |= failed
            q.put((proc, "failed", failed, _t.monotonic_ns(), [c.pred(n) for n in range(len(node_procs))]))
        _t.sleep(0.005)
    q.put((proc, "done", seen, c.dead_procs(), [c.pred(n) for n in range(len(node_procs))]))
    c.close()


def test_sigkill_of_a_relay_process_is_detected_by_heartbeat_and_the_chain_rebuilt():
    """"the rollout manager detects the failure via heartbeat monitoring and immediately
    reconstructs the broadcast chain ... a constant-time (O(1)) operation".  Four rank processes own
    node k (node 0 = the actor's slots on process 0, relays 1..3 on processes 1..3); process 2 is
    SIGKILLed.  The survivors' heartbeats must declare it dead within the limit (+ one period), fail
    exactly node 2 once, and relink node 3 to node 1; detection well under the paper's one second."""
    import signal
    import time as _t
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = f"lam_hb_test_{os.getpid()}"
    n = 4
    node_procs = [1 << k for k in range(n)]            # node k lives on process k
    owner = lam.Ctl(name, True, n, 2, 1)
    limit = 0.5
    stop = ctx.Event()
    procs = [ctx.Process(target=_hb_worker, args=(k, n, name, limit, node_procs, q, stop)) for k in range(n)]
    for pr in procs:
        pr.start()
    ready = [q.get(timeout=120) for _ in range(n)]     # every process stamped (spawn + import done)
    assert sorted(m[0] for m in ready) == list(range(n)) and all(m[1] == "ready" for m in ready)
    _t.sleep(0.5)
    kill_ns = _t.monotonic_ns()
    os.kill(procs[2].pid, signal.SIGKILL)
    procs[2].join(timeout=10)
    _t.sleep(1.5)                                      # 3 x the limit: detection must have happened
    stop.set()
    msgs = []
    t0 = _t.time()
    while sum(1 for m in msgs if m[1] == "done") < n - 1 and _t.time() - t0 < 60:
        msgs.append(q.get(timeout=60))
    for k in (0, 1, 3):
        procs[k].join(timeout=30)
    fails = [m for m in msgs if m[1] == "failed"]
    assert len(fails) == 1, fails                      # node 2 failed once, by whichever survivor saw it first
    proc, _, mask, t_ns, preds = fails[0]
    assert proc != 2 and mask == 1 << 2
    detect_s = (t_ns - kill_ns) / 1e9
    assert limit - 0.05 <= detect_s < 1.0, detect_s    # "less than one second"
    assert preds[3] == 1 and preds[2] == -1 and preds[1] == 0
    done = [m for m in msgs if m[1] == "done"]
    assert all(m[3] == 1 << 2 for m in done)           # every survivor sees process 2 (only) as dead
    assert owner.pred(3) == 1
    owner.close()


# ---------------------------------------------------------------- multicast (star) and tree topologies
def _publish(c, v):
    st, s = c.publish(v)
    assert st == lam.LAM_OK
    return s


def test_star_topology_every_relay_fed_by_node0():
    """LAM_HOP_MULTICAST (NEXT-2): every relay's predecessor is node 0, so all relays start a version as
    soon as node 0 holds it (the multicast pack feeds them at once), each pinning node 0's slot; a failed
    relay relinks nobody."""
    c = lam.Ctl("", True, n_nodes=4, slots=2, hop_mode=lam.LAM_HOP_MULTICAST)
    assert [c.pred(n) for n in (1, 2, 3)] == [0, 0, 0]
    s0 = _publish(c, 1)
    fills = {}
    for node in (1, 2, 3):                        # node 0 still FILLING: every relay starts v1 at once
        s, v, opened = c.start(node)
        assert (v, opened) == (1, True)
        fills[node] = s
    assert c.slot(0, s0)[2] == 3                  # pinned by the three fills
    c.pack_done(s0, 1)
    assert c.fail(2) and [c.pred(n) for n in (1, 3)] == [0, 0]
    assert c.slot(0, s0)[2] == 2                  # the dead relay's pin is gone
    for node in (1, 3):
        assert c.part_done(node, fills[node], 1)
    assert c.slot(0, s0)[2] == 0 and c.latest(1) == c.latest(3) == 1
    c.close()


def test_tree_gang_start_and_peer_pins():
    """LAM_HOP_TREE: the first relay to start a version opens it at every idle relay (gang start); each
    fill pins node 0's slot and the slot of the version at every other relay holding it; pins end with
    the fills; a relay that fails mid-broadcast releases its pins and restarts its readers' fills."""
    c = lam.Ctl("", True, n_nodes=4, slots=2, hop_mode=lam.LAM_HOP_TREE)
    assert [c.pred(n) for n in (1, 2, 3)] == [0, 0, 0]
    s0 = _publish(c, 1)
    s1, v, opened = c.start(1)                    # opens v1 at relays 1, 2 and 3 at once
    assert (v, opened) == (1, True)
    fills = {1: s1}
    for node in (2, 3):
        s, u, op = c.start(node)                  # already FILLING: returned, not reopened
        assert u == 1 and not op
        fills[node] = s
    assert c.slot(0, s0)[2] == 3                  # node 0 pinned by the three fills
    for node in (1, 2, 3):                        # each pinned by the other two
        assert c.slot(node, fills[node])[2] == 2
    c.pack_done(s0, 1)
    assert c.fail(3)                              # relay 3 dies mid-broadcast
    assert c.slot(0, s0)[2] == 2                  # its own pin of node 0 is gone
    assert c.slot(1, fills[1])[2] == 1 and c.slot(2, fills[2])[2] == 1   # and of its peers
    for node in (1, 2):                           # the survivors no longer pin relay 3
        assert c.part_done(node, fills[node], 1)
    assert c.slot(0, s0)[2] == 0 and c.latest(1) == c.latest(2) == 1
    assert [c.slot(n, fills[n])[2] for n in (1, 2)] == [0, 0]
    c.close()


def test_tree_late_relay_pins_only_holders():
    """A relay still filling the previous version misses the gang start of the next; it starts that
    version later and then pins the relays that hold it, while their earlier fills do not pin it."""
    c = lam.Ctl("", True, n_nodes=3, slots=2, hop_mode=lam.LAM_HOP_TREE)

    def filling(node, v):
        return [k for k in (0, 1) if c.slot(node, k)[:2] == (v, FILLING)][0]

    s = _publish(c, 1)
    c.pack_done(s, 1)
    c.start(1)                                    # gang: v1 at relays 1 and 2
    for node in (1, 2):
        assert c.part_done(node, filling(node, 1), 1)
    s = _publish(c, 2)
    c.pack_done(s, 2)
    c.start(1)                                    # gang: v2 at relays 1 and 2
    assert c.part_done(1, filling(1, 2), 2)       # relay 2 is still receiving v2
    s = _publish(c, 3)
    c.pack_done(s, 3)
    c.start(1)                                    # gang: only relay 1 is idle
    k13 = filling(1, 3)
    assert c.slot(1, k13)[2] == 0                 # relay 2 does not hold v3: nothing pinned
    assert c.part_done(2, filling(2, 2), 2)
    s2, u, opened = c.start(2)                    # late start of v3 at relay 2
    assert (u, opened) == (3, True)
    assert c.slot(1, k13)[2] == 1                 # relay 2 pins relay 1's v3 (it reads relay 1's chunks)
    assert c.slot(2, s2)[2] == 0                  # relay 1's fill did not pin relay 2
    assert c.part_done(1, k13, 3) and c.part_done(2, s2, 3)
    assert c.slot(1, k13)[2] == 0 and c.latest(1) == c.latest(2) == 3
    c.close()


@pytest.mark.parametrize("hop_mode,seed", [(m, s) for m in (lam.LAM_HOP_KERNEL, lam.LAM_HOP_MULTICAST, lam.LAM_HOP_TREE)
                                           for s in range(4)])
def test_random_interleavings_keep_the_slot_invariants(hop_mode, seed):
    """Seeded random publish / pack / fill / corrupt-fill / rollout pin-unpin interleavings in every
    topology (chain, star, two-level): latest never goes back, a pinned slot is COMPLETE at the
    pinned version, reader counts stay >= 0, and once progress runs without faults
    every relay serves the newest version and every pin (rollout, fill, peer) has been released."""
    rng = random.Random(seed)
    n = 4
    c = lam.Ctl("", True, n_nodes=n, slots=2, hop_mode=hop_mode)
    seen = [0] * n
    pins = []
    v = 0

    def check():
        for node in range(n):
            lt = c.latest(node)
            assert lt >= seen[node], (node, seen[node], lt)
            seen[node] = lt
            for k in range(2):
                assert c.slot(node, k)[2] >= 0

    def step(node, p_done, p_bad):
        s, u, _ = c.start(node)
        if s >= 0 and rng.random() < p_done:
            c.part_done(node, s, u, 1, lam.LAM_ECHECKSUM if rng.random() < p_bad else lam.LAM_OK)
        return s

    for _ in range(600):
        r = rng.random()
        if r < 0.15:
            st, s = c.publish(v + 1)
            if st == lam.LAM_OK:
                v += 1
                if rng.random() < 0.8:
                    c.pack_done(s, v)
                else:
                    pending = (s, v)
                    step(rng.randrange(1, n), 0.5, 0.0)   # relays may start v before the pack ends
                    c.pack_done(*pending)
        elif r < 0.75:
            step(rng.randrange(1, n), 0.6, 0.05)
        elif r < 0.9:
            node = rng.randrange(1, n)
            got, slot = c.pin(node)
            if got:
                assert c.slot(node, slot)[:2] == (got, COMPLETE)
                pins.append((node, slot))
        elif pins:
            c.unpin(*pins.pop(rng.randrange(len(pins))))
        check()
    while pins:
        c.unpin(*pins.pop())
    for _ in range(100):                                   # fault-free progress to quiescence
        if all(step(node, 1.0, 0.0) < 0 for node in range(1, n)):
            break
        check()
    assert [c.latest(node) for node in range(n)] == [v] * n
    assert [c.slot(node, k)[2] for node in range(n) for k in range(2)] == [0] * (2 * n)
    c.close()

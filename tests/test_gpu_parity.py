"""GPU parity: the CUDA path through the C ABI vs the oracle, bit-exact (copy/cast/index work).

Quiescent runs (publish -> relay_step until LAM_IDLE -> pull) must reproduce exactly:
  * every relay's slot bytes == IMG(v) and its chunk headers == the oracle's (S1, S2),
  * every pulled TP buffer == TP_r(RNE_bf16(W_v)).
Tiny: full comparison.  7B (the bench workload): sampled chunks and sampled destination elements,
computed one by one by the oracle.
"""
import time

import numpy as np
import pytest
import torch

from oracle.image import FSDP1_FLAT, FSDP2_DIM0, image_plan, publish, publish_chunk
from oracle.model import MODELS as OMODELS
from oracle.model import tensors as otensors
from oracle.tp import direct_pull, dst_elements
from paper_2510_12633_b200 import lam
from paper_2510_12633_b200.workload import MODELS, ActorShard, RolloutBuffers
from synth import SEED

pytestmark = pytest.mark.gpu
OLAYOUT = {lam.LAM_FSDP2_DIM0: FSDP2_DIM0, lam.LAM_FSDP1_FLAT: FSDP1_FLAT}


def ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def until_idle(ctx, timeout=120.0):
    t0 = time.time()
    while True:
        st, _ = ctx.relay_step()
        if st == lam.LAM_IDLE:
            return
        if time.time() - t0 > timeout:
            raise TimeoutError("relay never went idle")
        time.sleep(0.0005)


def check_image(ctx, node, v, oimg, ohdr, C):
    info = ctx.plan_info()
    assert info.total_chunks == len(ohdr)
    got = ctx.read_image(node, v, 0, info.image_bytes)
    assert got.size == oimg.size
    if not np.array_equal(got, oimg):
        bad = np.nonzero(got != oimg)[0]
        raise AssertionError(f"node {node}: {bad.size} image bytes differ, first at {bad[0]} (chunk {bad[0] // C})")
    hdr = ctx.read_headers(node, v)
    for g, (a, b) in enumerate(zip(hdr, ohdr)):
        assert a == b, (node, g, a, b)


def check_pull(ctx, rid, tp, rank, dev, v, specials, odims, transpose=False):
    rb = RolloutBuffers(MODELS_BY_DIMS[id(odims)], tp, rank, dev, transpose=transpose)
    rb.fill_(0xFFFF)
    s = torch.cuda.Stream(device=dev)
    got_v = ctx.pull(rid, rb.tp, s.cuda_stream)
    assert got_v == v
    s.synchronize()
    want = direct_pull(odims, tp, rank, SEED, v, specials=specials, transpose=transpose)
    for name, t in rb.bufs.items():
        g = t.view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(g, want[name].reshape(g.shape)), (name, rank)
    return rb


MODELS_BY_DIMS = {id(OMODELS[k]): MODELS[k] for k in OMODELS}


def make_ctx(model, fsdp, actor_devs, relays, rollouts, layout=lam.LAM_FSDP2_DIM0, C=1 << 20, **kw):
    return lam.Context(lam.Config(model=MODELS[model], fsdp_size=fsdp, actor_devices=actor_devs, relays=relays,
                                  rollouts=rollouts, actor_layout=layout, chunk_bytes=C, **kw))


def _memcpy(dst, src, n):
    import ctypes
    rc = ctypes.CDLL("libcudart.so.12").cudaMemcpy(ctypes.c_void_p(dst), ctypes.c_void_p(src), ctypes.c_size_t(n), 4)
    assert rc == 0, rc


def publish_all(ctx, shards, v, specials):
    torch.cuda.synchronize()
    for r, sh in enumerate(shards):
        sh.fill(SEED, v, specials)
    torch.cuda.synchronize()
    for r, sh in enumerate(shards):
        with torch.cuda.device(sh.device):
            st = ctx.publish(v, r, sh.shards(), torch.cuda.current_stream().cuda_stream)
        assert st == lam.LAM_OK


# ------------------------------------------------------------------------------------- tiny
@pytest.mark.parametrize("layout,N,C,tp", [(lam.LAM_FSDP2_DIM0, 1, 1 << 20, 1),
                                           (lam.LAM_FSDP2_DIM0, 1, 3 * 4096, 2),      # many ragged chunks
                                           (lam.LAM_FSDP2_DIM0, 4, 1 << 18, 4),
                                           (lam.LAM_FSDP1_FLAT, 3, 1 << 18, 2),       # mid-row cuts
                                           (lam.LAM_FSDP2_DIM0, 8, 4096, 8)])
def test_tiny_publish_pull_single_gpu(layout, N, C, tp):
    od = OMODELS["tiny"]
    ctx = make_ctx("tiny", N, [0] * N, [], [(0, 0)], layout=layout, C=C)
    shards = [ActorShard(MODELS["tiny"], N, r, 0, layout, misalign=(layout == lam.LAM_FSDP1_FLAT)) for r in range(N)]
    assert ctx.latest(0) == 0
    rb = RolloutBuffers(MODELS["tiny"], tp, 0, 0)
    assert ctx.pull(0, rb.tp, 0) == 0                                   # nothing complete yet
    publish_all(ctx, shards, 1, True)
    until_idle(ctx)
    assert ctx.latest(0) == 1
    plan = image_plan([s for _, s in otensors(od)], N, C, OLAYOUT[layout])
    oimg, ohdr = publish(plan, SEED, 1, specials=True)
    check_image(ctx, 0, 1, oimg, ohdr, C)
    for r in range(tp):
        check_pull(ctx, 0, tp, r, 0, 1, True, od)
    ctx.close()


@pytest.mark.parametrize("sms", [1, 16, 74])
def test_tiny_pack_confined_to_k_sms(sms):
    """lam_config.pack_sms (actor-stall control): the pack's CTAs outside SMs [0, k) leave at once and
    every unit comes from the work counter — the image, headers and a pull stay bit-exact (specials,
    ragged chunks, FSDP-4)."""
    od = OMODELS["tiny"]
    N, C = 4, 3 * 4096
    ctx = make_ctx("tiny", N, [0] * N, [], [(0, 0)], C=C, pack_sms=sms)
    shards = [ActorShard(MODELS["tiny"], N, r, 0) for r in range(N)]
    for v in (1, 2):
        publish_all(ctx, shards, v, True)
        until_idle(ctx)
        plan = image_plan([s for _, s in otensors(od)], N, C)
        oimg, ohdr = publish(plan, SEED, v, specials=True)
        check_image(ctx, 0, v, oimg, ohdr, C)
    check_pull(ctx, 0, 2, 1, 0, 2, True, od)
    ctx.close()


@pytest.mark.parametrize("model,layout,N,C,tps", [
    ("odd", lam.LAM_FSDP2_DIM0, 1, 4096, (1, 2, 4, 8)),      # KV-head replication, vocab padding
    ("odd", lam.LAM_FSDP1_FLAT, 3, 4096, (2, 8)),            # ... with mid-row FSDP1 cuts
    ("tiny", lam.LAM_FSDP2_DIM0, 4, 3 * 4096, (8,)),         # nkv = 4 < tp = 8
    ("tiny", lam.LAM_FSDP1_FLAT, 3, 1 << 18, (1, 2))])
@pytest.mark.parametrize("transpose", [False, True])
def test_pull_rules_and_k_major(model, layout, N, C, tps, transpose):
    """A6 beyond the configs (R14-R16): HEAD_DIM0 with KV heads replicated when tp > nkv,
    zero-filled vocabulary padding rows, and K-major (transposed) destinations — full comparison."""
    od = OMODELS[model]
    ctx = make_ctx(model, N, [0] * N, [], [(0, 0)], layout=layout, C=C)
    shards = [ActorShard(MODELS[model], N, r, 0, layout, misalign=(layout == lam.LAM_FSDP1_FLAT)) for r in range(N)]
    publish_all(ctx, shards, 2, True)
    until_idle(ctx)
    for tp in tps:
        for r in range(tp):
            check_pull(ctx, 0, tp, r, 0, 2, True, od, transpose=transpose)
    ctx.close()


def test_7b_k_major_tp2_sampled():
    """K-major TP=2 pull of the 7B bench workload: sampled elements of every destination vs the oracle."""
    od = OMODELS["7b"]
    ctx = make_ctx("7b", 1, [0], [], [(0, 0)], C=64 << 20)
    shard = ActorShard(MODELS["7b"], 1, 0, 0)
    publish_all(ctx, [shard], 4, False)
    until_idle(ctx)
    del shard
    torch.cuda.empty_cache()
    rng = np.random.default_rng(1)
    for rank in range(2):
        rb = RolloutBuffers(MODELS["7b"], 2, rank, 0, transpose=True)
        rb.fill_(0xFFFF)
        assert ctx.pull(0, rb.tp, 0) == 4
        torch.cuda.synchronize()
        for name, t in rb.bufs.items():
            idx = rng.integers(0, t.numel(), 512)
            got = t.view(-1).view(torch.int16).cpu().numpy().view(np.uint16)[idx]
            assert np.array_equal(got, dst_elements(od, 2, rank, name, idx, SEED, 4, transpose=True)), name
        del rb
    ctx.close()


HOP_MODES = [lam.LAM_HOP_KERNEL, lam.LAM_HOP_COPY_ENGINE]


@pytest.mark.parametrize("hop_mode", HOP_MODES)
def test_tiny_three_versions_chain_on_one_gpu(hop_mode):
    """Config 1: 1 actor, 2 relays, 2 rollouts TP=1, 3 versions — all on GPU 0 (stream-ordered hops)."""
    od = OMODELS["tiny"]
    C = 64 * 4096
    ctx = make_ctx("tiny", 1, [0], [[0], [0]], [(1, 0), (2, 0)], C=C, hop_mode=hop_mode)
    shard = ActorShard(MODELS["tiny"], 1, 0, 0)
    plan = image_plan([s for _, s in otensors(od)], 1, C)
    for v in (1, 2, 3):
        publish_all(ctx, [shard], v, True)
        until_idle(ctx)
        oimg, ohdr = publish(plan, SEED, v, specials=True)
        for node in (0, 1, 2):
            assert ctx.latest(node) == v
            check_image(ctx, node, v, oimg, ohdr, C)
        for rid in (0, 1):
            check_pull(ctx, rid, 1, 0, 0, v, True, od)
    st = ctx.stats()
    assert st["publishes"] == 3 and st["hops_launched"] == 6 and st["checksum_errors"] == 0
    ctx.close()


@pytest.mark.parametrize("hop_mode", HOP_MODES)
def test_tiny_host_memory_relay_tier(hop_mode):
    """NEXT-3: relay node 1 keeps its ring in pinned host memory (received by
    GPU 0's SMs or copy engines over PCIe), node 2 (HBM) is fed from it — its hop reads host memory —
    and rollouts pull from both; two versions, everything compared in full with the oracle."""
    od = OMODELS["tiny"]
    C = 16 * 4096
    ctx = make_ctx("tiny", 1, [0], [[0], [0]], [(1, 0), (2, 0)], C=C, hop_mode=hop_mode, host_relays=[1])
    shard = ActorShard(MODELS["tiny"], 1, 0, 0)
    plan = image_plan([s for _, s in otensors(od)], 1, C)
    for v in (1, 2):
        publish_all(ctx, [shard], v, True)
        until_idle(ctx)
        oimg, ohdr = publish(plan, SEED, v, specials=True)
        for node in (0, 1, 2):
            assert ctx.latest(node) == v
            check_image(ctx, node, v, oimg, ohdr, C)
        for r in range(2):
            check_pull(ctx, 0, 2, r, 0, v, True, od)            # TP=2 reshard straight from host memory
        check_pull(ctx, 1, 1, 0, 0, v, True, od)
    assert ctx.pull_bytes(0, RolloutBuffers(MODELS["tiny"], 1, 0, 0).tp)[0] == 0  # nothing from local HBM
    ctx.close()


def test_tiny_host_relay_read_by_other_gpus():
    """Host tier across devices: GPU 1 receives node 1 into host memory; GPU 0 pulls from it (portable
    registration) and node 2 on GPU 0 chains from it."""
    if ngpu() < 2:
        pytest.skip("needs >= 2 GPUs")
    od = OMODELS["tiny"]
    C = 8 * 4096
    ctx = make_ctx("tiny", 1, [0], [[1], [0]], [(1, 0), (2, 1)], C=C, host_relays=[1])
    shard = ActorShard(MODELS["tiny"], 1, 0, 0)
    plan = image_plan([s for _, s in otensors(od)], 1, C)
    publish_all(ctx, [shard], 1, True)
    until_idle(ctx)
    oimg, ohdr = publish(plan, SEED, 1, specials=True)
    for node in (1, 2):
        check_image(ctx, node, 1, oimg, ohdr, C)
    check_pull(ctx, 0, 1, 0, 0, 1, True, od)
    check_pull(ctx, 1, 2, 1, 1, 1, True, od)
    ctx.close()


@pytest.mark.parametrize("hop_mode", HOP_MODES)
def test_tiny_chain_across_gpus(hop_mode):
    n = ngpu()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    od = OMODELS["tiny"]
    C = 16 * 4096
    relays = [[d] for d in range(1, n)]
    ctx = make_ctx("tiny", 1, [0], relays, [(i + 1, i + 1) for i in range(n - 1)], C=C, hop_mode=hop_mode)
    shard = ActorShard(MODELS["tiny"], 1, 0, 0)
    plan = image_plan([s for _, s in otensors(od)], 1, C)
    for v in (1, 2):
        publish_all(ctx, [shard], v, True)
        until_idle(ctx)
        oimg, ohdr = publish(plan, SEED, v, specials=True)
        for node in range(n):
            check_image(ctx, node, v, oimg, ohdr, C)
        for rid in range(n - 1):
            check_pull(ctx, rid, 1, 0, rid + 1, v, True, od)
    ctx.close()


def test_sharded_relay_and_remote_pull():
    """FSDP-2 actor on GPUs 0,1; a range-sharded relay over GPUs 0,1; TP=2 pulls gather over NVLink."""
    if ngpu() < 2:
        pytest.skip("needs >= 2 GPUs")
    od = OMODELS["tiny"]
    C = 8 * 4096
    ctx = make_ctx("tiny", 2, [0, 1], [[1, 0]], [(1, 0), (1, 1), (0, 1)], C=C)
    shards = [ActorShard(MODELS["tiny"], 2, r, r) for r in range(2)]
    publish_all(ctx, shards, 1, False)
    until_idle(ctx)
    plan = image_plan([s for _, s in otensors(od)], 2, C)
    oimg, ohdr = publish(plan, SEED, 1)
    check_image(ctx, 0, 1, oimg, ohdr, C)
    check_image(ctx, 1, 1, oimg, ohdr, C)
    check_pull(ctx, 0, 2, 0, 0, 1, False, od)
    check_pull(ctx, 1, 2, 1, 1, 1, False, od)
    check_pull(ctx, 2, 1, 0, 1, 1, False, od)
    ctx.close()


# ---------------------------------------------------------------------------- semantics
def test_version_rules_and_busy():
    ctx = make_ctx("tiny", 1, [0], [], [(0, 0)])
    shard = ActorShard(MODELS["tiny"], 1, 0, 0)
    publish_all(ctx, [shard], 5, False)
    for stale in (5, 4):                                      # same rank again / older: rejected
        with pytest.raises(lam.LamError) as e:
            ctx.publish(stale, 0, shard.shards())
        assert e.value.status == lam.LAM_ESTALE
    until_idle(ctx)
    rb = RolloutBuffers(MODELS["tiny"], 1, 0, 0)
    # pin v5 with a pull whose stream is blocked, publish v6 (other slot), then v7 must be BUSY
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        torch.cuda._sleep(3_000_000_000)                 # ~1.5 s: keeps the pull (and its pin) in flight
    assert ctx.pull(0, rb.tp, s.cuda_stream) == 5
    # no device-wide synchronize from here on: it would drain stream s and release the pin
    assert ctx.publish(6, 0, shard.shards(), torch.cuda.current_stream().cuda_stream) == lam.LAM_OK
    until_busy = time.time()
    while ctx.latest(0) != 6 and time.time() - until_busy < 30:
        ctx.relay_step()
    assert ctx.latest(0) == 6
    assert ctx.publish(7, 0, shard.shards()) == lam.LAM_EBUSY   # slot of v5 pinned, v6 is latest
    s.synchronize()
    until_idle(ctx)
    assert ctx.publish(7, 0, shard.shards()) == lam.LAM_OK
    until_idle(ctx)
    assert ctx.latest(0) == 7
    ctx.close()


def test_tiny_multicast_broadcast():
    """NEXT-2: LAM_HOP_MULTICAST — the pack stores the image once through an NVSwitch
    multicast object; every relay (one per other GPU) verifies and commits it
    from its local replica.  Three versions with specials, full image/header compare at every node and
    TP=1 / TP=2 pulls at every relay against the oracle."""
    n = ngpu()
    if n < 2:
        pytest.skip("multicast needs >= 2 GPUs (a one-device multicast team is invalid)")
    od = OMODELS["tiny"]
    C = 8 * 4096
    relays = [[d] for d in range(1, n)]
    rollouts = [(i + 1, relays[i][0]) for i in range(len(relays))]
    try:
        ctx = make_ctx("tiny", 1, [0], relays, rollouts, C=C, hop_mode=lam.LAM_HOP_MULTICAST)
    except lam.LamError as e:
        if e.status == lam.LAM_EINVAL:
            pytest.skip("multicast objects not supported on this box (no NVSwitch / fabric manager)")
        raise
    shard = ActorShard(MODELS["tiny"], 1, 0, 0)
    plan = image_plan([s for _, s in otensors(od)], 1, C)
    for v in (1, 2, 3):
        publish_all(ctx, [shard], v, True)
        until_idle(ctx)
        oimg, ohdr = publish(plan, SEED, v, specials=True)
        for node in range(len(relays) + 1):
            assert ctx.latest(node) == v
            check_image(ctx, node, v, oimg, ohdr, C)
        for rid, (_, dev) in enumerate(rollouts):
            check_pull(ctx, rid, 1, 0, dev, v, True, od)
            check_pull(ctx, rid, 2, v % 2, dev, v, True, od)
    st = ctx.stats()
    assert st["publishes"] == 3 and st["hops_launched"] == 3 * len(relays) and st["checksum_errors"] == 0
    ctx.close()


def test_tiny_tree_broadcast():
    """LAM_HOP_TREE: each relay pulls its own share of the chunks from node 0 and the others from the
    relays that own them; three versions with specials, full image/header compare at every node and
    TP=1 / TP=2 pulls at every relay against the oracle."""
    n = ngpu()
    if n < 3:
        pytest.skip("needs >= 3 GPUs (two relays reading each other)")
    od = OMODELS["tiny"]
    C = 8 * 4096
    relays = [[d] for d in range(1, n)]
    rollouts = [(i + 1, relays[i][0]) for i in range(len(relays))]
    ctx = make_ctx("tiny", 1, [0], relays, rollouts, C=C, hop_mode=lam.LAM_HOP_TREE)
    shard = ActorShard(MODELS["tiny"], 1, 0, 0)
    plan = image_plan([s for _, s in otensors(od)], 1, C)
    for v in (1, 2, 3):
        publish_all(ctx, [shard], v, True)
        until_idle(ctx)
        oimg, ohdr = publish(plan, SEED, v, specials=True)
        for node in range(len(relays) + 1):
            assert ctx.latest(node) == v
            check_image(ctx, node, v, oimg, ohdr, C)
        for rid, (_, dev) in enumerate(rollouts):
            check_pull(ctx, rid, 1, 0, dev, v, True, od)
            check_pull(ctx, rid, 2, v % 2, dev, v, True, od)
    assert ctx.stats()["checksum_errors"] == 0
    ctx.close()


def test_multicast_corrupt_replica_is_never_committed():
    """A byte flipped in GPU 1's multicast replica of node 0's slot after the pack: relay 1's k_hop
    recomputes the checksum from that replica, rejects the version, and keeps serving v1;
    node 0 itself is intact."""
    if ngpu() < 2:
        pytest.skip("multicast needs >= 2 GPUs (a one-device multicast team is invalid)")
    C = 16 * 4096
    try:
        ctx = make_ctx("tiny", 1, [0], [[1]], [(1, 1)], C=C, hop_mode=lam.LAM_HOP_MULTICAST)
    except lam.LamError as e:
        if e.status == lam.LAM_EINVAL:
            pytest.skip("multicast objects not supported on this box")
        raise
    shard = ActorShard(MODELS["tiny"], 1, 0, 0)
    publish_all(ctx, [shard], 1, False)
    until_idle(ctx)
    assert ctx.latest(1) == 1
    publish_all(ctx, [shard], 2, False)
    torch.cuda.synchronize()                                # pack done, relay hop not launched yet
    ptr = ctx.debug_replica(1, 2, 0) + 5 * C + 1000
    with torch.cuda.device(1):
        byte = torch.empty(1, dtype=torch.uint8, device="cuda:1")
        _memcpy(byte.data_ptr(), ptr, 1)
        byte ^= 0xFF
        _memcpy(ptr, byte.data_ptr(), 1)
        torch.cuda.synchronize()
    with pytest.raises(lam.LamError) as e:
        until_idle(ctx)
    assert e.value.status == lam.LAM_ECHECKSUM
    until_idle(ctx)
    assert ctx.latest(0) == 2 and ctx.latest(1) == 1
    check_pull(ctx, 0, 1, 0, 1, 1, False, OMODELS["tiny"])
    ctx.close()


@pytest.mark.parametrize("hop_mode", HOP_MODES)
def test_corrupt_chunk_is_never_committed(hop_mode):
    """A byte flipped in the master's slot after packing: the relay's checksum rejects the version,
    the relay keeps serving the previous one."""
    C = 16 * 4096
    ctx = make_ctx("tiny", 1, [0], [[0]], [(1, 0)], C=C, hop_mode=hop_mode)
    shard = ActorShard(MODELS["tiny"], 1, 0, 0)
    publish_all(ctx, [shard], 1, False)
    until_idle(ctx)
    assert ctx.latest(1) == 1
    publish_all(ctx, [shard], 2, False)
    torch.cuda.synchronize()                                # pack done, relay hop not launched yet
    ptr = ctx.debug_region(0, 2, 0) + 5 * C + 1000
    byte = torch.empty(1, dtype=torch.uint8, device="cuda:0")
    _memcpy(byte.data_ptr(), ptr, 1)
    byte ^= 0xFF
    _memcpy(ptr, byte.data_ptr(), 1)
    torch.cuda.synchronize()
    with pytest.raises(lam.LamError) as e:
        until_idle(ctx)
    assert e.value.status == lam.LAM_ECHECKSUM
    until_idle(ctx)
    assert ctx.latest(0) == 2 and ctx.latest(1) == 1
    assert ctx.stats()["checksum_errors"] == 1
    od = OMODELS["tiny"]
    check_pull(ctx, 0, 1, 0, 0, 1, False, od)               # relay still serves v1 intact
    ctx.close()


# ------------------------------------------------------------------------- 7B (bench config)
_HDR = None


def _oracle_header(g):
    from oracle.checksum import chunk_checksum
    plan, v = _HDR
    want = publish_chunk(plan, g, SEED, v)
    return chunk_checksum(want), want.size


def oracle_headers(plan, v):
    """(S1, S2) and byte length of every chunk of IMG(v), computed by the oracle on a fork pool
    (publish_chunk + chunk_checksum per chunk, all host cores)."""
    import multiprocessing as mp
    import os
    global _HDR
    _HDR = (plan, v)
    with mp.get_context("fork").Pool(os.cpu_count() or 1) as pool:
        return pool.map(_oracle_header, range(plan.total_chunks), chunksize=1)


def test_7b_single_gpu_all_headers_sampled_elements():
    """The bench workload at full size on one GPU: EVERY chunk header (all 227 of the 64 MiB chunks:
    version, index, length, S1, S2) == the oracle's, the bytes of 3 whole chunks == the oracle's, and
    sampled TP=1 elements of every destination == the oracle's (element by element)."""
    od = OMODELS["7b"]
    ctx = make_ctx("7b", 1, [0], [], [(0, 0)], C=64 << 20)
    info = ctx.plan_info()
    C = info.chunk_bytes
    shard = ActorShard(MODELS["7b"], 1, 0, 0)
    publish_all(ctx, [shard], 3, False)
    until_idle(ctx)
    plan = image_plan([s for _, s in otensors(od)], 1, C)
    assert plan.total_chunks == info.total_chunks == 227
    hdr = ctx.read_headers(0, 3)
    want_hdr = oracle_headers(plan, 3)
    for g, ((s12, n), h) in enumerate(zip(want_hdr, hdr)):
        assert (h["s1"], h["s2"]) == s12 and h["bytes"] == n, g
        assert h["version"] == 3 and h["idx"] == g and h["n"] == plan.total_chunks, (g, h)
    for g in sorted({0, plan.total_chunks // 2, plan.total_chunks - 1}):
        want = publish_chunk(plan, g, SEED, 3)
        got = ctx.read_image(0, 3, g * C, want.size)
        assert np.array_equal(got, want), g
    del shard
    torch.cuda.empty_cache()
    rb = RolloutBuffers(MODELS["7b"], 1, 0, 0)
    assert ctx.pull(0, rb.tp, 0) == 3
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    for name, t in rb.bufs.items():
        idx = rng.integers(0, t.numel(), 256)
        got = t.view(-1).view(torch.int16).cpu().numpy().view(np.uint16)[idx]
        assert np.array_equal(got, dst_elements(od, 1, 0, name, idx, SEED, 3)), name
    ctx.close()

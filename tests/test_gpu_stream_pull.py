"""Streaming pulls (lam_pull_stream): a waiting rollout reshards a version chunk by chunk while its
relay is still receiving it; the result must be exactly the oracle's pull of that version, and a
version that fails at the relay must be reported, never served."""
import time

import numpy as np
import pytest
import torch

from oracle.model import MODELS as OMODELS
from oracle.tp import direct_pull, dst_elements
from paper_2510_12633_b200 import lam
from paper_2510_12633_b200.workload import MODELS, ActorShard, RolloutBuffers
from synth import SEED

pytestmark = pytest.mark.gpu


def drive(ctx, rid, timeout=120):
    t0 = time.time()
    while True:
        ctx.relay_step()
        v, st = ctx.pull_state(rid)
        if st <= 0:
            return v, st
        assert time.time() - t0 < timeout, "streaming pull never finished"


@pytest.mark.parametrize("tp", [1, 2])
def test_stream_pull_tiny_chain(tp):
    n = torch.cuda.device_count()
    devs = [1 % n, 2 % n]
    od = OMODELS["tiny"]
    ctx = lam.Context(lam.Config(model=MODELS["tiny"], relays=[[devs[0]], [devs[1]]],
                                 rollouts=[(2, devs[1]), (0, 0)], chunk_bytes=8 * 4096))
    shard = ActorShard(MODELS["tiny"], 1, 0, 0)
    rb = RolloutBuffers(MODELS["tiny"], tp, tp - 1, devs[1])
    s = torch.cuda.Stream(device=devs[1])
    for v in (1, 2, 3):
        shard.fill(SEED, v, specials=True)
        torch.cuda.synchronize()
        rb.fill_(0xFFFF)
        torch.cuda.synchronize()
        assert ctx.publish(v, 0, shard.shards()) == lam.LAM_OK
        got = 0
        t0 = time.time()
        while got == 0:                                     # wait until relay 2 starts receiving v
            ctx.relay_step()
            got = ctx.pull_stream(0, rb.tp, s.cuda_stream, None, v)
            assert time.time() - t0 < 60
        assert got == v
        assert drive(ctx, 0) == (v, 0)
        s.synchronize()
        want = direct_pull(od, tp, tp - 1, SEED, v, specials=True)
        for name, t in rb.bufs.items():
            g = t.view(torch.int16).cpu().numpy().view(np.uint16)
            assert np.array_equal(g, want[name].reshape(g.shape)), (v, name)
        for _ in range(100000):
            if ctx.relay_step()[0] == lam.LAM_IDLE:
                break
    ctx.close()


@pytest.mark.parametrize("model,tp,rank", [("odd", 8, 7), ("odd", 4, 1), ("tiny", 2, 0)])
def test_stream_pull_k_major(model, tp, rank):
    """Streaming pull into K-major buffers with zero-filled vocabulary padding and replicated KV heads:
    transposed tiles are cut at chunk boundaries in 8-row groups, zero tiles go with the first chunk."""
    n = torch.cuda.device_count()
    dev = 1 % n
    od = OMODELS[model]
    ctx = lam.Context(lam.Config(model=MODELS[model], fsdp_size=3, actor_devices=[0, 0, 0],
                                 actor_layout=lam.LAM_FSDP1_FLAT, relays=[[dev] * 3],
                                 rollouts=[(1, dev)], chunk_bytes=4096))
    shards = [ActorShard(MODELS[model], 3, r, 0, lam.LAM_FSDP1_FLAT) for r in range(3)]
    rb = RolloutBuffers(MODELS[model], tp, rank, dev, transpose=True)
    s = torch.cuda.Stream(device=dev)
    for v in (1, 2):
        for sh in shards:
            sh.fill(SEED, v, specials=True)
        rb.fill_(0xFFFF)
        torch.cuda.synchronize()
        for r, sh in enumerate(shards):
            assert ctx.publish(v, r, sh.shards()) == lam.LAM_OK
        got = 0
        t0 = time.time()
        while got == 0:
            ctx.relay_step()
            got = ctx.pull_stream(0, rb.tp, s.cuda_stream, None, v)
            assert time.time() - t0 < 60
        assert got == v
        assert drive(ctx, 0) == (v, 0)
        s.synchronize()
        want = direct_pull(od, tp, rank, SEED, v, specials=True, transpose=True)
        for name, t in rb.bufs.items():
            g = t.view(torch.int16).cpu().numpy().view(np.uint16)
            assert np.array_equal(g, want[name].reshape(g.shape)), (v, name)
        for _ in range(100000):
            if ctx.relay_step()[0] == lam.LAM_IDLE:
                break
    ctx.close()


def test_stream_pull_from_master_while_packing():
    od = OMODELS["7b"]
    ctx = lam.Context(lam.Config(model=MODELS["7b"], rollouts=[(0, 0)], chunk_bytes=128 << 20))
    shard = ActorShard(MODELS["7b"], 1, 0, 0)
    shard.fill(SEED, 4)
    rb = RolloutBuffers(MODELS["7b"], 1, 0, 0)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    done = torch.cuda.Event()
    done.record()                      # create the handle (torch makes it lazily)
    assert ctx.publish(4, 0, shard.shards()) == lam.LAM_OK
    assert ctx.pull_stream(0, rb.tp, s.cuda_stream, done.cuda_event, 4) == 4   # FILLING at node 0
    assert drive(ctx, 0) == (4, 0)
    done.synchronize()
    rng = np.random.default_rng(7)
    for name, t in rb.bufs.items():
        idx = rng.integers(0, t.numel(), 64)
        g = t.view(-1).view(torch.int16).cpu().numpy().view(np.uint16)[idx]
        assert np.array_equal(g, dst_elements(od, 1, 0, name, idx, SEED, 4)), name
    ctx.close()


@pytest.mark.parametrize("model,N", [("tiny", 1), ("tiny", 3), ("7b", 1)])
def test_colocated_subscription(model, N):
    """lam_subscribe: the pack writes the colocated TP=1 rollout in the same pass; the rollout's
    buffers equal the oracle's pull of that version, and the master slot is still IMG(v)."""
    od = OMODELS[model]
    C = 64 << 20 if model == "7b" else 16 * 4096
    ctx = lam.Context(lam.Config(model=MODELS[model], fsdp_size=N, actor_devices=[0] * N, rollouts=[(0, 0)],
                                 chunk_bytes=C))
    shards = [ActorShard(MODELS[model], N, r, 0) for r in range(N)]
    rb = RolloutBuffers(MODELS[model], 1, 0, 0)
    for v in (1, 2):
        for sh in shards:
            sh.fill(SEED, v, specials=model == "tiny")
        rb.fill_(0xFFFF)
        torch.cuda.synchronize()
        done = torch.cuda.Event()
        done.record()                  # create the handle (torch makes it lazily)
        ctx.subscribe(0, rb.tp, done.cuda_event)
        assert ctx.pull_state(0)[1] == 1
        for r, sh in enumerate(shards):
            assert ctx.publish(v, r, sh.shards()) == lam.LAM_OK
        assert ctx.pull_state(0) == (v, 0)
        done.synchronize()
        if model == "tiny":
            want = direct_pull(od, 1, 0, SEED, v, specials=True)
            for name, t in rb.bufs.items():
                g = t.view(torch.int16).cpu().numpy().view(np.uint16)
                assert np.array_equal(g, want[name].reshape(g.shape)), name
        else:
            rng = np.random.default_rng(v)
            for name, t in rb.bufs.items():
                idx = rng.integers(0, t.numel(), 64)
                g = t.view(-1).view(torch.int16).cpu().numpy().view(np.uint16)[idx]
                assert np.array_equal(g, dst_elements(od, 1, 0, name, idx, SEED, v)), name
        for _ in range(100000):
            if ctx.relay_step()[0] == lam.LAM_IDLE:
                break
        assert ctx.latest(0) == v
    if model == "tiny":                                     # the master slot is untouched by the fusion
        from oracle.image import image_plan, publish
        from oracle.model import tensors as otensors
        oimg, ohdr = publish(image_plan([s for _, s in otensors(od)], N, C), SEED, 2, specials=True)
        assert np.array_equal(ctx.read_image(0, 2, 0, oimg.size), oimg)
        assert ctx.read_headers(0, 2) == ohdr
    ctx.close()


def test_subscription_refused_when_actor_ranks_span_gpus():
    """the pack writes only the shards packed on the rollout's own GPU, so a colocated
    subscription is refused (LAM_EINVAL) unless every actor rank is on that GPU — the rollout would
    otherwise run with a partial version.  The same rollout pulls the version normally instead."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    od = OMODELS["tiny"]
    ctx = lam.Context(lam.Config(model=MODELS["tiny"], fsdp_size=2, actor_devices=[0, 1], rollouts=[(0, 0)],
                                 chunk_bytes=16 * 4096))
    rb = RolloutBuffers(MODELS["tiny"], 1, 0, 0)
    with pytest.raises(lam.LamError) as e:
        ctx.subscribe(0, rb.tp, None)
    assert e.value.status == lam.LAM_EINVAL
    shards = [ActorShard(MODELS["tiny"], 2, r, r) for r in range(2)]
    for sh in shards:
        sh.fill(SEED, 1, specials=True)
    torch.cuda.synchronize()
    for r, sh in enumerate(shards):
        with torch.cuda.device(r):
            assert ctx.publish(1, r, sh.shards(), torch.cuda.current_stream().cuda_stream) == lam.LAM_OK
    for _ in range(100000):
        if ctx.relay_step()[0] == lam.LAM_IDLE:
            break
    s = torch.cuda.Stream(device=0)
    assert ctx.pull(0, rb.tp, s.cuda_stream) == 1      # gathers rank 1's region from GPU 1 over NVLink
    s.synchronize()
    want = direct_pull(od, 1, 0, SEED, 1, specials=True)
    for name, t in rb.bufs.items():
        g = t.view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(g, want[name].reshape(g.shape)), name
    ctx.close()


def test_stream_pull_of_a_corrupt_version_fails():
    ctx = lam.Context(lam.Config(model=MODELS["tiny"], relays=[[0]], rollouts=[(1, 0)], chunk_bytes=16 * 4096))
    shard = ActorShard(MODELS["tiny"], 1, 0, 0)
    shard.fill(SEED, 1)
    torch.cuda.synchronize()
    assert ctx.publish(1, 0, shard.shards()) == lam.LAM_OK
    torch.cuda.synchronize()                                # packed; relay hop not launched yet
    ptr = ctx.debug_region(0, 1, 0) + 3 * 16 * 4096 + 100
    byte = torch.empty(1, dtype=torch.uint8, device="cuda:0")
    import ctypes
    cp = ctypes.CDLL("libcudart.so.12").cudaMemcpy
    assert cp(ctypes.c_void_p(byte.data_ptr()), ctypes.c_void_p(ptr), ctypes.c_size_t(1), 4) == 0
    byte ^= 0xFF
    assert cp(ctypes.c_void_p(ptr), ctypes.c_void_p(byte.data_ptr()), ctypes.c_size_t(1), 4) == 0
    rb = RolloutBuffers(MODELS["tiny"], 1, 0, 0)
    got = 0
    for _ in range(1000):
        try:
            ctx.relay_step()
        except lam.LamError:
            pass
        got = got or ctx.pull_stream(0, rb.tp, 0, None, 1)
        if got:
            break
    assert got == 1
    t0 = time.time()
    while ctx.pull_state(0)[1] == 1:
        try:
            ctx.relay_step()
        except lam.LamError as e:
            assert e.status == lam.LAM_ECHECKSUM
        assert time.time() - t0 < 60
    assert ctx.pull_state(0) == (1, lam.LAM_ECHECKSUM)
    assert ctx.latest(1) == 0
    ctx.close()

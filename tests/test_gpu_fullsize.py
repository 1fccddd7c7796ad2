"""GPU parity of the cast over EVERY fp32 bit pattern at full 7B size (R1).

The 7B actor shard (7.62 G fp32 elements, FSDP-1) is filled with its own element index mod 2^32 as
fp32 bits — not the generator, whose values sit in a narrow exponent band — so every one of the 2^32
patterns (all exponents, subnormals, +-inf, every NaN payload, every rounding tie) passes through k_pack
at least once.  The expected bf16 of pattern u is the oracle's `rne_bf16(u)` (the definition: nearest
of the two bracketing bf16 values, ties to even, NaN -> 0x7FC0), tabulated once over all 2^32 patterns
on a fork pool over the host cores.  Checked, every element:
  * the plain pack's bucket image (node 0's slot),
  * the colocated subscriber's TP=1 buffers written by the same pack pass (k_pack<true>),
  * the pack of a misaligned shard (odd element offsets: the scalar-load path).
"""
import mmap
import multiprocessing as mp
import os

import numpy as np
import pytest
import torch

from oracle.bf16 import rne_bf16
from oracle.image import image_plan
from oracle.model import MODELS as OMODELS
from oracle.model import tensors as otensors
from paper_2510_12633_b200 import lam
from paper_2510_12633_b200.workload import MODELS, ActorShard, RolloutBuffers

pytestmark = pytest.mark.gpu
TWO32 = 1 << 32
_TABLE = None


def _table_job(i):
    step = 1 << 25
    u = np.arange(i * step, (i + 1) * step, dtype=np.uint64).astype(np.uint32)
    _TABLE[i * step:(i + 1) * step] = rne_bf16(u)
    return i


def rne_table():
    """exp[u] = oracle rne_bf16(u) for every u in [0, 2^32) (8.6 GB, shared with the fork pool)."""
    global _TABLE
    m = mmap.mmap(-1, 2 * TWO32)
    _TABLE = np.frombuffer(m, dtype=np.uint16)
    with mp.get_context("fork").Pool(os.cpu_count() or 1) as pool:
        pool.map(_table_job, range(TWO32 >> 25), chunksize=1)
    return _TABLE


def fill_index_bits(shard: ActorShard):
    """fp32 bits of buffer element i = i mod 2^32 (int32 view, written on the GPU)."""
    b = shard.buf.view(torch.int32)
    step = 1 << 28
    for a in range(0, b.numel(), step):
        n = min(step, b.numel() - a)
        x = torch.arange(a, a + n, dtype=torch.int64, device=b.device) & 0xFFFFFFFF
        b[a:a + n] = torch.where(x >= (1 << 31), x - TWO32, x).to(torch.int32)
    torch.cuda.synchronize()


def want_of(table, start, count):
    """Expected bf16 of `count` consecutive buffer elements starting at buffer element `start`."""
    a = start % TWO32
    if a + count <= TWO32:
        return table[a:a + count]
    return np.concatenate([table[a:], table[:count - (TWO32 - a)]])


def until_idle(ctx):
    for _ in range(10_000_000):
        if ctx.relay_step()[0] == lam.LAM_IDLE:
            return
    raise TimeoutError


def check_image(ctx, v, shard, table):
    od = OMODELS["7b"]
    info = ctx.plan_info()
    plan = image_plan([s for _, s in otensors(od)], 1, info.chunk_bytes)
    img = ctx.read_image(0, v, 0, info.image_bytes).view(np.uint16)
    off = {t: o for (t, _, _), o in zip(shard.pieces, shard.offs)}
    n = 0
    for s in plan.segments:
        got = img[plan.image_offset(s) // 2: plan.image_offset(s) // 2 + s.count]
        want = want_of(table, off[s.tensor_id] + s.elem0, s.count)
        if not np.array_equal(got, want):
            bad = np.nonzero(got != want)[0]
            raise AssertionError(f"tensor {s.tensor_id}: {bad.size} elements differ, first at {bad[0]}")
        n += s.count
    return n


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_7b_every_fp32_bit_pattern_plain_subscriber_misaligned():
    table = rne_table()
    m = MODELS["7b"]
    ctx = lam.Context(lam.Config(model=m, rollouts=[(0, 0)], chunk_bytes=128 << 20))
    shard = ActorShard(m, 1, 0, 0)
    assert shard.buf.numel() >= TWO32              # every pattern occurs at least once
    fill_index_bits(shard)
    rb = RolloutBuffers(m, 1, 0, 0)
    rb.fill_(0xFFFF)
    done = torch.cuda.Event()
    done.record()
    ctx.subscribe(0, rb.tp, done.cuda_event)       # plain image + subscriber buffers in one pack pass
    assert ctx.publish(1, 0, shard.shards(), torch.cuda.current_stream().cuda_stream) == lam.LAM_OK
    until_idle(ctx)
    torch.cuda.synchronize()
    assert ctx.pull_state(0) == (1, 0)
    assert check_image(ctx, 1, shard, table) == shard.numel
    off = {t: o for (t, _, _), o in zip(shard.pieces, shard.offs)}
    for d in lam.vllm_layout(m, 1):                # TP=1: every part is a whole tensor, in part order
        got = rb.bufs[d.name].view(-1).view(torch.int16).cpu().numpy().view(np.uint16)
        want, a = [], 0
        for t, _ in d.parts:
            cnt = int(np.prod(lam.model_tensors(m)[t][1]))
            want.append(want_of(table, off[t], cnt))
            a += cnt
        assert np.array_equal(got, np.concatenate(want)), d.name
    del rb, shard
    torch.cuda.empty_cache()
    mis = ActorShard(m, 1, 0, 0, misalign=True)    # odd element offsets: unaligned (scalar-load) pack path
    assert any(o % 4 for o in mis.offs)
    fill_index_bits(mis)
    assert ctx.publish(2, 0, mis.shards(), torch.cuda.current_stream().cuda_stream) == lam.LAM_OK
    until_idle(ctx)
    assert check_image(ctx, 2, mis, table) == mis.numel
    ctx.close()

"""Config 5 (continuous-publish stress), scaled: the actor publishes every step while rollouts pull at
random times.  Which version a pull sees is timing-dependent, so only the invariants of SURVEY C8 are
checked (oracle/invariants.py): the version was published, per-rollout versions never decrease, a
pull returns at least the latest version complete when it started, and the pulled bytes equal the
oracle's pull of exactly that version (no torn or mixed version).  The actor side also checks the
stall contract: lam_publish returns in microseconds and never blocks on a relay."""
import random
import time

import numpy as np
import pytest
import torch

from oracle import invariants
from oracle.model import MODELS as OMODELS
from oracle.tp import direct_pull
from paper_2510_12633_b200 import lam
from paper_2510_12633_b200.workload import MODELS, ActorShard, RolloutBuffers
from synth import SEED

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [0, 1])
def test_stress_invariants(seed):
    n = torch.cuda.device_count()
    relay_devs = [1 % n, 2 % n] if n >= 3 else [0, 0]
    rng = random.Random(seed)
    od = OMODELS["tiny"]
    ctx = lam.Context(lam.Config(model=MODELS["tiny"], relays=[[relay_devs[0]], [relay_devs[1]]],
                                 rollouts=[(1, relay_devs[0]), (2, relay_devs[1]), (2, relay_devs[1])],
                                 chunk_bytes=32 * 4096, slots=2))
    shard = ActorShard(MODELS["tiny"], 1, 0, 0)
    actor = torch.cuda.Stream(device=0)
    busy = torch.randn(2048, 2048, device="cuda:0")
    bufs = [RolloutBuffers(MODELS["tiny"], tp, 0, relay_devs[[0, 1, 1][i]]) for i, tp in enumerate([1, 1, 2])]
    streams = [torch.cuda.Stream(device=b.bufs[next(iter(b.bufs))].device) for b in bufs]
    published, records, stalls, pending = set(), [], [], []
    reads_done = None
    oracle_cache = {}

    def expect(v, tp):
        if (v, tp) not in oracle_cache:
            oracle_cache[(v, tp)] = direct_pull(od, tp, 0, SEED, v, specials=True)
        return oracle_cache[(v, tp)]

    def verify(i, v, latest0):
        streams[i].synchronize()
        want = expect(v, [1, 1, 2][i]) if v else None
        ok = True
        if v:
            for name, t in bufs[i].bufs.items():
                g = t.view(torch.int16).cpu().numpy().view(np.uint16)
                ok &= bool(np.array_equal(g, want[name].reshape(g.shape)))
        records.append(invariants.PullRecord(i, v, latest0, ok))

    for v in range(1, 41):
        with torch.cuda.stream(actor):
            if reads_done is not None:
                actor.wait_event(reads_done)               # optimizer waits for the previous pack's reads
            for _ in range(rng.choice([0, 1, 4])):
                busy = busy @ busy * 1e-3                   # a "training step" of random length
            torch.cuda._sleep(rng.choice([0, 100_000, 2_000_000]))
        shard.fill(SEED, v, specials=True, stream=actor.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(actor)                   # create the handle (torch makes it lazily)
        t0 = time.perf_counter()
        st = ctx.publish(v, 0, shard.shards(), actor.cuda_stream, ev.cuda_event)
        stalls.append(time.perf_counter() - t0)
        if st == lam.LAM_OK:
            published.add(v)
            reads_done = ev
        for _ in range(rng.randint(0, 6)):
            ctx.relay_step()
            i = rng.randrange(3)
            if rng.random() < 0.5:
                node = [1, 2, 2][i]
                latest0 = ctx.latest(node)
                got = ctx.pull(i, bufs[i].tp, streams[i].cuda_stream)
                verify(i, got, latest0)
            time.sleep(rng.choice([0, 0.0005, 0.002]))
    for _ in range(200000):
        if ctx.relay_step()[0] == lam.LAM_IDLE:
            break
    for i in range(3):                                        # quiescent: everyone gets the newest
        node = [1, 2, 2][i]
        latest0 = ctx.latest(node)
        got = ctx.pull(i, bufs[i].tp, streams[i].cuda_stream)
        verify(i, got, latest0)
        assert got == max(published)
    errs = invariants.check(published, records)
    assert errs == [], errs[:10]
    assert len([r for r in records if r.version]) >= 20
    stalls.sort()
    assert stalls[len(stalls) // 2] < 2e-3, f"publish host time p50 {stalls[len(stalls) // 2] * 1e3:.2f} ms"
    st = ctx.stats()
    print(f"stress: published {len(published)}/40, busy {st['publish_busy']}, skipped {st['versions_skipped']}, "
          f"pulls {st['pulls']}, publish p50 {stalls[len(stalls) // 2] * 1e6:.0f} us max {stalls[-1] * 1e6:.0f} us")
    ctx.close()

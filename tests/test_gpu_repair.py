"""NEXT-1 on the GPU: fault-tolerant chain broadcast (detection, O(1) rebuild,
repair in under a second; SPEC L604-612, L634 digest agreement).

* one GPU: chain 0 -> 1 -> 2, relay 1 fails between versions; the next version reaches relay 2
  straight from the master and its pulls are bit-exact; the failed relay serves nothing.
* >= 2 GPUs, 7B-sized: relay 1 fails while the broadcast is in flight; relay 2 re-points to the
  master and resumes from its lowest missing chunk; every chunk header at relay 2 (the checksum
  of its own bytes) equals the master's, sampled chunks equal the oracle's IMG(v), repair < 1 s.
"""
import time

import numpy as np
import pytest
import torch

from oracle.image import image_plan, publish, publish_chunk
from oracle.model import MODELS as OMODELS
from oracle.model import tensors as otensors
from oracle.tp import direct_pull
from paper_2510_12633_b200 import lam
from paper_2510_12633_b200.workload import MODELS, ActorShard, RolloutBuffers
from synth import SEED

pytestmark = pytest.mark.gpu


def until_idle(ctx, timeout=120.0):
    t0 = time.time()
    while ctx.relay_step()[0] != lam.LAM_IDLE:
        if time.time() - t0 > timeout:
            raise TimeoutError("relay never went idle")


def test_failed_relay_is_bypassed_one_gpu():
    od = OMODELS["tiny"]
    C = 16 * 4096
    ctx = lam.Context(lam.Config(model=MODELS["tiny"], relays=[[0], [0]], rollouts=[(1, 0), (2, 0)], chunk_bytes=C))
    shard = ActorShard(MODELS["tiny"], 1, 0, 0)
    for v in (1, 2):
        shard.fill(SEED, v, specials=True)
        torch.cuda.synchronize()
        assert ctx.publish(v, 0, shard.shards()) == lam.LAM_OK
        until_idle(ctx)
        if v == 1:
            assert [ctx.latest(n) for n in range(3)] == [1, 1, 1]
            ctx.fail_node(1)
    assert [ctx.latest(n) for n in range(3)] == [2, 1, 2]
    plan = image_plan([s for _, s in otensors(od)], 1, C)
    oimg, ohdr = publish(plan, SEED, 2, specials=True)
    assert np.array_equal(ctx.read_image(2, 2, 0, oimg.size), oimg)
    assert ctx.read_headers(2, 2) == ohdr
    rb = RolloutBuffers(MODELS["tiny"], 1, 0, 0)
    assert ctx.pull(0, rb.tp, 0) == 0                       # relay 1 is out of the chain
    assert ctx.pull(1, rb.tp, 0) == 2
    torch.cuda.synchronize()
    want = direct_pull(od, 1, 0, SEED, 2, specials=True)
    for name, t in rb.bufs.items():
        g = t.view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(g, want[name].reshape(g.shape)), name
    assert ctx.stats()["chain_rebuilds"] == 1
    ctx.close()


@pytest.mark.parametrize("delay_ms", [2, 8])
def test_fail_mid_broadcast_resumes(delay_ms):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    od = OMODELS["7b"]
    C = 64 << 20
    # master on GPU 0 -> relay 1 on GPU 1 -> relay 2 on GPU 0 (relay 2 re-points to the master)
    ctx = lam.Context(lam.Config(model=MODELS["7b"], relays=[[1], [0]], rollouts=[(2, 0)], chunk_bytes=C))
    shard = ActorShard(MODELS["7b"], 1, 0, 0)
    shard.fill(SEED, 1)
    torch.cuda.synchronize()
    assert ctx.publish(1, 0, shard.shards()) == lam.LAM_OK
    ctx.relay_step()                                        # launches relay 1 and relay 2 (pipelined)
    time.sleep(delay_ms / 1e3)
    ctx.fail_node(1)
    until_idle(ctx)
    st = ctx.stats()
    assert ctx.latest(2) == 1 and ctx.latest(0) == 1
    assert st["chain_rebuilds"] == 1
    if st["chain_resumes"]:
        assert st["last_repair_ns"] < 1e9                   # repair in under a second
    info = ctx.plan_info()
    h0, h2 = ctx.read_headers(0, 1), ctx.read_headers(2, 1)
    assert h0 == h2                                         # digest agreement, every chunk
    plan = image_plan([s for _, s in otensors(od)], 1, C)
    for g in sorted({0, info.total_chunks // 3, info.total_chunks - 1}):
        want = publish_chunk(plan, g, SEED, 1)
        assert np.array_equal(ctx.read_image(2, 1, g * C, want.size), want), g
    print(f"fail after {delay_ms} ms: resumes={st['chain_resumes']} repair={st['last_repair_ns'] / 1e6:.2f} ms")
    ctx.close()


def test_sigkill_relay_process_mid_broadcast(tmp_path):
    """NEXT-1 end to end: three rank processes (actor GPU 0 -> relay 1 on GPU 1 ->
    relay 2 on GPU 2), 7B; the relay-1 PROCESS is SIGKILLed while its hop is running.  The survivors'
    heartbeats declare it dead, the chain is rebuilt in O(1) (node 2 <- node 0), node 2 resumes from its
    lowest missing chunk; digest agreement of every chunk header with node 0 and two chunks == the
    oracle's; repair (failure declared -> resumed hop launched) < 1 s."""
    import json
    import os
    import socket
    import subprocess
    import sys
    if torch.cuda.device_count() < 3:
        pytest.skip("needs >= 3 GPUs")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "kill")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    procs = []
    for r in range(3):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="3", LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(root, "tests", "kill_worker.py"), "--out", out,
                                       "--kill-after-ms", "80", "--hop-ctas", "2"], env=env, cwd=root,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = [p.communicate(timeout=400)[0] for p in procs]
    assert procs[1].returncode == -9, logs[1][-2000:]
    assert procs[0].returncode == 0 and procs[2].returncode == 0, (logs[0][-2000:], logs[2][-2000:])
    r2 = json.load(open(out + ".2"))
    assert r2["ok"] and r2["digest_agreement"], r2
    assert r2["latest"][2] == 1 and r2["latest"][0] == 1
    st = r2["stats"]
    assert st["chain_rebuilds"] == 1, st
    assert st["chain_resumes"] >= 1, st                      # killed mid-broadcast: node 2 resumed
    assert 0 < st["last_repair_ns"] < 1e9, st                # repair in under a second
    print(f"SIGKILL relay: repair {st['last_repair_ns'] / 1e6:.1f} ms, total {r2['t_total_s']:.2f} s")

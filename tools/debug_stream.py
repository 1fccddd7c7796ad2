"""Debug helper: streaming vs ordinary pull of the same version (tiny, TP=2 rank 1)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from oracle.model import MODELS as OMODELS
from oracle.tp import direct_pull
from paper_2510_12633_b200 import lam
from paper_2510_12633_b200.workload import MODELS, ActorShard, RolloutBuffers
from synth import SEED
n = torch.cuda.device_count(); devs = [1 % n, 2 % n]; tp = 2
od = OMODELS["tiny"]
ctx = lam.Context(lam.Config(model=MODELS["tiny"], relays=[[devs[0]], [devs[1]]], rollouts=[(2, devs[1]), (2, devs[1])], chunk_bytes=8 * 4096))
shard = ActorShard(MODELS["tiny"], 1, 0, 0)
rb = RolloutBuffers(MODELS["tiny"], tp, 1, devs[1]); rb2 = RolloutBuffers(MODELS["tiny"], tp, 1, devs[1])
s = torch.cuda.Stream(device=devs[1])
info = ctx.plan_info()
for v in range(1, 7):
    shard.fill(SEED, v, specials=True); torch.cuda.synchronize(); rb.fill_(0xFFFF); torch.cuda.synchronize()
    assert ctx.publish(v, 0, shard.shards()) == lam.LAM_OK
    got = 0; polls = 0
    while got == 0:
        ctx.relay_step(); got = ctx.pull_stream(0, rb.tp, s.cuda_stream, None, v); polls += 1
    st0 = ctx.latest(2)
    while ctx.pull_state(0)[1] == 1: ctx.relay_step()
    s.synchronize()
    while ctx.relay_step()[0] != lam.LAM_IDLE: pass
    assert ctx.pull(1, rb2.tp, s.cuda_stream) == v; s.synchronize()
    want = direct_pull(od, tp, 1, SEED, v, specials=True)
    bad = [k for k, t in rb.bufs.items() if not np.array_equal(t.view(torch.int16).cpu().numpy().view(np.uint16), want[k].reshape(t.shape))]
    bad2 = [k for k, t in rb2.bufs.items() if not np.array_equal(t.view(torch.int16).cpu().numpy().view(np.uint16), want[k].reshape(t.shape))]
    detail = ""
    if bad:
        t = rb.bufs[bad[0]].view(torch.int16).cpu().numpy().view(np.uint16); w = want[bad[0]].reshape(t.shape)
        rows = np.nonzero((t != w).any(axis=-1) if t.ndim == 2 else (t != w))[0]
        detail = f"rows {rows[:3]}..{rows[-1:]} n={rows.size}; stale==0xFFFF: {bool((t[rows[0]] == 0xFFFF).all() if t.ndim==2 else False)}"
    print(f"v={v} polls={polls} latest_at_start={st0} stream_bad={bad[:3]} ordinary_bad={bad2[:3]} {detail}", flush=True)
ctx.close()

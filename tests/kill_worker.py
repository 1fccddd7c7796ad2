"""Rank process of the SIGKILL-mid-broadcast test (tests/test_gpu_repair.py), one per GPU, started by
the test with RANK / WORLD_SIZE / MASTER_* in the environment (not torchrun: its agent would tear the
whole group down when a rank dies — here the survivors must carry on by themselves).

Chain: node 0 = the actor's slots (rank 0, GPU 0) -> relay 1 (rank 1, GPU 1) -> relay 2 (rank 2, GPU 2),
7B, heartbeat_timeout_s set, hops throttled (few CTAs) so that the broadcast lasts long enough to be
cut.  Rank 1 SIGKILLs itself once its hop has been running for `--kill-after-ms`.  The survivors keep
calling lam_relay_step (which runs the heartbeat check): they must declare process 1 dead, rebuild the
chain (node 2's predecessor becomes node 0) and node 2 must resume from its lowest missing chunk.
Rank 2 then checks, against the oracle, digest agreement of every chunk header with node 0 and two
whole chunks, and writes its verdict to `--out`.  No collective runs after the kill."""
import argparse
import json
import os
import signal
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.checksum import chunk_checksum  # noqa: E402
from oracle.image import image_plan, publish_chunk  # noqa: E402
from oracle.model import MODELS as OMODELS  # noqa: E402
from oracle.model import tensors as otensors  # noqa: E402
from paper_2510_12633_b200 import lam  # noqa: E402
from paper_2510_12633_b200.workload import MODELS, ActorShard  # noqa: E402
from synth import SEED  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kill-after-ms", type=float, default=60)
    ap.add_argument("--hop-ctas", type=int, default=2)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rank, N = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    C = 64 << 20
    cfg = lam.Config(model=MODELS["7b"], relays=[[1], [2]], rollouts=[], chunk_bytes=C, proc_rank=rank,
                     n_procs=N, proc_of_device={d: d for d in range(N)},
                     shm_name=f"lam_kill_{os.environ['MASTER_PORT']}", hop_ctas=a.hop_ctas,
                     heartbeat_timeout_s=0.3, spin_timeout_s=60)
    ctx = lam.Context(cfg)
    blobs = [None] * N
    dist.all_gather_object(blobs, ctx.export_ipc())
    for p, b in enumerate(blobs):
        if p != rank:
            ctx.import_ipc(p, b)
    ctx.connect()
    shard = ActorShard(MODELS["7b"], 1, 0, 0) if rank == 0 else None
    if shard:
        shard.fill(SEED, 1)
        torch.cuda.synchronize()
    dist.barrier()                                   # the last collective
    t0 = time.time()
    if rank == 0:
        assert ctx.publish(1, 0, shard.shards(), 0) == lam.LAM_OK
    t_hop = None
    while True:
        ctx.relay_step()                             # progress + heartbeat (every process)
        if rank == 1:
            if t_hop is None and ctx.stats()["hops_launched"] >= 1:
                t_hop = time.time()
            if t_hop is not None and time.time() - t_hop >= a.kill_after_ms / 1e3:
                os.kill(os.getpid(), signal.SIGKILL)     # the relay process dies mid-broadcast
        if rank in (0, 2) and ctx.latest(2) >= 1:
            break
        if time.time() - t0 > 120:
            json.dump(dict(rank=rank, ok=False, why="timeout", stats=ctx.stats(),
                           latest=[ctx.latest(n) for n in range(3)]), open(a.out + f".{rank}", "w"))
            os._exit(3)
    res = dict(rank=rank, ok=True, latest=[ctx.latest(n) for n in range(3)], stats=ctx.stats(),
               t_total_s=time.time() - t0)
    if rank == 2:
        od = OMODELS["7b"]
        plan = image_plan([s for _, s in otensors(od)], 1, C)
        h0, h2 = ctx.read_headers(0, 1), ctx.read_headers(2, 1)
        res["digest_agreement"] = h0 == h2
        chunks = sorted({1, plan.total_chunks - 1})
        ok = []
        for g in chunks:
            want = publish_chunk(plan, g, SEED, 1)
            ok.append(bool(np.array_equal(ctx.read_image(2, 1, g * C, want.size), want))
                      and (h2[g]["s1"], h2[g]["s2"]) == chunk_checksum(want))
        res["chunks_vs_oracle"] = dict(zip(map(str, chunks), ok))
        res["ok"] = res["digest_agreement"] and all(ok)
    json.dump(res, open(a.out + f".{rank}", "w"))
    if rank == 0:                                    # keep node 0's memory alive until rank 2 has read it
        t1 = time.time()
        while not os.path.exists(a.out + ".2") and time.time() - t1 < 180:
            time.sleep(0.05)
    sys.stdout.flush()
    os._exit(0)                                      # no collective: the group has a dead member


if __name__ == "__main__":
    main()

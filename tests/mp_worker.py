"""Multi-process parity worker (one process per GPU, launched by tests/test_gpu_multiproc.py via torchrun).

Runs bench.py's placement (`topology`) through the C ABI exactly as the bench does — ranks exchange CUDA
IPC handles, the version table lives in POSIX shared memory — publishes several versions and checks,
on every rank, against the oracle:
  * every node's image bytes and chunk headers == IMG(v) (tiny: full; 7B: sampled chunks),
  * every rollout's pulled TP buffers == TP_r(RNE_bf16(W_v)) (tiny: full; 7B: sampled elements).
Exit code 0 iff every check passed on this rank.
"""
import argparse
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle.checksum import chunk_checksum  # noqa: E402
from oracle.image import image_plan, publish, publish_chunk  # noqa: E402
from oracle.model import MODELS as OMODELS  # noqa: E402
from oracle.model import tensors as otensors  # noqa: E402
from oracle.tp import direct_pull, dst_elements  # noqa: E402
from paper_2510_12633_b200 import lam  # noqa: E402
from paper_2510_12633_b200.workload import MODELS, ActorShard, RolloutBuffers  # noqa: E402
from synth import SEED  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="chain")
    ap.add_argument("--model", default="tiny")
    ap.add_argument("--tp", type=int, default=0)
    ap.add_argument("--versions", type=int, default=2)
    ap.add_argument("--chunk-kb", type=int, default=64)
    ap.add_argument("--hop-mode", type=int, default=0)
    ap.add_argument("--stream", action="store_true", help="rollouts use lam_pull_stream during the broadcast")
    a = ap.parse_args()
    import faulthandler
    faulthandler.dump_traceback_later(float(os.environ.get("LAM_MP_WATCHDOG", "500")), exit=True)
    rank, N = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    T = bench.topology(a.config, N, a.tp)
    ro = T["rollouts"]
    specials = a.model == "tiny"
    cfg = lam.Config(model=MODELS[a.model], fsdp_size=T["fsdp"], actor_devices=T["actors"], relays=T["relays"],
                     rollouts=[(n, d) for n, d, _, _ in ro], chunk_bytes=a.chunk_kb << 10, proc_rank=rank,
                     n_procs=N, proc_of_device={d: d for d in range(N)},
                     shm_name=f"lam_mp_{os.environ.get('MASTER_PORT', '0')}_{os.getppid()}", spin_timeout_s=60,
                     hop_mode=a.hop_mode, host_relays=T.get("host_relays", []))
    ctx = lam.Context(cfg)
    blobs = [None] * N
    dist.all_gather_object(blobs, ctx.export_ipc())
    for p, b in enumerate(blobs):
        if p != rank:
            ctx.import_ipc(p, b)
    ctx.connect()
    dist.barrier()
    my_ranks = [r for r, d in enumerate(T["actors"]) if d == rank]
    shards = {r: ActorShard(MODELS[a.model], T["fsdp"], r, rank) for r in my_ranks}
    mine = [rid for rid, (_, d, _, _) in enumerate(ro) if d == rank]
    od = OMODELS[a.model]
    info = ctx.plan_info()
    C = info.chunk_bytes
    plan = image_plan([s for _, s in otensors(od)], T["fsdp"], C)
    failures = []
    for v in range(1, a.versions + 1):
        for r in my_ranks:
            shards[r].fill(SEED, v, specials)
        torch.cuda.synchronize()
        dist.barrier()
        for r in my_ranks:
            assert ctx.publish(v, r, shards[r].shards(), torch.cuda.current_stream().cuda_stream) == lam.LAM_OK
        t0 = time.time()
        streamed = {}
        if a.stream:                                # start every rollout's pull while v is in flight
            ss = torch.cuda.Stream()
            todo = list(mine)
            while todo or any(ctx.pull_state(rid)[1] == 1 for rid in streamed):
                ctx.relay_step()
                for rid in list(todo):
                    node, dev, tp, tr = ro[rid]
                    rb = RolloutBuffers(MODELS[a.model], tp, tr, dev) if rid not in streamed else streamed[rid]
                    streamed[rid] = rb
                    if ctx.pull_stream(rid, rb.tp, ss.cuda_stream, None, v):
                        todo.remove(rid)
                if time.time() - t0 > 120:
                    raise TimeoutError(f"rank {rank}: streaming pulls of v{v} never finished")
            ss.synchronize()
        while not all(ctx.latest(n) >= v for n in range(len(T["relays"]) + 1)):
            ctx.relay_step()
            if time.time() - t0 > 120:
                raise TimeoutError(f"rank {rank}: version {v} never completed everywhere")
        # every rank checks one node's image (spread the oracle work), rank 0 checks node 0
        nodes = list(range(len(T["relays"]) + 1))
        for node in nodes[rank::N]:
            if a.model == "tiny":
                oimg, ohdr = publish(plan, SEED, v, specials=True)
                got = ctx.read_image(node, v, 0, info.image_bytes)
                if not np.array_equal(got, oimg):
                    failures.append(f"node {node} v{v}: image differs at {np.nonzero(got != oimg)[0][:4]}")
                if ctx.read_headers(node, v) != ohdr:
                    failures.append(f"node {node} v{v}: headers differ")
            else:
                hdr = ctx.read_headers(node, v)
                for g in sorted({0, plan.total_chunks // 2, plan.total_chunks - 1}):
                    want = publish_chunk(plan, g, SEED, v)
                    if not np.array_equal(ctx.read_image(node, v, g * C, want.size), want):
                        failures.append(f"node {node} v{v}: chunk {g} differs")
                    if (hdr[g]["s1"], hdr[g]["s2"]) != chunk_checksum(want):
                        failures.append(f"node {node} v{v}: header {g} differs")
        s = torch.cuda.Stream()
        for rid in mine:
            node, dev, tp, tr = ro[rid]
            if rid in streamed:
                rb = streamed[rid]
                got_v = ctx.pull_state(rid)[0]
            else:
                rb = RolloutBuffers(MODELS[a.model], tp, tr, dev)
                got_v = ctx.pull(rid, rb.tp, s.cuda_stream)
                s.synchronize()
            if got_v != v:
                failures.append(f"rollout {rid}: pulled {got_v}, expected {v}")
            if a.model == "tiny":
                want = direct_pull(od, tp, tr, SEED, v, specials=True)
                for name, t in rb.bufs.items():
                    g = t.view(torch.int16).cpu().numpy().view(np.uint16)
                    if not np.array_equal(g, want[name].reshape(g.shape)):
                        failures.append(f"rollout {rid} v{v}: {name} differs")
            else:
                rng = np.random.default_rng(rid * 100 + v)
                for name, t in rb.bufs.items():
                    idx = rng.integers(0, t.numel(), 64)
                    g = t.view(-1).view(torch.int16).cpu().numpy().view(np.uint16)[idx]
                    if not np.array_equal(g, dst_elements(od, tp, tr, name, idx, SEED, v)):
                        failures.append(f"rollout {rid} v{v}: {name} sampled elements differ")
            del rb
        ctx.relay_step()
        dist.barrier()
    st = ctx.stats()
    ctx.close()
    dist.barrier()
    if failures:
        print(f"rank {rank} FAILED:\n  " + "\n  ".join(failures[:20]), flush=True)
        sys.exit(1)
    print(f"rank {rank} ok: {a.config} {a.model} N={N} versions={a.versions} stats={st}", flush=True)


if __name__ == "__main__":
    main()

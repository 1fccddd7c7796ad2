#!/usr/bin/env python
"""Comparator (not the product path): the paper's "GPU-based global synchronization" baseline
("each actor model partition is broadcast to the corresponding model shards on each
rollout ... uses NCCL"), on the bench's config-2 workload: actor FSDP-1 on GPU 0 casts its fp32
masters to bf16 with torch (`.to(bfloat16)` into one flat buffer) and NCCL-broadcasts the 15.23 GB
snapshot to every rank; TP=1 rollouts use the broadcast buffer in place (no reshard needed).

    python -m torch.distributed.run --nproc-per-node N tools/nccl_baseline.py --steps 5 --warmup 2

Prints one JSON line (max over ranks of CUDA-event time per step).  NCCL_ALGO / NCCL_PROTO from the
environment are reported.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_12633_b200 import lam  # noqa: E402
from paper_2510_12633_b200.workload import MODELS  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    rank, N = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    tensors = lam.model_tensors(MODELS[a.model])
    numels = [int(torch.tensor(s).prod()) for _, s in tensors]
    P = sum(numels)
    flat = torch.empty(P, dtype=torch.bfloat16, device="cuda")
    masters = []
    if rank == 0:
        for t, n in enumerate(numels):
            m = torch.empty(n, dtype=torch.float32, device="cuda")
            synth.fill_device(m.data_ptr(), n, synth.SEED, 1, t)
            masters.append(m)
    torch.cuda.synchronize()

    def step():
        if rank == 0:
            o = 0
            for m, n in zip(masters, numels):
                flat[o:o + n].copy_(m)               # torch fp32 -> bf16 cast (RNE)
                o += n
        dist.broadcast(flat, src=0)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.steps):
        step()
    e.record()
    torch.cuda.synchronize()
    ms = torch.tensor([s.elapsed_time(e) / a.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    # broadcast alone, for the bandwidth figure
    dist.barrier()
    s.record()
    for _ in range(a.steps):
        dist.broadcast(flat, src=0)
    e.record()
    torch.cuda.synchronize()
    bms = torch.tensor([s.elapsed_time(e) / a.steps], device="cuda")
    dist.all_reduce(bms, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps(dict(impl="nccl-broadcast (comparator)", model=a.model, n_gpus=N, params=P,
                              ms_per_step=ms.item(), broadcast_ms=bms.item(),
                              broadcast_GBps=2 * P / (bms.item() / 1e3) / 1e9,
                              nccl_algo=os.environ.get("NCCL_ALGO"), nccl_proto=os.environ.get("NCCL_PROTO"),
                              note="torch cast on rank 0 + NCCL broadcast of the flat bf16 snapshot; TP=1 "
                                   "rollouts use the buffer in place")))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

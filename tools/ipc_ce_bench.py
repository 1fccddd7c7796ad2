"""Copy-engine NVLink bandwidth through CUDA IPC (one process per GPU, as the relay runtime runs) vs
peer access inside one process: does the IPC mapping change what cudaMemcpyAsync reaches?

  python tools/ipc_ce_bench.py            (needs 2 GPUs)

Process A (GPU 0) owns a 2 GiB source buffer and exports it (torch CUDA IPC = cudaIpcGetMemHandle);
process B (GPU 1) copies it into local memory with cudaMemcpyAsync (copy engines, the CE hop's
pull direction) in pieces of 128 MiB / 1 GiB, then the reverse push (B writes into A's exported
buffer).  Single-process peer copies of the same sizes for comparison.  CUDA events, best of 5."""
import os
import sys

import torch
import torch.multiprocessing as mp

GB = 1 << 30


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def copy_pieces(dst, src, piece):
    n = src.numel()
    for o in range(0, n, piece):
        dst[o:o + piece].copy_(src[o:o + piece], non_blocking=True)


def receiver(q, res):
    torch.cuda.set_device(1)
    src, remote_dst = q.get()                      # IPC-mapped tensors of process A (GPU 0)
    dst = torch.empty(2 * GB, dtype=torch.uint8, device="cuda:1")
    own = torch.empty(2 * GB, dtype=torch.uint8, device="cuda:1")
    out = {}
    for piece in (128 << 20, GB):
        ms = timed(lambda: copy_pieces(dst, src, piece))
        out[f"ipc pull {piece >> 20} MiB"] = 2 * GB / (ms / 1e3) / 1e9
        ms = timed(lambda: copy_pieces(remote_dst, own, piece))
        out[f"ipc push {piece >> 20} MiB"] = 2 * GB / (ms / 1e3) / 1e9
    res.put(out)


def main():
    if torch.cuda.device_count() < 2:
        print("needs 2 GPUs")
        return
    # single process: peer access
    a = torch.empty(2 * GB, dtype=torch.uint8, device="cuda:0").fill_(1)
    b = torch.empty(2 * GB, dtype=torch.uint8, device="cuda:1")
    torch.cuda.set_device(1)
    for piece in (128 << 20, GB):
        ms = timed(lambda: copy_pieces(b, a, piece))
        print(f"peer pull (stream on receiver) {piece >> 20:5d} MiB pieces: {2 * GB / (ms / 1e3) / 1e9:7.1f} GB/s")
    torch.cuda.set_device(0)
    for piece in (128 << 20, GB):
        ms = timed(lambda: copy_pieces(b, a, piece))
        print(f"peer push (stream on sender)   {piece >> 20:5d} MiB pieces: {2 * GB / (ms / 1e3) / 1e9:7.1f} GB/s")
    del b
    ctx = mp.get_context("spawn")
    q, res = ctx.Queue(), ctx.Queue()
    p = ctx.Process(target=receiver, args=(q, res))
    p.start()
    rdst = torch.empty(2 * GB, dtype=torch.uint8, device="cuda:0")
    q.put((a, rdst))
    for k, v in res.get(timeout=300).items():
        print(f"{k:28s}: {v:7.1f} GB/s")
    p.join()


if __name__ == "__main__":
    sys.exit(main())

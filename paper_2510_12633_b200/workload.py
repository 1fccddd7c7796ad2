"""Workload plumbing for tests and bench.py: Qwen2.5-shaped model dims, the actor's fp32 FSDP shards in
HBM (filled on the GPU by synth's generator), and rollout TP destination buffers.

torch is used only for device memory and streams here; nothing of the method runs in this module.
The FSDP split below is the *caller's* layout (what torch FSDP would hand the actor); the library
re-derives its own image plan from the same rule and checks coverage at publish time.
"""
from __future__ import annotations

import torch

import synth

from . import lam

# Qwen2.5 public configs + our tiny model.
MODELS = {
    "tiny": lam.dims(256, 1024, 4, 8, 4, 32, 12288),
    "7b": lam.dims(3584, 18944, 28, 28, 4, 128, 152064),
    "32b": lam.dims(5120, 27648, 64, 40, 8, 128, 152064),
    "72b": lam.dims(8192, 29568, 80, 64, 8, 128, 152064),
    "odd": lam.dims(64, 192, 2, 8, 2, 8, 130),   # vocab padding + KV-head replication cases
}


def _numel(shape):
    n = 1
    for s in shape:
        n *= s
    return n


def fsdp_pieces(tensors, N: int, rank: int, layout: int):
    """(tensor_id, elem0, count) owned by `rank` (FSDP2: torch.chunk rows; FSDP1: flat equal split)."""
    out = []
    if layout == lam.LAM_FSDP2_DIM0:
        for t, (_, shp) in enumerate(tensors):
            d0, row = shp[0], _numel(shp) // shp[0]
            per = -(-d0 // N)
            a, b = rank * per, min(d0, (rank + 1) * per)
            if b > a:
                out.append((t, a * row, (b - a) * row))
    else:
        sizes = [_numel(s) for _, s in tensors]
        P = sum(sizes)
        each = -(-P // N)
        a, b = rank * each, min(P, (rank + 1) * each)
        start = 0
        for t, n in enumerate(sizes):
            lo, hi = max(a, start), min(b, start + n)
            if hi > lo:
                out.append((t, lo - start, hi - lo))
            start += n
    return out


class ActorShard:
    """fp32 master shard of one actor rank, one flat HBM buffer carved into 16-B aligned pieces."""

    def __init__(self, model: lam.lam_model_dims, N: int, rank: int, device: int,
                 layout: int = lam.LAM_FSDP2_DIM0, misalign: bool = False):
        self.tensors = lam.model_tensors(model)
        self.pieces = fsdp_pieces(self.tensors, N, rank, layout)
        self.device = device
        offs, o = [], 0
        for (_, _, cnt) in self.pieces:
            o += 1 if misalign else 0            # odd element offsets exercise the unaligned pack path
            offs.append(o)
            o += -(-cnt // 4) * 4
        self.buf = torch.empty(max(o, 1), dtype=torch.float32, device=f"cuda:{device}")
        self.offs = offs
        self.numel = sum(c for _, _, c in self.pieces)

    def fill(self, seed: int, version: int, specials: bool = False, stream: int = 0) -> None:
        base = self.buf.data_ptr()
        with torch.cuda.device(self.device):
            for (t, e0, cnt), o in zip(self.pieces, self.offs):
                synth.fill_device(base + 4 * o, cnt, seed, version, t, e0, specials, stream)

    def shards(self):
        base = self.buf.data_ptr()
        return [(t, e0, cnt, base + 4 * o) for (t, e0, cnt), o in zip(self.pieces, self.offs)]


class RolloutBuffers:
    """bf16 destination buffers of one rollout TP rank in the vLLM Qwen2 convention."""

    def __init__(self, model: lam.lam_model_dims, tp: int, rank: int, device: int, transpose: bool = False):
        """`transpose`: every 2-D buffer K-major, i.e. shaped (cols, rows) (R16)."""
        self.layout = lam.vllm_layout(model, tp)
        self.bufs = {}
        dsts = []
        for d in self.layout:
            two_d = d.cols > 1   # (a rows x 1 matrix has the same bytes either way)
            shape = ((d.cols, d.rows) if transpose else (d.rows, d.cols)) if two_d else (d.rows,)
            t = torch.empty(shape, dtype=torch.bfloat16, device=f"cuda:{device}")
            self.bufs[d.name] = t
            dsts.append((d.parts, t.data_ptr(), 0, transpose and two_d))
        self.tp = lam.TPLayout(tp, rank, dsts)
        self.bytes = sum(t.numel() * 2 for t in self.bufs.values())

    def fill_(self, value: int = 0xFFFF) -> None:
        for t in self.bufs.values():
            t.view(torch.int16).fill_(value - 65536 if value > 32767 else value)

"""Pull-time TP reshard rules and the pull itself (oracle).

Passages followed:
  * PAPER L654-655 (§4.2): the relay "reshards them according to the rollout sharding strategy
    (e.g., tensor parallelism among GPUs a rollout runs on)".  The north star moves this reshard
    from the master relay to pull time; the output bytes are the same (SURVEY reading 6).
  * PAPER L550 (§3.2 step 7) and L670: "A rollout can fetch the latest weights from its colocated
    relay at any time"; rollouts use TP 1/4/8 (L1357).

Reading (DESIGN.md §3 R9, R14-R16) — the vLLM Qwen2 convention for rank r of tp:
  embed_tokens / lm_head : VOCAB_DIM0 — the vocabulary is padded to Vp = 64*ceil(V/64) rows; rank r
                           owns padded rows [r*Vp/tp, (r+1)*Vp/tp): its real rows first, then zero
                           rows for the padding (R15)
  qkv_proj (weight, bias): [q_r; k_r; v_r] — HEAD_DIM0 of q (nh heads), k and v (nkv heads each),
                           concatenated along dim 0.  HEAD_DIM0 splits whole heads: with tp <= heads
                           rank r gets heads [r*heads/tp, (r+1)*heads/tp); with tp > heads (tp a
                           multiple of heads) the heads are replicated and rank r gets head
                           r // (tp/heads) (R14, KV-head replication)
  o_proj, down_proj      : SHARD_DIM1 — columns [r*C/tp, (r+1)*C/tp) of every row
  gate_up_proj           : [gate_r; up_r] — SHARD_DIM0 of gate and up concatenated
  norms                  : REPLICATE
  transpose (optional)   : a 2-D destination stored K-major: the (rows x cols) matrix above is
                           stored as its transpose, dst[c][i] = A[i][c] (R16); 1-D destinations are
                           unaffected.
The oracle pulls two ways that must agree: `direct_pull` (generator -> cast -> TP rule, no buckets)
and `pull_from_image` (inverse bucket map of IMG(v) -> TP rule).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from synth import gen_bits, gen_bits_at

from .bf16 import rne_bf16
from .image import ImagePlan, unpack_tensor
from .model import Dims, numel, tensors

REPLICATE, SHARD_DIM0, SHARD_DIM1, VOCAB_DIM0, HEAD_DIM0 = 0, 1, 2, 3, 4
VOCAB_PAD = 64   # vLLM's default vocabulary padding (DEFAULT_VOCAB_PADDING_SIZE), reading R15


@dataclass(frozen=True)
class Part:
    tensor: str
    rule: int
    heads: int = 0   # HEAD_DIM0: number of attention heads stacked along dim 0


@dataclass(frozen=True)
class Dst:
    name: str
    shape: tuple[int, ...]
    parts: tuple[Part, ...]


def part_slice(shape: tuple[int, ...], rule: int, tp: int, rank: int, heads: int = 0):
    """(row0, row1, col0, col1, pad) of the source tensor that rank `rank` receives (cols None for
    1-D); `pad` zero rows follow the real rows in the destination (vocabulary padding only)."""
    d0 = shape[0]
    d1 = shape[1] if len(shape) == 2 else None
    c0 = 0 if d1 else None
    if rule == REPLICATE:
        return 0, d0, c0, d1, 0
    if rule == SHARD_DIM0:
        if d0 % tp:
            raise ValueError(f"dim 0 ({d0}) not divisible by tp={tp}")
        n = d0 // tp
        return rank * n, (rank + 1) * n, c0, d1, 0
    if rule == HEAD_DIM0:
        if heads < 1 or d0 % heads:
            raise ValueError(f"dim 0 ({d0}) is not {heads} heads")
        hd = d0 // heads
        if tp <= heads:
            if heads % tp:
                raise ValueError(f"{heads} heads not divisible by tp={tp}")
            per = heads // tp
            return rank * per * hd, (rank + 1) * per * hd, c0, d1, 0
        if tp % heads:
            raise ValueError(f"tp={tp} not a multiple of {heads} heads")
        h = rank // (tp // heads)
        return h * hd, (h + 1) * hd, c0, d1, 0
    if rule == VOCAB_DIM0:
        vp = -(-d0 // VOCAB_PAD) * VOCAB_PAD
        if vp % tp:
            raise ValueError(f"padded vocab ({vp}) not divisible by tp={tp}")
        n = vp // tp
        r0, r1 = min(rank * n, d0), min((rank + 1) * n, d0)
        return r0, r1, c0, d1, n - (r1 - r0)
    if rule == SHARD_DIM1:
        if d1 is None or d1 % tp:
            raise ValueError(f"dim 1 ({d1}) not divisible by tp={tp}")
        n = d1 // tp
        return 0, d0, rank * n, (rank + 1) * n, 0
    raise ValueError(rule)


def vllm_dsts(d: Dims, tp: int) -> list[Dst]:
    """Destination buffers of one TP rank, in the vLLM Qwen2 convention (shapes per rank)."""
    shp = dict(tensors(d))

    def dst(name, parts):
        shapes = []
        for p in parts:
            r0, r1, c0, c1, pad = part_slice(shp[p.tensor], p.rule, tp, 0, p.heads)
            shapes.append((r1 - r0 + pad,) + ((c1 - c0,) if c0 is not None else ()))
        rows = sum(s[0] for s in shapes)
        return Dst(name, (rows,) + shapes[0][1:], tuple(parts))

    out = [dst("model.embed_tokens.weight", [Part("model.embed_tokens.weight", VOCAB_DIM0)])]
    for l in range(d.L):
        p = f"model.layers.{l}."
        a = p + "self_attn."
        m = p + "mlp."
        out += [
            dst(a + "qkv_proj.weight", [Part(a + x + "_proj.weight", HEAD_DIM0, h)
                                        for x, h in (("q", d.nh), ("k", d.nkv), ("v", d.nkv))]),
            dst(a + "qkv_proj.bias", [Part(a + x + "_proj.bias", HEAD_DIM0, h)
                                      for x, h in (("q", d.nh), ("k", d.nkv), ("v", d.nkv))]),
            dst(a + "o_proj.weight", [Part(a + "o_proj.weight", SHARD_DIM1)]),
            dst(m + "gate_up_proj.weight", [Part(m + "gate_proj.weight", SHARD_DIM0),
                                            Part(m + "up_proj.weight", SHARD_DIM0)]),
            dst(m + "down_proj.weight", [Part(m + "down_proj.weight", SHARD_DIM1)]),
            dst(p + "input_layernorm.weight", [Part(p + "input_layernorm.weight", REPLICATE)]),
            dst(p + "post_attention_layernorm.weight",
                [Part(p + "post_attention_layernorm.weight", REPLICATE)]),
        ]
    out += [dst("model.norm.weight", [Part("model.norm.weight", REPLICATE)]),
            dst("lm_head.weight", [Part("lm_head.weight", VOCAB_DIM0)])]
    return out


def _apply(full: np.ndarray, p: Part, tp: int, rank: int) -> np.ndarray:
    r0, r1, c0, c1, pad = part_slice(full.shape, p.rule, tp, rank, p.heads)
    x = full[r0:r1] if c0 is None else full[r0:r1, c0:c1]
    if pad:
        x = np.concatenate([x, np.zeros((pad,) + x.shape[1:], dtype=x.dtype)], axis=0)
    return x


def _finish(pieces: list[np.ndarray], transpose: bool) -> np.ndarray:
    a = np.concatenate(pieces, axis=0)
    return np.ascontiguousarray(a.T if transpose and a.ndim == 2 else a)


def direct_pull(d: Dims, tp: int, rank: int, seed: int, v: int, specials: bool = False,
                only: set[str] | None = None, transpose: bool = False) -> dict[str, np.ndarray]:
    """dst_r = TP_r(RNE_bf16(W_v)) straight from the generator (no buckets); `transpose` stores
    every 2-D destination K-major."""
    tl = tensors(d)
    tid = {n: i for i, (n, _) in enumerate(tl)}
    out = {}
    for dst in vllm_dsts(d, tp):
        if only is not None and dst.name not in only:
            continue
        pieces = []
        for p in dst.parts:
            shape = tl[tid[p.tensor]][1]
            w = rne_bf16(gen_bits(seed, v, tid[p.tensor], 0, numel(shape), specials)).reshape(shape)
            pieces.append(_apply(w, p, tp, rank))
        out[dst.name] = _finish(pieces, transpose)
    return out


def pull_from_image(read, plan: ImagePlan, d: Dims, tp: int, rank: int,
                    only: set[str] | None = None, transpose: bool = False) -> dict[str, np.ndarray]:
    """Step-by-step pull: inverse bucket map of the relay's image, then the TP rule."""
    tl = tensors(d)
    tid = {n: i for i, (n, _) in enumerate(tl)}
    out = {}
    for dst in vllm_dsts(d, tp):
        if only is not None and dst.name not in only:
            continue
        pieces = []
        for p in dst.parts:
            t = tid[p.tensor]
            pieces.append(_apply(unpack_tensor(read, plan, t, tl[t][1]), p, tp, rank))
        out[dst.name] = _finish(pieces, transpose)
    return out


def dst_elements(d: Dims, tp: int, rank: int, dst_name: str, flat_idx: np.ndarray, seed: int, v: int,
                 specials: bool = False, transpose: bool = False) -> np.ndarray:
    """Expected bf16 values at flat positions of one destination buffer, computed one by one
    (for parity at full model sizes, where whole tensors are too big for the oracle).  With
    `transpose`, flat positions index the K-major buffer: position c*rows + i holds element (i, c)."""
    tl = tensors(d)
    tid = {n: i for i, (n, _) in enumerate(tl)}
    dst = next(x for x in vllm_dsts(d, tp) if x.name == dst_name)
    flat_idx = np.asarray(flat_idx, dtype=np.int64)
    width = numel(dst.shape) // dst.shape[0]
    if transpose and len(dst.shape) == 2:
        col, row = flat_idx // dst.shape[0], flat_idx % dst.shape[0]
    else:
        row, col = flat_idx // width, flat_idx % width
    out = np.zeros(flat_idx.size, dtype=np.uint16)   # padding rows stay 0x0000
    row_base = 0
    for p in dst.parts:
        shape = tl[tid[p.tensor]][1]
        r0, r1, c0, _, pad = part_slice(shape, p.rule, tp, rank, p.heads)
        sel = (row >= row_base) & (row < row_base + (r1 - r0))
        src_row = row[sel] - row_base + r0
        if c0 is None:
            src = src_row
        else:
            src = src_row * shape[1] + col[sel] + c0
        out[sel] = rne_bf16(gen_bits_at(seed, v, tid[p.tensor], src.astype(np.uint64), specials))
        row_base += r1 - r0 + pad
    return out

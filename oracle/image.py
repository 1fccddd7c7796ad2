"""Actor partition layouts and the chunked bucket image IMG(v) (oracle).

Passages followed:
  * PAPER L548, L653 (§4.2): after an update the actor "pushes the new actor weights to the master
    relay"; L1521: in BF16.  => publish = cast the actor's fp32 shards to bf16 and pack them.
  * PAPER L693 (§4.3): the master relay "receives weights from the actor, chunks them";
    L1467 (App. D.1): "the total model weights, of size M bytes, are divided into k smaller chunks,
    each of size M/k".  SPEC L534: chunk sizes ceil(M/k) except possibly the last.
  * the actor is sharded with PyTorch FSDP.

Readings — the byte format is ours, not the paper's:
  * FSDP2 (default): each tensor is split along dim 0 with torch.chunk semantics: ceil(d0/N) rows
    per rank, trailing ranks short or empty.  FSDP1 (variant): all tensors flattened in order and
    concatenated, zero-padded to a multiple of N, equal contiguous split (cuts may fall mid-row).
    Padding is never published.
  * Rank region r holds rank r's segments in tensor order; every segment starts at a 256-byte
    aligned offset, gaps are zero; the region length is rounded up to 256 bytes.
  * Each region is cut into chunks of C bytes (C a multiple of 4 KiB), its last chunk short.
    Regions are placed chunk-aligned, in rank order: region r starts at image offset
    C * (number of chunks of regions < r).  Global chunk g covers [g*C, g*C + len_g).
  * One header per chunk: {version, idx, n, bytes, S1, S2} with (S1, S2) from checksum.py.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from synth import gen_bits

from .bf16 import rne_bf16
from .checksum import chunk_checksum
from .model import numel

SEG_ALIGN = 256
CHUNK_ALIGN = 4096
FSDP2_DIM0 = "fsdp2"
FSDP1_FLAT = "fsdp1"


def _cdiv(a: int, b: int) -> int:
    return -(-a // b)


def _align(x: int, a: int) -> int:
    return _cdiv(x, a) * a


def actor_shards(shapes: list[tuple[int, ...]], N: int, layout: str = FSDP2_DIM0
                 ) -> list[list[tuple[int, int, int]]]:
    """Per actor rank, the list of (tensor_id, elem0, count) it owns, in tensor order."""
    out: list[list[tuple[int, int, int]]] = [[] for _ in range(N)]
    if layout == FSDP2_DIM0:
        for t, shp in enumerate(shapes):
            d0 = shp[0]
            row = numel(shp) // d0
            per = _cdiv(d0, N)
            for r in range(N):
                r0, r1 = r * per, min(d0, (r + 1) * per)
                if r1 > r0:
                    out[r].append((t, r0 * row, (r1 - r0) * row))
    elif layout == FSDP1_FLAT:
        sizes = [numel(s) for s in shapes]
        P = sum(sizes)
        per = _cdiv(P, N)              # = P_pad / N with P_pad = ceil(P/N)*N
        starts = np.cumsum([0] + sizes)
        for r in range(N):
            a, b = r * per, min(P, (r + 1) * per)
            for t in range(len(shapes)):
                lo, hi = max(a, int(starts[t])), min(b, int(starts[t + 1]))
                if hi > lo:
                    out[r].append((t, lo - int(starts[t]), hi - lo))
    else:
        raise ValueError(layout)
    return out


@dataclass
class Segment:
    tensor_id: int
    rank: int
    elem0: int
    count: int
    off: int            # byte offset inside the rank region


@dataclass
class ImagePlan:
    C: int
    N: int
    segments: list[Segment]
    region_len: list[int]
    n_chunks: list[int]
    chunk_base: list[int]
    total_chunks: int
    by_tensor: dict[int, list[Segment]] = field(default_factory=dict)

    @property
    def image_bytes(self) -> int:
        return self.C * self.total_chunks

    def image_offset(self, seg: Segment) -> int:
        return self.chunk_base[seg.rank] * self.C + seg.off

    def chunk_rank(self, g: int) -> int:
        for r in range(self.N):
            if self.chunk_base[r] <= g < self.chunk_base[r] + self.n_chunks[r]:
                return r
        raise IndexError(g)

    def chunk_len(self, g: int) -> int:
        r = self.chunk_rank(g)
        j = g - self.chunk_base[r]
        return min(self.C, self.region_len[r] - j * self.C)


def image_plan(shapes: list[tuple[int, ...]], N: int, C: int, layout: str = FSDP2_DIM0) -> ImagePlan:
    if C <= 0 or C % CHUNK_ALIGN:
        raise ValueError("chunk bytes must be a positive multiple of 4 KiB")
    shards = actor_shards(shapes, N, layout)
    segs: list[Segment] = []
    region_len, n_chunks, chunk_base = [], [], []
    base = 0
    for r in range(N):
        off = 0
        for (t, e0, cnt) in shards[r]:
            off = _align(off, SEG_ALIGN)
            segs.append(Segment(t, r, e0, cnt, off))
            off += 2 * cnt
        L = _align(off, SEG_ALIGN)
        region_len.append(L)
        n_chunks.append(_cdiv(L, C))
        chunk_base.append(base)
        base += n_chunks[-1]
    plan = ImagePlan(C, N, segs, region_len, n_chunks, chunk_base, base)
    for s in segs:
        plan.by_tensor.setdefault(s.tensor_id, []).append(s)
    return plan


def segment_bf16(seg: Segment, seed: int, v: int, specials: bool = False) -> np.ndarray:
    """The bf16 bit patterns the segment holds: RNE of the actor's fp32 master values W_v."""
    return rne_bf16(gen_bits(seed, v, seg.tensor_id, seg.elem0, seg.count, specials))


def publish(plan: ImagePlan, seed: int, v: int, specials: bool = False):
    """IMG(v) as a uint8 array of image_bytes, plus the per-chunk header list."""
    img = np.zeros(plan.image_bytes, dtype=np.uint8)
    for s in plan.segments:
        o = plan.image_offset(s)
        img[o:o + 2 * s.count] = segment_bf16(s, seed, v, specials).view(np.uint8)
    return img, headers_of(plan, img, v)


def headers_of(plan: ImagePlan, img: np.ndarray, v: int) -> list[dict]:
    hdr = []
    for g in range(plan.total_chunks):
        n = plan.chunk_len(g)
        s1, s2 = chunk_checksum(img[g * plan.C: g * plan.C + n])
        hdr.append(dict(version=v, idx=g, n=plan.total_chunks, bytes=n, s1=s1, s2=s2))
    return hdr


def publish_chunk(plan: ImagePlan, g: int, seed: int, v: int, specials: bool = False) -> np.ndarray:
    """Bytes of chunk g of IMG(v) alone (generates only the segments it intersects)."""
    r = plan.chunk_rank(g)
    j = g - plan.chunk_base[r]
    a, n = j * plan.C, plan.chunk_len(g)
    out = np.zeros(n, dtype=np.uint8)
    for s in plan.segments:
        if s.rank != r:
            continue
        lo, hi = max(a, s.off), min(a + n, s.off + 2 * s.count)
        if hi <= lo:
            continue
        e_lo, e_hi = (lo - s.off) // 2, (hi - s.off) // 2       # offsets are even
        vals = rne_bf16(gen_bits(seed, v, s.tensor_id, s.elem0 + e_lo, e_hi - e_lo, specials))
        out[lo - a:hi - a] = vals.view(np.uint8)
    return out


def unpack_tensor(read, plan: ImagePlan, tensor_id: int, shape: tuple[int, ...]) -> np.ndarray:
    """Inverse bucket map: reassemble the full bf16 tensor from image bytes.

    `read(offset, nbytes) -> uint8 array` reads IMG bytes (from whatever stores them)."""
    flat = np.zeros(numel(shape), dtype=np.uint16)
    for s in plan.by_tensor.get(tensor_id, []):
        raw = read(plan.image_offset(s), 2 * s.count)
        flat[s.elem0:s.elem0 + s.count] = np.ascontiguousarray(raw).view(np.uint16)
    return flat.reshape(shape)

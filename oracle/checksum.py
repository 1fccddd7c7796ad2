"""Per-chunk checksum (oracle).

The paper gives no checksum; SPEC L643/L652 frames each chunk with one and treats a mismatch as
node failure.  Reading: over the chunk's bytes, zero-padded to a
multiple of 16, taken as little-endian u32 words w_0..w_{n-1}:

    S1 = sum_i w_i            mod 2^64
    S2 = sum_i (i + 1) * w_i  mod 2^64

Position-weighted so that swapped words change S2; associative so any thread mapping gives the
same result.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1


def words_of(buf: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(buf, dtype=np.uint8).ravel()
    pad = (-b.size) % 16
    if pad:
        b = np.concatenate([b, np.zeros(pad, dtype=np.uint8)])
    return b.view("<u4").astype(np.uint64)


def chunk_checksum(buf: np.ndarray) -> tuple[int, int]:
    """(S1, S2) of a byte buffer, per the definition above (numpy uint64 arithmetic wraps mod 2^64)."""
    w = words_of(buf)
    i1 = np.arange(1, w.size + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        s1 = int(w.sum(dtype=np.uint64))
        s2 = int((w * i1).sum(dtype=np.uint64))
    return s1 & MASK64, s2 & MASK64

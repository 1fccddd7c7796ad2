"""Seeded synthetic fp32 master weights — the ONE module shared by the oracle and the CUDA path.

It holds no arithmetic of the method (no cast, no checksum, no layout): it only defines the
values the actor's fp32 master shards hold, so that both sides can regenerate identical inputs
independently.  The paper's weights are Qwen2.5 bf16 checkpoints ("BF16");
their values are irrelevant to a copy/cast/index path, so ours are synthetic.

Counter-based generator (one value per (seed, version, tensor_id, flat element index)):

    key = seed ^ (v * 0x9E3779B97F4A7C15) ^ (tensor_id << 44) ^ idx        (all mod 2^64)
    x   = splitmix64(key)
    m   = (x >> 40) - 2^23                                                  (24-bit signed)
    w   = m * 2^-30      (exact in fp32; |w| < 2^-7)

The version enters the hash, so consecutive versions differ almost everywhere: a torn or mixed
pull is visible.  ``specials=True`` (tiny configuration only) substitutes, when
``(x & 0xFFF) == 0x5A5``, the pattern ``SPECIALS[(x >> 12) % 19]`` — NaNs, infinities,
subnormals, signed zeros and rounding ties — so the cast's edge cases occur in real buffers.

The CUDA twin is ``synth/synth.cuh`` (same definition, written again); ``tests/test_synth.py``
pins both to the published SplitMix64 test vector and to each other.
"""
from __future__ import annotations

import numpy as np

SEED = 0x251012633  # SURVEY §8(d) "Synthetic inputs": seed 0x251012633

GOLDEN_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# fp32 bit patterns substituted in "specials" mode (SURVEY §8(c) C2 special table + NaN/inf/zero).
SPECIALS = np.array([
    0x3F808000, 0x3F818000, 0xBF808000, 0x7F7F7FFF, 0x7F7F8000, 0x7F7FFFFF, 0xFF7F8000,
    0x00008000, 0x00018000, 0x00000001, 0x80000001, 0x007FFFFF, 0x80000000,
    0x7F800000, 0xFF800000, 0x7FC00000, 0x7F800001, 0xFFFFFFFF, 0x00000000,
], dtype=np.uint32)


def splitmix64(state: np.ndarray) -> np.ndarray:
    """SplitMix64 output for the given state(s): z = state + gamma, then the Stafford-13 mix."""
    with np.errstate(over="ignore"):
        z = np.asarray(state, dtype=np.uint64) + GOLDEN_GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def gen_bits(seed: int, version: int, tensor_id: int, idx0: int, count: int,
             specials: bool = False) -> np.ndarray:
    """fp32 bit patterns (uint32) of elements [idx0, idx0+count) of tensor `tensor_id` at `version`."""
    return gen_bits_at(seed, version, tensor_id, np.arange(idx0, idx0 + count, dtype=np.uint64), specials)


def gen_bits_at(seed: int, version: int, tensor_id: int, idx: np.ndarray,
                specials: bool = False) -> np.ndarray:
    """fp32 bit patterns (uint32) of the elements at flat indices `idx` of tensor `tensor_id`."""
    with np.errstate(over="ignore"):
        base = (np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
                ^ (np.uint64(version & 0xFFFFFFFFFFFFFFFF) * GOLDEN_GAMMA)
                ^ (np.uint64(tensor_id) << np.uint64(44)))
        x = splitmix64(base ^ np.asarray(idx, dtype=np.uint64))
    m = (x >> np.uint64(40)).astype(np.int64) - (1 << 23)
    w = (m.astype(np.float32) * np.float32(2.0 ** -30))  # exact: |m| < 2^24
    bits = w.view(np.uint32).copy()
    if specials:
        hit = (x & np.uint64(0xFFF)) == np.uint64(0x5A5)
        if hit.any():
            sel = ((x[hit] >> np.uint64(12)) % np.uint64(len(SPECIALS))).astype(np.int64)
            bits[hit] = SPECIALS[sel]
    return bits


def gen_f32(seed: int, version: int, tensor_id: int, idx0: int, count: int,
            specials: bool = False) -> np.ndarray:
    """Same as gen_bits, viewed as float32 (bit patterns preserved, NaN payloads included)."""
    return gen_bits(seed, version, tensor_id, idx0, count, specials).view(np.float32)

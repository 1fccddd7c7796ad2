"""Pins of oracle/bf16.py (RNE definition) and oracle/checksum.py against things other than themselves."""
import os

import numpy as np
import pytest
import torch

from oracle.bf16 import rne_bf16
from oracle.checksum import chunk_checksum

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "bf16_specials.txt")


def _torch_bf16(bits: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(bits.view(np.float32).copy())
    return t.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def _integer_formula(bits: np.ndarray) -> np.ndarray:
    # the classic bit trick, written here only as an independent cross-check
    u = bits.astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = (bits & 0x7FFFFFFF) > 0x7F800000
    r[nan] = 0x7FC0
    return r


def test_special_table_from_survey():
    rows = []
    for line in open(GOLDEN):
        line = line.split("#")[0].strip()
        if line:
            a, b = line.split()
            rows.append((int(a, 16), int(b, 16)))
    got = rne_bf16(np.array([a for a, _ in rows], dtype=np.uint32))
    for (a, b), g in zip(rows, got):
        assert int(g) == b, f"{a:08X}: got {int(g):04X} want {b:04X}"


def _structured_patterns():
    # every upper half (sign, exponent, 7 significand bits) x every decision-relevant lower half
    hi = np.arange(1 << 16, dtype=np.uint32) << 16
    lows = np.array([0x0000, 0x0001, 0x7FFE, 0x7FFF, 0x8000, 0x8001, 0xC000, 0xFFFF], dtype=np.uint32)
    return (hi[:, None] | lows[None, :]).ravel()


def test_vs_torch_structured_exhaustive():
    bits = _structured_patterns()
    ours = rne_bf16(bits)
    ref = _torch_bf16(bits)
    nan = (bits & 0x7FFFFFFF) > 0x7F800000
    assert np.array_equal(ours[~nan], ref[~nan])
    assert np.all(ours[nan] == 0x7FC0)


def test_vs_torch_and_integer_formula_random():
    rng = np.random.default_rng(12633)
    bits = rng.integers(0, 2 ** 32, size=1 << 22, dtype=np.uint64).astype(np.uint32)
    ours = rne_bf16(bits)
    nan = (bits & 0x7FFFFFFF) > 0x7F800000
    assert np.array_equal(ours[~nan], _torch_bf16(bits)[~nan])
    assert np.array_equal(ours, _integer_formula(bits))


@pytest.mark.slow
def test_exhaustive_2_pow_32_vs_torch():
    step = 1 << 26
    for start in range(0, 1 << 32, step):
        bits = np.arange(start, start + step, dtype=np.uint64).astype(np.uint32)
        ours = rne_bf16(bits)
        nan = (bits & 0x7FFFFFFF) > 0x7F800000
        assert np.array_equal(ours[~nan], _torch_bf16(bits)[~nan]), hex(start)
        assert np.all(ours[nan] == 0x7FC0)


# ------------------------------------------------------------------------------------ checksum
def _naive(buf: bytes):
    b = bytes(buf) + bytes((-len(buf)) % 16)
    s1 = s2 = 0
    for i in range(len(b) // 4):
        w = int.from_bytes(b[4 * i:4 * i + 4], "little")
        s1 += w
        s2 += (i + 1) * w
    return s1 % 2 ** 64, s2 % 2 ** 64


def test_checksum_closed_forms():
    assert chunk_checksum(np.zeros(4096, np.uint8)) == (0, 0)
    for i, w in [(0, 1), (5, 0xDEADBEEF), (1023, 0xFFFFFFFF)]:
        buf = np.zeros(4096, np.uint8)
        buf[4 * i:4 * i + 4] = np.frombuffer(w.to_bytes(4, "little"), np.uint8)
        assert chunk_checksum(buf) == (w, (i + 1) * w)


def test_checksum_concatenation_law_and_naive():
    rng = np.random.default_rng(1)
    for la, lb in [(16, 16), (256, 4096), (4096, 48), (160, 1 << 14)]:
        a = rng.integers(0, 256, la, dtype=np.uint8)
        b = rng.integers(0, 256, lb, dtype=np.uint8)
        A, B, AB = chunk_checksum(a), chunk_checksum(b), chunk_checksum(np.concatenate([a, b]))
        assert AB[0] == (A[0] + B[0]) % 2 ** 64
        assert AB[1] == (A[1] + B[1] + (la // 4) * B[0]) % 2 ** 64
        assert AB == _naive(np.concatenate([a, b]).tobytes())


def test_checksum_pads_to_16_and_detects_swaps():
    rng = np.random.default_rng(2)
    a = rng.integers(0, 256, 40, dtype=np.uint8)
    assert chunk_checksum(a) == _naive(a.tobytes()) == chunk_checksum(np.concatenate([a, np.zeros(8, np.uint8)]))
    w = a.view("<u4").copy()
    w[0], w[1] = w[1], w[0]
    if w[0] != w[1]:
        assert chunk_checksum(w.view(np.uint8))[1] != chunk_checksum(a)[1]
    big = np.empty(1 << 20, dtype=np.uint8)                    # S2 wraps mod 2^64 here
    big[:] = 0xFF
    assert chunk_checksum(big) == _naive(big.tobytes())

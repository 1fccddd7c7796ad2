"""fp32 -> bf16 round-to-nearest-even, written as the definition (oracle).

PAPER.md L1521: weights are synchronized "in BF16 precision"; the north star fixes the rounding
mode: fp32 -> bf16 round-to-nearest-even.  Readings:
  * nearest representable bf16, ties to the even significand;
  * subnormals kept (no flush to zero);
  * overflow rounds to +-inf (rounding as if the exponent range were unbounded: the value just
    above the largest finite bf16 is 2^128, whose significand is even);
  * every NaN -> the canonical quiet NaN 0x7FC0 (what PyTorch CPU's c10::BFloat16 produces).

Implementation: for each |x|, the two bf16 candidates bracketing it are lo = |x| with its low
16 bits cleared and hi = the next bf16 magnitude; the distances |x|-lo and hi-|x| are computed in
float64, where they are exact for fp32 operands.  No bit trick, so a test may pin it against the
integer formula without circularity.
"""
from __future__ import annotations

import numpy as np


def rne_bf16(bits: np.ndarray) -> np.ndarray:
    """uint32 fp32 bit patterns -> uint16 bf16 bit patterns (nearest, ties to even)."""
    u = np.ascontiguousarray(bits, dtype=np.uint32)
    sign = (u >> np.uint32(16)) & np.uint32(0x8000)
    mag = u & np.uint32(0x7FFFFFFF)
    is_nan = mag > np.uint32(0x7F800000)
    is_inf = mag == np.uint32(0x7F800000)
    fin = ~(is_nan | is_inf)

    lo = mag & np.uint32(0xFFFF0000)                       # largest bf16 magnitude <= |x|
    hi = lo + np.uint32(0x00010000)                        # next bf16 magnitude above lo
    with np.errstate(invalid="ignore", over="ignore"):
        x = mag.view(np.float32).astype(np.float64)
        lo_v = lo.view(np.float32).astype(np.float64)
        hi_v = np.where(hi == np.uint32(0x7F800000), 2.0 ** 128,
                        hi.view(np.float32).astype(np.float64))
        d_lo = x - lo_v                                    # exact in float64
        d_hi = hi_v - x
    lo_odd = ((lo >> np.uint32(16)) & np.uint32(1)) == np.uint32(1)
    take_hi = fin & ((d_hi < d_lo) | ((d_hi == d_lo) & lo_odd))
    out_mag = np.where(take_hi, hi, lo) >> np.uint32(16)   # inf stays inf (lo == 0x7F800000)
    out = (sign | out_mag).astype(np.uint16)
    out[is_nan] = np.uint16(0x7FC0)
    return out


def rne_bf16_scalar(bits: int) -> int:
    """Scalar convenience wrapper (tests)."""
    return int(rne_bf16(np.array([bits], dtype=np.uint32))[0])

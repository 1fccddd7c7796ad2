"""Seeded synthetic inputs shared by the oracle and the CUDA path (generator only; see synth.py)."""
from .synth import SEED, SPECIALS, gen_bits, gen_bits_at, gen_f32, splitmix64  # noqa: F401

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def gpu_lib():
    """ctypes handle of synth/libsynth.so (the CUDA twin's fill kernel); raises if not built."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libsynth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        lib.synth_fill_f32.restype = ctypes.c_int
        lib.synth_fill_f32.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
        _LIB = lib
    return _LIB


def fill_device(ptr: int, count: int, seed: int, version: int, tensor_id: int, idx0: int = 0,
                specials: bool = False, stream: int = 0) -> None:
    """Fill `count` fp32 at device pointer `ptr` with elements [idx0, idx0+count) of the tensor."""
    rc = gpu_lib().synth_fill_f32(ptr, count, seed, version, tensor_id, idx0, int(specials), stream)
    if rc != 0:
        raise RuntimeError(f"synth_fill_f32 failed: cudaError {rc}")

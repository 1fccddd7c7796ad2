"""B200-native relay-tier weight synchronization (arxiv 2510.12633): publish -> chain relay -> pull.

The product is liblam.so (include/lam.h, CUDA for sm_100a); `lam` is its thin ctypes binding and
`workload` the torch-memory plumbing used by tests and bench.py.
"""
from . import lam  # noqa: F401

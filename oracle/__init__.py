"""CPU oracle for the relay-tier weight synchronization path (arxiv 2510.12633) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
leg may import anything from this package.  The product path (``paper_2510_12633_b200``) never
does: it has no CPU fallback and fails loudly when its CUDA library is missing.

The oracle is plain, slow, and written from the paper plus SURVEY.md §8(c)'s readings,
in numpy/pure Python.  It shares no code with the CUDA path; the only common module is ``synth``
(the seeded input generator, which holds none of the method's arithmetic).

What it computes (the plain definition):
    for every pull that returns version v on TP rank r:  dst_r = TP_r(RNE_bf16(W_v))
and the relay slot bytes at every relay equal the canonical bucket image IMG(v).

Modules (each function cites the passage it follows):
    model.py      Qwen2.5 tensor tables (PAPER "Qwen2.5"; L1357 TP sizes)
    bf16.py       fp32 -> bf16 round-to-nearest-even, by the definition (PAPER "BF16")
    checksum.py   per-chunk position-weighted checksum (SURVEY C3 reading)
    image.py      actor FSDP layouts and the chunked bucket image IMG(v)
    tp.py         TP reshard rules and the pull
    relay.py      chain-pipelined relay rounds + Appendix D latency model
    invariants.py concurrent-pull invariant checker

Parity status: every function is pinned by a ``-m "not gpu"`` test in tests/test_oracle_*.py
against something other than itself, except the exact version sequence a *concurrent* pull sees,
which is nondeterministic by design ("parity unpinned" — only invariants are checked).
"""

"""Multi-process GPU parity (one process per GPU, torchrun): the bench's placements through the C ABI
with CUDA IPC + shared-memory version table, checked against the oracle (tests/mp_worker.py)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def run(n, *args, port=29900, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", "mp_worker.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count(" ok: ") == n, out[-4000:]


CASES = [  # (min GPUs, args)
    (2, ["--config", "chain", "--model", "tiny", "--versions", "3"]),
    (2, ["--config", "colocated", "--model", "tiny", "--tp", "2"]),
    (2, ["--config", "relay-tp", "--model", "tiny", "--tp", "1"]),
    (4, ["--config", "chain", "--model", "tiny", "--versions", "3", "--chunk-kb", "16"]),
    (4, ["--config", "colocated", "--model", "tiny", "--tp", "4"]),
    (4, ["--config", "colocated", "--model", "tiny", "--tp", "2"]),
    (4, ["--config", "relay-tp", "--model", "tiny", "--tp", "2"]),
    (2, ["--config", "chain", "--model", "7b", "--chunk-kb", str(128 << 10)]),
    (4, ["--config", "chain", "--model", "tiny", "--versions", "3", "--chunk-kb", "16", "--hop-mode", "1"]),
    (4, ["--config", "relay-tp", "--model", "tiny", "--tp", "2", "--hop-mode", "1"]),
    (4, ["--config", "chain", "--model", "tiny", "--versions", "3", "--chunk-kb", "16", "--stream"]),
    (4, ["--config", "colocated", "--model", "tiny", "--tp", "4", "--stream"]),
    (4, ["--config", "relay-tp", "--model", "tiny", "--tp", "2", "--stream"]),
    (2, ["--config", "chain", "--model", "7b", "--chunk-kb", str(128 << 10), "--stream"]),
    (2, ["--config", "host", "--model", "tiny", "--versions", "3"]),                 # NEXT-3 host tier
    (4, ["--config", "host", "--model", "tiny", "--tp", "2", "--stream"]),
    (4, ["--config", "host", "--model", "tiny", "--versions", "2", "--hop-mode", "1"]),
    (2, ["--config", "chain", "--model", "7b", "--chunk-kb", str(128 << 10), "--hop-mode", "1"]),   # CE, 7B
    # NEXT-2 multicast broadcast: the multicast object crosses processes (SCM_RIGHTS), every relay
    # verifies its replica
    (2, ["--config", "chain", "--model", "tiny", "--versions", "3", "--hop-mode", "2"]),
    (4, ["--config", "chain", "--model", "tiny", "--versions", "3", "--chunk-kb", "16", "--hop-mode", "2", "--stream"]),
    (4, ["--config", "chain", "--model", "7b", "--chunk-kb", str(128 << 10), "--hop-mode", "2"]),
    # two-level broadcast: relays read each other's slots across processes
    (4, ["--config", "chain", "--model", "tiny", "--versions", "3", "--chunk-kb", "16", "--hop-mode", "4", "--stream"]),
    (4, ["--config", "chain", "--model", "7b", "--chunk-kb", str(128 << 10), "--hop-mode", "4", "--stream"]),
]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_multiproc_parity(i):
    need, args = CASES[i]
    n = ngpu()
    if n < need:
        pytest.skip(f"needs {need} GPUs")
    run(need, *args, port=29900 + i)

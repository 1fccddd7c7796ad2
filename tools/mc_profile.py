"""Single-process 2-GPU multicast publish for ncu (NVLink counters of the multicast pack, NEXT-2): node 0
on GPU 0 packs the 7B snapshot through the multicast object; relay node 1 on GPU 1 verifies its
replica after the pack has completed (so no kernel spins while ncu replays the pack).

  ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,\
dram__bytes_write.sum -k regex:k_pack python tools/mc_profile.py

Prints the pack's own CUDA-event time and the relay's verify time (run once without ncu for that)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2510_12633_b200 import lam  # noqa: E402
from paper_2510_12633_b200.workload import MODELS, ActorShard  # noqa: E402
from synth import SEED  # noqa: E402


def main():
    model = sys.argv[1] if len(sys.argv) > 1 else "7b"
    ctx = lam.Context(lam.Config(model=MODELS[model], relays=[[1]], rollouts=[], chunk_bytes=128 << 20,
                                 hop_mode=lam.LAM_HOP_MULTICAST))
    sh = ActorShard(MODELS[model], 1, 0, 0)
    sh.fill(SEED, 1)
    torch.cuda.synchronize()
    ctx.set_profiling(True)
    M = ctx.plan_info().snapshot_bytes
    for v in (1, 2, 3):
        assert ctx.publish(v, 0, sh.shards(), 0) == lam.LAM_OK
        while ctx.latest(0) < v:            # the pack completes before the relay's verify is launched
            ctx.relay_step()
        t0 = time.time()
        while ctx.latest(1) < v:
            ctx.relay_step()
            if time.time() - t0 > 120:
                raise TimeoutError
        torch.cuda.synchronize()
        kt = ctx.kernel_times()
        pms, hms = kt["pack"][0] / max(kt["pack"][1], 1), kt["hop"][0] / max(kt["hop"][1], 1)
        print(f"v{v}: multicast pack {pms:.3f} ms = {M / (pms / 1e3) / 1e9:.1f} GB/s per receiver; relay verify+commit "
              f"from its replica {hms:.3f} ms = {2 * M / (hms / 1e3) / 1e9:.1f} GB/s HBM", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()

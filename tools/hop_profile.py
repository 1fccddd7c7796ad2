"""Single-process 2-GPU chain hop for ncu (NVLink counters of k_hop): the actor's pack on GPU 0
completes first, then relay node 1 on GPU 1 runs one k_hop over the whole 7B image — so the hop never
spins on a flag while ncu replays it.

  ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,\
dram__bytes_write.sum -k regex:k_hop python tools/hop_profile.py

Also prints the hop's own CUDA-event time (run it once without ncu for that)."""
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
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    model = args[0] if args else "7b"
    mode = lam.LAM_HOP_COPY_ENGINE if "--ce" in sys.argv else lam.LAM_HOP_KERNEL
    nrel = int(args[1]) if len(args) > 1 else 1
    ctx = lam.Context(lam.Config(model=MODELS[model], relays=[[d] for d in range(1, nrel + 1)], rollouts=[],
                                 chunk_bytes=128 << 20, hop_mode=mode))
    sh = ActorShard(MODELS[model], 1, 0, 0)
    sh.fill(SEED, 1)
    torch.cuda.synchronize()
    ctx.set_profiling(True)
    for v in (1, 2, 3):
        assert ctx.publish(v, 0, sh.shards(), 0) == lam.LAM_OK
        while ctx.latest(0) < v:            # the pack completes before the hop is launched
            ctx.relay_step()
        t0 = time.time()
        while ctx.latest(nrel) < v:
            ctx.relay_step()
            if time.time() - t0 > 120:
                raise TimeoutError
        t1 = time.time()
        torch.cuda.synchronize()
        kt = ctx.kernel_times()
        ms, n = kt["hop"]
        M = ctx.plan_info().snapshot_bytes
        print(f"v{v}: {nrel} relay(s), {'ce' if mode else 'kernel'}: hop avg {ms / max(n, 1):.3f} ms = "
              f"{M / (ms / max(n, 1) / 1e3) / 1e9:.1f} GB/s; master complete -> last relay {1e3 * (t1 - t0):.2f} ms "
              f"(pack {kt['pack'][0]:.3f} ms)", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Pull/reshard microbenchmark: k_pull alone on one GPU, per TP layout, row-major
vs K-major destinations, against the measured HBM copy peak.  Algorithmic bytes = 2 x the rank's
slice bytes (read from the relay slot + write into the rollout buffers).

  python tools/pull_bench.py [--model 7b] [--tps 1,2,4,8] [--reps 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b")
    ap.add_argument("--tps", default="1,2,4")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--pull-ctas", type=int, default=0)
    ap.add_argument("--layouts", default="row-major,k-major")
    a = ap.parse_args()
    import torch

    from paper_2510_12633_b200 import lam
    from paper_2510_12633_b200.workload import MODELS, ActorShard, RolloutBuffers
    from synth import SEED

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6542.7) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6542.7
    m = MODELS[a.model]
    ctx = lam.Context(lam.Config(model=m, rollouts=[(0, 0)], chunk_bytes=64 << 20, pull_ctas=a.pull_ctas))
    sh = ActorShard(m, 1, 0, 0)
    sh.fill(SEED, 1)
    torch.cuda.synchronize()
    assert ctx.publish(1, 0, sh.shards()) == lam.LAM_OK
    while ctx.relay_step()[0] != lam.LAM_IDLE:
        pass
    del sh
    torch.cuda.empty_cache()
    s = torch.cuda.Stream()
    for tp in [int(x) for x in a.tps.split(",")]:
        for tr in [x == "k-major" for x in a.layouts.split(",")]:
            rb = RolloutBuffers(m, tp, 0, 0, transpose=tr)
            assert ctx.pull(0, rb.tp, s.cuda_stream) == 1      # warm-up (builds the plan)
            s.synchronize()
            ctx.kernel_times()
            ctx.set_profiling(True)
            for _ in range(a.reps):
                ctx.pull(0, rb.tp, s.cuda_stream)
            s.synchronize()
            ctx.relay_step()
            kt = ctx.kernel_times()
            ctx.set_profiling(False)
            ms, n = kt["pull"]
            ms /= max(n, 1)
            gbs = 2 * rb.bytes / (ms / 1e3) / 1e9
            print(json.dumps(dict(model=a.model, tp=tp, layout="k-major" if tr else "row-major",
                                  slice_bytes=rb.bytes, ms=round(ms, 4), gbs=round(gbs, 1),
                                  frac_of_measured_hbm=round(gbs / peak, 3), launches=n)), flush=True)
            del rb
            torch.cuda.empty_cache()
    ctx.close()


if __name__ == "__main__":
    main()

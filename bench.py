#!/usr/bin/env python
"""bench.py — publish -> all-rollouts weight-sync latency of the relay tier (arxiv 2510.12633 §4).

One step = one pass of the whole hot path over a fresh version:
  lam_publish(v)   fp32 master shard -> bf16 RNE -> chunked bucket image in the master's slot
  lam_relay_step   chain-pipelined hops master -> relay 1 -> ... (N > 1), version commit
  lam_pull         every rollout pulls v and reshards it into its TP buffers
and the step's time is publish -> every rollout's pull completed.

Workload (BASELINE.json configs[1]): Qwen2.5-7B-shaped snapshot (7.62 G params, 15.23 GB bf16),
actor FSDP-1 on GPU 0.  N = 1: master node on GPU 0, one TP=1 rollout pulling from it.
N > 1 (torchrun, one process per GPU): relays on GPUs 1..N-1 in a chain, one TP=1 rollout per relay
GPU (config 2 at N = 8).  Weak scaling: each added GPU adds one relay + one rollout.

`--impl reference` times the CPU oracle (the reference arm of this tier) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "publish->all-rollouts sync latency"
UNIT = "s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lam", choices=["lam", "reference"])
    ap.add_argument("--model", default="7b")
    ap.add_argument("--config", default="chain", choices=["chain", "colocated", "relay-tp", "host"],
                    help="placement: chain (config 2), colocated (config 4), relay-tp (config 3), "
                         "host (NEXT-3: the paper's host-memory relay tier)")
    ap.add_argument("--tp", type=int, default=0, help="rollout TP size (colocated / relay-tp)")
    ap.add_argument("--chunk-mb", type=int, default=0, help="chunk size; 0 = Appendix D k*")
    ap.add_argument("--hop-ctas", type=int, default=0)
    ap.add_argument("--hop-mode", default="kernel", choices=["kernel", "ce"],
                    help="relay hop: TMA kernel or copy engines + k_verify")
    ap.add_argument("--stream-pull", default="auto", choices=["auto", "on", "off"],
                    help="on: rollouts reshard chunk by chunk while their relay receives (lam_pull_stream); "
                         "off: pull once the relay committed (lam_pull); auto: on for chain / relay-tp, off for "
                         "colocated (there the pull competes with the pack for HBM and gains nothing)")
    ap.add_argument("--no-stream-pull", action="store_true", help="same as --stream-pull off")
    ap.add_argument("--no-subscribe", action="store_true",
                    help="colocated rollouts pull after the pack instead of being written by it")
    ap.add_argument("--pack-ctas", type=int, default=0)
    ap.add_argument("--pull-ctas", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the oracle sample")
    ap.add_argument("--quick", action="store_true", help="profiling mode: no e2e, no cpu baseline, no clocks")
    return ap.parse_args()


# ------------------------------------------------------------------------------ CPU oracle leg
def oracle_sample(model: str, seconds: float, version: int = 1):
    """Time the oracle (as it stands) on a bounded sample of the workload, scaled to one full step.

    Sample: the leading segments of the 7B image (inputs pre-generated, like resident masters):
    publish = RNE cast + pack into the image + chunk checksums; pull = inverse bucket map + TP=1 rule.
    """
    import numpy as np

    from oracle.bf16 import rne_bf16
    from oracle.checksum import chunk_checksum
    from oracle.image import image_plan, unpack_tensor
    from oracle.model import MODELS, numel, tensors
    from synth import SEED, gen_bits

    d = MODELS[model]
    tl = tensors(d)
    shapes = [s for _, s in tl]
    P = sum(numel(s) for s in shapes)
    C = 64 << 20
    plan = image_plan(shapes, 1, C)
    # pick whole tensors from the start of the layer stack until ~seconds/6 of generation work
    budget_elems = int(1.5e7 * seconds)          # ~15 M params/s through the numpy oracle
    chosen, n = [], 0
    for t in range(1, len(tl)):               # skip the 545M-element embedding: keep the sample bounded
        if n >= budget_elems:
            break
        chosen.append(t)
        n += numel(shapes[t])
    segs = [s for s in plan.segments if s.tensor_id in set(chosen)]
    inputs = {s.tensor_id: gen_bits(SEED, version, s.tensor_id, s.elem0, s.count) for s in segs}
    lo = min(plan.image_offset(s) for s in segs)
    hi = max(plan.image_offset(s) + 2 * s.count for s in segs)
    img = np.zeros(hi - lo + 4096, dtype=np.uint8)
    t0 = time.perf_counter()
    for s in segs:                               # publish: cast + pack
        o = plan.image_offset(s) - lo
        img[o:o + 2 * s.count] = rne_bf16(inputs[s.tensor_id]).view(np.uint8)
    for a in range(0, img.size, C):              # checksums of the produced bytes
        chunk_checksum(img[a:a + C])
    t_pub = time.perf_counter() - t0
    rd = lambda o, k: img[o - lo:o - lo + k]
    t0 = time.perf_counter()
    for t in chosen:                             # pull at TP=1: inverse bucket map
        unpack_tensor(rd, plan, t, shapes[t]).copy()
    t_pull = time.perf_counter() - t0
    frac = n / P
    full = (t_pub + t_pull) / frac
    return full, dict(kind="oracle", cores=1, value=full, unit=UNIT,
                      sample=f"{len(chosen)} tensors / {n / 1e6:.1f} M params of {model} "
                             f"({100 * frac:.2f}%): publish {t_pub:.2f} s + pull {t_pull:.2f} s, "
                             f"scaled to the full snapshot; numpy, single thread")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    per = max(2.0, args.cpu_seconds / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        oracle_sample(args.model, per)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, info = oracle_sample(args.model, per)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = sum(vals) / len(vals)
    cpu = os.cpu_count()
    out = dict(metric=METRIC, value=value, unit=UNIT, impl="reference", n_gpus=args.gpus, steps=args.steps,
               warmup=args.warmup, ms_per_step=value * 1e3, higher_is_better=False, scaling="weak",
               vs_baseline=None, dtype="bf16", data="synthetic",
               config=dict(workload=f"{args.model} [{args.config}]: " + topology(args.config, args.gpus, args.tp)["desc"],
                           model=f"Qwen2.5-{args.model.upper()}-shaped",
                           reference="CPU oracle publish + TP=1 pull, bounded sample scaled to one step"),
               cpu_baseline=dict(info, value=value, host_cpus=cpu, wall_s=wall),
               e2e=dict(value=value, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(out))
    return 0


# ------------------------------------------------------------------------------------ clocks
class Clocks:
    def __init__(self, device: int):
        self.samples, self.proc = [], None
        self.device = device

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["unavailable"], samples=0)
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower().startswith("active")})
        return dict(sm_mhz=sm[len(sm) // 2] if sm else None, sm_max_mhz=mx, reasons=reasons, samples=len(self.samples))


# -------------------------------------------------------------------------------- GPU leg
def topology(config: str, N: int, tp_arg: int):
    """Placement of actor ranks, relay nodes and rollouts on N GPUs (BASELINE.json configs)."""
    if config == "host":
        # NEXT-3: actor FSDP-1 on GPU 0 -> one relay node in pinned host
        # memory (received by GPU min(1, N-1) over PCIe) -> TP rollouts on GPUs 1..N-1 (GPU 0 at N=1)
        # pull from host memory over their own PCIe links
        g = min(1, N - 1)
        tp = tp_arg or 1
        gpus = list(range(g, N))
        ro = [(1, gpus[k * tp + j], tp, j) for k in range(len(gpus) // tp) for j in range(tp)]
        return dict(fsdp=1, actors=[0], relays=[[g]], host_relays=[1], rollouts=ro,
                    desc=f"actor FSDP-1 on GPU0 -> host-memory relay (received by GPU{g}) -> "
                         f"{len(ro) // tp} TP={tp} rollout(s) on GPUs {g}..{N - 1} pulling over PCIe")
    if config == "chain" or N == 1:
        # config 2: actor FSDP-1 on GPU 0 -> chain of relays on GPUs 1..N-1, one TP=1 rollout each
        if N == 1:
            return dict(fsdp=1, actors=[0], relays=[], rollouts=[(0, 0, 1, 0)],
                        desc="actor FSDP-1 + master node + one TP=1 rollout on GPU0")
        return dict(fsdp=1, actors=[0], relays=[[d] for d in range(1, N)],
                    rollouts=[(i, i, 1, 0) for i in range(1, N)],
                    desc=f"actor FSDP-1 on GPU0 -> chain of {N - 1} relays (GPUs 1..{N - 1}), one TP=1 rollout per relay")
    if config == "colocated":
        # config 4: actor FSDP-N colocated on all GPUs; node 0 (the N colocated bf16 shards) serves
        # TP=tp rollouts that gather their slices over NVLink.  Replica k = GPUs {k + j*N/tp}.
        tp = tp_arg or N
        reps = N // tp
        ro = [(0, k + j * reps, tp, j) for k in range(reps) for j in range(tp)]
        return dict(fsdp=N, actors=list(range(N)), relays=[], rollouts=ro,
                    desc=f"actor FSDP-{N} colocated on GPUs 0..{N - 1}; {reps} TP={tp} rollout(s) gather from the colocated shards")
    if config == "relay-tp":
        # config 3: actor FSDP-N/2 on GPUs 0..N/2-1 -> one relay node range-sharded over GPUs N/2..N-1
        # (rank r's region on GPU N/2+r) -> TP=tp rollouts on the relay GPUs gather over NVLink
        h = N // 2
        tp = tp_arg or min(2, h)
        ro = [(1, h + k * tp + j, tp, j) for k in range(h // tp) for j in range(tp)]
        return dict(fsdp=h, actors=list(range(h)), relays=[[h + r for r in range(h)]], rollouts=ro,
                    desc=f"actor FSDP-{h} on GPUs 0..{h - 1} -> relay range-sharded over GPUs {h}..{N - 1} -> "
                         f"{h // tp} TP={tp} rollout(s) on the relay GPUs")
    raise SystemExit(f"unknown --config {config}")


def main():
    args = parse()
    if args.no_stream_pull or args.stream_pull == "off" or (args.stream_pull == "auto" and args.config == "colocated"):
        args.no_stream_pull = True
    if args.impl == "reference":
        return run_reference(args)
    if os.environ.get("LAM_BENCH_WATCHDOG"):      # debugging aid: dump every thread's stack, then exit
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["LAM_BENCH_WATCHDOG"]), exit=True)
    import torch
    import torch.distributed as dist

    from paper_2510_12633_b200 import lam
    from paper_2510_12633_b200.workload import MODELS, ActorShard, RolloutBuffers
    from synth import SEED

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    N = world
    if N != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}; using {N}", file=sys.stderr)
    torch.cuda.set_device(rank)
    gloo = None
    if N > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
        gloo = dist.new_group(backend="gloo")

    def barrier():
        if gloo is not None:
            dist.barrier(group=gloo)

    model = MODELS[args.model]
    T = topology(args.config, N, args.tp)
    rollouts = T["rollouts"]
    port = os.environ.get("MASTER_PORT", "0")
    cfg = lam.Config(model=model, fsdp_size=T["fsdp"], actor_devices=T["actors"], relays=T["relays"],
                     rollouts=[(n, d) for n, d, _, _ in rollouts], chunk_bytes=args.chunk_mb << 20,
                     proc_rank=rank, n_procs=N, proc_of_device={d: d for d in range(N)},
                     shm_name=f"lam_bench_{port}_{os.getppid()}", hop_ctas=args.hop_ctas,
                     pack_ctas=args.pack_ctas, pull_ctas=args.pull_ctas,
                     hop_mode=lam.LAM_HOP_COPY_ENGINE if args.hop_mode == "ce" else lam.LAM_HOP_KERNEL,
                     host_relays=T.get("host_relays", []))
    ctx = lam.Context(cfg)
    if N > 1:
        blobs = [None] * N
        dist.all_gather_object(blobs, ctx.export_ipc(), group=gloo)
        for p, b in enumerate(blobs):
            if p != rank:
                ctx.import_ipc(p, b)
        ctx.connect()
        barrier()
    info = ctx.plan_info()
    M = info.snapshot_bytes
    params = info.params

    my_ranks = [r for r, d in enumerate(T["actors"]) if d == rank]
    shards = {r: ActorShard(model, T["fsdp"], r, rank) for r in my_ranks}
    for sh in shards.values():
        sh.fill(SEED, 1)
    mine = [rid for rid, (_, dev, _, _) in enumerate(rollouts) if dev == rank]
    bufs = {rid: RolloutBuffers(model, rollouts[rid][2], rollouts[rid][3], rank) for rid in mine}
    pull_bytes = {rid: ctx.pull_bytes(rid, bufs[rid].tp) for rid in mine}
    stream = torch.cuda.Stream()
    actor_stream = torch.cuda.Stream()
    torch.cuda.synchronize()
    state = {"v": 0}
    pub_host = []                                   # host seconds inside lam_publish (actor stall part 1)

    # colocated rollouts (node 0, an actor GPU, TP=1) are written by the pack itself (lam_subscribe)
    subs = [] if args.no_subscribe else [rid for rid in mine if rollouts[rid][0] == 0 and rollouts[rid][2] == 1
                                          and rollouts[rid][1] in T["actors"]]
    sub_done = {rid: live_event(torch) for rid in subs}

    def step(h2d=None, d2h=None):
        state["v"] += 1
        v = state["v"]
        for rid in subs:
            ctx.subscribe(rid, bufs[rid].tp, sub_done[rid].cuda_event)
        for r in my_ranks:
            if h2d is not None:                        # e2e: the step's inputs arrive from host memory
                with torch.cuda.stream(actor_stream):
                    shards[r].buf.copy_(h2d[r], non_blocking=True)
            t_pub = time.perf_counter()
            while ctx.publish(v, r, shards[r].shards(), actor_stream.cuda_stream) == lam.LAM_EBUSY:
                ctx.relay_step()
            pub_host.append(time.perf_counter() - t_pub)
        pending, streaming = [rid for rid in mine if rid not in subs], list(subs)
        while True:
            ctx.relay_step()
            for rid in list(pending):
                if args.no_stream_pull:                     # classic: pull once the relay committed v
                    got = ctx.pull(rid, bufs[rid].tp, stream.cuda_stream) if ctx.latest(rollouts[rid][0]) >= v else 0
                else:                                       # reshard chunk by chunk while v arrives
                    got = ctx.pull_stream(rid, bufs[rid].tp, stream.cuda_stream, None, v)
                if got:
                    assert got >= v, (got, v)
                    pending.remove(rid)
                    streaming.append(rid)
            for rid in list(streaming):
                if (args.no_stream_pull and rid not in subs) or ctx.pull_state(rid)[1] == 0:
                    if rid in subs:                         # written by the pack on the side stream
                        stream.wait_event(sub_done[rid])
                    if d2h is not None:
                        with torch.cuda.stream(stream):
                            for name, t in bufs[rid].bufs.items():
                                d2h[rid][name].copy_(t, non_blocking=True)
                    streaming.remove(rid)
            if not pending and not streaming and (not my_ranks or ctx.latest(0) >= v):
                break
        stream.synchronize()
        ctx.relay_step()
        barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    pub_host.clear()
    ctx.kernel_times()
    ctx.set_profiling(True)
    st0 = ctx.stats()
    clk = Clocks(rank)
    barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lat = []
    with (clk if not args.quick else _Null()):
        start.record(stream)
        for _ in range(args.steps):
            t0 = time.perf_counter()
            step()
            lat.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        end.record(stream)
        end.synchronize()
    ms = start.elapsed_time(end)
    kt = ctx.kernel_times()
    ctx.set_profiling(False)
    st1 = ctx.stats()
    launches = sum(n for _, n in kt.values())

    def allreduce(x, op):
        if gloo is None:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=op, group=gloo)
        return float(t.item())

    allmax = lambda x: allreduce(x, dist.ReduceOp.MAX if gloo is not None else None)
    allsum = lambda x: allreduce(x, dist.ReduceOp.SUM if gloo is not None else None)
    ms_max = allmax(ms)
    launches_all = int(allsum(launches))
    avg = {k: (v / n if n else None) for k, (v, n) in kt.items()}
    # a streamed pull is many k_pull launches (one batch per arriving chunk): per pull = the sum of
    # this rank's pull launches / (timed steps x rollouts pulled here)
    n_pulled = len([rid for rid in mine if rid not in subs])
    if kt["pull"][1] and n_pulled:
        avg["pull"] = kt["pull"][0] / (args.steps * n_pulled)
    # per-rank roofline candidates of this rank's dominant kernel work
    cand = []
    if avg["pack"]:
        # 4 B fp32 read + 2 B bf16 slot write per param, + 2 B per param into a colocated subscriber
        b = (8.0 if subs else 6.0) * sum(sh.numel for sh in shards.values())
        cand.append(dict(kernel="k_pack" + ("+subscriber" if subs else ""), ms=avg["pack"], bound="hbm", bytes=b))
    if avg["hop"]:
        part_bytes = M if args.config in ("chain", "host") else M / max(1, T["fsdp"])
        cand.append(dict(kernel="k_hop", ms=avg["hop"], bound="pcie" if args.config == "host" else "nvlink",
                         bytes=float(part_bytes)))
    if avg["pull"] and mine:
        loc, rem = pull_bytes[mine[0]]
        if rem > 0:
            cand.append(dict(kernel="k_pull", ms=avg["pull"], bound="pcie" if args.config == "host" else "nvlink",
                             bytes=float(rem), local=loc, remote=rem))
        else:
            cand.append(dict(kernel="k_pull", ms=avg["pull"], bound="hbm", bytes=2.0 * loc, local=loc, remote=rem))
    per_rank = [None] * N
    mine_info = dict(rank=rank, ms=round(ms, 3), **{k: (round(v, 3) if v else None) for k, v in avg.items()},
                     cand=cand)
    if gloo is not None:
        dist.all_gather_object(per_rank, mine_info, group=gloo)
    else:
        per_rank = [mine_info]

    kmax = {k: allmax(v or 0.0) for k, v in avg.items()}   # collective: every rank, outside rank-0 code
    pcie_peak = measure_pcie(torch) if args.config == "host" and rank == 0 else None
    pub_timed = sorted(pub_host)
    e2e = None
    if not args.quick and not args.no_e2e:
        e2e = run_e2e(args, N, shards, bufs, mine, step, barrier, allmax, torch)
    stall = None
    if N == 1 and not args.quick and my_ranks:
        stall = actor_stall(ctx, lam, shards, state, actor_stream, torch)
    if stall is not None or pub_timed:
        stall = dict(stall or {}, publish_host_us=dict(
            p50=round(pub_timed[len(pub_timed) // 2] * 1e6, 1) if pub_timed else None,
            max=round(pub_timed[-1] * 1e6, 1) if pub_timed else None, n=len(pub_timed)))

    if rank == 0:
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        hbm_peak = peaks.get("hbm_gbs", 6650.0)
        nvl_peak = 770.0
        sec = ms_max / 1e3 / args.steps
        allc = [c for pr in per_rank for c in pr["cand"]]
        dom = max(allc, key=lambda c: c["ms"]) if allc else None
        roof = None
        if dom:
            if dom["bound"] == "pcie":
                peak, src = pcie_peak
            else:
                peak = hbm_peak if dom["bound"] == "hbm" else nvl_peak
                src = ("MEASURED_PEAKS.json hbm_gbs (burst copy)" if dom["bound"] == "hbm" and "hbm_gbs" in peaks
                       else "fallback 6.65 TB/s" if dom["bound"] == "hbm"
                       else "B200_PROFILING.md measured peer copy 770 GB/s/dir (nominal 900)")
            ach = dom["bytes"] / (dom["ms"] / 1e3) / 1e9
            nominal = {"hbm": 8000.0, "nvlink": 900.0}.get(dom["bound"])
            roof = dict(bound=dom["bound"], kernel=dom["kernel"], achieved=ach, peak=peak, unit="GB/s",
                        frac=ach / peak, frac_of_nominal=(ach / nominal if nominal else None), traffic=traffic_of(dom["kernel"], args.model, N, args.config),
                        algorithmic_bytes_per_launch=dom["bytes"], launch_ms=dom["ms"], peak_source=src)
        cpu = None
        if N == 1 and not args.quick and not args.no_cpu_baseline:
            _, cpu = oracle_sample(args.model, args.cpu_seconds)
        lat.sort()
        out = dict(
            metric=METRIC, value=sec, unit=UNIT, n_gpus=N, steps=args.steps, warmup=args.warmup,
            ms_per_step=sec * 1e3, higher_is_better=False, scaling="weak", vs_baseline=None, dtype="bf16",
            data="synthetic",
            config=dict(workload=f"{args.model} [{args.config}]: " + T["desc"],
                        model=f"Qwen2.5-{args.model.upper()}-shaped", params=params, snapshot_bytes=M,
                        chunk_bytes=info.chunk_bytes, chunks=info.total_chunks, global_batch=None, seq_len=None,
                        parallelism=f"{args.config} N={N}", l2="inputs (fp32 masters, slots) >> 126 MB L2"),
            roofline=roof,
            kernels_ms=kmax, per_rank=per_rank,
            host_latency_ms=dict(p50=lat[len(lat) // 2] * 1e3, max=lat[-1] * 1e3),
            paper_context="actor stall 0.64 s (32B) / 1.40 s (72B); 72B to 127 relays < 1.6 s on 128x8 H800 + RDMA",
            cpu_baseline=cpu, e2e=e2e, gpu_launches=launches_all, actor_stall=stall,
            stats=dict(publishes=st1["publishes"] - st0["publishes"], hops=st1["hops_launched"] - st0["hops_launched"],
                       pulls=st1["pulls"] - st0["pulls"], skipped=st1["versions_skipped"] - st0["versions_skipped"]),
            clocks=None if args.quick else clk.summary())
        print(json.dumps(out))
    ctx.close()
    if N > 1:
        dist.barrier(group=gloo)
        dist.destroy_process_group()
    return 0


def live_event(torch, timing=False):
    """A torch CUDA event with its handle created (torch creates it lazily at the first record; until
    then .cuda_event is 0 and liblam would be handed a NULL event)."""
    e = torch.cuda.Event(enable_timing=timing)
    e.record()
    return e


def actor_stall(ctx, lam, shards, state, actor_stream, torch, reps=5, target_ms=25.0):
    """Actor stall per publish, the trainer's view of step 5 ("pushes the new
    actor weights to the master relay and immediately resumes its next training iteration"):
      reads_done_wait_ms  actor-stream wait on reads_done before the next optimizer step, when that step
                          comes one synthetic training step after the publish;
      inflation_ms        that training step's slowdown from the concurrent pack (SM / HBM contention,
                          PAPER L401-402): synthetic step = a bf16 GEMM loop of ~target_ms on the actor
                          stream (torch/cuBLAS: it stands in for the trainer, it is not the path).
    Pack-only publishes (no subscriber), each committed before the next; medians over `reps`."""
    n = 8192
    a = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    ev = lambda: torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(actor_stream):
        for _ in range(3):
            torch.mm(a, b, out=c)
        e0, e1 = ev(), ev()
        e0.record()
        for _ in range(10):
            torch.mm(a, b, out=c)
        e1.record()
    e1.synchronize()
    iters = max(1, int(target_ms / (e0.elapsed_time(e1) / 10)))

    def train_step():
        with torch.cuda.stream(actor_stream):
            for _ in range(iters):
                torch.mm(a, b, out=c)

    alone, total, wait, busy = [], [], [], []
    for _ in range(reps):
        with torch.cuda.stream(actor_stream):
            s0, s1 = ev(), ev()
            s0.record()
        train_step()
        with torch.cuda.stream(actor_stream):
            s1.record()
        s1.synchronize()
        alone.append(s0.elapsed_time(s1))
    for _ in range(reps):
        state["v"] += 1
        v = state["v"]
        rd = {r: live_event(torch, timing=True) for r in shards}
        with torch.cuda.stream(actor_stream):
            t0, t_mid, t1 = ev(), ev(), ev()
            t0.record()
        for r, sh in shards.items():
            while ctx.publish(v, r, sh.shards(), actor_stream.cuda_stream, rd[r].cuda_event) == lam.LAM_EBUSY:
                ctx.relay_step()
        train_step()                                   # the next training iteration, concurrent with the pack
        with torch.cuda.stream(actor_stream):
            t_mid.record()
            for e in rd.values():
                actor_stream.wait_event(e)             # before the optimizer overwrites the fp32 masters
            t1.record()
        t1.synchronize()
        while ctx.relay_step()[0] != lam.LAM_IDLE:
            pass
        total.append(t0.elapsed_time(t_mid))
        wait.append(t_mid.elapsed_time(t1))
        busy.append(max(t0.elapsed_time(e) for e in rd.values()))
    med = lambda x: sorted(x)[len(x) // 2]
    del a, b, c
    return dict(step_ms_alone=round(med(alone), 3), step_ms_with_publish=round(med(total), 3),
                inflation_ms=round(med(total) - med(alone), 3),
                inflation_frac=round(med(total) / med(alone) - 1, 4),
                reads_done_wait_ms=round(med(wait), 4), masters_busy_ms=round(med(busy), 3),
                actor_step=f"bf16 GEMM {n}^3 x {iters} on the actor stream (~{target_ms:.0f} ms)", reps=reps)


def measure_pcie(torch):
    """Host-tier roofline: this box's pinned copy bandwidth, measured here (best of 5, 1 GiB each way);
    the host relay's dominant direction decides (receive = D2H, pull = H2D), so report the max."""
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    best = {}
    for name, (dst, src) in {"h2d": (d, h), "d2h": (h, d)}.items():
        t = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dst.copy_(src, non_blocking=True)
            b.record()
            b.synchronize()
            t.append(a.elapsed_time(b))
        best[name] = n / (min(t) / 1e3) / 1e9
    del h, d
    return max(best.values()), "measured in this run: pinned cudaMemcpy 1 GiB, H2D %.1f / D2H %.1f GB/s" % (
        best["h2d"], best["d2h"])


def traffic_of(kernel, model, N, config):
    """dram read+write bytes per launch from the committed ncu --set full capture, if one matches."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return t.get(f"{kernel}:{model}:{config}:{N}")
    except Exception:
        return None


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def run_e2e(args, N, shards, bufs, mine, step, barrier, allmax, torch):
    import psutil
    need = sum(sh.buf.numel() * 4 for sh in shards.values()) + sum(b.bytes for b in bufs.values())
    need_all = allsum_host(need, torch)          # every rank pins its share of the same host RAM
    ok = psutil.virtual_memory().available > 1.5 * need_all + (16 << 30)
    if allmax(0.0 if ok else 1.0) != 0.0:
        return dict(value=None, unit=UNIT, reason="not enough host RAM for pinned buffers")
    h2d = {r: sh.buf.to("cpu").pin_memory() for r, sh in shards.items()}
    d2h = {rid: {n: torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for n, t in bufs[rid].bufs.items()}
           for rid in mine}
    step(h2d, d2h)  # warm-up with host buffers
    torch.cuda.synchronize()
    barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream()
    s.record(st)
    for _ in range(args.e2e_steps):
        step(h2d, d2h)
    torch.cuda.synchronize()
    e.record(st)
    e.synchronize()
    ms = allmax(s.elapsed_time(e))
    hb = allsum_host(sum(sh.buf.numel() * 4 for sh in shards.values()), torch)
    db = allsum_host(sum(b.bytes for b in bufs.values()), torch)
    return dict(value=ms / 1e3 / args.e2e_steps, unit=UNIT, h2d_bytes_per_step=int(hb), d2h_bytes_per_step=int(db),
                steps=args.e2e_steps,
                note="pinned host fp32 masters -> H2D -> lam_publish -> relay -> lam_pull -> D2H of every rollout")


def allsum_host(x, torch):
    import torch.distributed as dist
    if not dist.is_initialized():
        return x
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=_gloo_group())
    return float(t.item())


_GLOO = None


def _gloo_group():
    global _GLOO
    import torch.distributed as dist
    if _GLOO is None:
        _GLOO = dist.new_group(backend="gloo")
    return _GLOO


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python
"""bench.py — publish -> all-rollouts weight-sync latency of the relay tier (arxiv 2510.12633 §4).

One step = one pass of the whole hot path over a fresh version:
  lam_publish(v)   fp32 master shard -> bf16 RNE -> chunked bucket image in the master's slot
  lam_relay_step   chain-pipelined hops master -> relay 1 -> ... (N > 1), version commit
  lam_pull         every rollout pulls v and reshards it into its TP buffers
and the step's time is publish -> every rollout's pull completed.

Workload (BASELINE.json configs[1]): Qwen2.5-7B-shaped snapshot (7.62 G params, 15.23 GB bf16),
actor FSDP-1 on GPU 0.  N = 1: master node on GPU 0, one TP=1 rollout pulling from it.
N > 1 (one process per GPU): relays on GPUs 1..N-1 in a chain, one TP=1 rollout per relay GPU
(config 2 at N = 8).  Weak scaling: each added GPU adds one relay + one rollout.

`python bench.py --gpus N` without torchrun's environment re-launches itself as N ranks
(torch.distributed.run, 127.0.0.1); under torchrun it runs as the rank it is given.

After the timed steps every run publishes one more, freshly generated version and checks it against
the oracle (outside the timed region): chunk headers of every node == node 0's (digest agreement),
two chunks per node == oracle.image.publish_chunk byte for byte, and sampled elements of every
rollout's buffers == oracle.tp.dst_elements; the line carries the counts under "parity".

At N = 8 (or with --headline on) the line also carries "headline": the full-size 8-GPU
configurations of the north star (32B x 8 colocated TP=2, 32B relay-tp TP=2, 72B TP=8 / TP=4), each
with its NVLink bound and ratio.  `--config stress` runs BASELINE configs[4] (continuous publish,
6 rollouts pulling at exponential intervals).

`--impl reference` times the CPU oracle (the reference arm of this tier).
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
NVL_NOMINAL = 900.0      # GB/s per direction per GPU (NVLink 5, 18 links x 50 GB/s)
NVL_MEASURED = 770.0     # B200_PROFILING.md measured peer copy per direction


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lam", choices=["lam", "reference"])
    ap.add_argument("--model", default="7b")
    ap.add_argument("--config", default="chain", choices=["chain", "colocated", "relay-tp", "host", "stress"],
                    help="placement: chain (config 2), colocated (config 4), relay-tp (config 3), "
                         "host (NEXT-3: the paper's host-memory relay tier), stress (config 5)")
    ap.add_argument("--tp", type=int, default=0, help="rollout TP size (colocated / relay-tp)")
    ap.add_argument("--chunk-mb", type=int, default=0, help="chunk size; 0 = Appendix D k*")
    ap.add_argument("--hop-ctas", type=int, default=0)
    ap.add_argument("--hop-mode", default="kernel", choices=["kernel", "ce", "mc", "tree"],
                    help="relay hop: TMA kernel, copy engines + k_verify, NVSwitch multicast (NEXT-2: the "
                         "pack stores once through a multicast object, every relay verifies its replica), or tree "
                         "(two-level: each relay pulls its 1/R of the chunks from node 0, the rest from their owners)")
    ap.add_argument("--stream-pull", default="auto", choices=["auto", "on", "off"],
                    help="on: rollouts reshard chunk by chunk while their relay receives (lam_pull_stream); "
                         "off: pull once the relay committed (lam_pull); auto: on for chain / relay-tp, off for "
                         "colocated (there the pull competes with the pack for HBM and gains nothing)")
    ap.add_argument("--no-stream-pull", action="store_true", help="same as --stream-pull off")
    ap.add_argument("--no-subscribe", action="store_true",
                    help="colocated rollouts pull after the pack instead of being written by it")
    ap.add_argument("--slots", type=int, default=0, help="ring slots per node (0: 2, stress: 3)")
    ap.add_argument("--pack-ctas", type=int, default=0)
    ap.add_argument("--pack-sms", type=int, default=0, help="confine the pack to this many SMs (0 = all)")
    ap.add_argument("--pull-ctas", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="skip the post-run oracle parity check")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the single-thread oracle sample")
    ap.add_argument("--headline", default="auto", choices=["auto", "on", "off"],
                    help="also run the full-size 8-GPU configurations (auto: at N = 8)")
    ap.add_argument("--extra-steps", type=int, default=5, help="timed steps of each headline configuration")
    ap.add_argument("--stress-steps", type=int, default=40, help="--config stress: actor steps")
    ap.add_argument("--stress-ms", type=float, default=25.0, help="--config stress: synthetic actor step (ms)")
    ap.add_argument("--quick", action="store_true", help="profiling mode: no e2e, no cpu baseline, no clocks")
    return ap.parse_args(argv)


# ------------------------------------------------------------------------------ CPU oracle leg
def host_info():
    cpu = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return dict(nproc=os.cpu_count(), cpu_model=cpu,
                affinity=len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())


def oracle_sample(model: str, seconds: float, version: int = 1):
    """Time the oracle (as it stands, one thread) on a bounded sample of the workload, scaled to one step.

    Sample: the leading segments of the image (inputs pre-generated, like resident masters):
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
    budget_elems = int(1.5e7 * seconds)          # ~15 M params/s through the numpy oracle
    chosen, n = [], 0
    for t in range(1, len(tl)):               # skip the embedding: keep the sample bounded
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
    return full, dict(kind="oracle", cores=1, value=full, unit=UNIT, measured="scaled sample",
                      sample=f"{len(chosen)} tensors / {n / 1e6:.1f} M params of {model} "
                             f"({100 * frac:.2f}%): publish {t_pub:.2f} s + pull {t_pull:.2f} s, "
                             f"scaled to the full snapshot; numpy, single thread")


class OracleStep:
    """The oracle's full step on all host cores (SURVEY §8(d) "the same code with a per-tensor thread
    pool over all cores"), measured, not scaled:

      publish  per chunk g (pool): every segment of g = rne_bf16(fp32 master values), chunk_checksum
      relay    per relay node and chunk (pool): copy the chunk from the predecessor's image, recompute
               chunk_checksum and compare with the header (A3/A4)
      pull     per tensor (pool): unpack_tensor through the inverse bucket map (TP=1 rule)

    Inputs (the fp32 masters, harness) and the images live in anonymous shared memory that the forked
    workers inherit.  The workers run only numpy + oracle/ code."""

    def __init__(self, model: str, relays: int = 0, workers: int | None = None, inputs_from=None,
                 chunk_bytes: int = 128 << 20):
        import mmap

        import numpy as np

        from oracle.image import image_plan
        from oracle.model import MODELS, numel, tensors
        self.model = model
        self.d = MODELS[model]
        tl = tensors(self.d)
        self.shapes = [s for _, s in tl]
        self.sizes = [numel(s) for s in self.shapes]
        self.base = np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int64)
        self.P = int(self.base[-1])
        self.plan = image_plan(self.shapes, 1, chunk_bytes)
        self.relays = relays
        self.workers = workers or os.cpu_count() or 1

        def shared(nbytes, dtype):
            m = mmap.mmap(-1, max(nbytes, 1))
            self._maps.append(m)
            return np.frombuffer(m, dtype=dtype)
        self._maps = []
        self.inputs = shared(4 * self.P, np.uint32)
        self.images = [shared(self.plan.image_bytes, np.uint8) for _ in range(2 if relays else 1)]
        self.out = shared(2 * self.P, np.uint16)
        self.hdr = [None] * self.plan.total_chunks
        t0 = time.perf_counter()
        if inputs_from is not None:
            inputs_from(self)                      # caller copies resident masters (e.g. from the GPU)
        else:
            self._pool_map(_oracle_gen, [(self, t) for t in range(len(self.shapes))])
        self.setup_s = time.perf_counter() - t0

    def _pool_map(self, fn, items):
        import multiprocessing as mp
        global _ORACLE
        _ORACLE = self
        if self.workers <= 1:
            return [fn(i[1]) for i in items]
        with mp.get_context("fork").Pool(self.workers) as pool:
            return pool.map(fn, [i[1] for i in items], chunksize=1)

    def step(self) -> dict:
        t0 = time.perf_counter()
        hdr = self._pool_map(_oracle_publish_chunk, [(self, g) for g in range(self.plan.total_chunks)])
        t1 = time.perf_counter()
        self.hdr = hdr
        for i in range(self.relays):
            ok = self._pool_map(_oracle_relay_chunk, [(self, (i, g)) for g in range(self.plan.total_chunks)])
            if not all(ok):
                raise RuntimeError("oracle relay: checksum mismatch")
        t2 = time.perf_counter()
        self._pool_map(_oracle_pull_tensor, [(self, t) for t in range(len(self.shapes))])
        t3 = time.perf_counter()
        return dict(total=t3 - t0, publish=t1 - t0, relay=t2 - t1, pull=t3 - t2)

    def close(self):
        for m in self._maps:
            try:
                m.close()
            except BufferError:
                pass
        self._maps = []


_ORACLE = None


def _oracle_gen(t):
    from synth import SEED, gen_bits
    o = _ORACLE
    step = 1 << 24
    for a in range(0, o.sizes[t], step):
        n = min(step, o.sizes[t] - a)
        o.inputs[o.base[t] + a:o.base[t] + a + n] = gen_bits(SEED, 1, t, a, n)
    return 0


def _oracle_publish_chunk(g):
    from oracle.bf16 import rne_bf16
    from oracle.checksum import chunk_checksum
    o = _ORACLE
    p = o.plan
    img = o.images[0]
    a, n = g * p.C, p.chunk_len(g)
    for s in p.segments:                         # segments intersecting chunk g (FSDP-1: one region)
        so = p.image_offset(s)
        lo, hi = max(a, so), min(a + n, so + 2 * s.count)
        if hi <= lo:
            continue
        e0 = (lo - so) // 2
        src = o.inputs[o.base[s.tensor_id] + s.elem0 + e0: o.base[s.tensor_id] + s.elem0 + e0 + (hi - lo) // 2]
        img[lo:hi] = rne_bf16(src).view("u1")
    return chunk_checksum(img[a:a + n])


def _oracle_relay_chunk(arg):
    from oracle.checksum import chunk_checksum
    i, g = arg
    o = _ORACLE
    p = o.plan
    src, dst = o.images[i % 2], o.images[(i + 1) % 2]
    a, n = g * p.C, p.chunk_len(g)
    dst[a:a + n] = src[a:a + n]
    return chunk_checksum(dst[a:a + n]) == o.hdr[g]


def _oracle_pull_tensor(t):
    from oracle.image import unpack_tensor
    o = _ORACLE
    img = o.images[o.relays % 2] if o.relays else o.images[0]
    read = lambda off, k: img[off:off + k]
    o.out[o.base[t]:o.base[t] + o.sizes[t]] = unpack_tensor(read, o.plan, t, o.shapes[t]).ravel()
    return 0


def line_config(args, N):
    """The `config` object of the JSON line — identical for the lam arm and the reference arm (the
    driver compares the two arms only on the same config)."""
    T = topology(args.config if args.config != "stress" else "chain", N, args.tp)
    return dict(workload=f"{args.model} [{args.config}]: " + T["desc"],
                model=f"Qwen2.5-{args.model.upper()}-shaped", params=int(P_params(args.model)),
                snapshot_bytes=int(2 * P_params(args.model)), global_batch=None, seq_len=None,
                parallelism=f"{args.config} N={N}" + ("" if args.hop_mode == "kernel" else f" hop={args.hop_mode}"),
                l2="inputs (fp32 masters, slots) >> 126 MB L2")


def run_reference(args):
    """The reference arm of this tier: the CPU oracle, as it stands, timed on the host cores on the lam
    arm's workload — every timed step a FULL publish -> relay -> TP=1 pull of the snapshot on a process
    pool over all cores (measured, not scaled).  Warm-up steps run on a bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    N = args.gpus
    relays = N - 1 if args.config == "chain" else 0
    hi = host_info()
    t_setup = time.perf_counter()
    o = OracleStep(args.model, relays=relays)
    for _ in range(args.warmup):                 # untimed, bounded
        oracle_sample(args.model, 2.0)
    times = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        times.append(o.step())
    wall = time.perf_counter() - t0
    o.close()
    value = sum(t["total"] for t in times) / len(times)
    desc = topology(args.config if args.config != "stress" else "chain", N, args.tp)["desc"]
    sample = (f"full {args.model} step: publish (cast+pack+checksum of every chunk) + {relays} relay hop(s) "
              f"(copy + checksum verify) + TP=1 pull (inverse bucket map) of all {o.P / 1e9:.2f} G params; "
              f"numpy oracle on a {o.workers}-process pool; inputs generated once (untimed, "
              f"{o.setup_s:.1f} s); warm-up steps on a bounded sample")
    out = dict(metric=METRIC, value=value, unit=UNIT, impl="reference", n_gpus=N, steps=args.steps,
               warmup=args.warmup, ms_per_step=value * 1e3, higher_is_better=False, scaling="weak",
               vs_baseline=None, dtype="bf16", data="synthetic",
               config=line_config(args, N),
               reference="CPU oracle publish -> relay -> TP=1 pull, full snapshot per step",
               cpu_baseline=dict(kind="oracle", cores=o.workers, value=value, unit=UNIT, sample=sample,
                                 measured="full step", host=hi, wall_s=round(wall, 2),
                                 setup_s=round(time.perf_counter() - t_setup - wall, 2),
                                 phases_s={k: round(sum(t[k] for t in times) / len(times), 3)
                                           for k in ("publish", "relay", "pull")}),
               e2e=dict(value=value, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0),
               consistency=dict(steps_x_value_s=round(value * args.steps, 2), timed_wall_s=round(wall, 2)))
    print(json.dumps(out), flush=True)
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


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


# -------------------------------------------------------------------------------- placements
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
    if config == "stress":
        # config 5 (BASELINE configs[4]): 7B actor on GPU 0 publishing every step; 6 TP=1 rollouts pull
        # staggered versions.  N=1: rollouts pull from the master node on GPU 0; N>1: relays on GPUs
        # 1..N-1 in a chain, rollouts round-robin over them
        if N == 1:
            return dict(fsdp=1, actors=[0], relays=[], rollouts=[(0, 0, 1, 0)] * 6,
                        desc="stress: actor FSDP-1 + master node on GPU0, 6 TP=1 rollouts pulling from it")
        relay_gpus = list(range(1, N))
        ro = [(1 + i % len(relay_gpus), relay_gpus[i % len(relay_gpus)], 1, 0) for i in range(6)]
        return dict(fsdp=1, actors=[0], relays=[[d] for d in relay_gpus], rollouts=ro,
                    desc=f"stress: actor FSDP-1 on GPU0 -> chain of {N - 1} relays, 6 TP=1 rollouts "
                         f"round-robin on GPUs 1..{N - 1}")
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


# The north star's full-size 8-GPU configurations, run as extra keys at N = 8.
HEADLINE = [
    ("32b_x8_colocated_tp2", "32b", "colocated", 2),   # "all 8 rollouts": 4 TP=2 replicas, replica k = {k, k+4}
    ("32b_relay_tp2", "32b", "relay-tp", 2),           # config 3: FSDP-4 -> relay on GPUs 4-7 -> 2 x TP=2
    ("72b_colocated_tp8", "72b", "colocated", 8),      # config 4
    ("72b_colocated_tp4", "72b", "colocated", 4),      # config 4
]


def nvlink_bound(T, N, P, pull_in=None, multicast=False):
    """Publish->all lower bound: max over GPUs of the bf16 bytes that must enter (or
    leave) that GPU over NVLink, / 900 GB/s (the stages pipeline).  Counted from the placement: chain
    hops between GPUs, plus `pull_in[d]` = bytes the rollouts on GPU d gather from other GPUs.
    multicast (NEXT-2): every relay receives from node 0 and the switch replicates, so the source's
    egress is each region once, whatever the number of relays."""
    n = T["fsdp"]
    region = 2.0 * P / n                    # bf16 bytes of one actor rank's region
    ing = {d: 0.0 for d in range(N)}
    egr = {d: 0.0 for d in range(N)}
    prev = {r: T["actors"][r] for r in range(n)}
    sent = set()
    for node in T["relays"]:                # chain hops: each relay part receives its rank's region
        for r, d in enumerate(node):
            src = T["actors"][r] if multicast else prev[r]
            if d != src:
                ing[d] += region
                if not multicast or r not in sent:
                    egr[src] += region
                    sent.add(r)
        prev = {r: node[r] for r in range(n)}
    for d, x in (pull_in or {}).items():
        ing[d] += x
    return ing, egr


def pull_remote_bytes(ctx, rid, tp_layout):
    loc, rem = ctx.pull_bytes(rid, tp_layout)
    return loc, rem


def live_event(torch, timing=False):
    """A torch CUDA event with its handle created (torch creates it lazily at the first record; until
    then .cuda_event is 0 and liblam would be handed a NULL event)."""
    e = torch.cuda.Event(enable_timing=timing)
    e.record()
    return e


class Dist:
    def __init__(self, torch, N, rank):
        import torch.distributed as dist
        self.dist, self.torch, self.N, self.rank = dist, torch, N, rank
        self.gloo = self.gloo_extra = None
        if N > 1:
            from datetime import timedelta
            dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
            self.gloo = dist.new_group(backend="gloo")
            # the extra (headline) configurations run on a group with a 15 min timeout: a rank that failed
            # alone turns the others' wait into an exception instead of a hang that would cost the line
            self.gloo_extra = dist.new_group(backend="gloo", timeout=timedelta(seconds=900))

    def barrier(self):
        if self.gloo is not None:
            self.dist.barrier(group=self.gloo)

    def reduce(self, x, op):
        if self.gloo is None:
            return x
        t = self.torch.tensor([float(x)], dtype=self.torch.float64)
        self.dist.all_reduce(t, op=op, group=self.gloo)
        return float(t.item())

    def max(self, x):
        return self.reduce(x, self.dist.ReduceOp.MAX if self.gloo is not None else None)

    def sum(self, x):
        return self.reduce(x, self.dist.ReduceOp.SUM if self.gloo is not None else None)

    def gather(self, obj):
        if self.gloo is None:
            return [obj]
        out = [None] * self.N
        self.dist.all_gather_object(out, obj, group=self.gloo)
        return out

    def close(self):
        if self.gloo is not None:
            self.dist.barrier(group=self.gloo)
            self.dist.destroy_process_group()


class Placement:
    """One placement set up through the C ABI on this rank: context, fp32 masters, rollout buffers."""

    def __init__(self, args, D: Dist, model: str, config: str, tp: int, tag: str):
        import torch

        from paper_2510_12633_b200 import lam
        from paper_2510_12633_b200.workload import MODELS, ActorShard, RolloutBuffers
        from synth import SEED
        self.torch, self.lam, self.D, self.args = torch, lam, D, args
        N, rank = D.N, D.rank
        self.N, self.rank = N, rank
        self.model_name, self.config, self.tag = model, config, tag
        self.model = MODELS[model]
        self.T = T = topology(config, N, tp)
        self.rollouts = T["rollouts"]
        port = os.environ.get("MASTER_PORT", "0")
        cfg = lam.Config(model=self.model, fsdp_size=T["fsdp"], actor_devices=T["actors"], relays=T["relays"],
                         rollouts=[(n, d) for n, d, _, _ in self.rollouts], chunk_bytes=args.chunk_mb << 20,
                         proc_rank=rank, n_procs=N, proc_of_device={d: d for d in range(N)},
                         shm_name=f"lam_bench_{port}_{os.getppid()}_{tag}", hop_ctas=args.hop_ctas,
                         pack_ctas=args.pack_ctas, pull_ctas=args.pull_ctas, pack_sms=args.pack_sms,
                         slots=args.slots or (3 if config == "stress" and N > 1 else 2),
                         hop_mode={"ce": lam.LAM_HOP_COPY_ENGINE, "mc": lam.LAM_HOP_MULTICAST,
                                   "tree": lam.LAM_HOP_TREE}.get(args.hop_mode, lam.LAM_HOP_KERNEL),
                         host_relays=T.get("host_relays", []))
        self.ctx = ctx = lam.Context(cfg)
        if N > 1:
            blobs = D.gather(ctx.export_ipc())
            for p, b in enumerate(blobs):
                if p != rank:
                    ctx.import_ipc(p, b)
            ctx.connect()
            D.barrier()
        self.info = ctx.plan_info()
        self.my_ranks = [r for r, d in enumerate(T["actors"]) if d == rank]
        self.shards = {r: ActorShard(self.model, T["fsdp"], r, rank) for r in self.my_ranks}
        self.data_version = 1
        for sh in self.shards.values():
            sh.fill(SEED, 1)
        self.mine = [rid for rid, (_, dev, _, _) in enumerate(self.rollouts) if dev == rank]
        self.bufs = {rid: RolloutBuffers(self.model, self.rollouts[rid][2], self.rollouts[rid][3], rank)
                     for rid in self.mine}
        self.pull_bytes = {rid: ctx.pull_bytes(rid, self.bufs[rid].tp) for rid in self.mine}
        self.stream = torch.cuda.Stream()
        self.rstream = {rid: torch.cuda.Stream() for rid in self.mine}   # one engine stream per rollout
        self.actor_stream = torch.cuda.Stream()
        torch.cuda.synchronize()
        self.v = 0
        self.pub_host = []
        ns = args.no_stream_pull or args.stream_pull == "off" or (args.stream_pull == "auto" and config == "colocated")
        self.no_stream_pull = ns
        # colocated rollouts (node 0, an actor GPU, TP=1) are written by the pack itself (lam_subscribe),
        # only when every actor rank packs on the rollout's GPU (the pack writes only its own shards)
        self.subs = [] if args.no_subscribe else [
            rid for rid in self.mine if self.rollouts[rid][0] == 0 and self.rollouts[rid][2] == 1
            and all(d == self.rollouts[rid][1] for d in T["actors"])]
        self.sub_done = {rid: live_event(torch) for rid in self.subs}

    def refill(self, version):
        """The optimizer's write of new master values: the generator at `version` (harness)."""
        from synth import SEED
        for sh in self.shards.values():
            sh.fill(SEED, version)
        self.data_version = version
        self.torch.cuda.synchronize()

    def step(self, h2d=None, d2h=None):
        lam, ctx = self.lam, self.ctx
        self.v += 1
        v = self.v
        for rid in self.subs:
            ctx.subscribe(rid, self.bufs[rid].tp, self.sub_done[rid].cuda_event)
        for r in self.my_ranks:
            if h2d is not None:                        # e2e: the step's inputs arrive from host memory
                with self.torch.cuda.stream(self.actor_stream):
                    self.shards[r].buf.copy_(h2d[r], non_blocking=True)
            t_pub = time.perf_counter()
            while ctx.publish(v, r, self.shards[r].shards(), self.actor_stream.cuda_stream) == lam.LAM_EBUSY:
                ctx.relay_step()
            self.pub_host.append(time.perf_counter() - t_pub)
        pending, streaming = [rid for rid in self.mine if rid not in self.subs], list(self.subs)
        got_v = {}
        while True:
            ctx.relay_step()
            for rid in list(pending):
                if self.no_stream_pull:                     # classic: pull once the relay committed v
                    got = (ctx.pull(rid, self.bufs[rid].tp, self.stream.cuda_stream)
                           if ctx.latest(self.rollouts[rid][0]) >= v else 0)
                else:                                       # reshard chunk by chunk while v arrives
                    got = ctx.pull_stream(rid, self.bufs[rid].tp, self.stream.cuda_stream, None, v)
                if got:
                    assert got >= v, (got, v)
                    got_v[rid] = got
                    pending.remove(rid)
                    streaming.append(rid)
            for rid in list(streaming):
                if (self.no_stream_pull and rid not in self.subs) or ctx.pull_state(rid)[1] == 0:
                    if rid in self.subs:                    # written by the pack on the side stream
                        self.stream.wait_event(self.sub_done[rid])
                        got_v[rid] = ctx.pull_state(rid)[0]
                    if d2h is not None:
                        with self.torch.cuda.stream(self.stream):
                            for name, t in self.bufs[rid].bufs.items():
                                d2h[rid][name].copy_(t, non_blocking=True)
                    streaming.remove(rid)
            if not pending and not streaming and (not self.my_ranks or ctx.latest(0) >= v):
                break
        self.stream.synchronize()
        ctx.relay_step()
        self.D.barrier()
        return got_v

    def quiesce(self, v):
        """Step the progress engine until every node committed v (every rank must call)."""
        t0 = time.time()
        n_nodes = len(self.T["relays"]) + 1
        while not all(self.ctx.latest(n) >= v for n in range(n_nodes)):
            self.ctx.relay_step()
            if time.time() - t0 > 300:
                raise TimeoutError(f"version {v} never completed at every node")
        self.D.barrier()

    def close(self):
        self.torch.cuda.synchronize()
        self.ctx.close()
        self.shards, self.bufs = {}, {}
        self.torch.cuda.empty_cache()
        self.D.barrier()


def timed_steps(P: Placement, steps, warmup, quick):
    """W warm-up steps, then exactly `steps` timed steps bracketed by barrier + synchronize; returns
    this rank's elapsed ms, per-step host latencies, kernel times and clocks."""
    torch, ctx = P.torch, P.ctx
    for _ in range(warmup):
        P.step()
    torch.cuda.synchronize()
    P.pub_host.clear()
    ctx.kernel_times()
    ctx.set_profiling(True)
    st0 = ctx.stats()
    clk = Clocks(P.rank)
    P.D.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lat = []
    with (clk if not quick else _Null()):
        start.record(P.stream)
        for _ in range(steps):
            t0 = time.perf_counter()
            P.step()
            lat.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        end.record(P.stream)
        end.synchronize()
    ms = start.elapsed_time(end)
    kt = ctx.kernel_times()
    ctx.set_profiling(False)
    st1 = ctx.stats()
    return dict(ms=ms, lat=lat, kt=kt, st0=st0, st1=st1, clocks=None if quick else clk.summary())


def roofline_of(P: Placement, kt, steps):
    """Per-rank roofline candidates (dominant kernel work of this rank) from liblam's own CUDA-event
    timings on the streams the kernels run on."""
    M = P.info.snapshot_bytes
    avg = {k: (v / n if n else None) for k, (v, n) in kt.items()}
    n_pulled = len([rid for rid in P.mine if rid not in P.subs])
    if kt["pull"][1] and n_pulled:      # a streamed pull = many launches: per pull = sum / (steps x rollouts)
        avg["pull"] = kt["pull"][0] / (steps * n_pulled)
    cand = []
    mc = P.args.hop_mode == "mc" and P.N > 1
    if avg["pack"] and mc:
        # NEXT-2: the pack's stores go through the NVSwitch multicast object — NVLink egress of the image
        # once (each relay GPU receives M), 4 B/param of HBM reads on the side
        cand.append(dict(kernel="k_pack(multicast)", ms=avg["pack"], bound="nvlink",
                         bytes=2.0 * sum(sh.numel for sh in P.shards.values())))
    elif avg["pack"]:
        b = (8.0 if P.subs else 6.0) * sum(sh.numel for sh in P.shards.values())
        cand.append(dict(kernel="k_pack" + ("+subscriber" if P.subs else ""), ms=avg["pack"], bound="hbm", bytes=b))
    if avg["hop"] and mc:   # verify + commit from the local replica: HBM read + write
        # it runs as long as the multicast pack feeds it (it waits on the chunk flags): reported, never
        # the dominant kernel
        cand.append(dict(kernel="k_hop(replica)", ms=avg["hop"], bound="hbm", bytes=2.0 * M, follows=True))
    elif avg["hop"]:
        part_bytes = M if P.config in ("chain", "host", "stress") else M / max(1, P.T["fsdp"])
        cand.append(dict(kernel="k_hop", ms=avg["hop"], bound="pcie" if P.config == "host" else "nvlink",
                         bytes=float(part_bytes)))
    if avg["pull"] and P.mine:
        loc, rem = P.pull_bytes[P.mine[0]]
        if rem > 0:
            cand.append(dict(kernel="k_pull", ms=avg["pull"], bound="pcie" if P.config == "host" else "nvlink",
                             bytes=float(rem), local=loc, remote=rem))
        else:
            cand.append(dict(kernel="k_pull", ms=avg["pull"], bound="hbm", bytes=2.0 * loc, local=loc, remote=rem))
    return avg, cand


def verify(P: Placement, chunk_mode="two"):
    """Parity of one fresh version against the oracle, outside the timed region (every rank calls).

    Publishes version v with master values W_v (generator at v), runs it to every node, then checks:
      digest   every node's chunk headers == node 0's (rank 0; SPEC L634 digest agreement)
      chunks   per node, chunk (7k+3) mod n and the last (short) chunk == oracle.image.publish_chunk,
               byte for byte, and the node's header (S1, S2) == oracle.checksum.chunk_checksum
      rollouts each rollout pulled exactly v; 512 sampled elements of every destination buffer ==
               oracle.tp.dst_elements (TP_r(RNE_bf16(W_v)) computed one element at a time)
    The oracle work of a rank runs on a small fork pool (numpy only)."""
    import numpy as np

    from oracle.checksum import chunk_checksum
    from oracle.image import image_plan
    from oracle.model import MODELS as OMODELS
    from oracle.model import tensors as otensors
    from oracle.tp import dst_elements
    from synth import SEED
    torch, ctx, D = P.torch, P.ctx, P.D
    t_start = time.time()
    v = P.v + 1
    P.refill(v)
    D.barrier()
    got = P.step()
    P.quiesce(v)
    fails = []
    n_nodes = len(P.T["relays"]) + 1
    total = P.info.total_chunks
    C = P.info.chunk_bytes
    nodes_ok = None
    if P.rank == 0:
        h0 = ctx.read_headers(0, v)
        nodes_ok = 0
        for k in range(n_nodes):
            hk = h0 if k == 0 else ctx.read_headers(k, v)
            if hk == h0 and all(h["version"] == v and h["idx"] == i for i, h in enumerate(hk)):
                nodes_ok += 1
            else:
                fails.append(f"node {k}: chunk headers differ from node 0's")
    od = OMODELS[P.model_name]
    plan = image_plan([s for _, s in otensors(od)], P.T["fsdp"], C)
    jobs = []
    for k in range(P.rank, n_nodes, P.N):
        for g in sorted({(7 * k + 3) % total, total - 1}):
            jobs.append((k, g))
    global _VERIFY
    _VERIFY = (plan, SEED, v)
    import multiprocessing as mp
    workers = max(1, min(len(jobs), (os.cpu_count() or 1) // P.N))
    if workers > 1:
        with mp.get_context("fork").Pool(workers) as pool:
            wants = pool.map(_verify_chunk, [g for _, g in jobs], chunksize=1)
    else:
        wants = [_verify_chunk(g) for _, g in jobs]
    chunks_ok = 0
    for (k, g), want in zip(jobs, wants):
        ok = np.array_equal(ctx.read_image(k, v, g * C, want.size), want)
        h = ctx.read_headers(k, v, g, 1)[0]
        ok = ok and (h["s1"], h["s2"]) == chunk_checksum(want) and h["bytes"] == want.size
        chunks_ok += ok
        if not ok:
            fails.append(f"node {k} chunk {g} differs from the oracle")
    elems = elems_ok = 0
    rollouts_ok = 0
    for rid in P.mine:
        node, dev, tp, tr = P.rollouts[rid]
        if got.get(rid) != v:
            fails.append(f"rollout {rid}: pulled {got.get(rid)}, expected {v}")
            continue
        rng = np.random.default_rng(1000 * rid + v)
        ok_all = True
        for name, t in P.bufs[rid].bufs.items():
            idx = rng.integers(0, t.numel(), 512)
            g_ = t.view(-1).view(torch.int16)[torch.from_numpy(idx).to(t.device)].cpu().numpy().view(np.uint16)
            w = dst_elements(od, tp, tr, name, idx, SEED, v)
            ok = int((g_ == w).sum())
            elems += idx.size
            elems_ok += ok
            if ok != idx.size:
                ok_all = False
                fails.append(f"rollout {rid}: {name}: {idx.size - ok} sampled elements differ")
        rollouts_ok += ok_all
    mine = dict(rank=P.rank, nodes_ok=nodes_ok, chunks=len(jobs), chunks_ok=chunks_ok, elements=elems,
                elements_ok=elems_ok, rollouts=len(P.mine), rollouts_ok=rollouts_ok, fails=fails[:8])
    allr = D.gather(mine)
    D.barrier()
    out = dict(version=v, nodes=n_nodes, nodes_digest_ok=allr[0]["nodes_ok"],
               chunks_checked=sum(a["chunks"] for a in allr), chunks_ok=sum(a["chunks_ok"] for a in allr),
               elements_checked=sum(a["elements"] for a in allr), elements_ok=sum(a["elements_ok"] for a in allr),
               rollouts_checked=sum(a["rollouts"] for a in allr), rollouts_ok=sum(a["rollouts_ok"] for a in allr),
               seconds=round(time.time() - t_start, 1))
    out["ok"] = (out["nodes_digest_ok"] == n_nodes and out["chunks_ok"] == out["chunks_checked"]
                 and out["elements_ok"] == out["elements_checked"] and out["rollouts_ok"] == len(P.rollouts))
    f = [x for a in allr for x in a["fails"]]
    if f:
        out["fails"] = f[:16]
    return out


_VERIFY = None


def _verify_chunk(g):
    from oracle.image import publish_chunk
    plan, seed, v = _VERIFY
    return publish_chunk(plan, g, seed, v)


def pull_latency(P: Placement, reps=5):
    """Rollout pull latency (north star; "fetch the latest weights ... at any time"): an
    on-demand lam_pull of the newest complete version, host call -> destination buffers valid, per
    rollout, after the broadcast (untimed phase).  Returns every rank's samples gathered."""
    torch, ctx = P.torch, P.ctx
    samples = []
    for rid in P.mine:
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(P.stream)
            v = ctx.pull(rid, P.bufs[rid].tp, P.stream.cuda_stream)
            e1.record(P.stream)
            e1.synchronize()
            host = time.perf_counter() - t0
            ctx.relay_step()
            loc, rem = P.pull_bytes[rid]
            if v:
                samples.append(dict(rid=rid, host_ms=host * 1e3, dev_ms=e0.elapsed_time(e1), bytes=loc + rem,
                                    remote=rem))
    allr = [s for r in P.D.gather(samples) for s in r]
    P.D.barrier()
    if not allr:
        return None
    h = sorted(s["host_ms"] for s in allr)
    dv = sorted(s["dev_ms"] for s in allr)
    b = allr[0]["bytes"]
    return dict(p50_ms=round(h[len(h) // 2], 3), max_ms=round(h[-1], 3), device_p50_ms=round(dv[len(dv) // 2], 3),
                bytes_per_pull=b, remote_bytes_per_pull=allr[0]["remote"],
                gbs_p50=round(b / (dv[len(dv) // 2] / 1e3) / 1e9, 1), n=len(allr),
                what="lam_pull of the newest complete version into the rollout's TP buffers, host call -> done")


def summarize(P: Placement, res, steps, rank0_extra=None):
    """Per-placement result (rank 0 assembles; every rank must call: collectives inside)."""
    D = P.D
    N = P.N
    ms_max = D.max(res["ms"])
    # every kernel liblam launched in the timed region (the stats block is shared by all ranks)
    launches_all = int(res["st1"]["kernel_launches"] - res["st0"]["kernel_launches"])
    avg, cand = roofline_of(P, res["kt"], steps)
    mine_info = dict(rank=P.rank, ms=round(res["ms"], 3), **{k: (round(v, 3) if v else None) for k, v in avg.items()},
                     cand=cand)
    per_rank = D.gather(mine_info)
    kmax = {k: D.max(v or 0.0) for k, v in avg.items()}
    sec = ms_max / 1e3 / steps
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    allc = [c for pr in per_rank for c in pr["cand"] if not c.get("follows")]
    dom = max(allc, key=lambda c: c["ms"]) if allc else None
    roof = None
    if dom:
        if dom["bound"] == "pcie":
            peak, src = (rank0_extra or {}).get("pcie_peak") or (None, "unmeasured")
        else:
            peak = hbm_peak if dom["bound"] == "hbm" else NVL_MEASURED
            src = ("MEASURED_PEAKS.json hbm_gbs (burst copy)" if dom["bound"] == "hbm" and "hbm_gbs" in peaks
                   else "fallback 6.65 TB/s" if dom["bound"] == "hbm"
                   else "B200_PROFILING.md measured peer copy 770 GB/s/dir (nominal 900)")
        ach = dom["bytes"] / (dom["ms"] / 1e3) / 1e9
        nominal = {"hbm": 8000.0, "nvlink": NVL_NOMINAL}.get(dom["bound"])
        roof = dict(bound=dom["bound"], kernel=dom["kernel"], achieved=ach, peak=peak, unit="GB/s",
                    frac=(ach / peak if peak else None), frac_of_nominal=(ach / nominal if nominal else None),
                    traffic=traffic_of(dom["kernel"], P.model_name, N, P.config),
                    algorithmic_bytes_per_launch=dom["bytes"], launch_ms=dom["ms"], peak_source=src)
        if dom["bound"] == "nvlink":
            roof["per_link_gbs"] = ach / 18.0       # 18 NVLink 5 links per GPU, 50 GB/s/dir each
            # what the fabric gives each transport on this pool (tools/chain_bench.cu, 1 GiB per hop, every
            # hop at once): a relay that also serves its successor tops out below a lone hop
            roof["transport_ceilings_gbs"] = dict(single_hop_tma_pull=782, middle_relay_tma_pull=668,
                                                  middle_relay_copy_engines=765, multicast_store=558,
                                                  source="profiles/r2/r2f_chain_bench_4gpu.txt, r2g_mc_bench.txt")
            nvl = traffic_of("nvlink:" + dom["kernel"], P.model_name, N, P.config)
            if nvl:   # ncu nvlrx/nvltx of the same kernel (raw link bytes incl. packet headers / read requests)
                roof["nvlink_traffic"] = dict(nvl, source="ncu nvlrx__bytes.sum / nvltx__bytes.sum per launch")
    rem = 0.0 if P.config == "host" else float(sum(P.pull_bytes[rid][1] for rid in P.mine))
    pull_in = {r: x for r, x in enumerate(D.gather(rem))}
    ing, egr = nvlink_bound(P.T, N, P.info.params, pull_in, multicast=P.args.hop_mode == "mc")
    worst = max(max(ing.values()), max(egr.values()))
    bound_s = worst / (NVL_NOMINAL * 1e9)
    lat = sorted(res["lat"])
    out = dict(sec=sec, ms_per_step=sec * 1e3, roofline=roof, kernels_ms=kmax, per_rank=per_rank,
               host_latency_ms=dict(p50=lat[len(lat) // 2] * 1e3, max=lat[-1] * 1e3),
               gpu_launches=launches_all,
               nvlink_bound=dict(seconds=bound_s, ratio=(sec / bound_s if bound_s else None),
                                 max_gpu_ingress_bytes=max(ing.values()), max_gpu_egress_bytes=max(egr.values()),
                                 at="900 GB/s/dir nominal"),
               stats=dict(publishes=res["st1"]["publishes"] - res["st0"]["publishes"],
                          hops=res["st1"]["hops_launched"] - res["st0"]["hops_launched"],
                          pulls=res["st1"]["pulls"] - res["st0"]["pulls"],
                          skipped=res["st1"]["versions_skipped"] - res["st0"]["versions_skipped"]),
               clocks=res["clocks"])
    return out


# ---------------------------------------------------------------------------------- main
def self_launch(args):
    """`bench.py --gpus N` outside torchrun: re-run this command as N ranks on 127.0.0.1."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "RANK" not in os.environ:
        return self_launch(args)
    if args.impl == "reference":
        return run_reference(args)
    if os.environ.get("LAM_BENCH_WATCHDOG"):      # debugging aid: dump every thread's stack, then exit
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["LAM_BENCH_WATCHDOG"]), exit=True)
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    N = world
    if N != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    if torch.cuda.device_count() < N:
        raise SystemExit(f"--gpus {N} but only {torch.cuda.device_count()} CUDA devices")
    torch.cuda.set_device(rank)
    D = Dist(torch, N, rank)
    if args.config == "stress":
        out = run_stress(args, D)
        if rank == 0:
            print(json.dumps(out), flush=True)
        D.close()
        return 0

    P = Placement(args, D, args.model, args.config, args.tp, "main")
    res = timed_steps(P, args.steps, args.warmup, args.quick)
    pcie = measure_pcie(torch) if args.config == "host" and rank == 0 else None
    summ = summarize(P, res, args.steps, dict(pcie_peak=pcie))
    parity = None if args.no_verify else verify(P)
    plat = pull_latency(P)
    e2e = None
    if not args.quick and not args.no_e2e:
        e2e = run_e2e(args, P)
    stall = None
    if N == 1 and not args.quick and P.my_ranks:
        stall = actor_stall(P)
    pub_timed = sorted(P.pub_host[:args.steps]) if P.pub_host else []
    if stall is not None or pub_timed:
        s0, s1 = res["st0"], res["st1"]
        npub = max(1, s1["publishes"] - s0["publishes"])
        stall = dict(stall or {}, publish_host_us=dict(
            p50=round(pub_timed[len(pub_timed) // 2] * 1e6, 1) if pub_timed else None,
            max=round(pub_timed[-1] * 1e6, 1) if pub_timed else None, n=len(pub_timed),
            what="Python caller: ctypes marshalling + lam_publish"),
            publish_lib_us=dict(mean=round((s1["publish_ns_total"] - s0["publish_ns_total"]) / npub / 1e3, 1),
                                max_since_start=round(s1["publish_ns_max"] / 1e3, 1),
                                what="inside lam_publish (steady clock, library stats)"))
    cpu = None
    if rank == 0 and N == 1 and not args.quick and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, P)
    P.close()
    del P

    headline = None
    if args.headline == "on" or (args.headline == "auto" and N == 8):
        headline = {}
        main_group, D.gloo = D.gloo, D.gloo_extra or D.gloo
        for name, model, config, tp in HEADLINE:
            if config == "relay-tp" and N < 2 or config == "colocated" and N % tp:
                continue
            need = hbm_need(topology(config, N, tp), N, P_params(model))
            if need > 175e9:
                if rank == 0:
                    headline[name] = dict(skipped=f"needs {need / 1e9:.0f} GB on one GPU at N={N}")
                continue
            # an extra configuration must not cost the main line: a failure is recorded in its entry (every
            # rank takes the same path, so the collectives stay matched)
            try:
                Q = Placement(args, D, model, config, tp, name)
                r = timed_steps(Q, args.extra_steps, 2, True)
                s = summarize(Q, r, args.extra_steps)
                par = None if args.no_verify else verify(Q)
                if rank == 0:
                    headline[name] = dict(workload=f"{model} [{config}]: " + Q.T["desc"], value=s["sec"], unit=UNIT,
                                          steps=args.extra_steps, warmup=2, nvlink_bound=s["nvlink_bound"],
                                          target_1_5x_bound_s=1.5 * s["nvlink_bound"]["seconds"],
                                          kernels_ms=s["kernels_ms"], roofline=s["roofline"],
                                          gpu_launches=s["gpu_launches"], parity=par)
                Q.close()
                del Q
            except Exception as e:   # noqa: BLE001
                if rank == 0:
                    headline[name] = dict(error=f"{type(e).__name__}: {e}"[:300])
                import torch
                torch.cuda.synchronize()
                torch.cuda.empty_cache()
        D.gloo = main_group

    if rank == 0:
        M = summ
        T = topology(args.config, N, args.tp)
        out = dict(
            metric=METRIC, value=M["sec"], unit=UNIT, n_gpus=N, steps=args.steps, warmup=args.warmup,
            ms_per_step=M["ms_per_step"], higher_is_better=False, scaling="weak", vs_baseline=None, dtype="bf16",
            data="synthetic",
            config=line_config(args, N),
            roofline=M["roofline"], nvlink_bound=M["nvlink_bound"], kernels_ms=M["kernels_ms"],
            per_rank=M["per_rank"], host_latency_ms=M["host_latency_ms"], pull_latency=plat,
            paper_context="actor stall 0.64 s (32B) / 1.40 s (72B); 72B to 127 relays < 1.6 s on 128x8 H800 + RDMA",
            cpu_baseline=cpu, e2e=e2e, gpu_launches=M["gpu_launches"], actor_stall=stall, parity=parity,
            stats=M["stats"], clocks=M["clocks"])
        out["config"].update(params=int(P_params(args.model)), snapshot_bytes=int(2 * P_params(args.model)))
        if headline is not None:
            out["headline"] = headline
        print(json.dumps(out), flush=True)
    D.close()
    return 0


def hbm_need(T, N, P):
    """Largest per-GPU footprint of a placement: fp32 master shards + 2 ring slots of every part a GPU
    stores + its rollouts' TP buffers (tests/test_abi_host.py checks the same count)."""
    n = T["fsdp"]
    per = {d: 0.0 for d in range(N)}
    for d in T["actors"]:
        per[d] += 4 * P / n + 2 * (2 * P / n)
    for node in T["relays"]:
        for d in node:
            per[d] += 2 * (2 * P / n)
    for _, dev, tpr, _ in T["rollouts"]:
        per[dev] += 2 * P / tpr
    return max(per.values())


def P_params(model):
    from oracle.model import MODELS, param_count
    return param_count(MODELS[model])


def cpu_baseline(args, P: Placement):
    """The oracle on this box's host cores (rank 0, N = 1): the full publish -> TP=1 pull step on a
    process pool over all cores (measured), plus the single-thread oracle on a bounded sample (scaled).
    The fp32 inputs are the resident masters of the timed run, copied from the GPU (harness)."""
    import numpy as np

    from oracle.model import MODELS, tensors
    hi = host_info()
    res = dict(kind="oracle", host=hi)
    try:
        import psutil
        need = 4.2 * P_params(args.model) + 8 * P_params(args.model)     # inputs + image + output (+ slack)
        if psutil.virtual_memory().available < need + (16 << 30):
            raise MemoryError(f"needs {need / 1e9:.0f} GB of host RAM")
        tl = tensors(MODELS[args.model])

        def from_gpu(o):
            sh = P.shards[0]
            buf = sh.buf
            for (t, e0, cnt), off in zip(sh.pieces, sh.offs):
                o.inputs[o.base[t] + e0:o.base[t] + e0 + cnt] = (
                    buf[off:off + cnt].cpu().numpy().view(np.uint32))
        assert len(tl) == len(P.shards[0].tensors)
        o = OracleStep(args.model, relays=0, inputs_from=from_gpu, chunk_bytes=P.info.chunk_bytes)
        t = o.step()
        o.close()
        res.update(value=t["total"], unit=UNIT, cores=o.workers, measured="full step",
                   sample=f"full {args.model} publish (cast+pack+checksum, {o.plan.total_chunks} chunks) + TP=1 "
                          f"pull of {o.P / 1e9:.2f} G params, numpy oracle on a {o.workers}-process pool",
                   phases_s={k: round(v, 3) for k, v in t.items()})
    except Exception as e:  # noqa: BLE001 - reported, the single-thread sample below still stands
        res.update(full_step_error=str(e)[:200])
    st, info = oracle_sample(args.model, args.cpu_seconds)
    res["single_thread"] = dict(value=st, cores=1, measured="scaled sample", sample=info["sample"])
    if "value" not in res:
        res.update(value=st, unit=UNIT, cores=1, measured="scaled sample", sample=info["sample"])
    return res


def actor_stall(P: Placement, reps=5, target_ms=25.0, sms_list=(0, 24, 40, 56, 74)):
    """Actor stall per publish, the trainer's view of step 5 ("pushes the new
    actor weights to the master relay and immediately resumes its next training iteration"):
      reads_done_wait_ms  actor-stream wait on reads_done before the next optimizer step, when that step
                          comes one synthetic training step after the publish;
      inflation_ms        that training step's slowdown from the concurrent pack (SM / HBM contention,
                          PAPER L401-402): synthetic step = a bf16 GEMM loop of ~target_ms on the actor
                          stream (torch/cuBLAS: it stands in for the trainer, it is not the path).
    Pack-only publishes (no subscriber), each committed before the next; medians over `reps`.
    pack_sms_sweep: the same with the pack confined to k SMs (lam_set_pack_sms), trading pack time for
    trainer SMs; the line's own numbers use --pack-sms."""
    torch, ctx, lam = P.torch, P.ctx, P.lam
    actor_stream = P.actor_stream
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

    alone = []
    for _ in range(reps):
        with torch.cuda.stream(actor_stream):
            s0, s1 = ev(), ev()
            s0.record()
        train_step()
        with torch.cuda.stream(actor_stream):
            s1.record()
        s1.synchronize()
        alone.append(s0.elapsed_time(s1))
    med = lambda x: sorted(x)[len(x) // 2]
    sweep = []
    for sms in sms_list:                               # pack confined to `sms` SMs (0 = all)
        ctx.set_pack_sms(sms)
        r = _stall_reps(P, reps, train_step, ev)
        sweep.append(dict(pack_sms=sms, inflation_ms=round(r[0] - med(alone), 3), masters_busy_ms=round(r[2], 3),
                          reads_done_wait_ms=round(r[1], 4)))
    ctx.set_pack_sms(P.args.pack_sms)
    tot, wt, bz = _stall_reps(P, reps, train_step, ev)
    del a, b, c
    return dict(step_ms_alone=round(med(alone), 3), step_ms_with_publish=round(tot, 3),
                inflation_ms=round(tot - med(alone), 3),
                inflation_frac=round(tot / med(alone) - 1, 4),
                reads_done_wait_ms=round(wt, 4), masters_busy_ms=round(bz, 3), pack_sms=P.args.pack_sms,
                pack_sms_sweep=sweep,
                actor_step=f"bf16 GEMM {n}^3 x {iters} on the actor stream (~{target_ms:.0f} ms)", reps=reps)


def _stall_reps(P, reps, train_step, ev):
    """Medians over `reps` of (step time with a concurrent publish, reads_done wait, pack duration)."""
    torch, ctx, lam = P.torch, P.ctx, P.lam
    actor_stream = P.actor_stream
    total, wait, busy = [], [], []
    for _ in range(reps):
        P.v += 1
        v = P.v
        rd = {r: live_event(torch, timing=True) for r in P.shards}
        with torch.cuda.stream(actor_stream):
            t0, t_mid, t1 = ev(), ev(), ev()
            t0.record()
        for r, sh in P.shards.items():
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
    return med(total), med(wait), med(busy)


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


def run_e2e(args, P: Placement):
    import psutil
    torch, D = P.torch, P.D
    need = sum(sh.buf.numel() * 4 for sh in P.shards.values()) + sum(b.bytes for b in P.bufs.values())
    need_all = D.sum(need)          # every rank pins its share of the same host RAM
    ok = psutil.virtual_memory().available > 1.5 * need_all + (16 << 30)
    if D.max(0.0 if ok else 1.0) != 0.0:
        return dict(value=None, unit=UNIT, reason="not enough host RAM for pinned buffers")
    h2d = {r: sh.buf.to("cpu").pin_memory() for r, sh in P.shards.items()}
    d2h = {rid: {n: torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for n, t in P.bufs[rid].bufs.items()}
           for rid in P.mine}
    P.step(h2d, d2h)  # warm-up with host buffers
    torch.cuda.synchronize()
    D.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream()
    s.record(st)
    for _ in range(args.e2e_steps):
        P.step(h2d, d2h)
    torch.cuda.synchronize()
    e.record(st)
    e.synchronize()
    ms = D.max(s.elapsed_time(e))
    hb = D.sum(sum(sh.buf.numel() * 4 for sh in P.shards.values()))
    db = D.sum(sum(b.bytes for b in P.bufs.values()))
    del h2d, d2h
    return dict(value=ms / 1e3 / args.e2e_steps, unit=UNIT, h2d_bytes_per_step=int(hb), d2h_bytes_per_step=int(db),
                steps=args.e2e_steps,
                note="pinned host fp32 masters -> H2D -> lam_publish -> relay -> lam_pull -> D2H of every rollout")


# ------------------------------------------------------------------------------ config 5: stress
def run_stress(args, D: Dist):
    """BASELINE configs[4]: the actor publishes every step while 6 rollouts pull staggered versions.

    Actor loop (GPU 0), per step v: synthetic forward/backward (bf16 GEMM loop of ~stress_ms, which
    overlaps the pack of v-1) -> the optimizer waits for reads_done of the previous publish, then writes
    the masters of version v (generator, harness) -> lam_publish(v).  Every rank drives lam_relay_step; rollout k pulls (lam_pull of the
    newest complete version at its node) at exponential intervals of mean 2 x stress_ms (seed k).
    Reported: publish -> every-node-committed latency per version (the line's value, p50), actor stall
    per publish (host time in lam_publish + actor-stream wait on reads_done), pull latency p50/p99,
    staleness (newest committed at the node when the pull returned - pulled), versions skipped, and the
    C8 invariants: every pulled version was published, is monotone per rollout, is >= the
    node's latest at call time, and 64 sampled elements per destination buffer ==
    oracle.tp.dst_elements at that version (no torn or mixed version)."""
    import numpy as np
    import torch

    from oracle.invariants import PullRecord, check
    from oracle.model import MODELS as OMODELS
    from oracle.tp import dst_elements
    from synth import SEED
    P = Placement(args, D, args.model, "stress", 1, "stress")
    ctx, lam = P.ctx, P.lam
    rank, N = P.rank, P.N
    od = OMODELS[args.model]
    steps = args.stress_steps
    n_nodes = len(P.T["relays"]) + 1
    gemm = None
    if P.my_ranks:                      # synthetic training step on the actor GPU (stands in for the trainer)
        n = 8192
        a = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
        c = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
        with torch.cuda.stream(P.actor_stream):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.mm(a, b, out=c)
            e0.record()
            for _ in range(5):
                torch.mm(a, b, out=c)
            e1.record()
        e1.synchronize()
        gemm = (a, b, c, max(1, int(args.stress_ms / (e0.elapsed_time(e1) / 5))))
    rng = {rid: np.random.default_rng(rid) for rid in P.mine}
    D.barrier()
    t_start = time.time()
    mean_s = 2 * args.stress_ms / 1e3
    next_pull = {rid: t_start + rng[rid].exponential(mean_s) for rid in P.mine}
    records, lat, samples, stale = [], [], [], []
    pub_host, rd_wait, pub_t, commit_t, pub_busy = [], [], {}, {}, []
    seen = [0] * n_nodes
    rd_prev = g_prev = None
    inflight = {}                # rid -> (version, event, t_call, latest_at_call)
    actor_v = 0
    while True:
        if P.my_ranks and actor_v < steps and (g_prev is None or g_prev.query()):
            # the trainer's pace: step v is enqueued once step v-1's compute is done; its optimizer
            # write of the masters waits (on the stream) for the previous pack's reads_done
            actor_v += 1
            v = actor_v
            A, B, Cc, iters = gemm
            with torch.cuda.stream(P.actor_stream):    # forward/backward of step v (overlaps pack v-1)
                for _ in range(iters):
                    torch.mm(A, B, out=Cc)
                g_prev = torch.cuda.Event()
                g_prev.record()
            if rd_prev is not None:                    # the optimizer may overwrite the masters only
                with torch.cuda.stream(P.actor_stream):    # once the previous pack has read them
                    w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    w0.record()
                    P.actor_stream.wait_event(rd_prev)
                    w1.record()
                    rd_wait.append((w0, w1))
            for sh in P.shards.values():              # optimizer: new master values (version v)
                sh.fill(SEED, v, stream=P.actor_stream.cuda_stream)
            rd = live_event(torch)
            t0 = time.perf_counter()
            busy = 0
            for r, sh in P.shards.items():
                while ctx.publish(v, r, sh.shards(), P.actor_stream.cuda_stream, rd.cuda_event) == lam.LAM_EBUSY:
                    busy += 1
                    ctx.relay_step()
            pub_host.append(time.perf_counter() - t0)
            pub_busy.append(busy)
            pub_t[v] = time.time()
            rd_prev = rd
        ctx.relay_step()
        if rank == 0:                   # publish -> committed at every node, per version
            for k in range(n_nodes):
                lv = ctx.latest(k)
                if lv > seen[k]:
                    seen[k] = lv
            low = min(seen)
            for v in range(max(commit_t.keys(), default=0) + 1, low + 1):
                commit_t[v] = time.time()
        for rid in P.mine:
            node = P.rollouts[rid][0]
            if rid in inflight:
                v, ev, tc, lat0 = inflight[rid]
                if ev.query():
                    lat.append((time.time() - tc) * 1e3)
                    stale.append(ctx.latest(node) - v)
                    chk = {}
                    g = np.random.default_rng(v * 7 + rid)
                    for name, buf in P.bufs[rid].bufs.items():
                        idx = g.integers(0, buf.numel(), 64)
                        got = buf.view(-1).view(torch.int16)[torch.from_numpy(idx).to(buf.device)].cpu().numpy()
                        chk[name] = (idx, got.view(np.uint16))
                    samples.append((rid, v, lat0, chk))
                    del inflight[rid]
            elif time.time() >= next_pull[rid]:
                lat0 = ctx.latest(node)
                tc = time.time()
                v = ctx.pull(rid, P.bufs[rid].tp, P.rstream[rid].cuda_stream)
                if v:
                    ev = torch.cuda.Event()
                    ev.record(P.rstream[rid])
                    inflight[rid] = (v, ev, tc, lat0)
                next_pull[rid] = time.time() + rng[rid].exponential(mean_s)
        if (actor_v >= steps or not P.my_ranks) and not inflight and ctx.latest(0) >= steps and \
                all(ctx.latest(k) >= steps for k in range(n_nodes)):
            break
        if time.time() - t_start > 900:
            raise TimeoutError("stress run did not finish")
    torch.cuda.synchronize()
    wall = time.time() - t_start
    for rid, v, lat0, chk in samples:       # C8 (iv) on sampled elements, against the oracle
        node, dev, tp, tr = P.rollouts[rid]
        ok = all(np.array_equal(got, dst_elements(od, tp, tr, name, idx, SEED, v)) for name, (idx, got) in chk.items())
        records.append(PullRecord(rollout=rid, version=v, latest_at_start=lat0, content_ok=ok))
    viol = check(set(range(1, steps + 1)), records)
    stats = ctx.stats()
    mine = dict(lat=lat, stale=stale, n=len(records), torn=sum(not r.content_ok for r in records), viol=viol[:8],
                nviol=len(viol), pub_host=pub_host, rd_wait=[w0.elapsed_time(w1) for w0, w1 in rd_wait],
                pub_t=pub_t, pub_busy=pub_busy)
    allr = D.gather(mine)
    out = None
    if rank == 0:
        pct = lambda xs, q: (round(xs[min(len(xs) - 1, int(q * len(xs)))], 3) if xs else None)
        pt = {v: t for a in allr for v, t in a["pub_t"].items()}
        commit = sorted((commit_t[v] - pt[v]) * 1e3 for v in commit_t if v in pt)
        lat_all = sorted(x for a in allr for x in a["lat"])
        st_all = sorted(x for a in allr for x in a["stale"])
        ph = [x * 1e3 for a in allr for x in a["pub_host"]]
        rw = [x for a in allr for x in a["rd_wait"]]
        stall = sorted(h + w for h, w in zip(ph[1:], rw))
        # the first publish of a shard list builds the pack plan (one-time set-up, reported apart)
        phs, rws = sorted(ph[1:]), sorted(rw)
        busy = [b for a in allr for b in a["pub_busy"][1:]]
        out = dict(metric=METRIC, value=(pct(commit, 0.5) / 1e3 if commit else None), unit=UNIT, n_gpus=N,
                   steps=steps, warmup=0, ms_per_step=pct(commit, 0.5), higher_is_better=False, scaling="weak",
                   vs_baseline=None, dtype="bf16", data="synthetic",
                   config=dict(workload=f"{args.model} [stress]: " + P.T["desc"],
                               model=f"Qwen2.5-{args.model.upper()}-shaped", actor_step_ms=args.stress_ms,
                               pull_mean_interval_ms=2 * args.stress_ms,
                               value="p50 over versions of publish -> committed at every node (host clock)"),
                   stress=dict(
                       wall_s=round(wall, 2), publishes=steps, versions_committed_everywhere=len(commit),
                       publish_to_all_nodes_ms=dict(p50=pct(commit, 0.5), p99=pct(commit, 0.99)),
                       actor_stall_ms=dict(p50=pct(stall, 0.5), p99=pct(stall, 0.99), max=stall[-1] if stall else None,
                                           what="host time in lam_publish + actor-stream wait on reads_done "
                                                "before the next optimizer write"),
                       publish_host_ms=dict(p50=pct(phs, 0.5), p99=pct(phs, 0.99), first=round(ph[0], 3) if ph else None,
                                            what="host time in lam_publish (+ LAM_EBUSY retries) after the first "
                                                 "publish; first = one-time pack-plan build"),
                       publish_busy=dict(publishes_that_waited=sum(1 for b in busy if b), of=len(busy),
                                         what="LAM_EBUSY: every node-0 slot was packing, latest, or being read "
                                              "by relay 1 — the publish waited for one (back-pressure)"),
                       reads_done_wait_ms=dict(p50=pct(rws, 0.5), p99=pct(rws, 0.99)),
                       pull_latency_ms=dict(p50=pct(lat_all, 0.5), p99=pct(lat_all, 0.99), n=len(lat_all)),
                       staleness_versions=dict(p50=pct(st_all, 0.5), p99=pct(st_all, 0.99),
                                               what="node's latest when the pull completed - pulled version"),
                       versions_skipped=stats["versions_skipped"],
                       c8=dict(pulls=sum(a["n"] for a in allr), violations=sum(a["nviol"] for a in allr),
                               torn=sum(a["torn"] for a in allr), sampled_elements_per_buffer=64,
                               examples=[x for a in allr for x in a["viol"]][:4])))
    P.close()
    return out


if __name__ == "__main__":
    sys.exit(main())

"""CPU tests of the C ABI library: it loads, exports every symbol include/lam.h declares, and its host
planner (model table, vLLM layout, image plan, pull copy plan, Appendix D) agrees with the oracle.
No compute call is made here: the copy plan is *executed* by a numpy loop in this test only to check
the planner's arithmetic; the product executes it in k_pull on the GPU."""
import os
import re

import numpy as np
import pytest
import torch

from oracle import relay as orelay
from oracle.image import FSDP1_FLAT, FSDP2_DIM0, image_plan, publish
from oracle.model import MODELS as OMODELS
from oracle.model import tensors as otensors
from oracle.tp import direct_pull, vllm_dsts
from paper_2510_12633_b200 import lam
from paper_2510_12633_b200.workload import MODELS
from synth import SEED

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LAYOUT = {FSDP2_DIM0: lam.LAM_FSDP2_DIM0, FSDP1_FLAT: lam.LAM_FSDP1_FLAT}


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "lam.h")).read()
    declared = set(re.findall(r"\b(lam_[a-z_]+)\s*\(", hdr))
    L = lam.load()
    missing = [s for s in sorted(declared) if not hasattr(L, s)]
    assert not missing, missing
    assert declared >= set(lam.EXPORTED)


def test_no_gpu_fails_loudly():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(lam.LamError) as e:
        lam.Context(lam.Config(model=MODELS["tiny"], rollouts=[(0, 0)]))
    assert e.value.status == lam.LAM_ECUDA


@pytest.mark.parametrize("name", ["tiny", "7b", "32b", "72b", "odd"])
def test_model_table_matches_oracle(name):
    assert lam.model_tensors(MODELS[name]) == otensors(OMODELS[name])


@pytest.mark.parametrize("name,tp", [("tiny", 1), ("tiny", 4), ("tiny", 8), ("7b", 2), ("72b", 8), ("odd", 1),
                                     ("odd", 4), ("odd", 8)])
def test_vllm_layout_matches_oracle(name, tp):
    ours = lam.vllm_layout(MODELS[name], tp)
    ref = vllm_dsts(OMODELS[name], tp)
    names = [n for n, _ in otensors(OMODELS[name])]
    assert [d.name for d in ours] == [d.name for d in ref]
    for a, b in zip(ours, ref):
        assert (a.rows,) + ((a.cols,) if len(b.shape) == 2 else ()) == b.shape
        assert [(names[t], r) for t, r in a.parts] == [(p.tensor, p.rule) for p in b.parts]


def test_appendix_d_matches_oracle():
    import random
    rng = random.Random(1)
    for _ in range(200):
        p, k = rng.randint(2, 300), rng.randint(1, 2000)
        M, tb, ts = rng.uniform(1e6, 2e11), 1 / rng.uniform(1e9, 1e12), rng.uniform(1e-7, 1e-3)
        assert lam.chain_latency(p, k, M, tb, ts) == pytest.approx(orelay.chain_latency(p, k, M, tb, ts), rel=1e-12)
        assert lam.optimal_chunks(p, M, tb, ts, 1024) == orelay.optimal_chunks(p, M, tb, ts, 1024)


@pytest.mark.parametrize("name,layout,N,C", [("tiny", FSDP2_DIM0, 1, 1 << 20), ("tiny", FSDP1_FLAT, 3, 1 << 18),
                                             ("7b", FSDP2_DIM0, 1, 96 << 20), ("32b", FSDP2_DIM0, 4, 64 << 20),
                                             ("72b", FSDP2_DIM0, 8, 128 << 20), ("7b", FSDP1_FLAT, 8, 1 << 22)])
def test_image_plan_matches_oracle(name, layout, N, C):
    ours = lam.plan_segments(MODELS[name], LAYOUT[layout], N, C)
    plan = image_plan([s for _, s in otensors(OMODELS[name])], N, C, layout)
    ref = [(s.tensor_id, s.rank, s.elem0, s.count, plan.image_offset(s)) for s in plan.segments]
    assert ours == ref


def _execute_plan(tiles, img_rank_base, img, out_base, out):
    """numpy executor of the library's copy plan (test-only: checks the plan's arithmetic)."""
    for t in tiles:
        for r in range(t.rows):
            if t.src_rank == lam.LAM_TILE_ZERO:
                d = t.dst - out_base + r * t.dst_pitch
                out[d:d + t.row_bytes] = 0
                continue
            s = img_rank_base[t.src_rank] + t.src_off + r * t.src_pitch
            if t.align & lam.LAM_TILE_TRANSPOSE:   # element k of row r -> dst + k*dst_pitch + 2r
                d = t.dst - out_base + 2 * r
                for k in range(t.row_bytes // 2):
                    out[d + k * t.dst_pitch:d + k * t.dst_pitch + 2] = img[s + 2 * k:s + 2 * k + 2]
                continue
            d = t.dst - out_base + r * t.dst_pitch
            out[d:d + t.row_bytes] = img[s:s + t.row_bytes]


@pytest.mark.parametrize("model,layout,N,C,tp,tr", [
    ("tiny", FSDP2_DIM0, 1, 1 << 20, 1, False), ("tiny", FSDP2_DIM0, 4, 1 << 18, 2, False),
    ("tiny", FSDP1_FLAT, 3, 1 << 18, 4, False), ("tiny", FSDP2_DIM0, 8, 4096 * 5, 4, False),
    ("tiny", FSDP1_FLAT, 8, 4096, 8, False), ("tiny", FSDP2_DIM0, 3, 4096 * 3, 2, False),
    ("odd", FSDP2_DIM0, 1, 4096, 8, False), ("odd", FSDP1_FLAT, 3, 4096, 4, False),
    ("tiny", FSDP2_DIM0, 1, 1 << 18, 1, True), ("tiny", FSDP1_FLAT, 3, 4096 * 3, 2, True),
    ("odd", FSDP1_FLAT, 3, 4096, 8, True), ("odd", FSDP2_DIM0, 4, 4096 * 2, 4, True)])
def test_copy_plan_reproduces_oracle_pull(model, layout, N, C, tp, tr):
    """The library's pull plan, executed by numpy, reproduces the oracle's pull: fused qkv/gate_up,
    dim-1 slices, KV-head replication, vocabulary padding (zero tiles), K-major destinations."""
    d = OMODELS[model]
    plan = image_plan([s for _, s in otensors(d)], N, C, layout)
    img, _ = publish(plan, SEED, 4, specials=True)
    rank_base = [plan.chunk_base[r] * C for r in range(N)]
    layout_c = lam.vllm_layout(MODELS[model], tp)
    for rank in range(tp):
        want = direct_pull(d, tp, rank, SEED, 4, specials=True, transpose=tr)
        base, offs, o = 1 << 40, {}, 0
        for x in layout_c:
            offs[x.name] = o
            o += -(-x.rows * x.cols * 2 // 256) * 256
        tpl = lam.TPLayout(tp, rank, [(x.parts, base + offs[x.name], 0) for x in layout_c], transpose=tr)
        tiles = lam.plan_copy_tiles(MODELS[model], LAYOUT[layout], N, C, tpl)
        # streaming pulls launch tiles chunk by chunk: every tile must lie inside one source chunk,
        # and tiles must come in launch order — chunk j of every rank before chunk j + 1, ranks
        # rotated by tp_rank * N / tp (zero tiles first: they read nothing)
        rot = rank * N // tp
        order = lambda g: (g - plan.chunk_base[plan.chunk_rank(g)], (plan.chunk_rank(g) - rot) % N)
        chunks = []
        for t in tiles:
            if t.src_rank == lam.LAM_TILE_ZERO:
                assert not chunks
                continue
            lo = t.src_off
            hi = t.src_off + (t.rows - 1) * t.src_pitch + t.row_bytes
            assert lo // C == (hi - 1) // C, (t.src_rank, lo, hi, C)
            chunks.append(plan.chunk_base[t.src_rank] + lo // C)
        assert chunks == sorted(chunks, key=order)
        out = np.full(o, 0xAB, dtype=np.uint8)
        _execute_plan(tiles, rank_base, img, base, out)
        for x in layout_c:
            got = out[offs[x.name]:offs[x.name] + x.rows * x.cols * 2].view(np.uint16)
            assert np.array_equal(got, want[x.name].ravel()), (x.name, rank)


def test_config_struct_size_matches_library():
    """The binding's lam_config layout is the library's (a stale .so fails loudly in lam.load)."""
    import ctypes
    L = lam.load()
    assert L.lam_config_size() == ctypes.sizeof(lam.lam_config)
    assert ctypes.sizeof(lam.lam_node_desc) == 4 * (lam.LAM_MAX_RANKS + 1)   # part_device[] + host_memory


@pytest.mark.parametrize("config,tp", [("chain", 0), ("colocated", 0), ("colocated", 2), ("relay-tp", 2),
                                       ("relay-tp", 1), ("host", 1), ("host", 2), ("stress", 0)])
@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_bench_placements_are_valid(config, tp, N):
    """bench.py placements at every N the driver's scaling run uses: devices in range, every rollout
    rank r of a TP group present exactly once, relays hold every actor rank, and the 7B chain fits HBM."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    if (config == "relay-tp" and (N < 2 or tp > N // 2) or config == "colocated" and tp and N % tp
            or config == "host" and tp > max(1, N - 1)):
        return                                   # not a placement the bench offers at this N
    T = bench.topology(config, N, tp)
    assert len(T["actors"]) == T["fsdp"] and all(0 <= d < N for d in T["actors"])
    for node in T["relays"]:
        assert len(node) == T["fsdp"] and all(0 <= d < N for d in node)
    assert set(T.get("host_relays", [])) <= set(range(1, len(T["relays"]) + 1))
    assert T["rollouts"], "every placement has at least one rollout"
    for node, dev, tpr, rank in T["rollouts"]:
        assert 0 <= node <= len(T["relays"]) and 0 <= dev < N and 0 <= rank < tpr
    ranks = sorted(r for _, _, _, r in T["rollouts"])
    tpr = T["rollouts"][0][2]
    assert ranks == sorted(list(range(tpr)) * (len(ranks) // tpr))
    if config == "stress":
        assert len(T["rollouts"]) == 6                       # BASELINE configs[4]: 6 rollouts
    if config in ("chain", "stress"):
        P = sum(int(np.prod(s)) for _, s in otensors(OMODELS["7b"]))
        per_gpu = {d: 0 for d in range(N)}
        per_gpu[0] += 4 * P + 2 * 2 * P                      # fp32 masters + 2 master slots
        for node in T["relays"]:
            per_gpu[node[0]] += 2 * 2 * P                    # 2 relay slots (full image)
        for _, dev, tpr, _ in T["rollouts"]:
            per_gpu[dev] += 2 * P // tpr                     # rollout buffers
        assert max(per_gpu.values()) < 180e9


@pytest.mark.parametrize("config,model,tp", [("colocated", "32b", 2),     # the 32B x 8 reading
                                              ("colocated", "72b", 8), ("colocated", "72b", 4),   # config 4
                                              ("relay-tp", "32b", 2)])   # config 3
def test_full_size_8gpu_placements_fit_hbm(config, model, tp):
    """The full-size 8-GPU configurations (only their 4-GPU scalings could be measured) fit 180 GB per
    GPU: fp32 master shards + 2 ring slots of every part a GPU stores + its rollout's TP buffers."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    N = 8
    T = bench.topology(config, N, tp)
    P = sum(int(np.prod(s)) for _, s in otensors(OMODELS[model]))
    n = T["fsdp"]
    per_gpu = {d: 0.0 for d in range(N)}
    for d in T["actors"]:
        per_gpu[d] += 4 * P / n + 2 * (2 * P / n)            # fp32 shard + 2 master slots of its bf16 region
    for node in T["relays"]:
        for d in node:
            per_gpu[d] += 2 * (2 * P / n)                    # 2 relay slots of one rank region
    for _, dev, tpr, _ in T["rollouts"]:
        per_gpu[dev] += 2 * P / tpr
    assert max(per_gpu.values()) < 180e9, per_gpu


@pytest.mark.parametrize("name,layout,N,C,R", [("tiny", FSDP2_DIM0, 1, 1 << 16, 3), ("tiny", FSDP1_FLAT, 2, 1 << 15, 4),
                                               ("odd", FSDP2_DIM0, 3, 1 << 16, 2)])
def test_tree_tile_order(name, layout, N, C, R):
    """LAM_HOP_TREE: every relay walks the same tiles, a chunk's tiles stay together, each
    group of R chunk runs (in the hop order, which interleaves the FSDP ranks' regions; relay 1 walks it
    unrotated) starts at the run the relay owns (the j-th run of a group belongs to relay j + 1), and a
    tile is read from its owner relay when that relay is pinned in the mask, else from node 0."""
    d, lay = MODELS[name], LAYOUT[layout]

    def runs_of(tiles):
        ch = [t[1] for t in tiles]
        return [c for i, c in enumerate(ch) if i == 0 or ch[i - 1] != c]

    base = lam.plan_tree_tiles(d, lay, N, C, R, 1, 0)
    base_runs = runs_of(base)
    assert len(base_runs) == len(set(base_runs)) > R    # contiguous per chunk, several groups
    assert sorted(base_runs) == list(range(len(base_runs)))
    owner = {c: i % R + 1 for i, c in enumerate(base_runs)}
    ref = sorted(t[:4] for t in base)
    assert len(set(ref)) == len(ref)
    # the tiles cover every chunk of the oracle's image exactly: rank r's chunk j is the
    # bytes [j C, j C + len) of r's region, cut into consecutive tiles
    op = image_plan([s for _, s in otensors(OMODELS[name])], N, C, layout)
    cover = {}
    for off, g, rank, nb, _ in base:
        cover.setdefault(g, []).append((off, nb, rank))
    assert sorted(cover) == list(range(op.total_chunks))
    for g, ts in cover.items():
        r = op.chunk_rank(g)
        pos = (g - op.chunk_base[r]) * C
        for off, nb, rank in sorted(ts):
            assert (off, rank) == (pos, r) and 0 < nb
            pos += nb
        assert pos == (g - op.chunk_base[r]) * C + op.chunk_len(g)
    for mask in (0, sum(1 << n for n in range(1, R + 1)), 1 << R):
        for node in range(1, R + 1):
            tiles = lam.plan_tree_tiles(d, lay, N, C, R, node, mask)
            assert sorted(t[:4] for t in tiles) == ref
            runs = runs_of(tiles)
            assert len(runs) == len(base_runs)
            for g in range(0, len(runs), R):
                grp, mine = base_runs[g:g + R], runs[g:g + R]
                assert mine == grp[(node - 1) % len(grp):] + grp[:(node - 1) % len(grp)]
            for _, c, rank, _, src in tiles:
                assert rank < N
                assert src == (owner[c] if owner[c] != node and mask >> owner[c] & 1 else 0)
    with pytest.raises(lam.LamError):
        lam.plan_tree_tiles(d, lay, N, C, R, R + 1, 0)

"""Pins of oracle/tp.py (TP=1 == torch cast, brute-force inverse, two pull paths agree) and
oracle/relay.py (Appendix D closed forms, SPEC worked numbers, discrete schedule = T(p,k),
relay invariants under seeded random interleavings)."""
import random

import numpy as np
import pytest
import torch

from oracle import invariants
from oracle.image import FSDP1_FLAT, FSDP2_DIM0, image_plan, publish
from oracle.model import MODELS, numel, tensors
from oracle.relay import (COMPLETE, RelayChain, chain_latency, k_star, latency_decomposition,
                          optimal_chunks)
from oracle.tp import (HEAD_DIM0, REPLICATE, SHARD_DIM0, SHARD_DIM1, VOCAB_DIM0, direct_pull,
                       dst_elements, part_slice, pull_from_image, vllm_dsts)
from synth import SEED, gen_f32

D = MODELS["tiny"]


def _torch_cast(name, v, d=D):
    tl = tensors(d)
    t = [n for n, _ in tl].index(name)
    w = torch.from_numpy(gen_f32(SEED, v, t, 0, numel(tl[t][1])).reshape(tl[t][1]))
    return w.to(torch.bfloat16)


def test_tp1_pull_is_torch_cast():
    got = direct_pull(D, 1, 0, SEED, 3)
    for dst in vllm_dsts(D, 1):
        ref = torch.cat([_torch_cast(p.tensor, 3) for p in dst.parts], 0)
        assert np.array_equal(got[dst.name], ref.view(torch.int16).numpy().view(np.uint16)), dst.name


def _rank_rows(rule, shape, heads, tp):
    """Rows of a part in one rank's destination, by the vLLM arithmetic written out: whole heads per
    rank (one replicated head when tp > heads), vocab padded to 64, dim-1 splits keep all rows."""
    if rule in (REPLICATE, SHARD_DIM1):
        return shape[0]
    if rule == SHARD_DIM0:
        return shape[0] // tp
    if rule == HEAD_DIM0:
        return shape[0] // heads * max(1, heads // tp)
    return (shape[0] + 63) // 64 * 64 // tp


@pytest.mark.parametrize("model,tp", [("tiny", 2), ("tiny", 4), ("tiny", 8), ("odd", 2), ("odd", 4),
                                      ("odd", 8)])
def test_brute_force_inverse(model, tp):
    """Undo the TP rule with torch (cat over ranks) and recover every full tensor's torch cast:
    replicated KV heads are identical across their rank group and one per group reassembles the
    tensor; vocabulary padding rows are zero and the real rows reassemble the tensor."""
    d = MODELS[model]
    ranks = [direct_pull(d, tp, r, SEED, 1) for r in range(tp)]
    shp = dict(tensors(d))
    for dst in vllm_dsts(d, tp):
        row = 0
        for p in dst.parts:
            n_rows = _rank_rows(p.rule, shp[p.tensor], p.heads, tp)
            per_rank = [torch.from_numpy(x[dst.name].view(np.int16))[row:row + n_rows] for x in ranks]
            want = _torch_cast(p.tensor, 1, d).view(torch.int16)
            if p.rule == SHARD_DIM1:
                full = torch.cat(per_rank, 1)
            elif p.rule == REPLICATE:
                assert all(torch.equal(per_rank[0], y) for y in per_rank)
                full = per_rank[0]
            elif p.rule == HEAD_DIM0 and tp > p.heads:
                g = tp // p.heads                        # ranks sharing one head
                for h in range(p.heads):
                    assert all(torch.equal(per_rank[h * g], per_rank[h * g + j]) for j in range(g))
                full = torch.cat(per_rank[::g], 0)
            else:
                full = torch.cat(per_rank, 0)
            if p.rule == VOCAB_DIM0:
                assert not full[shp[p.tensor][0]:].any()   # padding rows are zero
                full = full[:shp[p.tensor][0]]
            assert torch.equal(full, want), (dst.name, p.tensor)
            row += n_rows
        assert row == dst.shape[0]


@pytest.mark.parametrize("V,tp", [(130, 1), (130, 2), (130, 4), (130, 8), (12288, 8), (152064, 8),
                                  (151936, 4), (1000, 8), (65, 2), (64, 8)])
def test_vocab_padding_matches_vllm(V, tp):
    """VOCAB_DIM0 reproduces vLLM's VocabParallelEmbedding shard ranges (pad_vocab_size +
    vocab_range_from_global_vocab_size; rows past the vocabulary are zero-filled by its loader)."""
    vp = pytest.importorskip("vllm.model_executor.layers.vocab_parallel_embedding")
    padded = vp.pad_vocab_size(V, vp.DEFAULT_VOCAB_PADDING_SIZE)
    for r in range(tp):
        s, e = vp.vocab_range_from_global_vocab_size(padded, r, tp)
        r0, r1, _, _, pad = part_slice((V, 8), VOCAB_DIM0, tp, r)
        assert (r0, r1, r1 - r0 + pad) == (min(s, V), min(e, V), e - s)


@pytest.mark.parametrize("model,tp", [("tiny", 1), ("tiny", 4), ("odd", 8)])
def test_transposed_pull(model, tp):
    """K-major destinations: element (i, c) of the row-major pull sits at flat c*rows + i, checked
    one element at a time from the generator (dst_elements) and, at TP=1, against torch's cast and
    transpose of the concatenated tensors."""
    d = MODELS[model]
    rng = np.random.default_rng(11)
    for r in range(tp):
        a = direct_pull(d, tp, r, SEED, 6, specials=True)
        t = direct_pull(d, tp, r, SEED, 6, specials=True, transpose=True)
        for dst in vllm_dsts(d, tp):
            x, y = a[dst.name], t[dst.name]
            if x.ndim == 1:
                assert np.array_equal(x, y)
                continue
            assert y.shape == (x.shape[1], x.shape[0])
            idx = rng.integers(0, x.size, 256)
            assert np.array_equal(y.ravel()[idx], dst_elements(d, tp, r, dst.name, idx, SEED, 6, True,
                                                               transpose=True)), dst.name
            ii, cc = idx % x.shape[0], idx // x.shape[0]
            assert np.array_equal(y.ravel()[idx], x[ii, cc])
    if tp == 1:
        t = direct_pull(d, 1, 0, SEED, 6, transpose=True)
        for dst in vllm_dsts(d, 1):
            ref = torch.cat([_torch_cast(p.tensor, 6, d) for p in dst.parts], 0)
            ref = ref.t().contiguous() if ref.dim() == 2 else ref
            assert np.array_equal(t[dst.name], ref.view(torch.int16).numpy().view(np.uint16)), dst.name


@pytest.mark.parametrize("model,layout,N,C,tp,tr", [
    ("tiny", FSDP2_DIM0, 1, 1 << 20, 1, False), ("tiny", FSDP2_DIM0, 4, 1 << 18, 2, False),
    ("tiny", FSDP1_FLAT, 3, 1 << 18, 4, False), ("tiny", FSDP2_DIM0, 8, 4096 * 5, 4, True),
    ("odd", FSDP1_FLAT, 3, 4096, 8, True), ("odd", FSDP2_DIM0, 4, 4096 * 2, 4, False)])
def test_two_pull_paths_agree(model, layout, N, C, tp, tr):
    d = MODELS[model]
    plan = image_plan([s for _, s in tensors(d)], N, C, layout)
    img, _ = publish(plan, SEED, 5, specials=True)
    rd = lambda o, n: img[o:o + n]
    for r in range(tp):
        a = pull_from_image(rd, plan, d, tp, r, transpose=tr)
        b = direct_pull(d, tp, r, SEED, 5, specials=True, transpose=tr)
        assert a.keys() == b.keys()
        assert all(np.array_equal(a[k], b[k]) for k in a)


@pytest.mark.parametrize("model,tp,r", [("tiny", 4, 3), ("odd", 8, 7), ("odd", 8, 5), ("odd", 4, 3)])
def test_sampled_elements_match_direct(model, tp, r):
    d = MODELS[model]
    rng = np.random.default_rng(3)
    full = direct_pull(d, tp, r, SEED, 2)
    for dst in vllm_dsts(d, tp):
        idx = rng.integers(0, numel(dst.shape), 64)
        assert np.array_equal(dst_elements(d, tp, r, dst.name, idx, SEED, 2), full[dst.name].ravel()[idx])


# --------------------------------------------------------------------------------- Appendix D
def test_spec_worked_numbers():
    # SPEC L556-558 / L565-567 / L574-576 (evaluations of PAPER L1491/L1509/L1513)
    assert chain_latency(2, 1, 1e9, 1e-9, 1e-3) == pytest.approx(1.001, rel=1e-12)
    assert chain_latency(4, 2, 1e9, 1e-9, 1e-3) == pytest.approx(2.004, rel=1e-12)
    assert chain_latency(3, 32, 1e9, 1e-9, 1e-3) == pytest.approx(33 * (1 / 32 + 0.001), rel=1e-12)
    assert abs(chain_latency(3, 32, 1e9, 1e-9, 1e-3) - 1.0643) < 1e-4   # SPEC quotes 1.0643 (4 d.p.)
    assert optimal_chunks(3, 1e9, 1e-9, 1e-3) == 32
    assert optimal_chunks(2, 1e9, 1e-9, 1e-3) == 1
    bw, lat, pipe = latency_decomposition(128, 1.6, 1.0, 5e-6)
    assert (round(bw, 6), round(lat, 5), round(pipe, 4)) == (1.6, 0.00063, 0.0635)
    assert round((bw + lat + pipe) / bw, 3) == 1.040       # "< 1.6 s" to 127 relays


def test_optimum_by_brute_force():
    rng = random.Random(7)
    for _ in range(100):
        p = rng.randint(3, 200)
        M, Tb, Ts = rng.uniform(1e6, 1e11), 1 / rng.uniform(1e9, 1e12), rng.uniform(1e-7, 1e-3)
        ks = range(1, 4097)
        best = min(ks, key=lambda k: chain_latency(p, k, M, Tb, Ts))
        kk = optimal_chunks(p, M, Tb, Ts, k_cap=4096)
        # the integer optimum is floor or ceil of k*, round() picks one of them
        assert abs(kk - best) <= 1
        assert chain_latency(p, kk, M, Tb, Ts) <= min(chain_latency(p, k, M, Tb, Ts)
                                                       for k in (max(1, kk - 1), kk + 1)) * (1 + 1e-12)
        ks_ = k_star(p, M, Tb, Ts)
        if 1 <= ks_:
            cont = chain_latency(p, 1, M, Tb, Ts) if ks_ == 1 else (p + ks_ - 2) * (M / ks_ * Tb + Ts)
            assert sum(latency_decomposition(p, M, Tb, Ts)) == pytest.approx(cont, rel=1e-12)


# ------------------------------------------------------------------------------- relay rounds
@pytest.mark.parametrize("p", range(2, 17))
def test_tail_completes_at_round_p_plus_k_minus_2(p):
    for k in range(1, 17):
        ch = RelayChain(p, k)
        assert ch.publish(1) == "ok"
        ch.run_until_quiescent()
        assert ch.completion_round[(p - 1, 1)] == p + k - 2
        # rounds x t_chunk reproduces the closed form exactly
        M, Tb, Ts = 1e9, 1e-9, 1e-3
        assert (p + k - 2) * (M / k * Tb + Ts) == chain_latency(p, k, M, Tb, Ts)


def test_publish_rules():
    ch = RelayChain(3, 4)
    assert ch.publish(1) == "ok"
    assert ch.publish(1) == "stale"
    assert ch.publish(0) == "stale"
    assert ch.pin_latest(2) == (0, None)                       # fresh node: none
    ch.step()
    assert ch.nodes[1].latest == 0                             # partial versions never served
    ch.run_until_quiescent()
    assert all(n.latest == 1 for n in ch.nodes)


@pytest.mark.parametrize("seed", range(20))
def test_random_interleavings_keep_invariants(seed):
    rng = random.Random(seed)
    p, k = rng.randint(2, 6), rng.randint(1, 6)
    ch = RelayChain(p, k, slots=rng.choice([2, 3]))
    published, v, pins, records = set(), 0, [], []
    last_latest = [0] * p
    for _ in range(400):
        a = rng.random()
        if a < 0.15:
            v += 1
            if ch.publish(v) == "ok":
                published.add(v)
        elif a < 0.35:
            node = rng.randrange(p)
            latest = ch.nodes[node].latest
            got, slot = ch.pin_latest(node)
            if got:
                s = ch.nodes[node].slots[slot]
                assert s.state == COMPLETE and s.version == got and len(s.have) == k
                pins.append((node, slot, got))
            records.append(invariants.PullRecord(node, got, latest, True))
        elif a < 0.5 and pins:
            node, slot, got = pins.pop(rng.randrange(len(pins)))
            ch.unpin(node, slot)
        else:
            ch.step()
        for node, slot, got in pins:                               # pinned slots never overwritten
            assert ch.nodes[node].slots[slot].version == got
        for i, n in enumerate(ch.nodes):
            assert n.latest >= last_latest[i]                      # monotone
            last_latest[i] = n.latest
    for node, slot, _ in pins:
        ch.unpin(node, slot)
    ch.run_until_quiescent()
    newest = max(published) if published else 0
    assert all(n.latest == newest for n in ch.nodes)              # quiescent: everyone has the newest
    assert invariants.check(published, records) == []


def test_invariant_checker_flags_violations():
    recs = [invariants.PullRecord(0, 2, 0, True), invariants.PullRecord(0, 1, 0, True),
            invariants.PullRecord(1, 9, 0, True), invariants.PullRecord(1, 3, 3, False),
            invariants.PullRecord(2, 2, 3, True)]
    errs = invariants.check({1, 2, 3}, recs)
    assert len(errs) == 5     # back, unpublished, back+torn, behind-latest

"""Pins of oracle/model.py and oracle/image.py: library model definitions, torch.chunk semantics,
bijection / brute-force reassembly, image format invariants, and the cast reached through the image."""
import numpy as np
import pytest
import torch

from oracle.bf16 import rne_bf16
from oracle.checksum import chunk_checksum
from oracle.image import (FSDP1_FLAT, FSDP2_DIM0, SEG_ALIGN, actor_shards, headers_of, image_plan,
                          publish, publish_chunk, unpack_tensor)
from oracle.model import MODELS, numel, param_count, tensors
from synth import SEED, gen_bits

# Published parameter counts of the Qwen2.5 checkpoints' configs (untied embeddings) and our tiny model.
PUBLISHED = {"tiny": (10_227_968, 51), "7b": (7_615_616_512, 339), "32b": (32_763_876_352, 771),
             "72b": (72_706_203_648, 963),
             # odd: embed 130*64 + 2 layers * (q 64*64+64, k,v 2*(16*64+16), o 64*64, gate/up/down
             # 3*192*64, norms 2*64) + norm 64 + lm_head 130*64, counted by hand
             "odd": (111_360, 27)}


@pytest.mark.parametrize("name", ["tiny", "7b", "32b", "72b", "odd"])
def test_param_counts(name):
    d = MODELS[name]
    assert (param_count(d), len(tensors(d))) == PUBLISHED[name]


@pytest.mark.parametrize("name", ["tiny", "7b", "odd"])
def test_tensor_table_matches_transformers_qwen2(name):
    transformers = pytest.importorskip("transformers")
    d = MODELS[name]
    cfg = transformers.Qwen2Config(hidden_size=d.H, intermediate_size=d.I, num_hidden_layers=d.L,
                                   num_attention_heads=d.nh, num_key_value_heads=d.nkv, head_dim=d.hd,
                                   vocab_size=d.V, tie_word_embeddings=False)
    with torch.device("meta"):
        m = transformers.Qwen2ForCausalLM(cfg)
    ref = [(k, tuple(v.shape)) for k, v in m.state_dict().items()]
    assert ref == tensors(d)


SHAPES = [(7, 3), (5,), (1, 4), (12, 2), (3, 5), (9,)]   # ragged: d0 < N, d0 % N != 0, 1-D


@pytest.mark.parametrize("N", [1, 2, 3, 4, 8])
def test_fsdp2_is_torch_chunk(N):
    sh = actor_shards(SHAPES, N, FSDP2_DIM0)
    for t, shp in enumerate(SHAPES):
        ref = torch.arange(numel(shp)).reshape(shp).chunk(N, dim=0)
        for r in range(N):
            mine = [(e0, c) for (tt, e0, c) in sh[r] if tt == t]
            want = ref[r].reshape(-1).tolist() if r < len(ref) else []
            got = list(range(mine[0][0], mine[0][0] + mine[0][1])) if mine else []
            assert got == want


@pytest.mark.parametrize("N", [1, 2, 3, 4, 8])
def test_fsdp1_is_flat_pad_split(N):
    sh = actor_shards(SHAPES, N, FSDP1_FLAT)
    flat = torch.cat([torch.full((numel(s),), t) * 1000 + torch.arange(numel(s)) for t, s in enumerate(SHAPES)])
    P = flat.numel()
    padded = torch.cat([flat, torch.full(((-P) % N,), -1)])
    for r, piece in enumerate(padded.chunk(N)):
        want = [int(x) for x in piece.tolist() if x >= 0]
        got = [t * 1000 + e for (t, e0, c) in sh[r] for e in range(e0, e0 + c)]
        assert got == want


@pytest.mark.parametrize("layout", [FSDP2_DIM0, FSDP1_FLAT])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 8])
def test_shards_are_a_bijection(layout, N):
    shapes = [s for _, s in tensors(MODELS["tiny"])]
    seen = [np.zeros(numel(s), np.int32) for s in shapes]
    for r, lst in enumerate(actor_shards(shapes, N, layout)):
        for t, e0, c in lst:
            seen[t][e0:e0 + c] += 1
    assert all(np.all(x == 1) for x in seen)


def _tiny_shapes():
    return [s for _, s in tensors(MODELS["tiny"])]


@pytest.mark.parametrize("layout,N,C", [(FSDP2_DIM0, 1, 1 << 20), (FSDP2_DIM0, 3, 3 * 4096 * 37),
                                        (FSDP1_FLAT, 4, 1 << 18), (FSDP2_DIM0, 8, 4096)])
def test_image_format_invariants(layout, N, C):
    shapes = _tiny_shapes()
    plan = image_plan(shapes, N, C, layout)
    assert sum(s.count for s in plan.segments) == sum(numel(s) for s in shapes)
    for r in range(N):
        segs = [s for s in plan.segments if s.rank == r]
        for a, b in zip(segs, segs[1:]):
            assert a.off + 2 * a.count <= b.off                  # disjoint, in tensor order
            assert a.tensor_id < b.tensor_id or layout == FSDP1_FLAT
        assert all(s.off % SEG_ALIGN == 0 for s in segs)
        assert plan.region_len[r] % SEG_ALIGN == 0 and plan.region_len[r] <= plan.n_chunks[r] * C
    lens = [plan.chunk_len(g) for g in range(plan.total_chunks)]
    assert all(0 < n <= C and n % 16 == 0 for n in lens)


def test_publish_image_unpacks_to_cast_of_masters():
    shapes = _tiny_shapes()
    for layout, N, C in [(FSDP2_DIM0, 2, 1 << 19), (FSDP1_FLAT, 3, 1 << 18)]:
        plan = image_plan(shapes, N, C, layout)
        img, hdr = publish(plan, SEED, 2, specials=True)
        covered = np.zeros(img.size, bool)
        for s in plan.segments:
            o = plan.image_offset(s)
            covered[o:o + 2 * s.count] = True
        assert not img[~covered].any()                           # pads and gaps are zero
        rd = lambda o, n: img[o:o + n]
        for t, shp in enumerate(shapes):
            want = rne_bf16(gen_bits(SEED, 2, t, 0, numel(shp), True)).reshape(shp)
            assert np.array_equal(unpack_tensor(rd, plan, t, shp), want)
        assert len(hdr) == plan.total_chunks
        for g, h in enumerate(hdr):
            assert (h["s1"], h["s2"]) == chunk_checksum(img[g * C:g * C + h["bytes"]])
            assert np.array_equal(publish_chunk(plan, g, SEED, 2, True), img[g * C:g * C + h["bytes"]])


def test_versions_differ_everywhere_that_matters():
    plan = image_plan(_tiny_shapes(), 1, 1 << 20)
    a, ha = publish(plan, SEED, 1)
    b, hb = publish(plan, SEED, 2)
    assert all((x["s1"], x["s2"]) != (y["s1"], y["s2"]) for x, y in zip(ha, hb))
    assert headers_of(plan, a, 1) == ha

"""Pin the oracle's TP reshard rules (oracle/tp.py, R7/R14/R15) against vLLM's own weight
loaders — the code a rollout engine runs to shard a full checkpoint for TP rank r ("reshards
them according to the rollout sharding strategy (e.g., tensor parallelism ...)"; L1357 TP 1/4/8).

For every destination of the Qwen2 layout, vLLM's layer for (tp, rank) is built on CPU (the layers'
TP-group queries answer (rank, tp) instead of asking a process group) and loaded with the FULL source
tensors through its weight_loader; the parameter it ends up holding must equal the oracle's rule applied
to the same tensors (`tp._apply` + concatenation, i.e. what `direct_pull` and `pull_from_image` produce
before the cast).  This pins the fused row orders [q_r; k_r; v_r] and [gate_r; up_r] (QKVParallelLinear,
MergedColumnParallelLinear), KV-head replication when tp > nkv, the dim-1 slices of RowParallelLinear,
and the padded vocabulary rows of VocabParallelEmbedding / ParallelLMHead — none of them by the
oracle's own arithmetic.  Values: distinct fp32 per element (harness generator), so any misplaced row
shows."""
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
L = pytest.importorskip("vllm.model_executor.layers.linear")
VE = pytest.importorskip("vllm.model_executor.layers.vocab_parallel_embedding")

from oracle.model import MODELS, tensors  # noqa: E402
from oracle.tp import _apply, vllm_dsts  # noqa: E402
from synth import SEED, gen_f32  # noqa: E402


def _set_tp(monkeypatch, tp, rank):
    for mod in list(sys.modules.values()):
        if mod is None or not getattr(mod, "__name__", "").startswith("vllm"):
            continue
        if hasattr(mod, "get_tensor_model_parallel_rank"):
            monkeypatch.setattr(mod, "get_tensor_model_parallel_rank", lambda: rank, raising=False)
        if hasattr(mod, "get_tensor_model_parallel_world_size"):
            monkeypatch.setattr(mod, "get_tensor_model_parallel_world_size", lambda: tp, raising=False)


def _full(d, name, shape):
    tid = [n for n, _ in tensors(d)].index(name)
    return gen_f32(SEED, 1, tid, 0, int(np.prod(shape))).reshape(shape).copy()


def _vllm_param(d, dst_name, tp, full):
    """The parameter vLLM's layer for this destination holds after loading the full tensors."""
    f32 = torch.float32
    T = lambda a: torch.from_numpy(a)
    base = dst_name.rsplit(".", 2)[0] + "." if dst_name.startswith("model.layers.") else ""
    if "qkv_proj" in dst_name:
        layer = L.QKVParallelLinear(d.H, d.hd, d.nh, d.nkv, bias=True, params_dtype=f32, prefix="qkv")
        what = "weight" if dst_name.endswith("weight") else "bias"
        param = getattr(layer, what)
        for sid in ("q", "k", "v"):
            src = base.replace("qkv_proj.", "") + f"{sid}_proj.{what}"
            layer.weight_loader(param, T(full[src]), sid)
        return param.detach().numpy()
    if "gate_up_proj" in dst_name:
        layer = L.MergedColumnParallelLinear(d.H, [d.I, d.I], bias=False, params_dtype=f32, prefix="gu")
        for sid, x in enumerate(("gate_proj", "up_proj")):
            layer.weight_loader(layer.weight, T(full[base.replace("gate_up_proj.", "") + f"{x}.weight"]), sid)
        return layer.weight.detach().numpy()
    if "o_proj" in dst_name or "down_proj" in dst_name:
        inp, out = (d.nh * d.hd, d.H) if "o_proj" in dst_name else (d.I, d.H)
        layer = L.RowParallelLinear(inp, out, bias=False, params_dtype=f32, prefix="row")
        layer.weight_loader(layer.weight, T(full[dst_name]))
        return layer.weight.detach().numpy()
    if dst_name in ("model.embed_tokens.weight", "lm_head.weight"):
        cls = VE.VocabParallelEmbedding if dst_name.startswith("model.") else VE.ParallelLMHead
        layer = cls(d.V, d.H, params_dtype=f32, prefix="vocab")
        layer.weight.data.zero_()
        layer.weight_loader(layer.weight, T(full[dst_name]))
        return layer.weight.detach().numpy()
    return None   # norms: REPLICATE, no TP layer


@pytest.mark.parametrize("model,tp", [("tiny", 1), ("tiny", 2), ("tiny", 4), ("tiny", 8),
                                      ("odd", 2), ("odd", 4), ("odd", 8)])
def test_tp_rules_equal_vllm_weight_loaders(monkeypatch, model, tp):
    d = MODELS[model]
    shapes = dict(tensors(d))
    layer0 = {n for n in shapes if not n.startswith("model.layers.") or n.startswith("model.layers.0.")}
    full = {n: _full(d, n, shapes[n]) for n in layer0}
    checked = 0
    for rank in range(tp):
        _set_tp(monkeypatch, tp, rank)
        for dst in vllm_dsts(d, tp):
            if dst.name.startswith("model.layers.") and not dst.name.startswith("model.layers.0."):
                continue
            got = _vllm_param(d, dst.name, tp, full)
            if got is None:
                continue
            want = np.concatenate([_apply(full[p.tensor], p, tp, rank) for p in dst.parts], axis=0)
            assert got.shape == want.shape, (dst.name, rank, got.shape, want.shape)
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (dst.name, tp, rank)
            checked += 1
    assert checked == tp * 7     # embed, qkv weight, qkv bias, o, gate_up, down, lm_head per rank


def test_kv_replication_case_is_exercised():
    """odd: nkv = 2 < tp = 4, 8 — the vLLM loader replicates KV heads; the oracle rule is HEAD_DIM0."""
    assert MODELS["odd"].nkv < 4 and MODELS["odd"].V % 64 != 0

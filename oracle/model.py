"""Qwen2.5-shaped tensor tables (oracle copy; the CUDA path has its own, independently written).

PAPER.md L963 ("Qwen2.5") and L1354 name the models; their public configs give the dimensions.
Tensor order is the Hugging Face Qwen2 state-dict order (SURVEY §8 "Per layer there are 12
tensors ..."); every nn.Parameter is published, rotary buffers are not (SURVEY reading 8);
embeddings are untied (reading 9).  Pinned in tests against transformers' own Qwen2ForCausalLM
(state_dict names, shapes, order) and against the published parameter counts.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Dims:
    H: int      # hidden size
    I: int      # MLP intermediate size
    L: int      # layers
    nh: int     # attention heads
    nkv: int    # key/value heads
    hd: int     # head dim
    V: int      # vocab


MODELS = {
    "tiny": Dims(H=256, I=1024, L=4, nh=8, nkv=4, hd=32, V=12288),      # SURVEY §8 "tiny (ours)"
    "7b": Dims(H=3584, I=18944, L=28, nh=28, nkv=4, hd=128, V=152064),  # Qwen2.5-7B
    "32b": Dims(H=5120, I=27648, L=64, nh=40, nkv=8, hd=128, V=152064),  # Qwen2.5-32B
    "72b": Dims(H=8192, I=29568, L=80, nh=64, nkv=8, hd=128, V=152064),  # Qwen2.5-72B
    # Edge-case model (ours): V = 130 needs vocabulary padding (to 192, so at
    # TP=8 ranks 6-7 hold only padding) and nkv = 2 < tp = 4, 8 needs KV-head replication.
    "odd": Dims(H=64, I=192, L=2, nh=8, nkv=2, hd=8, V=130),
}


def tensors(d: Dims) -> list[tuple[str, tuple[int, ...]]]:
    """(name, shape) of every published parameter, in state-dict order; tensor_id = list index."""
    out = [("model.embed_tokens.weight", (d.V, d.H))]
    q, kv = d.nh * d.hd, d.nkv * d.hd
    for l in range(d.L):
        p = f"model.layers.{l}."
        out += [
            (p + "self_attn.q_proj.weight", (q, d.H)),
            (p + "self_attn.q_proj.bias", (q,)),
            (p + "self_attn.k_proj.weight", (kv, d.H)),
            (p + "self_attn.k_proj.bias", (kv,)),
            (p + "self_attn.v_proj.weight", (kv, d.H)),
            (p + "self_attn.v_proj.bias", (kv,)),
            (p + "self_attn.o_proj.weight", (d.H, q)),
            (p + "mlp.gate_proj.weight", (d.I, d.H)),
            (p + "mlp.up_proj.weight", (d.I, d.H)),
            (p + "mlp.down_proj.weight", (d.H, d.I)),
            (p + "input_layernorm.weight", (d.H,)),
            (p + "post_attention_layernorm.weight", (d.H,)),
        ]
    out += [("model.norm.weight", (d.H,)), ("lm_head.weight", (d.V, d.H))]
    return out


def numel(shape: tuple[int, ...]) -> int:
    n = 1
    for s in shape:
        n *= s
    return n


def param_count(d: Dims) -> int:
    return sum(numel(s) for _, s in tensors(d))

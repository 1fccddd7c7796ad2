// Model table, vLLM TP destination layout, and the Appendix D chunk model (library side).
//
// Tensor table: Qwen2 state-dict order ("Qwen2.5").  TP rules follow
// vLLM's Qwen2 convention ("reshards them according to the rollout sharding strategy";
// SURVEY §8(c) C7): qkv = [q_r; k_r; v_r], gate_up = [gate_r; up_r] (dim-0 shards), o/down split on
// dim 1, embed/lm_head split by padded vocab rows, norms replicated; q/k/v split by whole heads with
// KV heads replicated when tp > kv_heads (R14, R15).
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>

#include "lam_internal.h"

namespace lam {

bool model_valid(const lam_model_dims& d) {
  return d.hidden > 0 && d.intermediate > 0 && d.layers > 0 && d.heads > 0 && d.kv_heads > 0 &&
         d.head_dim > 0 && d.vocab > 0 && d.heads % d.kv_heads == 0;
}

std::vector<Tensor> model_tensors(const lam_model_dims& d) {
  std::vector<Tensor> t;
  const int64_t H = d.hidden, I = d.intermediate, q = d.heads * d.head_dim, kv = d.kv_heads * d.head_dim;
  t.push_back({"model.embed_tokens.weight", d.vocab, H, 2});
  char p[96];
  for (int64_t l = 0; l < d.layers; ++l) {
    snprintf(p, sizeof p, "model.layers.%lld.", (long long)l);
    std::string s(p);
    t.push_back({s + "self_attn.q_proj.weight", q, H, 2, d.heads});
    t.push_back({s + "self_attn.q_proj.bias", q, 1, 1, d.heads});
    t.push_back({s + "self_attn.k_proj.weight", kv, H, 2, d.kv_heads});
    t.push_back({s + "self_attn.k_proj.bias", kv, 1, 1, d.kv_heads});
    t.push_back({s + "self_attn.v_proj.weight", kv, H, 2, d.kv_heads});
    t.push_back({s + "self_attn.v_proj.bias", kv, 1, 1, d.kv_heads});
    t.push_back({s + "self_attn.o_proj.weight", H, q, 2});
    t.push_back({s + "mlp.gate_proj.weight", I, H, 2});
    t.push_back({s + "mlp.up_proj.weight", I, H, 2});
    t.push_back({s + "mlp.down_proj.weight", H, I, 2});
    t.push_back({s + "input_layernorm.weight", H, 1, 1});
    t.push_back({s + "post_attention_layernorm.weight", H, 1, 1});
  }
  t.push_back({"model.norm.weight", H, 1, 1});
  t.push_back({"lm_head.weight", d.vocab, H, 2});
  return t;
}

bool part_slice(const Tensor& t, int rule, int tp, int rank, int64_t* r0, int64_t* r1, int64_t* c0,
                int64_t* c1, int64_t* pad) {
  *r0 = 0; *r1 = t.d0; *c0 = 0; *c1 = t.d1; *pad = 0;
  switch (rule) {
    case LAM_REPLICATE: return true;
    case LAM_SHARD_DIM0:
      if (t.d0 % tp) return false;
      *r0 = rank * (t.d0 / tp); *r1 = *r0 + t.d0 / tp;
      return true;
    case LAM_VOCAB_DIM0: {   // padded rows [rank*n, (rank+1)*n) of Vp; rows >= d0 are zero
      const int64_t vp = (t.d0 + kVocabPad - 1) / kVocabPad * kVocabPad;
      if (vp % tp) return false;
      const int64_t n = vp / tp;
      *r0 = std::min<int64_t>(rank * n, t.d0);
      *r1 = std::min<int64_t>((rank + 1) * n, t.d0);
      *pad = n - (*r1 - *r0);
      return true;
    }
    case LAM_HEAD_DIM0: {    // whole heads; KV heads replicated when tp > heads
      if (t.heads < 1 || t.d0 % t.heads) return false;
      const int64_t hd = t.d0 / t.heads;
      int64_t h0, nh;
      if (tp <= t.heads) {
        if (t.heads % tp) return false;
        nh = t.heads / tp;
        h0 = rank * nh;
      } else {
        if (tp % t.heads) return false;
        nh = 1;
        h0 = rank / (tp / t.heads);
      }
      *r0 = h0 * hd; *r1 = (h0 + nh) * hd;
      return true;
    }
    case LAM_SHARD_DIM1:
      if (t.ndim != 2 || t.d1 % tp) return false;
      *c0 = rank * (t.d1 / tp); *c1 = *c0 + t.d1 / tp;
      return true;
    default: return false;
  }
}

bool vllm_layout(const lam_model_dims& d, int tp, std::vector<VllmDst>* out) {
  if (tp < 1 || !model_valid(d)) return false;
  std::vector<Tensor> ts = model_tensors(d);
  out->clear();
  auto add = [&](const std::string& name, std::vector<DstPart> parts) -> bool {
    VllmDst v{name, 0, 0, parts};
    for (auto& p : parts) {
      int64_t r0, r1, c0, c1, pad;
      if (!part_slice(ts[p.tensor], p.rule, tp, 0, &r0, &r1, &c0, &c1, &pad)) return false;
      if (v.cols && v.cols != c1 - c0) return false;
      v.cols = c1 - c0;
      v.rows += r1 - r0 + pad;
    }
    out->push_back(v);
    return true;
  };
  uint32_t id = 0;
  bool ok = add("model.embed_tokens.weight", {{id++, LAM_VOCAB_DIM0}});
  char p[96];
  for (int64_t l = 0; l < d.layers && ok; ++l) {
    snprintf(p, sizeof p, "model.layers.%lld.", (long long)l);
    std::string s(p);
    uint32_t q = id, qb = id + 1, k = id + 2, kb = id + 3, v = id + 4, vb = id + 5, o = id + 6,
             g = id + 7, u = id + 8, dn = id + 9, n1 = id + 10, n2 = id + 11;
    id += 12;
    ok = ok && add(s + "self_attn.qkv_proj.weight", {{q, LAM_HEAD_DIM0}, {k, LAM_HEAD_DIM0}, {v, LAM_HEAD_DIM0}});
    ok = ok && add(s + "self_attn.qkv_proj.bias", {{qb, LAM_HEAD_DIM0}, {kb, LAM_HEAD_DIM0}, {vb, LAM_HEAD_DIM0}});
    ok = ok && add(s + "self_attn.o_proj.weight", {{o, LAM_SHARD_DIM1}});
    ok = ok && add(s + "mlp.gate_up_proj.weight", {{g, LAM_SHARD_DIM0}, {u, LAM_SHARD_DIM0}});
    ok = ok && add(s + "mlp.down_proj.weight", {{dn, LAM_SHARD_DIM1}});
    ok = ok && add(s + "input_layernorm.weight", {{n1, LAM_REPLICATE}});
    ok = ok && add(s + "post_attention_layernorm.weight", {{n2, LAM_REPLICATE}});
  }
  ok = ok && add("model.norm.weight", {{id++, LAM_REPLICATE}});
  ok = ok && add("lm_head.weight", {{id++, LAM_VOCAB_DIM0}});
  return ok;
}

}  // namespace lam

using namespace lam;

extern "C" int32_t lam_model_n_tensors(const lam_model_dims* d) {
  if (!d || !model_valid(*d)) return -1;
  return (int32_t)(3 + 12 * d->layers);
}

extern "C" lam_status lam_model_tensor(const lam_model_dims* d, int32_t id, char* name, int32_t cap,
                                       int64_t shape[2], int32_t* ndim) {
  if (!d || !model_valid(*d)) return LAM_EINVAL;
  std::vector<Tensor> ts = model_tensors(*d);
  if (id < 0 || id >= (int32_t)ts.size()) return LAM_EINVAL;
  if (name && cap > 0) snprintf(name, cap, "%s", ts[id].name.c_str());
  if (shape) { shape[0] = ts[id].d0; shape[1] = ts[id].ndim == 2 ? ts[id].d1 : 0; }
  if (ndim) *ndim = ts[id].ndim;
  return LAM_OK;
}

extern "C" int32_t lam_vllm_layout(const lam_model_dims* d, int32_t tp, lam_dst* dsts, int32_t cap_dsts,
                                   lam_part* parts, int32_t cap_parts, char* names, int32_t name_cap,
                                   int64_t* rows, int64_t* cols) {
  if (!d) return LAM_EINVAL;
  std::vector<VllmDst> v;
  if (!vllm_layout(*d, tp, &v)) return LAM_EINVAL;
  if (!dsts) return (int32_t)v.size();
  int32_t np = 0;
  for (size_t i = 0; i < v.size() && (int32_t)i < cap_dsts; ++i) {
    if (np + (int32_t)v[i].parts.size() > cap_parts) return LAM_EINVAL;
    dsts[i].parts = parts + np;
    dsts[i].n_parts = (int32_t)v[i].parts.size();
    dsts[i].transpose = 0;
    dsts[i].dst = nullptr;
    dsts[i].dst_row_pitch_bytes = 0;
    for (auto& p : v[i].parts) parts[np++] = lam_part{p.tensor, p.rule};
    if (names && name_cap > 0) snprintf(names + (size_t)i * name_cap, name_cap, "%s", v[i].name.c_str());
    if (rows) rows[i] = v[i].rows;
    if (cols) cols[i] = v[i].cols;
  }
  return (int32_t)v.size();
}

// Appendix D: library-side implementation used to pick the chunk size.
extern "C" double lam_chain_latency(int32_t p, int64_t k, double M, double tb, double ts) {
  if (p < 2 || k < 1) return -1.0;
  return (double)(p + k - 2) * (M / (double)k * tb + ts);
}

extern "C" int64_t lam_optimal_chunks(int32_t p, double M, double tb, double ts, int64_t cap) {
  if (p < 2 || cap < 1) return -1;
  if (ts <= 0) return cap;
  double k = sqrt((double)(p - 2) * M * tb / ts);
  int64_t r = (int64_t)llround(k);
  return r < 1 ? 1 : (r > cap ? cap : r);
}

// Model derivation, config validation, the analytic operator model and the
// contention-aware cost model.
//
// Parity notes: every floating-point expression below
// keeps the reference's operand order (domain.cpp:7-24, opcost.cpp:56-189,
// costmodel.cpp:8-102) because the controller compares latencies with `>`
// and a last-ulp difference would flip a split decision.
#include <algorithm>
#include <cstdio>

#include "core.hpp"

namespace nxb {

// ModelConfig::derive (domain.cpp:7-24): kv = 2*L*d*elem; dense params
// 4d^2 + 2*d*d_ff per layer; attention-internal weights d per layer.
nx_model_config derive_model(int64_t hidden, int64_t ffn, int32_t layers, int32_t heads,
                             int32_t elem) {
  nx_model_config m{};
  m.hidden_dim = hidden;
  m.ffn_dim = ffn;
  m.num_layers = layers;
  m.num_heads = heads;
  m.element_bytes = elem;
  m.kv_bytes_per_token = int64_t{2} * layers * hidden * elem;
  const int64_t dense_params = 4 * hidden * hidden + 2 * hidden * ffn;
  m.weight_bytes_per_layer_dense = dense_params * elem;
  m.weight_bytes_per_layer_attn = hidden * elem;
  return m;
}

namespace {

struct Violations {
  std::string text;
  int count = 0;
  void require(bool ok, const std::string& field, const char* why) {
    if (ok) return;
    if (count++) text += "; ";
    text += field + ": " + why;
  }
};

void check_curve(Violations& v, const nx_saturation_curve& c, const char* name) {
  const std::string base = std::string("profile.") + name;
  v.require(c.r_sat > 0.0 && c.r_sat <= 1.0, base + ".r_sat", "must lie in (0, 1]");
  v.require(c.lambda >= 0.0, base + ".lambda", "must be >= 0");
}

}  // namespace

// validate_config (domain.cpp:42-86): all violations, in the reference order.
std::string validate(const nx_model_config& m, const nx_gpu_spec& g,
                     const nx_controller_config& c, const nx_kernel_profile& p, int* count) {
  Violations v;
  v.require(m.hidden_dim > 0, "model.hidden_dim", "must be > 0");
  v.require(m.ffn_dim > 0, "model.ffn_dim", "must be > 0");
  v.require(m.ffn_dim >= m.hidden_dim, "model.ffn_dim", "must be >= hidden_dim");
  v.require(m.num_layers > 0, "model.num_layers", "must be > 0");
  v.require(m.num_heads > 0, "model.num_heads", "must be > 0");
  v.require(m.element_bytes > 0, "model.element_bytes", "must be > 0");
  v.require(m.kv_bytes_per_token > 0, "model.kv_bytes_per_token", "must be > 0");
  if (m.hidden_dim > 0 && m.num_layers > 0 && m.element_bytes > 0) {
    const int64_t want = int64_t{2} * m.num_layers * m.hidden_dim * m.element_bytes;
    v.require(m.kv_bytes_per_token == want, "model.kv_bytes_per_token",
              "must equal 2 * num_layers * hidden_dim * element_bytes");
  }
  v.require(m.weight_bytes_per_layer_dense > 0, "model.weight_bytes_per_layer_dense",
            "must be > 0");
  v.require(m.weight_bytes_per_layer_attn > 0, "model.weight_bytes_per_layer_attn",
            "must be > 0");
  v.require(g.total_sm >= 2, "gpu.total_sm", "must be >= 2 so both phases are allocatable");
  v.require(g.peak_compute > 0, "gpu.peak_compute", "must be > 0");
  v.require(g.peak_bandwidth > 0, "gpu.peak_bandwidth", "must be > 0");
  v.require(g.kv_capacity_bytes > 0, "gpu.kv_capacity_bytes", "must be > 0");
  v.require(c.alpha > 1.0, "controller.alpha", "must exceed 1");
  v.require(c.beta > 1.0, "controller.beta", "must exceed 1");
  v.require(c.kv_switch_fraction > 0.0 && c.kv_switch_fraction < 1.0,
            "controller.kv_switch_fraction", "must lie in (0, 1)");
  v.require(c.delta_pp >= 0, "controller.delta_pp", "must be >= 0");
  v.require(c.gamma >= 0.0, "controller.gamma", "must be >= 0");
  v.require(c.chunk_size >= 1, "controller.chunk_size", "must be >= 1");
  v.require(c.max_decode_batch >= 1, "controller.max_decode_batch", "must be >= 1");
  v.require(c.token_budget >= 1, "controller.token_budget", "must be >= 1");
  check_curve(v, p.qkv_proj, "qkv_proj");
  check_curve(v, p.attn_prefill, "attn_prefill");
  check_curve(v, p.attn_decode, "attn_decode");
  check_curve(v, p.attn_out_proj, "attn_out_proj");
  check_curve(v, p.ffn, "ffn");
  if (count) *count = v.count;
  return v.text;
}

const nx_saturation_curve& curve_of(const nx_kernel_profile& p, int kind) {
  switch (kind) {
    case NX_OP_QKV_PROJ: return p.qkv_proj;
    case NX_OP_ATTN_PREFILL: return p.attn_prefill;
    case NX_OP_ATTN_DECODE: return p.attn_decode;
    case NX_OP_ATTN_OUT_PROJ: return p.attn_out_proj;
    default: return p.ffn;
  }
}

static const char* const kOpNames[5] = {"qkv_proj", "attn_prefill", "attn_decode",
                                        "attn_out_proj", "ffn"};

const char* op_name(int kind) { return (kind >= 0 && kind < 5) ? kOpNames[kind] : "unknown"; }

int op_from_name(const std::string& name) {
  for (int k = 0; k < 5; ++k)
    if (name == kOpNames[k]) return k;
  return -1;
}

// ---------------------------------------------------------------------------
// Operator model.
// ---------------------------------------------------------------------------
namespace {

// Per-iteration bytes of each dense operator: the dense weight budget
// L * weight_bytes_per_layer_dense apportioned by parameter count
// (opcost.cpp:56-71).
struct DenseBytes {
  double qkv, out, ffn;
};

DenseBytes dense_bytes(const nx_model_config& m) {
  const double d = static_cast<double>(m.hidden_dim);
  const double dff = static_cast<double>(m.ffn_dim);
  const double p_qkv = 3.0 * d * d;
  const double p_out = d * d;
  const double p_ffn = 2.0 * d * dff;
  const double p_all = p_qkv + p_out + p_ffn;
  const double bytes = static_cast<double>(m.num_layers) *
                       static_cast<double>(m.weight_bytes_per_layer_dense);
  return {bytes * (p_qkv / p_all), bytes * (p_out / p_all), bytes * (p_ffn / p_all)};
}

double attention_weight_bytes(const nx_model_config& m) {
  return static_cast<double>(m.num_layers) * static_cast<double>(m.weight_bytes_per_layer_attn);
}

// GEMM FLOPs use the 2*m*n*k convention, summed over layers (opcost.cpp:73-87).
void push_qkv(OpList& ops, const nx_model_config& m, double n) {
  const double d = static_cast<double>(m.hidden_dim);
  const double L = static_cast<double>(m.num_layers);
  ops.push(NX_OP_QKV_PROJ, 6.0 * n * d * d * L, dense_bytes(m).qkv, 0, false);
}

void push_out_and_ffn(OpList& ops, const nx_model_config& m, double n) {
  const double d = static_cast<double>(m.hidden_dim);
  const double dff = static_cast<double>(m.ffn_dim);
  const double L = static_cast<double>(m.num_layers);
  const DenseBytes w = dense_bytes(m);
  ops.push(NX_OP_ATTN_OUT_PROJ, 2.0 * n * d * d * L, w.out, 0, false);
  ops.push(NX_OP_FFN, 4.0 * n * d * dff * L, w.ffn, 0, false);
}

// Accumulates chunk tokens, attention FLOPs (scores + aggregation, full
// context) and attended KV bytes, in chunk order.
struct PrefillSums {
  double tokens = 0, flops = 0, kv = 0;
};

PrefillSums sum_chunks(const nx_model_config& m, const Chunk* c, size_t n, const char* who) {
  const double d = static_cast<double>(m.hidden_dim);
  const double L = static_cast<double>(m.num_layers);
  PrefillSums s;
  for (size_t i = 0; i < n; ++i) {
    if (c[i].tokens < 1 || c[i].context < c[i].tokens)
      throw InvalidArg(std::string(who) + ": bad chunk shape");
    s.tokens += static_cast<double>(c[i].tokens);
    s.flops += 4.0 * static_cast<double>(c[i].tokens) * static_cast<double>(c[i].context) * d * L;
    s.kv += static_cast<double>(c[i].context) * static_cast<double>(m.kv_bytes_per_token);
  }
  return s;
}

struct DecodeSums {
  double flops = 0, kv = 0;
};

DecodeSums sum_decode(const nx_model_config& m, const int64_t* ctx, size_t n, const char* who) {
  const double d = static_cast<double>(m.hidden_dim);
  const double L = static_cast<double>(m.num_layers);
  DecodeSums s;
  for (size_t i = 0; i < n; ++i) {
    if (ctx[i] < 1) throw InvalidArg(std::string(who) + ": context_len must be >= 1");
    s.flops += 4.0 * static_cast<double>(ctx[i]) * d * L;
    s.kv += static_cast<double>(ctx[i]) * static_cast<double>(m.kv_bytes_per_token);
  }
  return s;
}

}  // namespace

// prefill_batch_workloads (opcost.cpp:99-126): [QKV, AttnPrefill, OutProj, FFN].
OpList prefill_ops(const nx_model_config& m, const Chunk* chunks, size_t n) {
  if (n == 0) throw InvalidArg("prefill_batch_workloads: empty batch");
  const PrefillSums s = sum_chunks(m, chunks, n, "prefill_batch_workloads");
  OpList ops;
  push_qkv(ops, m, s.tokens);
  ops.push(NX_OP_ATTN_PREFILL, s.flops, s.kv + attention_weight_bytes(m), s.kv, true);
  push_out_and_ffn(ops, m, s.tokens);
  return ops;
}

// decode_op_workloads (opcost.cpp:128-148): [QKV, AttnDecode, OutProj, FFN].
OpList decode_ops(const nx_model_config& m, const int64_t* ctx, size_t n) {
  if (n == 0) throw InvalidArg("decode_op_workloads: empty batch");
  const DecodeSums s = sum_decode(m, ctx, n, "decode_op_workloads");
  OpList ops;
  push_qkv(ops, m, static_cast<double>(n));
  ops.push(NX_OP_ATTN_DECODE, s.flops, s.kv + attention_weight_bytes(m), s.kv, true);
  push_out_and_ffn(ops, m, static_cast<double>(n));
  return ops;
}

// mixed_batch_workloads (opcost.cpp:150-189): the token count starts from the
// decode batch size, then adds every chunk — the same accumulation order.
OpList mixed_ops(const nx_model_config& m, const Chunk* chunks, size_t n, const int64_t* ctx,
                 size_t nd) {
  if (n == 0 && nd == 0) throw InvalidArg("mixed_batch_workloads: empty batch");
  if (n == 0) return decode_ops(m, ctx, nd);
  if (nd == 0) return prefill_ops(m, chunks, n);
  // The fused token count starts at the decode batch size and then adds the
  // chunks (opcost.cpp:159-170), so accumulate onto it directly.
  PrefillSums p = sum_chunks(m, chunks, n, "mixed_batch_workloads");
  p.tokens = static_cast<double>(nd);
  for (size_t i = 0; i < n; ++i) p.tokens += static_cast<double>(chunks[i].tokens);
  const DecodeSums dsum = sum_decode(m, ctx, nd, "mixed_batch_workloads");
  const double aw = attention_weight_bytes(m);
  OpList ops;
  push_qkv(ops, m, p.tokens);
  ops.push(NX_OP_ATTN_PREFILL, p.flops, p.kv + aw, p.kv, true);
  ops.push(NX_OP_ATTN_DECODE, dsum.flops, dsum.kv + aw, dsum.kv, true);
  push_out_and_ffn(ops, m, p.tokens);
  return ops;
}

// ---------------------------------------------------------------------------
// Cost model.
// ---------------------------------------------------------------------------

// Eq. 5 (costmodel.cpp:8-14): 1/share scaling up to r_sat, then a linear
// decay penalty lambda per unit of extra share.
double compute_latency(double flops, double share, const nx_saturation_curve& c, double peak) {
  if (!(share > 0.0)) throw InvalidArg("compute_latency: share must be > 0");
  if (flops < 0) throw InvalidArg("compute_latency: flops must be >= 0");
  if (share <= c.r_sat) return flops / (share * peak);
  return flops / (c.r_sat * peak) * (1.0 + c.lambda * (share - c.r_sat));
}

// Sum over operators of max(compute, memory) (costmodel.cpp:18-41).
nx_breakdown breakdown(const OpList& ops, double share, const nx_gpu_spec& g,
                       const nx_kernel_profile& p, double decode_bw, const nx_cost_ext* ext) {
  if (ops.empty()) throw InvalidArg("phase latency: empty operator list");
  const bool use_ext = ext != nullptr && ext->enabled != 0;
  nx_breakdown out{};
  out.n_ops = ops.n;
  for (int i = 0; i < ops.n; ++i) {
    const nx_op_workload& w = ops.op[i];
    const bool contended = w.kind == NX_OP_ATTN_DECODE && decode_bw > 0;
    nx_op_latency& o = out.per_op[i];
    o.kind = w.kind;
    o.compute_s = compute_latency(w.flops, share, curve_of(p, w.kind), g.peak_compute);
    double bw = contended ? decode_bw : g.peak_bandwidth;
    if (use_ext) {
      const double sat = ext->bw_sat[w.kind];
      if (sat > 0 && share < sat) bw = bw * (share / sat);  // SM-share-limited HBM bandwidth
    }
    o.mem_s = w.mem_bytes / bw;
    o.memory_bound = o.mem_s > o.compute_s ? 1 : 0;
    const double t = o.compute_s < o.mem_s ? o.mem_s : o.compute_s;  // std::max order
    out.total_s += t;
    if (w.is_attention && o.memory_bound) out.attn_mem_time_s += t;
  }
  return out;
}

// B_decode (costmodel.cpp:56-64).
double effective_decode_bw(double p_attn, double m_d, double m_p1, double m_p2, double peak) {
  if (!(m_d > 0)) throw InvalidArg("effective_decode_bandwidth: m_d must be > 0");
  if (m_p1 < 0 || m_p2 < 0)
    throw InvalidArg("effective_decode_bandwidth: m_p1/m_p2 must be >= 0");
  const double share_attn = m_d / (m_d + m_p1);
  const double share_dense = m_d / (m_d + m_p2);
  return share_attn * p_attn * peak + share_dense * (1.0 - p_attn) * peak;
}

// decode_latency_contended (costmodel.cpp:66-96): only the decode attention
// operator sees the contended bandwidth; P_attn comes from the in-flight
// prefill breakdown.
nx_breakdown decode_contended(const OpList& dec, double share, const nx_breakdown* pre_bd,
                              const OpList& pre, const nx_gpu_spec& g,
                              const nx_kernel_profile& p, const nx_cost_ext* ext) {
  if (pre_bd == nullptr) return isolated(dec, share, g, p, ext);
  if (ext != nullptr && ext->enabled != 0 && ext->contention != 0) {
    // measured co-location slowdown vs the prefill lane's share (flagged ext)
    nx_breakdown b = isolated(dec, share, g, p, ext);
    const double pp = 1.0 - share;
    const double f = ext->contention_c[0] + ext->contention_c[1] * pp + ext->contention_c[2] * pp * pp;
    for (int i = 0; i < b.n_ops; ++i) {
      b.per_op[i].compute_s *= f;
      b.per_op[i].mem_s *= f;
    }
    b.total_s *= f;
    b.attn_mem_time_s *= f;
    return b;
  }
  const double p_attn = pre_bd->total_s <= 0 ? 0.0 : pre_bd->attn_mem_time_s / pre_bd->total_s;
  double m_p1 = 0, m_p2 = 0, m_d = 0;
  for (int i = 0; i < pre.n; ++i) {
    if (pre.op[i].is_attention)
      m_p1 += pre.op[i].kv_bytes;
    else
      m_p2 += pre.op[i].mem_bytes;
  }
  for (int i = 0; i < dec.n; ++i)
    if (dec.op[i].kind == NX_OP_ATTN_DECODE) m_d += dec.op[i].kv_bytes;
  const double bw = m_d > 0 ? effective_decode_bw(p_attn, m_d, m_p1, m_p2, g.peak_bandwidth)
                            : g.peak_bandwidth;
  return breakdown(dec, share, g, p, bw, ext);
}

}  // namespace nxb

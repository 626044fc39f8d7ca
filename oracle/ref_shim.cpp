// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the *unmodified* reference library (nexussim core,
// compiled from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libnexussim_ref.so). It lets pytest (ctypes) drive the
// reference with the same POD structs the product's C-ABI uses
// (include/nexus_b200.h), so parity tests compare like with like.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs load this library.

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <unistd.h>
#include <vector>

#include "nexus_b200.h"
#include "nexussim/costmodel.hpp"
#include "nexussim/domain.hpp"
#include "nexussim/eventlog.hpp"
#include "nexussim/metrics.hpp"
#include "nexussim/opcost.hpp"
#include "nexussim/optimizer.hpp"
#include "nexussim/presets.hpp"
#include "nexussim/schedulers.hpp"
#include "nexussim/simulator.hpp"
#include "nexussim/workload.hpp"

using namespace nexus;

namespace {

thread_local std::string g_err;

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

ModelConfig to_ref(const nx_model_config& m) {
  ModelConfig r;
  r.hidden_dim = m.hidden_dim;
  r.ffn_dim = m.ffn_dim;
  r.num_layers = m.num_layers;
  r.num_heads = m.num_heads;
  r.element_bytes = m.element_bytes;
  r.kv_bytes_per_token = m.kv_bytes_per_token;
  r.weight_bytes_per_layer_dense = m.weight_bytes_per_layer_dense;
  r.weight_bytes_per_layer_attn = m.weight_bytes_per_layer_attn;
  return r;
}

GpuSpec to_ref(const nx_gpu_spec& g) {
  return GpuSpec{g.total_sm, g.peak_compute, g.peak_bandwidth, g.kv_capacity_bytes};
}

KernelProfile to_ref(const nx_kernel_profile& p) {
  KernelProfile r;
  r.qkv_proj = {p.qkv_proj.r_sat, p.qkv_proj.lambda};
  r.attn_prefill = {p.attn_prefill.r_sat, p.attn_prefill.lambda};
  r.attn_decode = {p.attn_decode.r_sat, p.attn_decode.lambda};
  r.attn_out_proj = {p.attn_out_proj.r_sat, p.attn_out_proj.lambda};
  r.ffn = {p.ffn.r_sat, p.ffn.lambda};
  return r;
}

ControllerConfig to_ref(const nx_controller_config& c) {
  ControllerConfig r;
  r.alpha = c.alpha;
  r.beta = c.beta;
  r.kv_switch_fraction = c.kv_switch_fraction;
  r.delta_pp = c.delta_pp;
  r.gamma = c.gamma;
  r.chunk_size = c.chunk_size;
  r.max_decode_batch = c.max_decode_batch;
  r.token_budget = c.token_budget;
  return r;
}

std::vector<OperatorWorkload> to_ref(const nx_op_workload* ops, size_t n) {
  std::vector<OperatorWorkload> v;
  for (size_t i = 0; i < n; ++i)
    v.push_back({static_cast<OperatorKind>(ops[i].kind), ops[i].flops, ops[i].mem_bytes,
                 ops[i].kv_bytes, ops[i].is_attention != 0});
  return v;
}

void from_ref(const std::vector<OperatorWorkload>& v, nx_op_workload* out, size_t* n) {
  for (size_t i = 0; i < v.size(); ++i) {
    out[i].kind = static_cast<int32_t>(v[i].kind);
    out[i].is_attention = v[i].is_attention ? 1 : 0;
    out[i].flops = v[i].flops;
    out[i].mem_bytes = v[i].mem_bytes;
    out[i].kv_bytes = v[i].kv_bytes;
  }
  *n = v.size();
}

void from_ref(const PhaseLatencyBreakdown& b, nx_breakdown* out) {
  std::memset(out, 0, sizeof(*out));
  out->total_s = b.total_s;
  out->attn_mem_time_s = b.attn_mem_time_s;
  out->n_ops = static_cast<int32_t>(b.per_op.size());
  for (size_t i = 0; i < b.per_op.size() && i < NX_MAX_OPS; ++i) {
    out->per_op[i].kind = static_cast<int32_t>(b.per_op[i].kind);
    out->per_op[i].memory_bound = b.per_op[i].memory_bound ? 1 : 0;
    out->per_op[i].compute_s = b.per_op[i].compute_s;
    out->per_op[i].mem_s = b.per_op[i].mem_s;
  }
}

PhaseLatencyBreakdown to_ref(const nx_breakdown& b) {
  PhaseLatencyBreakdown r;
  r.total_s = b.total_s;
  r.attn_mem_time_s = b.attn_mem_time_s;
  for (int i = 0; i < b.n_ops; ++i)
    r.per_op.push_back({static_cast<OperatorKind>(b.per_op[i].kind), b.per_op[i].compute_s,
                        b.per_op[i].mem_s, b.per_op[i].memory_bound != 0});
  return r;
}

void write_plan(const BatchPlan& p, nx_batch_member* out, size_t cap, size_t* n_out,
                int64_t* total) {
  size_t k = 0;
  for (const BatchMember& m : p.members) {
    if (k < cap) out[k] = {m.id, m.tokens};
    ++k;
  }
  *n_out = k;
  *total = p.total_tokens;
}

PhaseModel wrap(const nx_phase_model* m) {
  PhaseModel pm;
  pm.active = m->active != 0;
  const nx_phase_model copy = *m;
  pm.latency_at = [copy](int pct) { return copy.latency_at(copy.user, pct); };
  return pm;
}

std::string temp_path(const char* tag) {
  char buf[256];
  std::snprintf(buf, sizeof(buf), "/tmp/nxref_%s_%d_%p", tag, static_cast<int>(getpid()),
                static_cast<void*>(&buf));
  return buf;
}

}  // namespace

#define REF_TRY try {
#define REF_CATCH                   \
  }                                 \
  catch (const std::exception& e) { \
    g_err = e.what();               \
    return NX_EINVAL;               \
  }

extern "C" {

const char* nxref_last_error(void) { return g_err.c_str(); }
void nxref_free(void* p) { std::free(p); }

nx_model_config nxref_model_derive(int64_t d, int64_t dff, int32_t L, int32_t H, int32_t e) {
  ModelConfig m = ModelConfig::derive(d, dff, L, H, e);
  nx_model_config o{};
  o.hidden_dim = m.hidden_dim;
  o.ffn_dim = m.ffn_dim;
  o.num_layers = m.num_layers;
  o.num_heads = m.num_heads;
  o.element_bytes = m.element_bytes;
  o.kv_bytes_per_token = m.kv_bytes_per_token;
  o.weight_bytes_per_layer_dense = m.weight_bytes_per_layer_dense;
  o.weight_bytes_per_layer_attn = m.weight_bytes_per_layer_attn;
  return o;
}

// Reference default-constructed ControllerConfig / KernelProfile / EngineConfig
// (domain.hpp:45-89, simulator.hpp:36-45), so a caller can build a SimConfig
// without the product library.
void nxref_defaults(nx_controller_config* c, nx_kernel_profile* p, nx_engine_config* e) {
  const ControllerConfig rc{};
  std::memset(c, 0, sizeof(*c));
  c->alpha = rc.alpha;
  c->beta = rc.beta;
  c->kv_switch_fraction = rc.kv_switch_fraction;
  c->delta_pp = rc.delta_pp;
  c->gamma = rc.gamma;
  c->chunk_size = rc.chunk_size;
  c->max_decode_batch = rc.max_decode_batch;
  c->token_budget = rc.token_budget;
  const KernelProfile rp{};
  auto put = [](nx_saturation_curve& d, const SaturationCurve& s) {
    d.r_sat = s.r_sat;
    d.lambda = s.lambda;
  };
  put(p->qkv_proj, rp.qkv_proj);
  put(p->attn_prefill, rp.attn_prefill);
  put(p->attn_decode, rp.attn_decode);
  put(p->attn_out_proj, rp.attn_out_proj);
  put(p->ffn, rp.ffn);
  const EngineConfig re{};
  std::memset(e, 0, sizeof(*e));
  e->kind = NX_ENGINE_NEXUS;
  e->static_r_p = re.static_r_p;
  e->prefill_policy = re.prefill_policy == PrefillPolicy::Fcfs ? NX_PREFILL_FCFS : NX_PREFILL_SPF;
  e->clock_mode = NX_CLOCK_VIRTUAL;
  e->timeout_sim_s = re.timeout_sim_s;
  e->max_events = re.max_events;
}

int nxref_model_preset(const char* name, nx_model_config* out) {
  auto m = model_preset(name);
  if (!m) return NX_EINVAL;
  *out = nxref_model_derive(m->hidden_dim, m->ffn_dim, m->num_layers, m->num_heads,
                            m->element_bytes);
  return NX_OK;
}

int nxref_gpu_preset(const char* name, nx_gpu_spec* out) {
  auto g = gpu_preset(name);
  if (!g) return NX_EINVAL;
  std::memset(out, 0, sizeof(*out));
  out->total_sm = g->total_sm;
  out->peak_compute = g->peak_compute;
  out->peak_bandwidth = g->peak_bandwidth;
  out->kv_capacity_bytes = g->kv_capacity_bytes;
  return NX_OK;
}

int nxref_validate_config(const nx_model_config* m, const nx_gpu_spec* g,
                          const nx_controller_config* c, const nx_kernel_profile* p, char* msg,
                          size_t cap) {
  auto errs = validate_config(to_ref(*m), to_ref(*g), to_ref(*c), to_ref(*p));
  std::string s = describe(errs);
  if (msg && cap) {
    std::snprintf(msg, cap, "%s", s.c_str());
  }
  return static_cast<int>(errs.size());
}

int nxref_prefill_batch_workloads(const nx_model_config* m, const int64_t* tok,
                                  const int64_t* ctx, size_t n, nx_op_workload* out,
                                  size_t* n_ops) {
  REF_TRY
  std::vector<PrefillChunk> ch;
  for (size_t i = 0; i < n; ++i) ch.push_back({tok[i], ctx[i]});
  from_ref(prefill_batch_workloads(to_ref(*m), ch), out, n_ops);
  return NX_OK;
  REF_CATCH
}

int nxref_decode_op_workloads(const nx_model_config* m, const int64_t* ctx, size_t n,
                              nx_op_workload* out, size_t* n_ops) {
  REF_TRY
  std::vector<long> v(ctx, ctx + n);
  from_ref(decode_op_workloads(to_ref(*m), v), out, n_ops);
  return NX_OK;
  REF_CATCH
}

int nxref_mixed_batch_workloads(const nx_model_config* m, const int64_t* tok, const int64_t* ctx,
                                size_t n, const int64_t* dctx, size_t nd, nx_op_workload* out,
                                size_t* n_ops) {
  REF_TRY
  std::vector<PrefillChunk> ch;
  for (size_t i = 0; i < n; ++i) ch.push_back({tok[i], ctx[i]});
  std::vector<long> v(dctx, dctx + nd);
  from_ref(mixed_batch_workloads(to_ref(*m), ch, v), out, n_ops);
  return NX_OK;
  REF_CATCH
}

int nxref_compute_latency(double flops, double share, nx_saturation_curve c, double peak,
                          double* out) {
  REF_TRY
  *out = compute_latency(flops, share, SaturationCurve{c.r_sat, c.lambda}, peak);
  return NX_OK;
  REF_CATCH
}

int nxref_phase_latency_isolated(const nx_op_workload* ops, size_t n, double share,
                                 const nx_gpu_spec* g, const nx_kernel_profile* p,
                                 nx_breakdown* out) {
  REF_TRY
  from_ref(phase_latency_isolated(to_ref(ops, n), share, to_ref(*g), to_ref(*p)), out);
  return NX_OK;
  REF_CATCH
}

int nxref_effective_decode_bandwidth(double p_attn, double m_d, double m_p1, double m_p2,
                                     double peak, double* out) {
  REF_TRY
  ContentionContext c;
  c.p_attn = p_attn;
  c.m_d = m_d;
  c.m_p1 = m_p1;
  c.m_p2 = m_p2;
  *out = effective_decode_bandwidth(c, peak);
  return NX_OK;
  REF_CATCH
}

int nxref_decode_latency_contended(const nx_op_workload* dops, size_t nd, double share,
                                   const nx_breakdown* pbd, const nx_op_workload* pops,
                                   size_t np, const nx_gpu_spec* g, const nx_kernel_profile* p,
                                   nx_breakdown* out) {
  REF_TRY
  PhaseLatencyBreakdown bd;
  if (pbd) bd = to_ref(*pbd);
  from_ref(decode_latency_contended(to_ref(dops, nd), share, pbd ? &bd : nullptr,
                                    to_ref(pops, np), to_ref(*g), to_ref(*p)),
           out);
  return NX_OK;
  REF_CATCH
}

double nxref_min_phase_latency(const nx_op_workload* ops, size_t n, const nx_gpu_spec* g,
                               const nx_kernel_profile* p) {
  return min_phase_latency(to_ref(ops, n), to_ref(*g), to_ref(*p));
}

int nxref_select_mode(int64_t used, int64_t cap, double frac) {
  try {
    return select_mode(used, cap, frac) == ObjectiveMode::DecodePrioritized ? NX_MODE_DECODE
                                                                            : NX_MODE_PREFILL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int nxref_adjust_partition(int32_t target, const nx_partition_state* cur,
                           const nx_phase_model* pre, const nx_phase_model* dec,
                           const nx_controller_config* cfg, nx_adjust_outcome* out) {
  REF_TRY
  PartitionState s{cur->r_p, cur->r_d, cur->last_applied_r_p};
  AdjustOutcome o = adjust_partition(target == NX_PHASE_PREFILL ? Phase::Prefill : Phase::Decode,
                                     s, wrap(pre), wrap(dec), to_ref(*cfg));
  out->r_p = o.r_p;
  out->r_d = o.r_d;
  out->infeasible = o.infeasible ? 1 : 0;
  out->queries = o.queries;
  return NX_OK;
  REF_CATCH
}

struct nxref_controller {
  PartitionController pc;
};

int nxref_controller_create(const nx_partition_state* init, const nx_controller_config* cfg,
                            nxref_controller** out) {
  *out = new nxref_controller{
      PartitionController(PartitionState{init->r_p, init->r_d, init->last_applied_r_p},
                          to_ref(*cfg))};
  return NX_OK;
}

void nxref_controller_destroy(nxref_controller* c) { delete c; }

int nxref_controller_decide(nxref_controller* c, int64_t used, int64_t cap,
                            const nx_phase_model* pre, const nx_phase_model* dec,
                            nx_decision* out) {
  REF_TRY
  PartitionDecision d = c->pc.decide(used, cap, wrap(pre), wrap(dec));
  std::memset(out, 0, sizeof(*out));
  out->r_p = d.r_p;
  out->r_d = d.r_d;
  out->mode = d.mode == ObjectiveMode::DecodePrioritized ? NX_MODE_DECODE : NX_MODE_PREFILL;
  out->switched = d.switched ? 1 : 0;
  out->infeasible = d.infeasible ? 1 : 0;
  out->candidate_r_p = d.candidate_r_p;
  out->iterations_searched = d.iterations_searched;
  return NX_OK;
  REF_CATCH
}

int nxref_spf_schedule(const nx_prefill_entry* q, size_t n, int64_t budget, double gamma,
                       double now, int32_t skip, nx_batch_member* out, size_t cap, size_t* n_out,
                       int64_t* total) {
  REF_TRY
  std::vector<PrefillQueueEntry> v;
  for (size_t i = 0; i < n; ++i) v.push_back({q[i].id, q[i].remaining, q[i].arrival_s});
  write_plan(spf_schedule(v, budget, gamma, now, skip != 0), out, cap, n_out, total);
  return NX_OK;
  REF_CATCH
}

int nxref_fcfs_prefill_schedule(const nx_prefill_entry* q, size_t n, int64_t budget,
                                nx_batch_member* out, size_t cap, size_t* n_out, int64_t* total) {
  REF_TRY
  std::vector<PrefillQueueEntry> v;
  for (size_t i = 0; i < n; ++i) v.push_back({q[i].id, q[i].remaining, q[i].arrival_s});
  write_plan(fcfs_prefill_schedule(v, budget), out, cap, n_out, total);
  return NX_OK;
  REF_CATCH
}

int nxref_fcfs_decode_schedule(const nx_decode_candidate* a, size_t n, int32_t maxb,
                               nx_batch_member* out, size_t cap, size_t* n_out, int64_t* total) {
  REF_TRY
  std::vector<DecodeCandidate> v;
  for (size_t i = 0; i < n; ++i) v.push_back({a[i].id, a[i].arrival_s});
  write_plan(fcfs_decode_schedule(v, maxb), out, cap, n_out, total);
  return NX_OK;
  REF_CATCH
}

int nxref_chunked_mixed_schedule(const nx_prefill_entry* q, size_t nq,
                                 const nx_decode_candidate* a, size_t na, int64_t budget,
                                 int32_t maxb, int64_t chunk, nx_batch_member* out, size_t cap,
                                 size_t* n_out, int64_t* total) {
  REF_TRY
  std::vector<PrefillQueueEntry> v;
  for (size_t i = 0; i < nq; ++i) v.push_back({q[i].id, q[i].remaining, q[i].arrival_s});
  std::vector<DecodeCandidate> d;
  for (size_t i = 0; i < na; ++i) d.push_back({a[i].id, a[i].arrival_s});
  write_plan(chunked_mixed_schedule(v, d, budget, maxb, chunk), out, cap, n_out, total);
  return NX_OK;
  REF_CATCH
}

int nxref_workload_preset_trace(const char* name, double rate, int64_t count, uint64_t seed,
                                nx_request* out, size_t cap, size_t* n_out) {
  REF_TRY
  auto p = workload_preset(name, rate, count, seed);
  if (!p) {
    g_err = "unknown workload preset";
    return NX_EINVAL;
  }
  auto tr = realize(*p);
  size_t k = 0;
  for (const Request& r : tr) {
    if (k < cap) out[k] = {r.id, r.arrival_s, r.prompt_len, r.output_len};
    ++k;
  }
  *n_out = k;
  return NX_OK;
  REF_CATCH
}

// save_trace -> text, through a temp file (the reference only writes files).
int nxref_trace_text(const nx_request* t, size_t n, char** text) {
  REF_TRY
  std::vector<Request> tr;
  for (size_t i = 0; i < n; ++i) {
    Request r;
    r.id = t[i].id;
    r.arrival_s = t[i].arrival_s;
    r.prompt_len = t[i].prompt_len;
    r.output_len = t[i].output_len;
    tr.push_back(r);
  }
  const std::string path = temp_path("trace");
  save_trace(path, tr);
  std::ifstream in(path);
  std::stringstream ss;
  ss << in.rdbuf();
  std::remove(path.c_str());
  *text = dup_string(ss.str());
  return NX_OK;
  REF_CATCH
}

int nxref_kernel_profile_text(const nx_kernel_profile* p, char** text) {
  *text = dup_string(kernel_profile_text(to_ref(*p)));
  return NX_OK;
}

int nxref_kernel_profile_load_text(const char* text, nx_kernel_profile* out, char** warnings) {
  const std::string path = temp_path("prof");
  {
    std::ofstream f(path);
    f << text;
  }
  try {
    std::vector<std::string> w;
    KernelProfile p = load_kernel_profile(path, &w);
    std::remove(path.c_str());
    auto put = [](nx_saturation_curve& d, const SaturationCurve& s) {
      d.r_sat = s.r_sat;
      d.lambda = s.lambda;
    };
    put(out->qkv_proj, p.qkv_proj);
    put(out->attn_prefill, p.attn_prefill);
    put(out->attn_decode, p.attn_decode);
    put(out->attn_out_proj, p.attn_out_proj);
    put(out->ffn, p.ffn);
    std::string all;
    for (auto& s : w) all += s + "\n";
    *warnings = dup_string(all);
    return NX_OK;
  } catch (const std::exception& e) {
    std::remove(path.c_str());
    g_err = e.what();
    return NX_ERUNTIME;
  }
}

// nexus::run (simulator.cpp:760) with the three intra-GPU engines.
int nxref_run(const nx_sim_config* cfg, const nx_request* t, size_t n, char** events,
              char** decisions, char** summary, double* sim_end_s, int32_t* timed_out) {
  REF_TRY
  SimConfig sc;
  sc.model = to_ref(cfg->model);
  sc.gpu = to_ref(cfg->gpu);
  sc.ctrl = to_ref(cfg->ctrl);
  sc.profile = to_ref(cfg->profile);
  switch (cfg->engine.kind) {
    case NX_ENGINE_NEXUS: sc.engine.kind = EngineKind::NexusDisagg; break;
    case NX_ENGINE_MONOLITHIC: sc.engine.kind = EngineKind::MonolithicChunked; break;
    case NX_ENGINE_STATIC: sc.engine.kind = EngineKind::StaticPartition; break;
    default: g_err = "unsupported engine kind"; return NX_EINVAL;
  }
  sc.engine.static_r_p = cfg->engine.static_r_p;
  sc.engine.prefill_policy =
      cfg->engine.prefill_policy == NX_PREFILL_FCFS ? PrefillPolicy::Fcfs : PrefillPolicy::Spf;
  sc.engine.timeout_sim_s = cfg->engine.timeout_sim_s;
  sc.engine.max_events = cfg->engine.max_events;
  std::vector<Request> tr;
  for (size_t i = 0; i < n; ++i) {
    Request r;
    r.id = t[i].id;
    r.arrival_s = t[i].arrival_s;
    r.prompt_len = t[i].prompt_len;
    r.output_len = t[i].output_len;
    tr.push_back(r);
  }
  SimResult res = nexus::run(sc, tr);
  if (events) *events = dup_string(serialize_event_log(res.events));
  if (decisions) *decisions = dup_string(decision_log_text(res.decisions));
  if (summary)
    *summary = dup_string(res.metrics.completed ? summary_json(res.metrics, to_string(sc.engine.kind))
                                                : std::string());
  if (sim_end_s) *sim_end_s = res.sim_end_s;
  if (timed_out) *timed_out = res.timed_out ? 1 : 0;
  return NX_OK;
  REF_CATCH
}

// replay_report over an event log text (eventlog.cpp:147-193) -> summary JSON.
int nxref_replay_summary(const char* log_text, const char* label, char** summary) {
  const std::string path = temp_path("events");
  {
    std::ofstream f(path);
    f << log_text;
  }
  try {
    auto ev = read_event_log(path);
    std::remove(path.c_str());
    *summary = dup_string(summary_json(replay_report(ev), label));
    return NX_OK;
  } catch (const std::exception& e) {
    std::remove(path.c_str());
    g_err = e.what();
    return NX_ERUNTIME;
  }
}

}  // extern "C"

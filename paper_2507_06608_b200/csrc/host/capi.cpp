// extern "C" boundary (include/nexus_b200.h). Every entry point converts
// exceptions into status codes + a thread-local message; nothing throws
// across the ABI.
#include <cstring>
#include <string>

#include "capi_internal.hpp"
#include "core.hpp"
#include "engine.hpp"

using namespace nxb;

namespace nxb {
std::string& last_error() {
  thread_local std::string s;
  return s;
}
}  // namespace nxb

namespace {
#define g_last_error (::nxb::last_error())

int fail(int code, const char* what) {
  g_last_error = what;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    g_last_error.clear();
    return f();
  } catch (const InvalidArg& e) {
    return fail(NX_EINVAL, e.what());
  } catch (const RuntimeErr& e) {
    return fail(NX_ERUNTIME, e.what());
  } catch (const std::bad_alloc&) {
    return fail(NX_ENOMEM, "out of memory");
  } catch (const std::out_of_range& e) {
    return fail(NX_EINVAL, e.what());
  } catch (const std::exception& e) {
    return fail(NX_ERUNTIME, e.what());
  }
}

// Copies text into a caller buffer. buf == NULL is a size query.
int put_text(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (!buf) return NX_OK;
  if (cap == 0) return fail(NX_EINVAL, "buffer too small");
  const size_t n = std::min(s.size(), cap - 1);
  std::memcpy(buf, s.data(), n);
  buf[n] = '\0';
  return s.size() < cap ? NX_OK : fail(NX_EINVAL, "buffer too small");
}

int put_ops(const OpList& ops, nx_op_workload* out, size_t* n) {
  for (int i = 0; i < ops.n; ++i) out[i] = ops.op[i];
  *n = static_cast<size_t>(ops.n);
  return NX_OK;
}

OpList to_ops(const nx_op_workload* ops, size_t n) {
  if (n > NX_MAX_OPS) throw InvalidArg("too many operators");
  OpList l;
  for (size_t i = 0; i < n; ++i) l.op[l.n++] = ops[i];
  return l;
}

std::vector<Chunk> to_chunks(const int64_t* tok, const int64_t* ctx, size_t n) {
  std::vector<Chunk> c(n);
  for (size_t i = 0; i < n; ++i) c[i] = {tok[i], ctx[i]};
  return c;
}

int put_plan(const Plan& p, nx_batch_member* out, size_t cap, size_t* n_out, int64_t* total) {
  for (size_t i = 0; i < p.members.size() && i < cap; ++i) out[i] = p.members[i];
  *n_out = p.members.size();
  *total = p.total;
  return p.members.size() <= cap ? NX_OK : fail(NX_EINVAL, "member buffer too small");
}

}  // namespace

struct nx_controller {
  Controller c;
};

namespace {
thread_local nx_cost_ext g_ext{};
}

extern "C" {

const char* nx_last_error(void) { return g_last_error.c_str(); }
const char* nx_version(void) { return "nexus_b200 0.1 sm_100a"; }
size_t nx_sim_config_size(void) { return sizeof(nx_sim_config); }

nx_model_config nx_model_derive(int64_t d, int64_t dff, int32_t L, int32_t H, int32_t e) {
  return derive_model(d, dff, L, H, e);
}

nx_controller_config nx_controller_config_default(void) {
  nx_controller_config c{};
  c.alpha = 1.3;
  c.beta = 1.1;
  c.kv_switch_fraction = 0.7;
  c.gamma = 15.0;
  c.delta_pp = 5;
  c.max_decode_batch = 64;
  c.chunk_size = 2048;
  c.token_budget = 2048;
  return c;
}

nx_kernel_profile nx_kernel_profile_default(void) {
  nx_kernel_profile p{};
  p.qkv_proj = {0.6, 0.1};
  p.attn_prefill = {0.4, 0.05};
  p.attn_decode = {0.4, 0.05};
  p.attn_out_proj = {0.6, 0.1};
  p.ffn = {0.6, 0.1};
  return p;
}

nx_engine_config nx_engine_config_default(void) {
  nx_engine_config e{};
  e.kind = NX_ENGINE_NEXUS;
  e.static_r_p = 50;
  e.prefill_policy = NX_PREFILL_SPF;
  e.clock_mode = NX_CLOCK_VIRTUAL;
  e.timeout_sim_s = 3600.0;
  e.max_events = 10000000ULL;
  return e;
}

int nx_validate_config(const nx_model_config* m, const nx_gpu_spec* g,
                       const nx_controller_config* c, const nx_kernel_profile* p, char* msg,
                       size_t cap) {
  int n = 0;
  const std::string s = validate(*m, *g, *c, *p, &n);
  if (msg && cap) put_text(s, msg, cap, nullptr);
  return n;
}

int nx_prefill_batch_workloads(const nx_model_config* m, const int64_t* tok, const int64_t* ctx,
                               size_t n, nx_op_workload* out, size_t* n_ops) {
  return guarded([&] {
    const auto ch = to_chunks(tok, ctx, n);
    return put_ops(prefill_ops(*m, ch.data(), n), out, n_ops);
  });
}

int nx_decode_op_workloads(const nx_model_config* m, const int64_t* ctx, size_t n,
                           nx_op_workload* out, size_t* n_ops) {
  return guarded([&] { return put_ops(decode_ops(*m, ctx, n), out, n_ops); });
}

int nx_mixed_batch_workloads(const nx_model_config* m, const int64_t* tok, const int64_t* ctx,
                             size_t n, const int64_t* dctx, size_t nd, nx_op_workload* out,
                             size_t* n_ops) {
  return guarded([&] {
    const auto ch = to_chunks(tok, ctx, n);
    return put_ops(mixed_ops(*m, ch.data(), n, dctx, nd), out, n_ops);
  });
}

int nx_compute_latency(double flops, double share, nx_saturation_curve c, double peak,
                       double* out) {
  return guarded([&] {
    *out = compute_latency(flops, share, c, peak);
    return NX_OK;
  });
}

int nx_phase_latency_isolated(const nx_op_workload* ops, size_t n, double share,
                              const nx_gpu_spec* g, const nx_kernel_profile* p,
                              nx_breakdown* out) {
  return guarded([&] {
    *out = isolated(to_ops(ops, n), share, *g, *p, &g_ext);
    return NX_OK;
  });
}

int nx_effective_decode_bandwidth(double p_attn, double m_d, double m_p1, double m_p2,
                                  double peak, double* out) {
  return guarded([&] {
    *out = effective_decode_bw(p_attn, m_d, m_p1, m_p2, peak);
    return NX_OK;
  });
}

int nx_decode_latency_contended(const nx_op_workload* dops, size_t nd, double share,
                                const nx_breakdown* pbd, const nx_op_workload* pops, size_t np,
                                const nx_gpu_spec* g, const nx_kernel_profile* p,
                                nx_breakdown* out) {
  return guarded([&] {
    *out = decode_contended(to_ops(dops, nd), share, pbd, to_ops(pops, np), *g, *p, &g_ext);
    return NX_OK;
  });
}

int nx_set_cost_ext(const nx_cost_ext* ext) {
  if (ext) {
    for (double s : ext->bw_sat)
      if (ext->enabled && !(s > 0.0 && s <= 1.0)) return fail(NX_EINVAL, "bw_sat must lie in (0, 1]");
    g_ext = *ext;
  } else {
    g_ext = nx_cost_ext{};
  }
  return NX_OK;
}

double nx_min_phase_latency(const nx_op_workload* ops, size_t n, const nx_gpu_spec* g,
                            const nx_kernel_profile* p) {
  if (n == 0) return 0.0;  // a vacuous phase imposes no constraint
  try {
    return isolated(to_ops(ops, n), 1.0, *g, *p, &g_ext).total_s;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return -1.0;
  }
}

int nx_select_mode(int64_t used, int64_t cap, double frac) {
  try {
    return select_mode(used, cap, frac);
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return -1;
  }
}

int nx_adjust_partition(int32_t target, const nx_partition_state* cur, const nx_phase_model* pre,
                        const nx_phase_model* dec, const nx_controller_config* cfg,
                        nx_adjust_outcome* out) {
  return guarded([&] {
    *out = adjust(target, *cur, *pre, *dec, *cfg);
    return NX_OK;
  });
}

int nx_controller_create(const nx_partition_state* init, const nx_controller_config* cfg,
                         nx_controller** out) {
  return guarded([&] {
    *out = new nx_controller{Controller(*init, *cfg)};
    return NX_OK;
  });
}

void nx_controller_destroy(nx_controller* c) { delete c; }

int nx_controller_decide(nx_controller* c, int64_t used, int64_t cap, const nx_phase_model* pre,
                         const nx_phase_model* dec, nx_decision* out) {
  return guarded([&] {
    *out = c->c.decide(used, cap, *pre, *dec);
    return NX_OK;
  });
}

int nx_controller_state(const nx_controller* c, nx_partition_state* out) {
  *out = c->c.state();
  return NX_OK;
}

int nx_spf_schedule(const nx_prefill_entry* q, size_t n, int64_t budget, double gamma, double now,
                    int32_t skip, nx_batch_member* out, size_t cap, size_t* n_out,
                    int64_t* total) {
  return guarded([&] {
    return put_plan(spf(std::vector<nx_prefill_entry>(q, q + n), budget, gamma, now, skip != 0),
                    out, cap, n_out, total);
  });
}

int nx_fcfs_prefill_schedule(const nx_prefill_entry* q, size_t n, int64_t budget,
                             nx_batch_member* out, size_t cap, size_t* n_out, int64_t* total) {
  return guarded([&] {
    return put_plan(fcfs_prefill(std::vector<nx_prefill_entry>(q, q + n), budget), out, cap,
                    n_out, total);
  });
}

int nx_fcfs_decode_schedule(const nx_decode_candidate* a, size_t n, int32_t max_batch,
                            nx_batch_member* out, size_t cap, size_t* n_out, int64_t* total) {
  return guarded([&] {
    return put_plan(fcfs_decode(std::vector<nx_decode_candidate>(a, a + n), max_batch), out, cap,
                    n_out, total);
  });
}

int nx_chunked_mixed_schedule(const nx_prefill_entry* q, size_t nq, const nx_decode_candidate* a,
                              size_t na, int64_t budget, int32_t max_batch, int64_t chunk,
                              nx_batch_member* out, size_t cap, size_t* n_out, int64_t* total) {
  return guarded([&] {
    return put_plan(chunked_mixed(std::vector<nx_prefill_entry>(q, q + nq),
                                  std::vector<nx_decode_candidate>(a, a + na), budget, max_batch,
                                  chunk),
                    out, cap, n_out, total);
  });
}

int nx_workload_preset_trace(const char* preset, double rate, int64_t count, uint64_t seed,
                             nx_request* out, size_t cap, size_t* n_out) {
  return guarded([&] {
    const auto t = preset_trace(preset, rate, count, seed);
    for (size_t i = 0; i < t.size() && i < cap; ++i) out[i] = t[i];
    *n_out = t.size();
    return NX_OK;
  });
}

int nx_trace_to_text(const nx_request* t, size_t n, char* buf, size_t cap, size_t* len) {
  return guarded([&] { return put_text(trace_text(t, n), buf, cap, len); });
}

int nx_trace_from_text(const char* text, nx_request* out, size_t cap, size_t* n_out) {
  return guarded([&] {
    const auto t = parse_trace(text);
    for (size_t i = 0; i < t.size() && i < cap; ++i) out[i] = t[i];
    *n_out = t.size();
    return NX_OK;
  });
}

int nx_kernel_profile_to_text(const nx_kernel_profile* p, char* buf, size_t cap, size_t* len) {
  return guarded([&] { return put_text(profile_text(*p), buf, cap, len); });
}

int nx_kernel_profile_from_text(const char* text, nx_kernel_profile* out, char* warnings,
                                size_t warn_cap) {
  return guarded([&] {
    std::string w;
    *out = parse_profile(text, &w);
    if (warnings && warn_cap) put_text(w, warnings, warn_cap, nullptr);
    return NX_OK;
  });
}

// ---- engine ----------------------------------------------------------------

int nx_engine_create(const nx_sim_config* cfg, nx_engine** out) {
  return guarded([&] {
    *out = new nx_engine(*cfg);
    return NX_OK;
  });
}

void nx_engine_destroy(nx_engine* eng) { delete eng; }

const char* nx_engine_last_error(const nx_engine* eng) { return eng->err.c_str(); }

#define ENGINE_CALL(eng, body)     \
  do {                             \
    const int rc_ = guarded(body); \
    if (rc_ != NX_OK && rc_ != NX_EDONE && rc_ != NX_EAGAIN) (eng)->err = g_last_error; \
    return rc_;                    \
  } while (0)

int nx_submit(nx_engine* eng, const nx_request* r) {
  ENGINE_CALL(eng, [&] {
    eng->e.submit(*r, nullptr);
    return NX_OK;
  });
}

int nx_submit_trace(nx_engine* eng, const nx_request* r, size_t n) {
  ENGINE_CALL(eng, [&] {
    for (size_t i = 0; i < n; ++i) eng->e.submit(r[i], nullptr);
    return NX_OK;
  });
}

int nx_submit_with_tokens(nx_engine* eng, const nx_request* r, const int32_t* tokens) {
  ENGINE_CALL(eng, [&] {
    eng->e.submit(*r, tokens);
    return NX_OK;
  });
}

int nx_step(nx_engine* eng) {
  ENGINE_CALL(eng, [&] { return eng->e.step(); });
}

int nx_run(nx_engine* eng) {
  ENGINE_CALL(eng, [&] { return eng->e.run(); });
}

int nx_engine_set_replay_latencies(nx_engine* eng, const double* lat, size_t n) {
  eng->e.set_replay(lat, n);
  return NX_OK;
}

int nx_engine_set_logging(nx_engine* eng, int32_t events, int32_t pages) {
  eng->e.set_logging(events != 0, pages != 0);
  return NX_OK;
}

int nx_engine_set_slo(nx_engine* eng, double ttft_s, double tbt_s) {
  eng->e.set_slo(ttft_s, tbt_s);
  return NX_OK;
}

int nx_engine_set_launch_observer(nx_engine* eng, nx_launch_observer fn, void* user) {
  eng->e.set_launch_observer(fn, user);
  return NX_OK;
}

int nx_engine_get_stats(const nx_engine* eng, nx_engine_stats* out) {
  *out = eng->e.stats();
  return NX_OK;
}

int nx_engine_event_log(const nx_engine* eng, char* buf, size_t cap, size_t* len) {
  return guarded([&] { return put_text(eng->e.event_log(), buf, cap, len); });
}

int nx_engine_decision_log(const nx_engine* eng, char* buf, size_t cap, size_t* len) {
  return guarded([&] { return put_text(eng->e.decision_log(), buf, cap, len); });
}

int nx_engine_summary_json(const nx_engine* eng, const char* label, char* buf, size_t cap,
                           size_t* len) {
  return guarded([&] {
    const Report r = eng->e.report();
    return put_text(r.completed ? summary_json(r, label ? label : "nexus") : std::string(), buf,
                    cap, len);
  });
}

int nx_engine_goodput(const nx_engine* eng, nx_goodput* out) {
  return guarded([&] {
    const Report r = eng->e.report();
    out->completed = r.completed;
    out->slo_met = r.slo_met;
    out->makespan_s = r.makespan;
    out->goodput_tok_s = r.goodput_tok_s;
    out->ttft_p50 = r.ttft.p50;
    out->ttft_p99 = r.ttft.p99;
    out->tbt_p50 = r.tbt_pooled.p50;
    out->tbt_p99 = r.tbt_pooled.p99;
    double tokens = 0;
    for (size_t i = 0; i < eng->e.num_requests(); ++i)
      if (eng->e.request(i).finished)
        tokens += static_cast<double>(eng->e.request(i).token_times.size());
    out->output_tokens = tokens;
    return NX_OK;
  });
}

int nx_engine_launch_latencies(const nx_engine* eng, double* out, size_t cap, size_t* n) {
  const auto& v = eng->e.launch_latencies();
  for (size_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
  *n = v.size();
  return NX_OK;
}

int nx_engine_launch_device_ms(const nx_engine* eng, double* out, size_t cap, size_t* n) {
  const auto& v = eng->e.launch_device_ms();
  for (size_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
  *n = v.size();
  return NX_OK;
}

int nx_engine_requests(const nx_engine* eng, nx_request_state* out, size_t cap, size_t* n) {
  const size_t m = eng->e.num_requests();
  for (size_t i = 0; i < m && i < cap; ++i) {
    const ReqRecord& r = eng->e.request(i);
    out[i] = {r.id,        r.arrival,  r.prompt,
              r.output,    r.prefilled, r.decoded,
              r.has_first ? r.first : -1.0, r.finished ? r.finish : -1.0};
  }
  *n = m;
  return NX_OK;
}

int nx_engine_token_times(const nx_engine* eng, uint64_t id, double* out, size_t cap, size_t* n) {
  const ReqRecord* r = eng->e.find(id);
  if (!r) return fail(NX_EINVAL, "unknown request id");
  for (size_t i = 0; i < r->token_times.size() && i < cap; ++i) out[i] = r->token_times[i];
  *n = r->token_times.size();
  return NX_OK;
}

int nx_engine_tokens(const nx_engine* eng, uint64_t id, int32_t* out, size_t cap, size_t* n) {
  const std::vector<int32_t>* t = eng->e.tokens_of(id);
  if (!t) return fail(NX_EINVAL, "unknown request id");
  for (size_t i = 0; i < t->size() && i < cap; ++i) out[i] = (*t)[i];
  *n = t->size();
  return NX_OK;
}

int nx_kv_usage(const nx_engine* eng, int64_t* used, int64_t* reserved, int64_t* capacity) {
  const nx_engine_stats s = eng->e.stats();
  *used = s.kv_used;
  *reserved = s.kv_reserved;
  *capacity = s.kv_capacity;
  return NX_OK;
}

int nx_kv_block_table(const nx_engine* eng, uint64_t id, int32_t* pages, size_t cap, size_t* n) {
  const std::vector<int32_t>* t = eng->e.pages().table(id);
  if (!t) {
    *n = 0;
    return NX_OK;
  }
  for (size_t i = 0; i < t->size() && i < cap; ++i) pages[i] = (*t)[i];
  *n = t->size();
  return NX_OK;
}

int nx_kv_page_log(const nx_engine* eng, char* buf, size_t cap, size_t* len) {
  return guarded([&] { return put_text(eng->e.pages().log(), buf, cap, len); });
}

int nx_kv_configure(nx_engine* eng, int32_t page_tokens, int32_t num_pages) {
  if (page_tokens < 1 || num_pages < 1) return fail(NX_EINVAL, "bad page geometry");
  if (eng->e.num_requests() > 0) return fail(NX_EINVAL, "configure pages before submitting");
  eng->e.configure_pages(page_tokens, num_pages);
  return NX_OK;
}

}  // extern "C"

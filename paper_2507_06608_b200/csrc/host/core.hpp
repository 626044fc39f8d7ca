// Internal C++ declarations of the host side of the Nexus B200 executor.
//
// The POD types of include/nexus_b200.h are used directly as the value types
// (no parallel C++ hierarchy), so the C-ABI layer is a thin pass-through.
// Arithmetic that feeds scheduling decisions restates the reference
// expression-for-expression (same operand order, doubles, no FMA
// contraction: the library is built with -ffp-contract=off) so decisions are
// bit-identical to nexussim.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "nexus_b200.h"

namespace nxb {

// Precondition failure; maps to NX_EINVAL at the ABI.
struct InvalidArg : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
// I/O / parse / device failure; maps to NX_ERUNTIME at the ABI.
struct RuntimeErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---- model / validation (reference domain.cpp) ---------------------------
nx_model_config derive_model(int64_t hidden, int64_t ffn, int32_t layers, int32_t heads,
                             int32_t elem);
std::string validate(const nx_model_config& m, const nx_gpu_spec& g,
                     const nx_controller_config& c, const nx_kernel_profile& p, int* count);
const nx_saturation_curve& curve_of(const nx_kernel_profile& p, int kind);
const char* op_name(int kind);
int op_from_name(const std::string& name);  // -1 if unknown

// ---- operator model (reference opcost.cpp) --------------------------------
// Small fixed-capacity op list (at most 5 ops per iteration).
struct OpList {
  int n = 0;
  nx_op_workload op[NX_MAX_OPS];
  void push(int kind, double flops, double mem, double kv, bool attn) {
    nx_op_workload& w = op[n++];
    w.kind = kind;
    w.is_attention = attn ? 1 : 0;
    w.flops = flops;
    w.mem_bytes = mem;
    w.kv_bytes = kv;
  }
  bool empty() const { return n == 0; }
};

struct Chunk {
  int64_t tokens;
  int64_t context;
};

OpList prefill_ops(const nx_model_config& m, const Chunk* chunks, size_t n);
OpList decode_ops(const nx_model_config& m, const int64_t* ctx, size_t n);
OpList mixed_ops(const nx_model_config& m, const Chunk* chunks, size_t n, const int64_t* ctx,
                 size_t nd);

// ---- cost model (reference costmodel.cpp) ---------------------------------
double compute_latency(double flops, double share, const nx_saturation_curve& c, double peak);
// decode_bw <= 0 means "all operators at peak bandwidth". ext == nullptr or
// !ext->enabled is the reference model exactly.
nx_breakdown breakdown(const OpList& ops, double share, const nx_gpu_spec& g,
                       const nx_kernel_profile& p, double decode_bw,
                       const nx_cost_ext* ext = nullptr);
inline nx_breakdown isolated(const OpList& ops, double share, const nx_gpu_spec& g,
                             const nx_kernel_profile& p, const nx_cost_ext* ext = nullptr) {
  return breakdown(ops, share, g, p, 0.0, ext);
}
double effective_decode_bw(double p_attn, double m_d, double m_p1, double m_p2, double peak);
nx_breakdown decode_contended(const OpList& dec, double share, const nx_breakdown* pre_bd,
                              const OpList& pre, const nx_gpu_spec& g,
                              const nx_kernel_profile& p, const nx_cost_ext* ext = nullptr);

// ---- controller (reference optimizer.cpp) ---------------------------------
int select_mode(int64_t used, int64_t cap, double frac);
nx_adjust_outcome adjust(int target_phase, const nx_partition_state& cur,
                         const nx_phase_model& pre, const nx_phase_model& dec,
                         const nx_controller_config& cfg);

// Decode-step target of the prefill-priority search (nx_cost_ext
// .decode_target_s; off = reference). `slowdown` maps the prefill share to
// the co-location factor (1 without the contention term).
struct DecodeTarget {
  double target_s = 0.0;
  int contention = 0;
  double c[3] = {0.0, 0.0, 0.0};
  bool on() const { return target_s > 0.0; }
  double slowdown(double prefill_share) const {
    return contention ? c[0] + c[1] * prefill_share + c[2] * prefill_share * prefill_share : 1.0;
  }
};
DecodeTarget decode_target_of(const nx_cost_ext& ext);
nx_adjust_outcome adjust(int target_phase, const nx_partition_state& cur,
                         const nx_phase_model& pre, const nx_phase_model& dec,
                         const nx_controller_config& cfg, const DecodeTarget& dt);

class Controller {
 public:
  Controller(nx_partition_state s, nx_controller_config c, DecodeTarget dt = {})
      : st_(s), cfg_(c), dt_(dt) {}
  nx_decision decide(int64_t used, int64_t cap, const nx_phase_model& pre,
                     const nx_phase_model& dec);
  const nx_partition_state& state() const { return st_; }

 private:
  nx_partition_state st_;
  nx_controller_config cfg_;
  DecodeTarget dt_;
};

// ---- schedulers (reference schedulers.cpp) --------------------------------
struct Plan {
  std::vector<nx_batch_member> members;
  int64_t total = 0;
};
Plan spf(const std::vector<nx_prefill_entry>& q, int64_t budget, double gamma, double now,
         bool skip_non_fitting);
Plan fcfs_prefill(const std::vector<nx_prefill_entry>& q, int64_t budget);
Plan fcfs_decode(const std::vector<nx_decode_candidate>& a, int32_t max_batch);
Plan chunked_mixed(const std::vector<nx_prefill_entry>& q,
                   const std::vector<nx_decode_candidate>& a, int64_t budget, int32_t max_batch,
                   int64_t chunk);

// ---- workload / text formats (reference workload.cpp, presets.cpp) --------
std::vector<nx_request> preset_trace(const std::string& preset, double rate, int64_t count,
                                     uint64_t seed);
std::string trace_text(const nx_request* t, size_t n);
std::vector<nx_request> parse_trace(const std::string& text);
std::string profile_text(const nx_kernel_profile& p);
nx_kernel_profile parse_profile(const std::string& text, std::string* warnings);
uint64_t splitmix64(uint64_t x);

// ---- metrics / logs (reference metrics.cpp, eventlog.cpp) ----------------
struct ReqRecord {
  uint64_t id = 0;
  double arrival = 0;
  int64_t prompt = 0, output = 0;
  int64_t prefilled = 0, decoded = 0;
  bool has_first = false, finished = false;
  double first = 0, finish = 0;
  std::vector<double> token_times;
};

struct Agg {
  double mean = 0, p50 = 0, p95 = 0, p99 = 0;
  size_t count = 0;
};
struct Report {
  Agg ttft, tbt_pooled, tbt_mean, e2e, normalized;
  double makespan = 0, throughput = 0;
  size_t completed = 0;
  // Goodput (new, not in the reference): output tokens of requests meeting
  // both SLOs divided by the makespan.
  double goodput_tok_s = 0;
  size_t slo_met = 0;
};
Report make_report(const std::vector<const ReqRecord*>& done, double slo_ttft, double slo_tbt);
std::string summary_json(const Report& r, const std::string& engine);

}  // namespace nxb

// The Nexus step executor: two lanes (prefill, decode) sharing one GPU under
// a per-launch SM split, or one fused lane (monolithic chunked prefill).
//
// Semantics restate IntraGpuSim (reference simulator.cpp:142-501); the event
// and decision logs are byte-compatible with the reference's. What differs
// is where a batch's latency comes from (clock mode, nx_engine_config):
//   virtual — the cost model (reference behaviour, optionally with the
//             device executing every batch so tokens are real);
//   device  — measured: a lane completes when its device work finishes,
//             observed by polling; latency = observation - launch clock;
//   replay  — caller-supplied latencies in launch order (the replay oracle
//             for device runs).
#pragma once

#include <chrono>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "core.hpp"
#include "executor.hpp"
#include "kvpages.hpp"

namespace nxb {

struct EvMember {
  uint64_t id;
  int64_t tokens;
  int32_t emitted;
};

struct EvRecord {
  double t;
  int32_t lane, kind, r_p;
  int64_t kv_used;
  double latency;
  uint32_t first, count;  // slice of Engine::ev_members_
};

struct DecisionRec {
  double t, kv_frac;
  int32_t mode, candidate, applied, switched, queries;
};

class Engine {
 public:
  explicit Engine(const nx_sim_config& cfg);

  void submit(const nx_request& r, const int32_t* prompt_tokens);
  int step();  // NX_OK / NX_EDONE / NX_EAGAIN
  int run();

  void bind(Executor* ex, bool owns);
  void set_replay(const double* lat, size_t n) { replay_.assign(lat, lat + n); }
  void configure_pages(int32_t page_tokens, int32_t num_pages) {
    pages_.configure(page_tokens, num_pages);
  }
  void set_logging(bool events, bool pages) {
    log_events_ = events;
    pages_.set_logging(pages);
  }
  void set_slo(double ttft, double tbt) {
    slo_ttft_ = ttft;
    slo_tbt_ = tbt;
  }
  void set_prompt_seed(uint64_t s) { prompt_seed_ = s; }
  // Called on every launch, before the device sees it, with the batch as the
  // device ABI describes it (TP followers replay rank 0's launches from it).
  using LaunchObserver = void (*)(void* user, const nx_batch_desc* batch);
  void set_launch_observer(LaunchObserver fn, void* user) {
    obs_ = fn;
    obs_user_ = user;
  }

  // Introspection.
  std::string event_log() const;
  std::string decision_log() const;
  Report report() const;
  nx_engine_stats stats() const;
  const std::vector<double>& launch_latencies() const { return launch_lat_; }
  const std::vector<double>& launch_device_ms() const { return launch_dev_ms_; }
  const PagePool& pages() const { return pages_; }
  const ReqRecord* find(uint64_t id) const;
  const std::vector<int32_t>* tokens_of(uint64_t id) const;
  size_t num_requests() const { return reqs_.size(); }
  const ReqRecord& request(size_t i) const { return reqs_[i].rec; }

 private:
  struct Live {
    ReqRecord rec;
    bool admitted = false;
    bool in_flight = false;
    std::vector<int32_t> tokens;  // prompt ids followed by generated ids
  };
  struct Lane {
    bool busy = false;
    bool revealed = true;  // device clock: completion observed
    double done_at = 0;
    double launch_clock = 0;
    double latency = 0;       // drives done_at and the log
    size_t launch_event = SIZE_MAX;  // index of the launch record (device clock patch)
    size_t launch_index = 0;         // index into launch_lat_ / launch_dev_ms_
    std::vector<nx_batch_member> dec, pre;
    OpList ops;
    nx_breakdown bd{};
    int r_p = 0;
  };

  // candidate queues (simulator.cpp:198-218)
  std::vector<nx_prefill_entry> prefill_queue() const;
  std::vector<nx_decode_candidate> decode_queue() const;
  std::vector<nx_batch_member> admit(const std::vector<nx_batch_member>& m, bool commit);
  std::vector<int64_t> decode_ctx(const std::vector<nx_batch_member>& m) const;
  std::vector<Chunk> chunks_of(const std::vector<nx_batch_member>& m) const;
  Plan prefill_plan(const std::vector<nx_prefill_entry>& q) const;

  // control
  OpList provisional_prefill();
  OpList provisional_decode();
  int decide(int launching_phase, const OpList& launching_ops);
  void launches();
  bool launch_decode();
  bool launch_prefill();
  bool launch_mixed();
  void begin(Lane& lane, int slot, int lane_kind, double predicted);
  void complete(Lane& lane, int slot, int lane_id);
  void finish(uint64_t id, int r_p);

  void log(int lane, int kind, const std::vector<EvMember>& m, int r_p, double lat);
  int current_r_p() const { return monolithic_ ? 100 : ctl_.state().r_p; }
  Live& live(uint64_t id) { return reqs_[index_.at(id)]; }
  const Live& live(uint64_t id) const { return reqs_[index_.at(id)]; }
  int64_t footprint(const Live& l) const {
    return (l.rec.prompt + l.rec.output) * cfg_.model.kv_bytes_per_token;
  }
  double now_s() const;
  void dispatch_device(Lane& lane, int slot, int lane_kind);
  int device_share(const Lane& lane, int lane_kind) const;
  void notify_observer(const Lane& lane, int slot, int lane_kind) const;

  nx_sim_config cfg_;
  bool dynamic_, monolithic_;
  bool decode_full_when_idle_ = true;  // NX_DECODE_FULL_IDLE=0 disables (A/B)
  Controller ctl_;
  std::vector<Live> reqs_;
  std::unordered_map<uint64_t, size_t> index_;
  std::vector<size_t> active_;
  size_t next_arrival_ = 0;
  double clock_ = 0;
  uint64_t events_ = 0;
  bool timed_out_ = false;
  int64_t kv_used_ = 0, kv_reserved_ = 0;
  Lane prefill_, decode_;

  std::vector<EvRecord> ev_;
  std::vector<EvMember> ev_members_;
  std::vector<DecisionRec> decisions_;
  uint64_t switches_ = 0, launches_ = 0, completed_ = 0;
  bool log_events_ = true;

  PagePool pages_;
  std::vector<double> replay_;
  std::vector<double> launch_lat_, launch_dev_ms_;
  Executor* exec_ = nullptr;
  std::unique_ptr<Executor> owned_exec_;
  bool started_ = false;
  std::chrono::steady_clock::time_point t0_;
  double slo_ttft_ = 1.0, slo_tbt_ = 0.05;
  uint64_t prompt_seed_ = 1;
  LaunchObserver obs_ = nullptr;
  void* obs_user_ = nullptr;
};

}  // namespace nxb

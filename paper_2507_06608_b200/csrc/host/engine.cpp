// Step executor: the event loop of the Nexus engine.
//
// Reference semantics (simulator.cpp:142-501), restated:
//   * one event per loop iteration; lanes are (re)launched between events,
//     decode before prefill (try_launches, :328-335);
//   * ties retire prefill completion, then decode completion, then arrival;
//   * the controller is consulted on every Nexus launch with the other lane's
//     in-flight ops, or a provisional plan with a dry-run admission;
//   * admission reserves the whole KV footprint in bytes; kv_used grows by a
//     chunk's tokens, and by one token per emitted token (first included);
//   * a decode batch launched while prefill is in flight is costed with the
//     contended decode bandwidth, prefill never is.
#include "engine.hpp"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <thread>

namespace nxb {

namespace {
constexpr double kInf = std::numeric_limits<double>::infinity();

const char* lane_str(int lane) {
  switch (lane) {
    case NX_LANE_PREFILL: return "prefill";
    case NX_LANE_DECODE: return "decode";
    case NX_LANE_MIXED: return "mixed";
    default: return "-";
  }
}

const char* kind_str(int k) {
  static const char* const names[] = {"arrival", "launch", "complete", "finish", "timeout"};
  return (k >= 0 && k < 5) ? names[k] : "arrival";
}
}  // namespace

Engine::Engine(const nx_sim_config& cfg)
    : cfg_(cfg),
      dynamic_(cfg.engine.kind == NX_ENGINE_NEXUS),
      monolithic_(cfg.engine.kind == NX_ENGINE_MONOLITHIC),
      ctl_(nx_partition_state{50, 50, 50}, cfg.ctrl, decode_target_of(cfg.ext)) {
  int n_bad = 0;
  const std::string why = validate(cfg.model, cfg.gpu, cfg.ctrl, cfg.profile, &n_bad);
  if (n_bad) throw InvalidArg("invalid simulation config: " + why);
  if (cfg.engine.kind != NX_ENGINE_NEXUS && cfg.engine.kind != NX_ENGINE_STATIC &&
      cfg.engine.kind != NX_ENGINE_MONOLITHIC)
    throw InvalidArg("unsupported engine kind");
  if (cfg.engine.kind == NX_ENGINE_STATIC) {
    const int r = cfg.engine.static_r_p;
    if (r < 1 || r > 99) throw InvalidArg("static partition share must lie in [1, 99]");
    ctl_ = Controller(nx_partition_state{r, 100 - r, r}, cfg.ctrl);
  }
  if (const char* e = std::getenv("NX_DECODE_FULL_IDLE")) decode_full_when_idle_ = std::atoi(e) != 0;
  if (cfg.engine.clock_mode < NX_CLOCK_VIRTUAL || cfg.engine.clock_mode > NX_CLOCK_REPLAY)
    throw InvalidArg("unknown clock mode");
  // Default page pool: enough pages for the whole byte capacity plus one
  // partial page per concurrently admitted request.
  const int64_t cap_tokens = cfg.gpu.kv_capacity_bytes / cfg.model.kv_bytes_per_token;
  const int32_t page = 16;
  pages_.configure(page, static_cast<int32_t>(std::min<int64_t>(
                             cap_tokens / page + 4096, std::numeric_limits<int32_t>::max())));
}

void Engine::bind(Executor* ex, bool owns) {
  if (!reqs_.empty()) throw InvalidArg("bind the device before submitting requests");
  exec_ = ex;
  if (owns) owned_exec_.reset(ex);
  pages_.configure(ex->page_tokens(), ex->num_pages());
}

// Arrival admission checks of the SimBase constructor (simulator.cpp:72-93).
void Engine::submit(const nx_request& r, const int32_t* prompt_tokens) {
  if (!reqs_.empty() && r.arrival_s < reqs_.back().rec.arrival)
    throw InvalidArg("trace must be sorted by arrival time");
  if (r.prompt_len < 1 || r.output_len < 1)
    throw InvalidArg("trace token counts must be >= 1");
  if ((r.prompt_len + r.output_len) * cfg_.model.kv_bytes_per_token > cfg_.gpu.kv_capacity_bytes)
    throw InvalidArg("request " + std::to_string(r.id) + ": KV footprint exceeds device capacity");
  if (index_.count(r.id)) throw InvalidArg("duplicate request id in trace");
  Live l;
  l.rec.id = r.id;
  l.rec.arrival = r.arrival_s;
  l.rec.prompt = r.prompt_len;
  l.rec.output = r.output_len;
  if (exec_) {
    l.tokens.resize(static_cast<size_t>(r.prompt_len));
    const uint64_t vocab = static_cast<uint64_t>(exec_->vocab());
    for (int64_t i = 0; i < r.prompt_len; ++i)
      l.tokens[i] = prompt_tokens ? prompt_tokens[i]
                                  : static_cast<int32_t>(
                                        splitmix64(prompt_seed_ ^ splitmix64(r.id * 1000003ULL +
                                                                             uint64_t(i))) %
                                        vocab);
  }
  index_[r.id] = reqs_.size();
  reqs_.push_back(std::move(l));
}

double Engine::now_s() const {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
}

// ---- queues --------------------------------------------------------------

std::vector<nx_prefill_entry> Engine::prefill_queue() const {
  std::vector<nx_prefill_entry> q;
  for (size_t i : active_) {
    const Live& l = reqs_[i];
    const int64_t rem = l.rec.prompt - l.rec.prefilled;
    if (!l.in_flight && rem > 0) q.push_back({l.rec.id, rem, l.rec.arrival});
  }
  return q;
}

std::vector<nx_decode_candidate> Engine::decode_queue() const {
  std::vector<nx_decode_candidate> q;
  for (size_t i : active_) {
    const Live& l = reqs_[i];
    if (!l.in_flight && l.rec.prefilled == l.rec.prompt && l.rec.decoded < l.rec.output)
      q.push_back({l.rec.id, l.rec.arrival});
  }
  return q;
}

// filter_admissible (simulator.cpp:223-244): unadmitted prefill members
// reserve their whole footprint; the first misfit stops admission.
std::vector<nx_batch_member> Engine::admit(const std::vector<nx_batch_member>& m, bool commit) {
  std::vector<nx_batch_member> kept;
  int64_t reserved = kv_reserved_;
  for (const nx_batch_member& b : m) {
    Live& l = live(b.id);
    if (l.rec.prefilled >= l.rec.prompt || l.admitted) {
      kept.push_back(b);
      continue;
    }
    const int64_t need = footprint(l);
    if (reserved + need > cfg_.gpu.kv_capacity_bytes) break;
    reserved += need;
    if (commit) {
      l.admitted = true;
      kv_reserved_ = reserved;
    }
    kept.push_back(b);
  }
  return kept;
}

std::vector<int64_t> Engine::decode_ctx(const std::vector<nx_batch_member>& m) const {
  std::vector<int64_t> ctx;
  ctx.reserve(m.size());
  for (const nx_batch_member& b : m) {
    const Live& l = live(b.id);
    ctx.push_back(l.rec.prompt + l.rec.decoded);
  }
  return ctx;
}

std::vector<Chunk> Engine::chunks_of(const std::vector<nx_batch_member>& m) const {
  std::vector<Chunk> c;
  c.reserve(m.size());
  for (const nx_batch_member& b : m) c.push_back({b.tokens, live(b.id).rec.prefilled + b.tokens});
  return c;
}

Plan Engine::prefill_plan(const std::vector<nx_prefill_entry>& q) const {
  return cfg_.engine.prefill_policy == NX_PREFILL_FCFS
             ? fcfs_prefill(q, cfg_.ctrl.token_budget)
             : spf(q, cfg_.ctrl.token_budget, cfg_.ctrl.gamma, clock_, false);
}

// ---- partition control (simulator.cpp:268-324) ---------------------------

OpList Engine::provisional_prefill() {
  const auto q = prefill_queue();
  if (q.empty()) return {};
  const auto kept = admit(prefill_plan(q).members, /*commit=*/false);
  if (kept.empty()) return {};
  const auto ch = chunks_of(kept);
  return prefill_ops(cfg_.model, ch.data(), ch.size());
}

OpList Engine::provisional_decode() {
  const auto q = decode_queue();
  if (q.empty()) return {};
  const Plan p = fcfs_decode(q, cfg_.ctrl.max_decode_batch);
  if (p.members.empty()) return {};
  const auto ctx = decode_ctx(p.members);
  return decode_ops(cfg_.model, ctx.data(), ctx.size());
}

namespace {
struct ModelCtx {
  const OpList* ops;
  const nx_gpu_spec* gpu;
  const nx_kernel_profile* prof;
  const nx_cost_ext* ext;
};
// Planning latencies are isolated (simulator.cpp:299-314).
double latency_at(void* user, int32_t pct) {
  const ModelCtx* m = static_cast<const ModelCtx*>(user);
  return isolated(*m->ops, pct / 100.0, *m->gpu, *m->prof, m->ext).total_s;
}
}  // namespace

int Engine::decide(int launching, const OpList& launching_ops) {
  const OpList pre = prefill_.busy ? prefill_.ops
                                   : (launching == NX_PHASE_PREFILL ? launching_ops
                                                                    : provisional_prefill());
  const OpList dec = decode_.busy ? decode_.ops
                                  : (launching == NX_PHASE_DECODE ? launching_ops
                                                                  : provisional_decode());
  ModelCtx pc{&pre, &cfg_.gpu, &cfg_.profile, &cfg_.ext}, dc{&dec, &cfg_.gpu, &cfg_.profile, &cfg_.ext};
  const nx_phase_model pm{pre.empty() ? 0 : 1, latency_at, &pc};
  const nx_phase_model dm{dec.empty() ? 0 : 1, latency_at, &dc};
  const nx_decision d = ctl_.decide(kv_used_, cfg_.gpu.kv_capacity_bytes, pm, dm);
  decisions_.push_back({clock_,
                        static_cast<double>(kv_used_) /
                            static_cast<double>(cfg_.gpu.kv_capacity_bytes),
                        d.mode, d.candidate_r_p, d.r_p, d.switched, d.iterations_searched});
  if (d.switched) ++switches_;
  return d.r_p;
}

// ---- launches ------------------------------------------------------------

void Engine::launches() {
  if (monolithic_) {
    if (!prefill_.busy) launch_mixed();
    return;
  }
  if (!decode_.busy) launch_decode();
  if (!prefill_.busy) launch_prefill();
}

void Engine::begin(Lane& lane, int slot, int lane_kind, double predicted) {
  const int mode = cfg_.engine.clock_mode;
  lane.busy = true;
  lane.launch_clock = clock_;
  if (mode == NX_CLOCK_REPLAY) {
    if (launches_ >= replay_.size()) throw RuntimeErr("replay: latency list exhausted");
    lane.latency = replay_[launches_];
  } else {
    lane.latency = predicted;
  }
  lane.revealed = mode != NX_CLOCK_DEVICE;
  lane.done_at = lane.revealed ? clock_ + lane.latency : kInf;
  for (const auto& m : lane.dec) live(m.id).in_flight = true;
  for (const auto& m : lane.pre) live(m.id).in_flight = true;
  // Pages for every position this launch writes.
  for (const auto& m : lane.dec) {
    const Live& l = live(m.id);
    if (!pages_.ensure(m.id, l.rec.prompt + l.rec.decoded, nullptr))
      throw RuntimeErr("KV page pool exhausted");
  }
  for (const auto& m : lane.pre) {
    if (!pages_.ensure(m.id, live(m.id).rec.prefilled + m.tokens, nullptr))
      throw RuntimeErr("KV page pool exhausted");
  }
  if (obs_) notify_observer(lane, slot, lane_kind);
  if (exec_) dispatch_device(lane, slot, lane_kind);
  std::vector<EvMember> ev;
  for (const auto& m : lane.dec) ev.push_back({m.id, m.tokens, 0});
  for (const auto& m : lane.pre) ev.push_back({m.id, m.tokens, 0});
  lane.launch_event = log_events_ ? ev_.size() : SIZE_MAX;
  log(lane_kind, NX_EV_LAUNCH, ev, lane.r_p, lane.latency);
  lane.launch_index = launch_lat_.size();
  launch_lat_.push_back(lane.latency);
  launch_dev_ms_.push_back(0.0);
  ++launches_;
}

// The SM share a launch runs on. Device layout only (the decision log keeps
// the controller's r_p): a decode batch launched while the prefill lane is
// idle and no prompt waits runs on the whole GPU instead of leaving the
// prefill SMs dark. A prefill batch launched before it finishes is ordered
// after it by the executor (Model::launch), so the two never share SMs.
int Engine::device_share(const Lane& lane, int lane_kind) const {
  if (lane_kind == NX_LANE_MIXED) return 100;
  if (lane_kind == NX_LANE_PREFILL) return lane.r_p;
  if (decode_full_when_idle_ && !prefill_.busy && prefill_queue().empty()) return 100;
  return 100 - lane.r_p;
}

// nx_batch_desc of a launch (members in log order: decode first, then prefill
// chunks) for the launch observer.
void Engine::notify_observer(const Lane& lane, int slot, int lane_kind) const {
  std::vector<int32_t> ntok, sample, toks, npg, pages;
  std::vector<int64_t> start;
  auto add = [&](uint64_t id, int32_t n, int64_t s0, int32_t smp) {
    const Live& l = live(id);
    ntok.push_back(n);
    start.push_back(s0);
    sample.push_back(smp);
    if (!l.tokens.empty()) toks.insert(toks.end(), l.tokens.begin() + s0, l.tokens.begin() + s0 + n);
    const std::vector<int32_t>* pt = pages_.table(id);
    npg.push_back(pt ? static_cast<int32_t>(pt->size()) : 0);
    if (pt) pages.insert(pages.end(), pt->begin(), pt->end());
  };
  for (const auto& m : lane.dec) {
    const Live& l = live(m.id);
    add(m.id, 1, l.rec.prompt + l.rec.decoded - 1, 1);
  }
  for (const auto& m : lane.pre) {
    const Live& l = live(m.id);
    add(m.id, static_cast<int32_t>(m.tokens), l.rec.prefilled, l.rec.prefilled + m.tokens == l.rec.prompt ? 1 : 0);
  }
  nx_batch_desc d{};
  d.lane = slot;
  d.sm_pct = device_share(lane, lane_kind);
  d.n_members = static_cast<int32_t>(ntok.size());
  d.n_tokens = ntok.data();
  d.start_pos = start.data();
  d.sample = sample.data();
  d.tokens = toks.size() == 0 ? nullptr : toks.data();
  d.n_pages = npg.data();
  d.pages = pages.data();
  obs_(obs_user_, &d);
}

void Engine::dispatch_device(Lane& lane, int slot, int lane_kind) {
  ExecBatch b;
  b.lane_kind = lane_kind;
  b.sm_pct = device_share(lane, lane_kind);
  for (const auto& m : lane.dec) {
    const Live& l = live(m.id);
    const std::vector<int32_t>* pt = pages_.table(m.id);
    ExecMember e;
    e.id = m.id;
    e.n_tokens = 1;
    e.start_pos = l.rec.prompt + l.rec.decoded - 1;
    e.sample = 1;
    e.is_prefill = 0;
    e.tokens = &l.tokens[static_cast<size_t>(e.start_pos)];
    e.pages = pt->data();
    e.n_pages = static_cast<int32_t>(pt->size());
    b.members.push_back(e);
  }
  for (const auto& m : lane.pre) {
    const Live& l = live(m.id);
    const std::vector<int32_t>* pt = pages_.table(m.id);
    ExecMember e;
    e.id = m.id;
    e.n_tokens = static_cast<int32_t>(m.tokens);
    e.start_pos = l.rec.prefilled;
    e.sample = l.rec.prefilled + m.tokens == l.rec.prompt ? 1 : 0;
    e.is_prefill = 1;
    e.tokens = &l.tokens[static_cast<size_t>(e.start_pos)];
    e.pages = pt->data();
    e.n_pages = static_cast<int32_t>(pt->size());
    b.members.push_back(e);
  }
  exec_->launch(slot, b);
}

// launch_decode (simulator.cpp:348-375).
bool Engine::launch_decode() {
  const auto q = decode_queue();
  if (q.empty()) return false;
  Plan plan = fcfs_decode(q, cfg_.ctrl.max_decode_batch);
  if (plan.members.empty()) return false;
  const auto ctx = decode_ctx(plan.members);
  OpList ops = decode_ops(cfg_.model, ctx.data(), ctx.size());
  int r_p = ctl_.state().r_p;
  if (dynamic_) r_p = decide(NX_PHASE_DECODE, ops);
  const double share = (100 - r_p) / 100.0;
  decode_.bd = prefill_.busy ? decode_contended(ops, share, &prefill_.bd, prefill_.ops,
                                                cfg_.gpu, cfg_.profile, &cfg_.ext)
                             : isolated(ops, share, cfg_.gpu, cfg_.profile, &cfg_.ext);
  decode_.dec = std::move(plan.members);
  decode_.pre.clear();
  decode_.ops = ops;
  decode_.r_p = r_p;
  begin(decode_, kLaneDecode, NX_LANE_DECODE, decode_.bd.total_s);
  return true;
}

// launch_prefill (simulator.cpp:377-402).
bool Engine::launch_prefill() {
  const auto q = prefill_queue();
  if (q.empty()) return false;
  auto kept = admit(prefill_plan(q).members, /*commit=*/true);
  if (kept.empty()) return false;
  const auto ch = chunks_of(kept);
  OpList ops = prefill_ops(cfg_.model, ch.data(), ch.size());
  int r_p = ctl_.state().r_p;
  if (dynamic_) r_p = decide(NX_PHASE_PREFILL, ops);
  prefill_.bd = isolated(ops, r_p / 100.0, cfg_.gpu, cfg_.profile, &cfg_.ext);
  prefill_.pre = std::move(kept);
  prefill_.dec.clear();
  prefill_.ops = ops;
  prefill_.r_p = r_p;
  begin(prefill_, kLanePrefill, NX_LANE_PREFILL, prefill_.bd.total_s);
  return true;
}

// launch_mixed (simulator.cpp:404-439): one fused batch at full share.
bool Engine::launch_mixed() {
  const auto q = prefill_queue();
  const auto c = decode_queue();
  if (q.empty() && c.empty()) return false;
  const Plan plan = chunked_mixed(q, c, cfg_.ctrl.token_budget, cfg_.ctrl.max_decode_batch,
                                  cfg_.ctrl.chunk_size);
  if (plan.members.empty()) return false;
  std::vector<nx_batch_member> dec, pre;
  for (const auto& m : plan.members)
    (live(m.id).rec.prefilled == live(m.id).rec.prompt ? dec : pre).push_back(m);
  pre = admit(pre, /*commit=*/true);
  if (dec.empty() && pre.empty()) return false;
  const auto ch = chunks_of(pre);
  const auto ctx = decode_ctx(dec);
  OpList ops = mixed_ops(cfg_.model, ch.data(), ch.size(), ctx.data(), ctx.size());
  prefill_.bd = isolated(ops, 1.0, cfg_.gpu, cfg_.profile, &cfg_.ext);
  prefill_.dec = std::move(dec);
  prefill_.pre = std::move(pre);
  prefill_.ops = ops;
  prefill_.r_p = 100;
  begin(prefill_, kLanePrefill, NX_LANE_MIXED, prefill_.bd.total_s);
  return true;
}

// ---- completions (simulator.cpp:443-492) ---------------------------------

void Engine::complete(Lane& lane, int slot, int lane_id) {
  const std::vector<int32_t>* sampled = nullptr;
  if (exec_) {
    exec_->wait(slot);
    sampled = &exec_->sampled(slot);
    launch_dev_ms_[lane.launch_index] = exec_->device_ms(slot);
  }
  size_t next_tok = 0;
  auto take_token = [&](Live& l) {
    if (sampled && next_tok < sampled->size()) l.tokens.push_back((*sampled)[next_tok++]);
  };
  const int64_t kv = cfg_.model.kv_bytes_per_token;
  std::vector<EvMember> ev;
  std::vector<uint64_t> finished;
  for (const auto& m : lane.dec) {
    Live& l = live(m.id);
    l.in_flight = false;
    l.rec.decoded += 1;
    l.rec.token_times.push_back(clock_);
    take_token(l);
    kv_used_ += kv;
    ev.push_back({m.id, m.tokens, 1});
    if (l.rec.decoded == l.rec.output) finished.push_back(m.id);
  }
  for (const auto& m : lane.pre) {
    Live& l = live(m.id);
    l.in_flight = false;
    l.rec.prefilled += m.tokens;
    kv_used_ += m.tokens * kv;
    int emitted = 0;
    if (l.rec.prefilled == l.rec.prompt) {
      // The completed prompt yields the first token; its KV joins the cache.
      emitted = 1;
      l.rec.decoded = 1;
      l.rec.has_first = true;
      l.rec.first = clock_;
      l.rec.token_times.push_back(clock_);
      take_token(l);
      kv_used_ += kv;
      if (l.rec.output == 1) finished.push_back(m.id);
    }
    ev.push_back({m.id, m.tokens, emitted});
  }
  lane.busy = false;
  lane.dec.clear();
  lane.pre.clear();
  log(lane_id, NX_EV_COMPLETE, ev, lane.r_p, lane.latency);
  for (uint64_t id : finished) finish(id, lane.r_p);
}

void Engine::finish(uint64_t id, int r_p) {
  Live& l = live(id);
  l.rec.finished = true;
  l.rec.finish = clock_;
  kv_used_ -= (l.rec.prompt + l.rec.decoded) * cfg_.model.kv_bytes_per_token;
  kv_reserved_ -= footprint(l);
  l.admitted = false;
  const size_t idx = index_.at(id);
  active_.erase(std::remove(active_.begin(), active_.end(), idx), active_.end());
  pages_.release(id);
  ++completed_;
  log(NX_LANE_NONE, NX_EV_FINISH, {{id, 0, 0}}, r_p, 0);
}

void Engine::log(int lane, int kind, const std::vector<EvMember>& m, int r_p, double lat) {
  if (!log_events_) return;
  EvRecord r{clock_, lane, kind, r_p, kv_used_, lat, static_cast<uint32_t>(ev_members_.size()),
             static_cast<uint32_t>(m.size())};
  ev_members_.insert(ev_members_.end(), m.begin(), m.end());
  ev_.push_back(r);
}

// ---- the loop (simulator.cpp:150-179) ------------------------------------

int Engine::step() {
  if (timed_out_) return NX_EDONE;
  const bool device_clock = cfg_.engine.clock_mode == NX_CLOCK_DEVICE;
  if (!started_) {
    started_ = true;
    t0_ = std::chrono::steady_clock::now();
  }
  launches();
  for (;;) {
    const double now = device_clock ? now_s() : 0.0;
    if (device_clock) {
      Lane* lanes[2] = {&prefill_, &decode_};
      for (int s = 0; s < 2; ++s) {
        Lane& ln = *lanes[s];
        if (!ln.busy || ln.revealed || !exec_->done(s)) continue;
        // Completion observed at `now` (sampled before the probe).
        ln.latency = now - ln.launch_clock;
        ln.done_at = ln.launch_clock + ln.latency;
        ln.revealed = true;
        if (ln.launch_event < ev_.size()) ev_[ln.launch_event].latency = ln.latency;
        launch_lat_[ln.launch_index] = ln.latency;
      }
    }
    const double tp = prefill_.busy && prefill_.revealed ? prefill_.done_at : kInf;
    const double td = decode_.busy && decode_.revealed ? decode_.done_at : kInf;
    const double ta = next_arrival_ < reqs_.size() ? reqs_[next_arrival_].rec.arrival : kInf;
    const double t = std::min({tp, td, ta});
    const bool hidden = (prefill_.busy && !prefill_.revealed) || (decode_.busy && !decode_.revealed);
    if (t == kInf && !hidden) return NX_EDONE;
    if (device_clock && !(t <= now)) {  // nothing due yet: keep polling
      std::this_thread::yield();
      continue;
    }
    if (t > cfg_.engine.timeout_sim_s || ++events_ > cfg_.engine.max_events) {
      timed_out_ = true;
      log(NX_LANE_NONE, NX_EV_TIMEOUT, {}, current_r_p(), 0);
      return NX_EDONE;
    }
    clock_ = t;
    if (prefill_.busy && prefill_.done_at == t) {
      complete(prefill_, kLanePrefill, monolithic_ ? NX_LANE_MIXED : NX_LANE_PREFILL);
    } else if (decode_.busy && decode_.done_at == t) {
      complete(decode_, kLaneDecode, NX_LANE_DECODE);
    } else {
      Live& l = reqs_[next_arrival_++];
      active_.push_back(index_.at(l.rec.id));
      log(NX_LANE_NONE, NX_EV_ARRIVAL, {{l.rec.id, 0, 0}}, current_r_p(), 0);
    }
    return NX_OK;
  }
}

int Engine::run() {
  for (;;) {
    const int rc = step();
    if (rc != NX_OK) return rc == NX_EDONE ? NX_OK : rc;
  }
}

// ---- introspection -------------------------------------------------------

std::string Engine::event_log() const {
  std::string s;
  s.reserve(ev_.size() * 64);
  char buf[128];
  for (const EvRecord& r : ev_) {
    std::snprintf(buf, sizeof buf, "%.17g\t%s\t%s\t", r.t, lane_str(r.lane), kind_str(r.kind));
    s += buf;
    if (r.count == 0) s += '-';
    for (uint32_t i = 0; i < r.count; ++i) {
      const EvMember& m = ev_members_[r.first + i];
      std::snprintf(buf, sizeof buf, "%s%llu:%ld:%d", i ? "," : "",
                    static_cast<unsigned long long>(m.id), static_cast<long>(m.tokens),
                    m.emitted);
      s += buf;
    }
    std::snprintf(buf, sizeof buf, "\t%d\t%lld\t%.17g\n", r.r_p, static_cast<long long>(r.kv_used),
                  r.latency);
    s += buf;
  }
  return s;
}

std::string Engine::decision_log() const {
  std::string s = "# time_s\tkv_frac\tmode\tcandidate_r_p\tapplied_r_p\tswitched\tqueries\n";
  char buf[160];
  for (const DecisionRec& d : decisions_) {
    std::snprintf(buf, sizeof buf, "%.17g\t%.17g\t%s\t%d\t%d\t%d\t%d\n", d.t, d.kv_frac,
                  d.mode == NX_MODE_DECODE ? "decode" : "prefill", d.candidate, d.applied,
                  d.switched, d.queries);
    s += buf;
  }
  return s;
}

Report Engine::report() const {
  std::vector<const ReqRecord*> done;
  for (const Live& l : reqs_)
    if (l.rec.finished) done.push_back(&l.rec);
  return make_report(done, slo_ttft_, slo_tbt_);
}

nx_engine_stats Engine::stats() const {
  nx_engine_stats s{};
  s.events = ev_.size();
  s.decisions = decisions_.size();
  s.switches = switches_;
  s.launches = launches_;
  s.completed_requests = completed_;
  s.timed_out = timed_out_ ? 1 : 0;
  s.current_r_p = current_r_p();
  s.clock_s = clock_;
  s.kv_used = kv_used_;
  s.kv_reserved = kv_reserved_;
  s.kv_capacity = cfg_.gpu.kv_capacity_bytes;
  return s;
}

const ReqRecord* Engine::find(uint64_t id) const {
  auto it = index_.find(id);
  return it == index_.end() ? nullptr : &reqs_[it->second].rec;
}

const std::vector<int32_t>* Engine::tokens_of(uint64_t id) const {
  auto it = index_.find(id);
  return it == index_.end() ? nullptr : &reqs_[it->second].tokens;
}

}  // namespace nxb

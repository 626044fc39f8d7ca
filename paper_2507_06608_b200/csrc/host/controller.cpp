// SM-split controller (Algorithm 1 + hysteresis) and the phase schedulers
// (SPF with aging for prefill, FCFS for decode, chunked-mixed baseline).
//
// Reference: optimizer.cpp:13-99 and schedulers.cpp:13-125. The search
// visits exactly the same shares in the same order, so the number of
// latency queries (logged per decision) matches too.
#include <algorithm>
#include <cstdlib>

#include "core.hpp"

namespace nxb {

// KV-pressure objective selection (optimizer.cpp:13-20): decode-prioritized
// iff used > frac * capacity (strict, in doubles).
int select_mode(int64_t used, int64_t cap, double frac) {
  if (used < 0 || used > cap) throw InvalidArg("select_mode: kv_used must lie in [0, capacity]");
  return static_cast<double>(used) > frac * static_cast<double>(cap) ? NX_MODE_DECODE
                                                                     : NX_MODE_PREFILL;
}

DecodeTarget decode_target_of(const nx_cost_ext& ext) {
  DecodeTarget dt;
  if (ext.enabled == 0 || !(ext.decode_target_s > 0.0)) return dt;
  dt.target_s = ext.decode_target_s;
  dt.contention = ext.contention;
  for (int i = 0; i < 3; ++i) dt.c[i] = ext.contention_c[i];
  return dt;
}

// Algorithm 1 (optimizer.cpp:22-61). The target phase's share walks down
// from its current value until the other phase fits slack * T_other(100),
// then up while the next step still fits. Shares stay in [1, 99].
nx_adjust_outcome adjust(int target_phase, const nx_partition_state& cur,
                         const nx_phase_model& pre, const nx_phase_model& dec,
                         const nx_controller_config& cfg) {
  return adjust(target_phase, cur, pre, dec, cfg, DecodeTarget{});
}

// With a decode-step target (prefill-priority mode only) a prefill share
// also fits when the decode batch's co-located step on the remaining SMs
// stays within the target: one latency query per probe, as in the reference.
nx_adjust_outcome adjust(int target_phase, const nx_partition_state& cur,
                         const nx_phase_model& pre, const nx_phase_model& dec,
                         const nx_controller_config& cfg, const DecodeTarget& dt) {
  const bool prefill_target = target_phase == NX_PHASE_PREFILL;
  const nx_phase_model& other = prefill_target ? dec : pre;
  nx_adjust_outcome out{};
  auto result = [&](int share, bool infeasible, int queries) {
    out.r_p = prefill_target ? share : 100 - share;
    out.r_d = 100 - out.r_p;
    out.infeasible = infeasible ? 1 : 0;
    out.queries = queries;
    return out;
  };
  if (!other.active) return result(99, false, 0);

  int queries = 1;
  const double bound = (prefill_target ? cfg.beta : cfg.alpha) * other.latency_at(other.user, 100);
  const bool use_target = prefill_target && dt.on();
  auto fits = [&](int target_share) {
    ++queries;
    const double t = other.latency_at(other.user, 100 - target_share);
    if (!(t > bound)) return true;
    return use_target && !(t * dt.slowdown(target_share / 100.0) > dt.target_s);
  };
  int share = std::clamp(prefill_target ? cur.r_p : cur.r_d, 1, 99);
  for (;;) {  // phase 1: shrink until the other phase meets its bound
    if (fits(share)) break;
    if (share == 1) return result(1, true, queries);
    --share;
  }
  while (share < 99 && fits(share + 1)) ++share;  // phase 2: grow while feasible
  return result(share, false, queries);
}

// PartitionController::decide (optimizer.cpp:63-99).
nx_decision Controller::decide(int64_t used, int64_t cap, const nx_phase_model& pre,
                               const nx_phase_model& dec) {
  nx_decision d{};
  d.mode = select_mode(used, cap, cfg_.kv_switch_fraction);
  const int target = d.mode == NX_MODE_DECODE ? NX_PHASE_DECODE : NX_PHASE_PREFILL;
  const nx_phase_model& tm = target == NX_PHASE_PREFILL ? pre : dec;
  d.r_p = st_.r_p;
  d.r_d = st_.r_d;
  if (!tm.active) {  // nothing to prioritize: keep the split
    d.candidate_r_p = st_.r_p;
    return d;
  }
  const nx_adjust_outcome a = adjust(target, st_, pre, dec, cfg_, dt_);
  d.candidate_r_p = a.r_p;
  d.infeasible = a.infeasible;
  d.iterations_searched = a.queries;
  if (std::abs(a.r_p - st_.last_applied_r_p) < cfg_.delta_pp) return d;  // hysteresis band
  st_.r_p = a.r_p;
  st_.r_d = a.r_d;
  st_.last_applied_r_p = a.r_p;
  d.r_p = a.r_p;
  d.r_d = a.r_d;
  d.switched = 1;
  return d;
}

// ---------------------------------------------------------------------------
// Schedulers.
// ---------------------------------------------------------------------------
namespace {

// Budget fill over an already-ordered queue (schedulers.cpp:13-32): take
// whole remainders while they fit; a head longer than the budget contributes
// a budget-sized chunk; the first misfit ends the scan unless skipping.
Plan fill_budget(const std::vector<nx_prefill_entry>& ordered, int64_t budget, bool skip) {
  Plan plan;
  for (const nx_prefill_entry& e : ordered) {
    if (plan.total + e.remaining <= budget) {
      plan.members.push_back({e.id, e.remaining});
      plan.total += e.remaining;
    } else if (plan.members.empty()) {
      plan.members.push_back({e.id, budget});
      plan.total = budget;
    } else if (!skip) {
      break;
    }
  }
  return plan;
}

bool arrival_order(double a_t, uint64_t a_id, double b_t, uint64_t b_id) {
  if (a_t < b_t) return true;
  if (b_t < a_t) return false;
  return a_id < b_id;
}

std::vector<nx_prefill_entry> by_arrival(std::vector<nx_prefill_entry> q) {
  std::sort(q.begin(), q.end(), [](const nx_prefill_entry& a, const nx_prefill_entry& b) {
    return arrival_order(a.arrival_s, a.id, b.arrival_s, b.id);
  });
  return q;
}

std::vector<nx_decode_candidate> by_arrival(std::vector<nx_decode_candidate> a) {
  std::sort(a.begin(), a.end(), [](const nx_decode_candidate& x, const nx_decode_candidate& y) {
    return arrival_order(x.arrival_s, x.id, y.arrival_s, y.id);
  });
  return a;
}

}  // namespace

// Shortest-prompt-first with aging (schedulers.cpp:43-64, Eq. 9):
// score = remaining - gamma * (now - arrival), ascending; ties on
// (arrival, id).
Plan spf(const std::vector<nx_prefill_entry>& q, int64_t budget, double gamma, double now,
         bool skip_non_fitting) {
  if (budget < 1) throw InvalidArg("spf_schedule: token_budget must be >= 1");
  struct Keyed {
    double score;
    nx_prefill_entry e;
  };
  std::vector<Keyed> k;
  k.reserve(q.size());
  for (const nx_prefill_entry& e : q) {
    const double age = now - e.arrival_s;
    k.push_back({static_cast<double>(e.remaining) - gamma * age, e});
  }
  std::sort(k.begin(), k.end(), [](const Keyed& a, const Keyed& b) {
    if (a.score < b.score) return true;
    if (b.score < a.score) return false;
    return arrival_order(a.e.arrival_s, a.e.id, b.e.arrival_s, b.e.id);
  });
  std::vector<nx_prefill_entry> ordered;
  ordered.reserve(k.size());
  for (const Keyed& x : k) ordered.push_back(x.e);
  return fill_budget(ordered, budget, skip_non_fitting);
}

// FCFS prefill ablation (schedulers.cpp:66-75).
Plan fcfs_prefill(const std::vector<nx_prefill_entry>& q, int64_t budget) {
  if (budget < 1) throw InvalidArg("fcfs_prefill_schedule: token_budget must be >= 1");
  return fill_budget(by_arrival(q), budget, false);
}

// FCFS decode (schedulers.cpp:77-88): earliest max_batch, one token each.
Plan fcfs_decode(const std::vector<nx_decode_candidate>& a, int32_t max_batch) {
  Plan plan;
  const std::vector<nx_decode_candidate> ordered = by_arrival(a);
  const size_t take = std::min(ordered.size(), static_cast<size_t>(std::max(max_batch, 0)));
  for (size_t i = 0; i < take; ++i) plan.members.push_back({ordered[i].id, 1});
  plan.total = static_cast<int64_t>(take);
  return plan;
}

// Monolithic chunked-prefill batch (schedulers.cpp:90-125): decode tokens
// first (FCFS, capped by max_batch and the budget), then FCFS prefill chunks
// of at most chunk tokens each until the budget is spent.
Plan chunked_mixed(const std::vector<nx_prefill_entry>& q,
                   const std::vector<nx_decode_candidate>& a, int64_t budget, int32_t max_batch,
                   int64_t chunk) {
  if (budget < 1) throw InvalidArg("chunked_mixed_schedule: token_budget must be >= 1");
  if (chunk < 1) throw InvalidArg("chunked_mixed_schedule: chunk_size must be >= 1");
  Plan plan;
  int64_t left = budget;
  const std::vector<nx_decode_candidate> dec = by_arrival(a);
  size_t take = std::min(dec.size(), static_cast<size_t>(std::max(max_batch, 0)));
  take = std::min(take, static_cast<size_t>(left));
  for (size_t i = 0; i < take; ++i) plan.members.push_back({dec[i].id, 1});
  plan.total += static_cast<int64_t>(take);
  left -= static_cast<int64_t>(take);
  for (const nx_prefill_entry& e : by_arrival(q)) {
    if (left <= 0) break;
    const int64_t t = std::min({e.remaining, chunk, left});
    if (t <= 0) continue;
    plan.members.push_back({e.id, t});
    plan.total += t;
    left -= t;
  }
  return plan;
}

}  // namespace nxb

// Serving metrics: TTFT, TBT (pooled and per-request mean), end-to-end and
// normalized latency, nearest-rank percentiles (reference metrics.cpp:13-91),
// the summary JSON (metrics.cpp:114-150), plus SLO goodput (new).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numeric>

#include "core.hpp"

namespace nxb {
namespace {

// p-th percentile, nearest rank: sorted[ceil(p/100 * n) - 1], clamped.
double nearest_rank(std::vector<double> v, double pct) {
  std::sort(v.begin(), v.end());
  const size_t n = v.size();
  size_t rank = static_cast<size_t>(std::ceil(pct / 100.0 * static_cast<double>(n)));
  rank = std::min(std::max<size_t>(rank, 1), n);
  return v[rank - 1];
}

Agg summarize(const std::vector<double>& v) {
  Agg a;
  a.count = v.size();
  if (v.empty()) return a;
  a.mean = std::accumulate(v.begin(), v.end(), 0.0) / static_cast<double>(v.size());
  a.p50 = nearest_rank(v, 50);
  a.p95 = nearest_rank(v, 95);
  a.p99 = nearest_rank(v, 99);
  return a;
}

}  // namespace

Report make_report(const std::vector<const ReqRecord*>& done_in, double slo_ttft,
                   double slo_tbt) {
  std::vector<const ReqRecord*> done = done_in;
  std::sort(done.begin(), done.end(),
            [](const ReqRecord* a, const ReqRecord* b) { return a->id < b->id; });
  Report r;
  if (done.empty()) return r;
  std::vector<double> ttft, e2e, norm, pooled, per_mean;
  double first_arrival = done.front()->arrival, last_finish = done.front()->finish;
  double good_tokens = 0;
  for (const ReqRecord* q : done) {
    const double t_first = q->first - q->arrival;
    const double t_e2e = q->finish - q->arrival;
    const double n_out = static_cast<double>(q->token_times.size());
    ttft.push_back(t_first);
    e2e.push_back(t_e2e);
    norm.push_back(t_e2e / n_out);
    first_arrival = std::min(first_arrival, q->arrival);
    last_finish = std::max(last_finish, q->finish);
    std::vector<double> gaps;
    for (size_t i = 1; i < q->token_times.size(); ++i)
      gaps.push_back(q->token_times[i] - q->token_times[i - 1]);
    if (!gaps.empty()) {
      double sum = 0;
      for (double g : gaps) {
        pooled.push_back(g);
        sum += g;
      }
      per_mean.push_back(sum / static_cast<double>(gaps.size()));
    }
    const bool ok_ttft = t_first <= slo_ttft;
    const bool ok_tbt = gaps.empty() || nearest_rank(gaps, 99) <= slo_tbt;
    if (ok_ttft && ok_tbt) {
      good_tokens += n_out;
      ++r.slo_met;
    }
  }
  r.ttft = summarize(ttft);
  r.e2e = summarize(e2e);
  r.normalized = summarize(norm);
  r.tbt_pooled = summarize(pooled);
  r.tbt_mean = summarize(per_mean);
  r.completed = done.size();
  r.makespan = last_finish - first_arrival;
  r.throughput = r.makespan > 0 ? static_cast<double>(r.completed) / r.makespan : 0.0;
  r.goodput_tok_s = r.makespan > 0 ? good_tokens / r.makespan : 0.0;
  return r;
}

std::string summary_json(const Report& r, const std::string& engine) {
  char buf[320];
  std::string s = "{\n  \"engine\": \"" + engine + "\",\n";
  std::snprintf(buf, sizeof buf,
                "  \"completed\": %zu,\n  \"makespan_s\": %.17g,\n  \"throughput_rps\": %.17g,\n",
                r.completed, r.makespan, r.throughput);
  s += buf;
  const std::pair<const char*, const Agg*> rows[] = {{"ttft_s", &r.ttft},
                                                     {"tbt_pooled_s", &r.tbt_pooled},
                                                     {"tbt_per_request_mean_s", &r.tbt_mean},
                                                     {"e2e_s", &r.e2e},
                                                     {"normalized_s_per_token", &r.normalized}};
  for (size_t i = 0; i < 5; ++i) {
    const Agg& a = *rows[i].second;
    std::snprintf(buf, sizeof buf,
                  "  \"%s\": {\"mean\": %.17g, \"p50\": %.17g, \"p95\": %.17g, \"p99\": %.17g, "
                  "\"count\": %zu}%s\n",
                  rows[i].first, a.mean, a.p50, a.p95, a.p99, a.count, i < 4 ? "," : "");
    s += buf;
  }
  s += "}\n";
  return s;
}

}  // namespace nxb

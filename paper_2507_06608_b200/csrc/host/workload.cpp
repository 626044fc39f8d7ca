// Synthetic traces and the shared text formats (trace file, calibration file).
//
// Traces are generated exactly as the reference does (workload.cpp:12-198,
// presets.cpp:38-105): one seed, splitmix64-derived mt19937_64 streams,
// lognormal lengths fitted to (mean, p50). The transforms use glibc
// log/exp/cos, so oracle and device runs should share trace *files*
// (SURVEY §8(c)); generating on both sides is exact only on the same libm.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <set>
#include <sstream>

#include "core.hpp"

namespace nxb {

uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

namespace {

// One independent random stream per (seed, tag) (workload.hpp:22-33).
class Stream {
 public:
  Stream(uint64_t seed, uint64_t tag) : g_(splitmix64(seed ^ splitmix64(tag))) {}
  double uniform() {  // 53-bit draw in (0, 1)
    const uint64_t bits = g_() >> 11;
    return (static_cast<double>(bits) + 0.5) * 0x1.0p-53;
  }
  double exponential(double rate) { return -std::log(uniform()) / rate; }
  double gaussian() {  // Box-Muller, cosine branch
    const double u1 = uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }
  // Gamma(shape, 1): Marsaglia-Tsang for shape >= 1, boosted for shape < 1.
  double gamma(double shape) {
    if (shape < 1.0) return gamma(shape + 1.0) * std::pow(uniform(), 1.0 / shape);
    const double d = shape - 1.0 / 3.0, c = 1.0 / std::sqrt(9.0 * d);
    for (;;) {
      double x, v;
      do {
        x = gaussian();
        v = 1.0 + c * x;
      } while (v <= 0.0);
      v = v * v * v;
      const double u = uniform();
      if (std::log(u) < 0.5 * x * x + d - d * v + d * std::log(v)) return d * v;
    }
  }

 private:
  std::mt19937_64 g_;
};

// Lognormal fitted to (mean, median): mu = ln p50, sigma^2 = 2 (ln mean - mu)
// (workload.cpp:55-68); samples are rounded and floored at one token.
struct Lengths {
  double mu = 0, sigma = 0;
  static Lengths fit(double mean, double p50) {
    Lengths l;
    l.mu = std::log(p50);
    const double s2 = 2.0 * (std::log(mean) - l.mu);
    l.sigma = s2 > 0 ? std::sqrt(s2) : 0.0;
    return l;
  }
  int64_t draw(Stream& s) const {
    const double v = std::exp(mu + sigma * s.gaussian());
    const long t = static_cast<long>(std::llround(v));
    return t < 1 ? 1 : t;
  }
};

struct Component {
  Lengths in, out;
};

// Summary statistics from the paper's workload table (presets.cpp:38-68).
Component sharegpt() { return {Lengths::fit(496, 432), Lengths::fit(97, 37)}; }
Component long_data() { return {Lengths::fit(5905, 5461), Lengths::fit(180, 159)}; }
Component arxiv() { return {Lengths::fit(3832, 3575), Lengths::fit(200, 181)}; }

constexpr uint64_t kArrivals = 0, kChoice = 1, kLengths = 2;

std::vector<nx_request> single(const Component& c, double rate, int64_t count, uint64_t seed) {
  Stream arr(seed, kArrivals), len(seed, kLengths);
  std::vector<nx_request> out;
  out.reserve(static_cast<size_t>(count));
  double t = 0;
  for (int64_t i = 0; i < count; ++i) {
    t += arr.exponential(rate);
    nx_request r{};
    r.id = static_cast<uint64_t>(i);
    r.arrival_s = t;
    r.prompt_len = c.in.draw(len);
    r.output_len = c.out.draw(len);
    out.push_back(r);
  }
  return out;
}

// mix_traces (workload.cpp:152-198): one arrival stream, a choice stream and
// one length stream per component.
std::vector<nx_request> mixture(const std::vector<Component>& cs, const std::vector<double>& w,
                                double rate, int64_t count, uint64_t seed) {
  Stream arr(seed, kArrivals), pick_s(seed, kChoice);
  std::vector<Stream> len;
  for (size_t i = 0; i < cs.size(); ++i) len.emplace_back(seed, kLengths + i);
  std::vector<nx_request> out;
  out.reserve(static_cast<size_t>(count));
  double t = 0;
  for (int64_t i = 0; i < count; ++i) {
    t += arr.exponential(rate);
    const double u = pick_s.uniform();
    size_t pick = 0;
    double acc = 0;
    for (size_t k = 0; k < w.size(); ++k) {
      pick = k;
      acc += w[k];
      if (u <= acc) break;
    }
    nx_request r{};
    r.id = static_cast<uint64_t>(i);
    r.arrival_s = t;
    r.prompt_len = cs[pick].in.draw(len[pick]);
    r.output_len = cs[pick].out.draw(len[pick]);
    out.push_back(r);
  }
  return out;
}

// New shapes (not in the reference presets): LongBench-shaped long prompts
// (uniform 4096..16384 tokens, ShareGPT-shaped outputs) and
// bursty arrivals (Gamma inter-arrival times with CV = 4, i.e. shape 1/16,
// over the "mixed" length mix; C4).
std::vector<nx_request> longbench(double rate, int64_t count, uint64_t seed) {
  Stream arr(seed, kArrivals), len(seed, kLengths);
  const Lengths out = sharegpt().out;
  std::vector<nx_request> v;
  double t = 0;
  for (int64_t i = 0; i < count; ++i) {
    t += arr.exponential(rate);
    nx_request r{};
    r.id = static_cast<uint64_t>(i);
    r.arrival_s = t;
    r.prompt_len = 4096 + static_cast<int64_t>(len.uniform() * (16384 - 4096 + 1));
    r.output_len = out.draw(len);
    v.push_back(r);
  }
  return v;
}

std::vector<nx_request> bursty(double rate, int64_t count, uint64_t seed, double cv) {
  std::vector<nx_request> v = mixture({sharegpt(), long_data()}, {0.6, 0.4}, rate, count, seed);
  Stream arr(seed, 7);  // separate stream: lengths stay those of "mixed"
  const double shape = 1.0 / (cv * cv), scale = 1.0 / (rate * shape);
  double t = 0;
  for (nx_request& r : v) {
    t += arr.gamma(shape) * scale;
    r.arrival_s = t;
  }
  return v;
}

}  // namespace

std::vector<nx_request> preset_trace(const std::string& preset, double rate, int64_t count,
                                     uint64_t seed) {
  if (!(rate > 0)) throw InvalidArg("workload.rate_rps: must be > 0");
  if (count < 0) throw InvalidArg("workload.count: must be >= 0");
  if (preset == "sharegpt") return single(sharegpt(), rate, count, seed);
  if (preset == "long-data") return single(long_data(), rate, count, seed);
  if (preset == "arxiv") return single(arxiv(), rate, count, seed);
  if (preset == "mixed") return mixture({sharegpt(), long_data()}, {0.6, 0.4}, rate, count, seed);
  if (preset == "longbench") return longbench(rate, count, seed);
  if (preset == "bursty") return bursty(rate, count, seed, 4.0);
  throw InvalidArg("unknown workload preset '" + preset + "'");
}

// "# nexustrace v1" + "id\tarrival\tprompt\toutput" lines (workload.cpp:200-243).
static const char kTraceHeader[] = "# nexustrace v1";

std::string trace_text(const nx_request* t, size_t n) {
  std::string s = std::string(kTraceHeader) + "\n";
  char line[160];
  for (size_t i = 0; i < n; ++i) {
    std::snprintf(line, sizeof line, "%llu\t%.17g\t%ld\t%ld\n",
                  static_cast<unsigned long long>(t[i].id), t[i].arrival_s,
                  static_cast<long>(t[i].prompt_len), static_cast<long>(t[i].output_len));
    s += line;
  }
  return s;
}

std::vector<nx_request> parse_trace(const std::string& text) {
  std::istringstream in(text);
  std::string line;
  if (!std::getline(in, line) || line != kTraceHeader)
    throw RuntimeErr("trace: bad or missing header (expected '# nexustrace v1')");
  std::vector<nx_request> out;
  int no = 1;
  while (std::getline(in, line)) {
    ++no;
    if (line.empty()) continue;
    unsigned long long id = 0;
    long p = 0, o = 0;
    double a = 0;
    if (std::sscanf(line.c_str(), "%llu\t%lg\t%ld\t%ld", &id, &a, &p, &o) != 4)
      throw RuntimeErr("trace line " + std::to_string(no) + ": malformed record");
    if (p < 1 || o < 1)
      throw RuntimeErr("trace line " + std::to_string(no) + ": token counts must be >= 1");
    out.push_back({id, a, p, o});
  }
  return out;
}

// Calibration file (presets.cpp:109-170).
std::string profile_text(const nx_kernel_profile& p) {
  std::string s = "# op\tr_sat\tlambda\n";
  char line[96];
  for (int k = 0; k < 5; ++k) {
    const nx_saturation_curve& c = curve_of(p, k);
    std::snprintf(line, sizeof line, "%s\t%.17g\t%.17g\n", op_name(k), c.r_sat, c.lambda);
    s += line;
  }
  return s;
}

nx_kernel_profile parse_profile(const std::string& text, std::string* warnings) {
  nx_kernel_profile p = nx_kernel_profile_default();
  std::istringstream in(text);
  std::string line;
  std::set<int> seen;
  int no = 0;
  while (std::getline(in, line)) {
    ++no;
    const size_t hash = line.find('#');
    if (hash != std::string::npos) line.erase(hash);
    std::istringstream ls(line);
    std::string op;
    if (!(ls >> op)) continue;
    double r_sat = 0, lambda = 0;
    const std::string where = "calibration line " + std::to_string(no);
    if (!(ls >> r_sat >> lambda)) throw RuntimeErr(where + ": expected '<op> <r_sat> <lambda>'");
    const int k = op_from_name(op);
    if (k < 0) throw RuntimeErr(where + ": unknown operator kind '" + op + "'");
    if (!(r_sat > 0.0 && r_sat <= 1.0)) throw RuntimeErr(where + ": r_sat must lie in (0, 1]");
    if (!(lambda >= 0.0)) throw RuntimeErr(where + ": lambda must be >= 0");
    nx_saturation_curve& c = const_cast<nx_saturation_curve&>(curve_of(p, k));
    c.r_sat = r_sat;
    c.lambda = lambda;
    seen.insert(k);
  }
  if (warnings) {
    for (int k = 0; k < 5; ++k)
      if (!seen.count(k))
        *warnings += std::string("calibration has no entry for '") + op_name(k) +
                     "'; using the default curve\n";
  }
  return p;
}

}  // namespace nxb

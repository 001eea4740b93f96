// Host-side workload synthesis for replica sweeps: a restatement of the
// reference's realize() (workload.cpp:319-372) for its built-in QA / RG / CG
// templates (workload.cpp:462-560), producing the flattened realization the
// device replica engine consumes. The random stream is the reference's:
// std::mt19937_64 (fully specified by the C++ standard), the hand-rolled
// samplers of rng.hpp:17-60 and glibc libm, compiled with
// -ffp-contract=off, so a given seed yields the reference's realization bit
// for bit (checked against realize() itself in tests/test_workload_port.py).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/kairos_b200.h"

namespace {

// rng.hpp:12-64
class Rng {
 public:
  explicit Rng(uint64_t seed) : gen_(seed) {}
  uint64_t next_u64() { return gen_(); }
  double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  int64_t uniform_int(int64_t lo, int64_t hi) {
    const auto span = static_cast<uint64_t>(hi - lo) + 1;
    return lo + static_cast<int64_t>(gen_() % span);
  }
  double exponential(double rate) {
    const double u = uniform();
    return -std::log1p(-u) / rate;
  }
  double normal() {
    double u1 = uniform();
    const double u2 = uniform();
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    constexpr double kTwoPi = 6.283185307179586476925286766559;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(kTwoPi * u2);
  }
  double lognormal(double mu, double sigma) { return std::exp(mu + sigma * normal()); }
  static uint64_t derive(uint64_t seed, uint64_t stream) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }

 private:
  std::mt19937_64 gen_;
};

// LengthSpec (workload.hpp:18-33, workload.cpp:13-59)
struct Length {
  int kind;  // 0 fixed, 1 uniform, 2 lognormal
  double a, b;
  int64_t lo, hi;
  int64_t sample(Rng& rng) const {
    int64_t v = 1;
    if (kind == 0) v = static_cast<int64_t>(a);
    else if (kind == 1) v = rng.uniform_int(static_cast<int64_t>(a), static_cast<int64_t>(b));
    else v = static_cast<int64_t>(std::llround(rng.lognormal(a, b)));
    return v < lo ? lo : (v > hi ? hi : v);
  }
};

Length uniform(int64_t lo, int64_t hi) { return {1, double(lo), double(hi), lo, hi}; }
Length lognormal(double median, double sigma, int64_t cap) { return {2, std::log(median), sigma, 1, cap}; }

struct Agent {
  int id;  // index in the built-in agent list (KX_AGENT_*)
  Length prompt, output;
  std::vector<std::pair<int, double>> choice;
  std::vector<int> parallel;
  int fb_target = -1;
  double fb_p = 0.0;
  int fb_max = 0;
};

struct App {
  int entry;
  double weight;
};

// Built-in agents, fixed order (kx_builtin_agent_name).
const char* kNames[10] = {"Router",         "Math",      "Humanities",     "Researcher", "Writer",
                          "ProductManager", "Architect", "ProjectManager", "Engineer",   "QAEngineer"};

std::vector<Agent> builtin_agents() {
  std::vector<Agent> a(10);
  for (int i = 0; i < 10; ++i) a[i].id = i;
  a[0].prompt = uniform(40, 80);   a[0].output = lognormal(10.0, 0.25, 40);
  a[0].choice = {{1, 0.5}, {2, 0.5}};
  a[1].prompt = uniform(60, 120);  a[1].output = lognormal(70.0, 0.35, 400);
  a[2].prompt = uniform(60, 120);  a[2].output = lognormal(240.0, 0.35, 900);
  a[3].prompt = uniform(80, 160);  a[3].output = lognormal(150.0, 0.35, 700);
  a[3].choice = {{4, 1.0}};
  a[4].prompt = uniform(120, 240); a[4].output = lognormal(380.0, 0.30, 1100);
  a[5].prompt = uniform(80, 160);  a[5].output = lognormal(70.0, 0.35, 300);  a[5].choice = {{6, 1.0}};
  a[6].prompt = uniform(80, 160);  a[6].output = lognormal(110.0, 0.35, 450); a[6].choice = {{7, 1.0}};
  a[7].prompt = uniform(80, 160);  a[7].output = lognormal(50.0, 0.30, 200);  a[7].choice = {{8, 1.0}};
  a[8].prompt = uniform(100, 200); a[8].output = lognormal(300.0, 0.40, 1100); a[8].choice = {{9, 1.0}};
  a[9].prompt = uniform(80, 160);  a[9].output = lognormal(40.0, 0.30, 160);
  a[9].fb_target = 8; a[9].fb_p = 0.3; a[9].fb_max = 3;
  return a;
}

}  // namespace

struct kx_realization {
  std::vector<double> arrival;
  std::vector<int32_t> app;
  std::vector<int64_t> wf_offsets{0};
  std::vector<int32_t> agent, parent;
  std::vector<int64_t> prompt, target;
  std::vector<double> pure_exec, remaining;
  std::vector<uint64_t> uid;
};

namespace {

thread_local std::string g_wl_error;

void realize_impl(uint32_t app_mask, double rate, double duration, uint64_t seed, double prefill,
                  double decode, kx_realization* r) {
  if (!(rate > 0.0)) throw std::invalid_argument("poisson rate must be positive");
  if (!(duration > 0.0)) throw std::invalid_argument("duration must be positive");
  if (!(prefill > 0.0 && decode > 0.0)) throw std::invalid_argument("rates must be positive");
  const auto agents = builtin_agents();
  std::vector<App> apps;
  if (app_mask & KX_APPS_QA) apps.push_back({0, 1.0});
  if (app_mask & KX_APPS_RG) apps.push_back({3, 1.0});
  if (app_mask & KX_APPS_CG) apps.push_back({5, 1.0});
  if (apps.empty()) throw std::invalid_argument("no applications configured");
  // Feedback loop budget per feedback-owning agent of the configured apps.
  const bool has_cg = (app_mask & KX_APPS_CG) != 0;

  std::vector<double> arrivals;  // workload.cpp:326-333
  {
    Rng arr(Rng::derive(seed, 0));
    double t = 0.0;
    while (true) {
      t += arr.exponential(rate);
      if (t > duration) break;
      arrivals.push_back(t);
    }
  }
  Rng entry_rng(Rng::derive(seed, 1));
  double weight_sum = 0.0;
  for (const auto& a : apps) weight_sum += a.weight;
  uint64_t next_uid = 1;
  for (size_t i = 0; i < arrivals.size(); ++i) {
    // Weighted entry selection (workload.cpp:347-360)
    int app = -1;
    double u = entry_rng.uniform() * weight_sum;
    for (size_t k = 0; k < apps.size(); ++k) {
      if (u < apps[k].weight) {
        app = static_cast<int>(k);
        break;
      }
      u -= apps[k].weight;
    }
    if (app < 0) app = static_cast<int>(apps.size()) - 1;
    Rng rng(Rng::derive(seed, 1000 + i));
    // instantiate_workflow (workload.cpp:227-288)
    int loops_qa_engineer = has_cg ? agents[9].fb_max : 0;
    struct Call {
      int agent, parent;
      int64_t prompt, target;
    };
    std::vector<Call> calls;
    auto add_call = [&](int agent, int parent) {
      Call c;
      c.agent = agent;
      c.parent = parent;
      c.prompt = agents[agent].prompt.sample(rng);
      c.target = agents[agent].output.sample(rng);
      calls.push_back(c);
      return static_cast<int>(calls.size() - 1);
    };
    auto expand = [&](auto&& self, int node) -> void {
      const Agent& spec = agents[calls[node].agent];
      if (spec.fb_target >= 0 && loops_qa_engineer > 0 && rng.uniform() < spec.fb_p) {
        --loops_qa_engineer;
        self(self, add_call(spec.fb_target, node));
        return;
      }
      if (!spec.parallel.empty()) {
        for (int to : spec.parallel) self(self, add_call(to, node));
      } else if (!spec.choice.empty()) {
        double v = rng.uniform();
        int chosen = spec.choice.back().first;
        for (const auto& [to, p] : spec.choice) {
          if (v < p) {
            chosen = to;
            break;
          }
          v -= p;
        }
        self(self, add_call(chosen, node));
      }
    };
    expand(expand, add_call(apps[app].entry, -1));
    // finalize_instance (workload.cpp:292-315)
    const size_t n = calls.size();
    const size_t b = r->agent.size();
    std::vector<double> rem(n, 0.0), pure(n);
    for (size_t c = 0; c < n; ++c) {
      pure[c] = static_cast<double>(calls[c].prompt) / prefill + static_cast<double>(calls[c].target) / decode;
    }
    for (size_t c = n; c-- > 0;) {
      double tail = 0.0;
      for (size_t ch = c + 1; ch < n; ++ch)
        if (calls[ch].parent == static_cast<int>(c) && tail < rem[ch]) tail = rem[ch];
      rem[c] = pure[c] + tail;
    }
    for (size_t c = 0; c < n; ++c) {
      r->agent.push_back(calls[c].agent);
      r->parent.push_back(calls[c].parent);
      r->prompt.push_back(calls[c].prompt);
      r->target.push_back(calls[c].target);
      r->pure_exec.push_back(pure[c]);
      r->remaining.push_back(rem[c]);
      r->uid.push_back(next_uid++);
    }
    (void)b;
    r->arrival.push_back(arrivals[i]);
    r->app.push_back(app);
    r->wf_offsets.push_back(static_cast<int64_t>(r->agent.size()));
  }
}

}  // namespace

extern "C" {

const char* kx_builtin_agent_name(int32_t agent) {
  return (agent >= 0 && agent < 10) ? kNames[agent] : nullptr;
}

int kx_realize_builtin(uint32_t app_mask, double rate, double duration, uint64_t seed,
                       double prefill_rate, double decode_rate, kx_realization** out) {
  try {
    if (!out) throw std::invalid_argument("null argument");
    auto* r = new kx_realization();
    try {
      realize_impl(app_mask, rate, duration, seed, prefill_rate, decode_rate, r);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
    return KX_OK;
  } catch (const std::invalid_argument& e) {
    g_wl_error = e.what();
    return KX_ERR_INVALID;
  } catch (const std::exception& e) {
    g_wl_error = e.what();
    return KX_ERR_RUNTIME;
  }
}

int kx_realization_sizes(const kx_realization* r, int64_t* n_workflows, int64_t* n_calls) {
  if (!r) return KX_ERR_INVALID;
  if (n_workflows) *n_workflows = static_cast<int64_t>(r->arrival.size());
  if (n_calls) *n_calls = static_cast<int64_t>(r->agent.size());
  return KX_OK;
}

int kx_realization_copy(const kx_realization* r, double* arrival, int32_t* app, int64_t* wf_offsets,
                        int32_t* agent, int32_t* parent, int64_t* prompt, int64_t* target,
                        double* pure_exec, double* remaining, uint64_t* uid) {
  if (!r) return KX_ERR_INVALID;
  auto cp = [](auto* dst, const auto& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
  };
  cp(arrival, r->arrival);
  cp(app, r->app);
  cp(wf_offsets, r->wf_offsets);
  cp(agent, r->agent);
  cp(parent, r->parent);
  cp(prompt, r->prompt);
  cp(target, r->target);
  cp(pure_exec, r->pure_exec);
  cp(remaining, r->remaining);
  cp(uid, r->uid);
  return KX_OK;
}

void kx_realization_free(kx_realization* r) { delete r; }

}  // extern "C"

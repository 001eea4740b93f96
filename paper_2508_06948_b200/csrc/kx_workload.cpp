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

namespace kx {
void set_last_error(const char* m);  // kx_abi.cu
}

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

// AgentSpec (workload.hpp:39-52) over dense agent indices.
struct Agent {
  Length prompt, output;
  std::vector<std::pair<int, double>> choice;
  std::vector<int> parallel;
  int fb_target = -1;
  double fb_p = 0.0;
  int fb_max = 0;
};

// AppSpec (workload.hpp:55-60): its agents (members) and entry.
struct App {
  std::vector<int> members;
  int entry;
  double weight;
};

// WorkloadConfig (workload.hpp:69-83) with the arrival times already
// materialised for TraceFile arrivals (ingest_arrival_trace is file I/O).
struct Config {
  std::vector<Agent> agents;
  std::vector<App> apps;
  int arrival_kind = 0;  // 0 Poisson, 1 explicit (scaled) trace timestamps
  double rate = 1.0;
  std::vector<double> trace;  // raw timestamps (kind 1)
  double trace_scale = 1.0;
  double duration = 60.0;
  int entry_cycle = 0;  // EntrySelection::Cycle
};

// Built-in agents, fixed order (kx_builtin_agent_name).
const char* kNames[10] = {"Router",         "Math",      "Humanities",     "Researcher", "Writer",
                          "ProductManager", "Architect", "ProjectManager", "Engineer",   "QAEngineer"};

// qa_app / rg_app / cg_app (workload.cpp:462-531).
std::vector<Agent> builtin_agents() {
  std::vector<Agent> a(10);
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

Length from_abi(const kx_length_spec& l) {
  if (l.kind < 0 || l.kind > 2) throw std::invalid_argument("unknown length spec kind");
  return {l.kind, l.a, l.b, l.min_tokens, l.max_tokens};
}

Config config_from_abi(const kx_workload_config* c) {
  if (!c || c->n_agents < 0 || c->n_apps < 0) throw std::invalid_argument("null argument");
  Config cfg;
  cfg.agents.resize(static_cast<size_t>(c->n_agents));
  auto agent_ok = [&](int32_t a) { return a >= 0 && a < c->n_agents; };
  for (int32_t i = 0; i < c->n_agents; ++i) {
    const kx_agent_spec& s = c->agents[i];
    Agent& a = cfg.agents[i];
    a.prompt = from_abi(s.prompt_len);
    a.output = from_abi(s.output_len);
    for (int32_t j = 0; j < s.n_choice; ++j) {
      if (!agent_ok(s.choice_to[j])) throw std::invalid_argument("agent " + std::to_string(i) + ": unknown downstream");
      a.choice.emplace_back(s.choice_to[j], s.choice_p[j]);
    }
    for (int32_t j = 0; j < s.n_parallel; ++j) {
      if (!agent_ok(s.parallel_to[j])) throw std::invalid_argument("agent " + std::to_string(i) + ": unknown downstream");
      a.parallel.push_back(s.parallel_to[j]);
    }
    if (s.feedback_target >= 0) {
      if (!agent_ok(s.feedback_target)) throw std::invalid_argument("agent " + std::to_string(i) + ": unknown feedback target");
      a.fb_target = s.feedback_target;
      a.fb_p = s.feedback_probability;
      a.fb_max = s.feedback_max_iterations;
    }
  }
  for (int32_t k = 0; k < c->n_apps; ++k) {
    const kx_app_spec& s = c->apps[k];
    App app;
    for (int32_t j = 0; j < s.n_members; ++j) {
      if (!agent_ok(s.members[j])) throw std::invalid_argument("app member out of range");
      app.members.push_back(s.members[j]);
    }
    if (!agent_ok(s.entry)) throw std::invalid_argument("entry agent not defined");
    app.entry = s.entry;
    app.weight = s.weight;
    cfg.apps.push_back(std::move(app));
  }
  cfg.arrival_kind = c->arrival_kind;
  cfg.rate = c->rate;
  if (c->arrival_kind == KX_ARRIVAL_TRACE) {
    if (c->n_trace < 0 || (c->n_trace > 0 && !c->trace)) throw std::invalid_argument("null argument");
    cfg.trace.assign(c->trace, c->trace + c->n_trace);
  } else if (c->arrival_kind != KX_ARRIVAL_POISSON) {
    throw std::invalid_argument("unknown arrival kind");
  }
  cfg.trace_scale = c->trace_scale;
  cfg.duration = c->duration;
  cfg.entry_cycle = c->entry_selection == KX_ENTRY_CYCLE ? 1 : 0;
  return cfg;
}

// WorkloadConfig::validate (workload.cpp:97-192) minus the name checks
// (agents are dense indices here, so names cannot be empty, reserved or
// duplicated; the caller owns the names).
void validate(const Config& c) {
  if (c.apps.empty()) throw std::invalid_argument("no applications configured");
  if (!(c.duration > 0.0)) throw std::invalid_argument("duration must be positive");
  if (c.arrival_kind == KX_ARRIVAL_POISSON && !(c.rate > 0.0))
    throw std::invalid_argument("poisson rate must be positive");
  for (const App& app : c.apps)
    if (!(app.weight > 0.0)) throw std::invalid_argument("app weight must be positive");
  for (const App& app : c.apps) {
    for (int m : app.members) {
      const Agent& a = c.agents[m];
      const std::string nm = "agent " + std::to_string(m);
      if (!a.choice.empty() && !a.parallel.empty())
        throw std::invalid_argument(nm + ": choice and parallel are exclusive");
      double p_sum = 0.0;
      for (const auto& [to, p] : a.choice) {
        (void)to;
        if (p < 0.0) throw std::invalid_argument("negative probability");
        p_sum += p;
      }
      if (!a.choice.empty() && std::abs(p_sum - 1.0) > 1e-9)
        throw std::invalid_argument(nm + ": choice probabilities must sum to 1");
      if (a.fb_target >= 0) {
        if (a.fb_max < 1) throw std::invalid_argument(nm + ": max_iterations < 1");
        if (a.fb_p < 0.0 || a.fb_p > 1.0) throw std::invalid_argument(nm + ": feedback probability");
      }
    }
    // choice/parallel structure acyclic; loops only through feedback edges
    std::vector<int> color(c.agents.size(), 0);
    auto dfs = [&](auto&& self, int node) -> void {
      color[node] = 1;
      const Agent& a = c.agents[node];
      std::vector<int> next;
      for (const auto& [to, p] : a.choice) {
        (void)p;
        next.push_back(to);
      }
      for (int to : a.parallel) next.push_back(to);
      for (int to : next) {
        if (color[to] == 1) throw std::invalid_argument("cycle is not a declared feedback edge");
        if (color[to] == 0) self(self, to);
      }
      color[node] = 2;
    };
    for (int m : app.members)
      if (color[m] == 0) dfs(dfs, m);
  }
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


// scale_arrival_gaps (workload.cpp:194-214)
std::vector<double> scale_gaps(const std::vector<double>& ts, double scale) {
  if (!(scale > 0.0)) throw std::invalid_argument("scale must be positive");
  std::vector<double> out;
  out.reserve(ts.size());
  double prev = 0.0, t = 0.0;
  for (size_t i = 0; i < ts.size(); ++i) {
    if (i > 0) {
      const double gap = ts[i] - prev;
      if (gap < 0.0) throw std::invalid_argument("non-monotone timestamp at index " + std::to_string(i));
      t += gap * scale;
    }
    prev = ts[i];
    out.push_back(t);
  }
  return out;
}

// realize (workload.cpp:319-372) with instantiate_workflow (227-288) and
// finalize_instance (292-315).
void realize_impl(const Config& cfg, uint64_t seed, double prefill, double decode, kx_realization* r) {
  validate(cfg);
  if (!(prefill > 0.0 && decode > 0.0)) throw std::invalid_argument("rates must be positive");
  const auto& agents = cfg.agents;
  const auto& apps = cfg.apps;
  std::vector<double> arrivals;
  if (cfg.arrival_kind == KX_ARRIVAL_POISSON) {
    Rng arr(Rng::derive(seed, 0));
    double t = 0.0;
    while (true) {
      t += arr.exponential(cfg.rate);
      if (t > cfg.duration) break;
      arrivals.push_back(t);
    }
  } else {
    for (double t : scale_gaps(cfg.trace, cfg.trace_scale))
      if (t <= cfg.duration) arrivals.push_back(t);
  }
  // Feedback loop budget: every feedback-owning agent of every app
  // (workload.cpp:233-240), reset per instance.
  std::vector<int> fb_agents;
  for (const App& app : apps)
    for (int m : app.members)
      if (agents[m].fb_target >= 0) fb_agents.push_back(m);
  std::vector<int> loops_left(agents.size(), 0);
  Rng entry_rng(Rng::derive(seed, 1));
  double weight_sum = 0.0;
  for (const auto& a : apps) weight_sum += a.weight;
  uint64_t next_uid = 1;
  struct Call {
    int agent, parent;
    int64_t prompt, target;
  };
  std::vector<Call> calls;
  std::vector<double> rem, pure;
  for (size_t i = 0; i < arrivals.size(); ++i) {
    int app = -1;
    if (cfg.entry_cycle) {
      app = static_cast<int>(i % apps.size());
    } else {  // weighted entry selection (workload.cpp:347-360)
      double u = entry_rng.uniform() * weight_sum;
      for (size_t k = 0; k < apps.size(); ++k) {
        if (u < apps[k].weight) {
          app = static_cast<int>(k);
          break;
        }
        u -= apps[k].weight;
      }
      if (app < 0) app = static_cast<int>(apps.size()) - 1;
    }
    Rng rng(Rng::derive(seed, 1000 + i));
    for (int m : fb_agents) loops_left[m] = agents[m].fb_max;
    calls.clear();
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
      const int ai = calls[node].agent;
      const Agent& spec = agents[ai];
      if (spec.fb_target >= 0 && loops_left[ai] > 0 && rng.uniform() < spec.fb_p) {
        --loops_left[ai];
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
    // finalize_instance: calls are parents-first, so a reverse sweep sees
    // every child before its parent (max over children = max of pushes).
    const size_t n = calls.size();
    pure.assign(n, 0.0);
    rem.assign(n, 0.0);
    std::vector<double> tail(n, 0.0);
    for (size_t c = 0; c < n; ++c)
      pure[c] = static_cast<double>(calls[c].prompt) / prefill + static_cast<double>(calls[c].target) / decode;
    for (size_t c = n; c-- > 0;) {
      rem[c] = pure[c] + tail[c];
      const int p = calls[c].parent;
      if (p >= 0) tail[p] = std::max(tail[p], rem[c]);
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
    r->arrival.push_back(arrivals[i]);
    r->app.push_back(app);
    r->wf_offsets.push_back(static_cast<int64_t>(r->agent.size()));
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    kx::set_last_error("");
    return KX_OK;
  } catch (const std::invalid_argument& e) {
    kx::set_last_error(e.what());
    return KX_ERR_INVALID;
  } catch (const std::bad_alloc&) {
    kx::set_last_error("out of host memory");
    return KX_ERR_CAPACITY;
  } catch (const std::exception& e) {
    kx::set_last_error(e.what());
    return KX_ERR_RUNTIME;
  }
}

int realize_to(const Config& cfg, uint64_t seed, double prefill, double decode, kx_realization** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null argument");
    auto* r = new kx_realization();
    try {
      realize_impl(cfg, seed, prefill, decode, r);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
  });
}

}  // namespace

extern "C" {

const char* kx_builtin_agent_name(int32_t agent) {
  return (agent >= 0 && agent < 10) ? kNames[agent] : nullptr;
}

int kx_realize_builtin(uint32_t app_mask, double rate, double duration, uint64_t seed,
                       double prefill_rate, double decode_rate, kx_realization** out) {
  // colocated_workload / qa_workload / ... (workload.cpp:536-560): the
  // selected apps in QA, RG, CG order, weight 1, Poisson arrivals.
  Config cfg;
  cfg.agents = builtin_agents();
  if (app_mask & KX_APPS_QA) cfg.apps.push_back({{0, 1, 2}, 0, 1.0});
  if (app_mask & KX_APPS_RG) cfg.apps.push_back({{3, 4}, 3, 1.0});
  if (app_mask & KX_APPS_CG) cfg.apps.push_back({{5, 6, 7, 8, 9}, 5, 1.0});
  cfg.rate = rate;
  cfg.duration = duration;
  return realize_to(cfg, seed, prefill_rate, decode_rate, out);
}

int kx_realize(const kx_workload_config* config, uint64_t seed, double prefill_rate, double decode_rate,
               kx_realization** out) {
  Config cfg;
  const int st = guarded([&] { cfg = config_from_abi(config); });
  if (st != KX_OK) return st;
  return realize_to(cfg, seed, prefill_rate, decode_rate, out);
}

int kx_realization_sizes(const kx_realization* r, int64_t* n_workflows, int64_t* n_calls) {
  if (!r) {
    kx::set_last_error("null realization");
    return KX_ERR_INVALID;
  }
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

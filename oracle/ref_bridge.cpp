// TEST / BASELINE INFRASTRUCTURE ONLY. A C-ABI bridge around the UNMODIFIED
// reference (libkairos_ref.a built from /root/reference/proj by
// oracle/Makefile) so bench.py can time the reference's own CPU
// implementation of the scheduling tick:
//   ordering  std::sort with the ReadyQueue comparator over
//             SchedulerPolicy::order_key (harness.cpp:92-100, priority.hpp:95-98)
//   placement the dispatch_loop sequence of engine.cpp:220-268 over the
//             ordered queue with the reference Dispatcher
//             (collect_live -> choose -> overload check -> commit -> admit)
//             and Dispatcher::gc (engine.cpp:212).
// The ordered-prefix walk replaces the reference's repeated best_index
// scans (O(D*N) per round), which only makes the baseline faster.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "kairos/dispatcher.hpp"
#include "kairos/priority.hpp"
#include "kairos/scheduler.hpp"

using namespace kairos;

namespace {

struct TablePolicy : SchedulerPolicy {
  // KairosScheduler::order_key (scheduler.hpp:111-113) over a fixed table.
  PriorityTable table;
  std::string name() const override { return "kairos"; }
  OrderKey order_key(const PendingRequest& r) const override {
    return {table.priority_key(r.agent), r.app_start, r.queue_enter};
  }
};

struct RefPool {
  std::unique_ptr<SchedulerPolicy> policy;
  std::vector<InstanceId> ids;
  std::vector<double> caps, ks;
  std::vector<int> max_batch;
  DispatcherConfig dcfg;
  std::unique_ptr<Dispatcher> pristine_disp, disp;
  std::vector<double> live0, live;
  std::vector<int> running0, running, waiting0, waiting;
  std::map<AgentId, double> T;
  std::vector<PendingRequest> queue0, queue;
  int64_t last_admitted = 0;
  int64_t last_decisions = 0;
  // Decision log of the last tick (engine.cpp:242-246 DecisionLogRow plus
  // DispatchDecision::candidate_peaks), filled only when `record` is set so
  // the timed baseline does not pay for it.
  bool record = false;
  std::vector<uint64_t> log_uid;
  std::vector<int32_t> log_target, log_admitted;
  std::vector<double> log_peak, log_cand;
};

}  // namespace

extern "C" {

// sched_kind: 0 kairos, 1 fcfs, 2 topo_depth, 3 oracle (the latter unused).
void* kxref_pool_new(int n_inst, const int32_t* ids, const double* caps, const double* ks,
                     const int32_t* max_batch, double slot_len, double watermark, int sched_kind,
                     int n_agents, const char* const* agent_names, const double* pk,
                     const uint8_t* pk_known, const int32_t* depth, const double* T) {
  auto* p = new RefPool();
  for (int i = 0; i < n_inst; ++i) {
    p->ids.push_back(ids[i]);
    p->caps.push_back(caps[i]);
    p->ks.push_back(ks[i]);
    p->max_batch.push_back(max_batch[i]);
  }
  p->dcfg.policy = DispatchPolicy::TimeSlot;
  p->dcfg.slot_len = slot_len;
  p->dcfg.resume_watermark = watermark;
  p->pristine_disp = std::make_unique<Dispatcher>(p->dcfg, p->ids, p->caps, p->ks);
  std::map<AgentId, int> depths;
  auto tp = std::make_unique<TablePolicy>();
  tp->table.anchor_coord = 0.0;
  for (int a = 0; a < n_agents; ++a) {
    const std::string name = agent_names[a];
    if (pk_known[a]) tp->table.coord[name] = pk[a];  // |coord - 0| = pk
    depths[name] = depth[a];
    p->T[name] = T[a];
  }
  switch (sched_kind) {
    case 1: p->policy = std::make_unique<FcfsScheduler>(); break;
    case 2: p->policy = std::make_unique<TopoDepthScheduler>(depths); break;
    default: p->policy = std::move(tp); break;
  }
  p->live0.assign(n_inst, 0.0);
  p->running0.assign(n_inst, 0);
  p->waiting0.assign(n_inst, 0);
  return p;
}

void kxref_pool_free(void* h) { delete static_cast<RefPool*>(h); }

void kxref_pool_set_live(void* h, const double* live, const int32_t* running, const int32_t* waiting) {
  auto* p = static_cast<RefPool*>(h);
  p->live0.assign(live, live + p->ids.size());
  p->running0.assign(running, running + p->ids.size());
  p->waiting0.assign(waiting, waiting + p->ids.size());
}

// SlotLedger preload through Dispatcher::commit (dispatcher.cpp:252-262).
int kxref_pool_commit(void* h, int32_t instance_id, uint64_t uid, int64_t prompt, double t0, double T) {
  auto* p = static_cast<RefPool*>(h);
  DispatchDecision d;
  d.request.uid = uid;
  d.request.prompt_tokens = prompt;
  d.target = instance_id;
  try {
    p->pristine_disp->commit(d, t0, T);
  } catch (...) {
    return 1;
  }
  return 0;
}

// Dispatcher::gc on the pre-tick state (the previous round ended at `now`).
void kxref_pool_gc(void* h, double now) { static_cast<RefPool*>(h)->pristine_disp->gc(now); }

// Queue contents; msg ids are "m-<msg_counter>" (MessageIdFactory, types.hpp:46-57).
void kxref_pool_set_queue(void* h, int64_t n, const int32_t* agent, const int64_t* prompt,
                          const double* app, const double* qe, const uint64_t* msg_counter,
                          const uint64_t* uid, const char* const* agent_names) {
  auto* p = static_cast<RefPool*>(h);
  p->queue0.clear();
  p->queue0.reserve(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    PendingRequest r;
    r.msg_id = "m-" + std::to_string(msg_counter[i]);
    r.agent = agent_names[agent[i]];
    r.prompt_tokens = prompt[i];
    r.app_start = app[i];
    r.queue_enter = qe[i];
    r.uid = uid[i];
    p->queue0.push_back(std::move(r));
  }
}

// Untimed: restore the pre-tick state (unsorted queue, pristine ledgers, live).
void kxref_pool_reset(void* h) {
  auto* p = static_cast<RefPool*>(h);
  p->queue = p->queue0;
  p->disp = std::make_unique<Dispatcher>(*p->pristine_disp);
  p->live = p->live0;
  p->running = p->running0;
  p->waiting = p->waiting0;
}

// Timed: one scheduling tick (order + dispatch + gc). Returns admitted count.
int64_t kxref_pool_tick(void* h, double now) {
  auto* p = static_cast<RefPool*>(h);
  const SchedulerPolicy& s = *p->policy;
  p->log_uid.clear();
  p->log_target.clear();
  p->log_admitted.clear();
  p->log_peak.clear();
  p->log_cand.clear();
  std::sort(p->queue.begin(), p->queue.end(), [&](const PendingRequest& a, const PendingRequest& b) {
    const auto ka = s.order_key(a);
    const auto kb = s.order_key(b);
    return std::tie(ka, a.app_start, a.queue_enter, a.msg_id, a.uid) <
           std::tie(kb, b.app_start, b.queue_enter, b.msg_id, b.uid);
  });
  int64_t admitted = 0, decisions = 0;
  const std::size_t ni = p->ids.size();
  std::size_t pos = 0;
  while (pos < p->queue.size()) {
    const PendingRequest& head = p->queue[pos];
    auto it = p->T.find(head.agent);
    const double T = it == p->T.end() ? p->dcfg.default_expected_time : it->second;
    std::vector<InstanceLive> live(ni);
    for (std::size_t i = 0; i < ni; ++i) {
      p->disp->on_live_usage(p->ids[i], p->live[i]);
      live[i].live_kv = p->live[i];
      live[i].running = p->running[i];
      live[i].waiting = p->waiting[i];
      live[i].batch_full = live[i].running + live[i].waiting >= p->max_batch[i];
    }
    DispatchDecision d = p->disp->choose(head, now, T, live);
    ++decisions;
    if (p->record) {
      p->log_uid.push_back(head.uid);
      p->log_target.push_back(d.target ? *d.target : -1);
      p->log_peak.push_back(d.target ? d.predicted_peak : 0.0);
      p->log_admitted.push_back(0);
      for (std::size_t i = 0; i < ni; ++i)
        p->log_cand.push_back(i < d.candidate_peaks.size() ? d.candidate_peaks[i] : -1.0);
    }
    if (!d.target) break;
    const std::size_t ti =
        static_cast<std::size_t>(std::find(p->ids.begin(), p->ids.end(), *d.target) - p->ids.begin());
    if (p->live[ti] + static_cast<double>(head.prompt_tokens) > p->caps[ti]) {
      p->disp->on_overload(*d.target);
      if (decisions > static_cast<int64_t>(p->queue.size() + 4 * ni + 16)) break;  // H6 guard
      continue;
    }
    p->disp->commit(d, now, T);
    if (p->record) p->log_admitted.back() = 1;
    p->live[ti] += static_cast<double>(head.prompt_tokens);
    p->running[ti] += 1;
    ++admitted;
    ++pos;
  }
  p->disp->gc(now);
  p->last_admitted = admitted;
  p->last_decisions = decisions;
  return admitted;
}

int64_t kxref_pool_last_decisions(void* h) { return static_cast<RefPool*>(h)->last_decisions; }

// Decision logging for parity checks (off by default: the timed baseline
// does not record).
void kxref_pool_record(void* h, int on) { static_cast<RefPool*>(h)->record = on != 0; }

// Rows logged by the last tick; copies them out (any pointer may be NULL;
// cand is rows x n_inst, Dispatcher ids_ order).
int64_t kxref_pool_log(void* h, uint64_t* uid, int32_t* target, int32_t* admitted, double* peak,
                       double* cand) {
  auto* p = static_cast<RefPool*>(h);
  const std::size_t n = p->log_uid.size();
  for (std::size_t j = 0; j < n; ++j) {
    if (uid) uid[j] = p->log_uid[j];
    if (target) target[j] = p->log_target[j];
    if (admitted) admitted[j] = p->log_admitted[j];
    if (peak) peak[j] = p->log_peak[j];
  }
  if (cand)
    for (std::size_t j = 0; j < p->log_cand.size(); ++j) cand[j] = p->log_cand[j];
  return static_cast<int64_t>(n);
}

// uids of the queue in the order the last tick sorted it (the reference
// comparator's permutation, harness.cpp:92-100); returns the queue length.
int64_t kxref_pool_order(void* h, uint64_t* uid) {
  auto* p = static_cast<RefPool*>(h);
  if (uid)
    for (std::size_t j = 0; j < p->queue.size(); ++j) uid[j] = p->queue[j].uid;
  return static_cast<int64_t>(p->queue.size());
}

// Ticks `n` pools concurrently on up to `threads` threads (the reference's
// std::async-per-cell model, harness.cpp:189-206); returns wall seconds.
double kxref_pools_tick(void** pools, int n, double now, int threads) {
  for (int i = 0; i < n; ++i) kxref_pool_reset(pools[i]);
  const auto t0 = std::chrono::steady_clock::now();
  if (threads <= 1) {
    for (int i = 0; i < n; ++i) kxref_pool_tick(pools[i], now);
  } else {
    for (int start = 0; start < n; start += threads) {
      std::vector<std::thread> ts;
      for (int i = start; i < std::min(n, start + threads); ++i)
        ts.emplace_back([=] { kxref_pool_tick(pools[i], now); });
      for (auto& t : ts) t.join();
    }
  }
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"

// ---- full replica simulation (tests of the device replica engine) -------
// Runs the reference Simulator (engine.cpp:85-123) on a flattened
// realization whose agents are the built-in template agents, exactly as
// run_cell wires it (harness.cpp:104-150), and returns completion-order
// records, counters and compute_metrics (metrics.cpp:13-88).
#include "kairos/engine.hpp"
#include "kairos/metrics.hpp"
#include "kairos/workflow.hpp"

#ifdef KX_DROPIN
extern "C" void kx_dropin_release(const void* dispatcher);
#endif

namespace {
const char* kBuiltin[10] = {"Router", "Math", "Humanities", "Researcher", "Writer",
                            "ProductManager", "Architect", "ProjectManager", "Engineer", "QAEngineer"};
}

extern "C" int kxref_sim_run(
    int64_t n_wf, const double* arrival, const int64_t* wf_off, const int32_t* agent,
    const int32_t* parent, const int64_t* prompt, const int64_t* target, const double* pure,
    const double* rem, const uint64_t* uid, int n_inst, const int32_t* ids, const double* caps,
    const double* ks, const double* prefill, const int32_t* max_batch, int sched_kind,
    int dispatch_policy, int oracle_T, double slot_len, double watermark, double static_threshold,
    double default_T, double dispatch_period, double recompute_fraction, const int32_t* topo_depth,
    uint64_t* c_uid, double* c_exec_start, double* c_exec_end, int32_t* c_instance,
    double* c_first_enqueue, double* c_queue_seconds, int32_t* c_episodes, int32_t* c_preemptions,
    int64_t* w_index, double* w_finish, int64_t* w_output_tokens, int64_t* w_calls,
    double* scalars, int64_t* n_calls_done, int64_t* n_wf_done, double* pk_out,
    int64_t* table_version_out) {
  try {
    WorkloadRealization real;
    for (int64_t w = 0; w < n_wf; ++w) {
      PlannedInstance inst;
      inst.msg_id = "m-" + std::to_string(w);
      inst.arrival = arrival[w];
      for (int64_t c = wf_off[w]; c < wf_off[w + 1]; ++c) {
        PlannedCall pc;
        pc.node_id = static_cast<int>(c - wf_off[w]);
        pc.agent = kBuiltin[agent[c]];
        if (parent[c] >= 0) pc.parents.push_back(parent[c]);
        pc.prompt_tokens = prompt[c];
        pc.target_tokens = target[c];
        pc.pure_exec = pure[c];
        pc.remaining_exec = rem[c];
        pc.uid = uid[c];
        real.remaining_by_uid[pc.uid] = rem[c];
        inst.calls.push_back(pc);
      }
      inst.entry = inst.calls.empty() ? "" : inst.calls[0].agent;
      real.total_calls += inst.calls.size();
      real.instances.push_back(std::move(inst));
    }
    EngineConfig ecfg;
    std::vector<InstanceId> vid;
    std::vector<double> vcap, vk;
    for (int i = 0; i < n_inst; ++i) {
      InstanceProfile p;
      p.id = ids[i];
      p.capacity_tokens = caps[i];
      p.decode_rate = ks[i];
      p.prefill_rate = prefill[i];
      p.max_batch = max_batch[i];
      ecfg.instances.push_back(p);
      vid.push_back(ids[i]);
      vcap.push_back(caps[i]);
      vk.push_back(ks[i]);
    }
    ecfg.dispatch_period = dispatch_period;
    ecfg.recompute_fraction = recompute_fraction;
    ecfg.default_expected_time = default_T;
    DispatcherConfig dcfg;
    dcfg.policy = static_cast<DispatchPolicy>(dispatch_policy);
    dcfg.slot_len = slot_len;
    dcfg.resume_watermark = watermark;
    dcfg.static_threshold = static_threshold;
    dcfg.default_expected_time = default_T;
    dcfg.oracle_expected_time = oracle_T != 0;
    std::map<AgentId, int> depths;
    for (int a = 0; a < 10; ++a) depths[kBuiltin[a]] = topo_depth[a];
    std::unique_ptr<SchedulerPolicy> sched;
    switch (sched_kind) {
      case 1: sched = std::make_unique<FcfsScheduler>(); break;
      case 2: sched = std::make_unique<TopoDepthScheduler>(depths); break;
      case 3: sched = std::make_unique<OracleScheduler>(&real.remaining_by_uid); break;
      default: {
        KairosSchedulerConfig kc;
        sched = std::make_unique<KairosScheduler>(kc);
      }
    }
    Dispatcher disp(dcfg, vid, vcap, vk);
    LatencyProfiler profiler;
    WorkflowAnalyzer analyzer;
    Simulator sim(ecfg, real, *sched, disp, profiler, analyzer);
    RunResult run = sim.run();
#ifdef KX_DROPIN
    kx_dropin_release(&disp);  // the drop-in build's device state of this Dispatcher
#endif
    for (std::size_t j = 0; j < run.calls.size(); ++j) {
      const auto& c = run.calls[j];
      c_uid[j] = c.uid;
      c_exec_start[j] = c.record.exec_start;
      c_exec_end[j] = c.record.exec_end;
      c_instance[j] = c.instance;
      c_first_enqueue[j] = c.first_enqueue;
      c_queue_seconds[j] = c.queue_seconds;
      c_episodes[j] = c.episodes;
      c_preemptions[j] = c.preemptions;
    }
    for (std::size_t j = 0; j < run.instances.size(); ++j) {
      const auto& w = run.instances[j];
      w_index[j] = std::stoll(w.msg_id.substr(2));
      w_finish[j] = w.finish;
      w_output_tokens[j] = w.output_tokens;
      w_calls[j] = static_cast<int64_t>(w.calls);
    }
    *n_calls_done = static_cast<int64_t>(run.calls.size());
    *n_wf_done = static_cast<int64_t>(run.instances.size());
    const MetricsReport m = compute_metrics("x", 0, run);
    const double s[] = {static_cast<double>(run.preemption_events),
                        static_cast<double>(run.preempted_requests),
                        run.wasted_kv_tokens,
                        run.completed_kv_tokens,
                        run.prefill_seconds,
                        run.decode_seconds,
                        static_cast<double>(run.total_events),
                        run.end_time,
                        m.mean_token_latency,
                        m.p90_token_latency,
                        m.p95_token_latency,
                        m.p99_token_latency,
                        m.mean_request_token_latency,
                        m.mean_queueing_ratio,
                        m.preemption_rate,
                        m.wasted_memory_fraction,
                        m.decode_time_fraction,
                        m.total_queue_seconds};
    for (std::size_t j = 0; j < sizeof(s) / sizeof(s[0]); ++j) scalars[j] = s[j];
    // KairosScheduler's final table (scheduler.hpp:120-122): priority_key per
    // built-in agent index and the table version (= tables built).
    if (const PriorityTable* t = sched->table()) {
      if (pk_out)
        for (int a = 0; a < 10; ++a) pk_out[a] = t->priority_key(kBuiltin[a]);
      if (table_version_out) *table_version_out = static_cast<int64_t>(t->version);
    }
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "kxref_sim_run: %s\n", e.what());
    return 1;
  }
}

// ---- realize() for a general WorkloadConfig (tests of kx_realize) -------
// Builds the reference WorkloadConfig (workload.hpp:69-83) from the C ABI's
// flat description (include/kairos_b200.h kx_workload_config), agent i named
// "a<i>", app k named "app<k>", and runs the reference realize()
// (workload.cpp:319-372). TraceFile arrivals go through a temporary file so
// the reference's own ingest_arrival_trace parses them.
#include <cstdlib>
#include <fstream>
#include <unistd.h>

#include "kairos/workload.hpp"
#include "../include/kairos_b200.h"

namespace {
LengthSpec ref_length(const kx_length_spec& l) {
  LengthSpec s;
  s.kind = static_cast<LengthSpec::Kind>(l.kind);
  s.a = l.a;
  s.b = l.b;
  s.min_tokens = l.min_tokens;
  s.max_tokens = l.max_tokens;
  return s;
}
struct RefRealization {
  std::vector<double> arrival;
  std::vector<int64_t> wf_offsets{0};
  std::vector<int32_t> agent, parent;
  std::vector<int64_t> prompt, target;
  std::vector<double> pure, rem, rem_map;
  std::vector<uint64_t> uid;
  std::string error;
};
}  // namespace

extern "C" void* kxref_realize(const kx_workload_config* c, uint64_t seed, double prefill, double decode) {
  auto* out = new RefRealization();
  std::string trace_path;
  try {
    WorkloadConfig cfg;
    auto name = [](int i) { return "a" + std::to_string(i); };
    for (int k = 0; k < c->n_apps; ++k) {
      AppSpec app;
      app.name = "app" + std::to_string(k);
      app.entry = name(c->apps[k].entry);
      app.weight = c->apps[k].weight;
      for (int j = 0; j < c->apps[k].n_members; ++j) {
        const int i = c->apps[k].members[j];
        const kx_agent_spec& s = c->agents[i];
        AgentSpec a;
        a.name = name(i);
        a.prompt_len = ref_length(s.prompt_len);
        a.output_len = ref_length(s.output_len);
        for (int t = 0; t < s.n_choice; ++t) a.choice.emplace_back(name(s.choice_to[t]), s.choice_p[t]);
        for (int t = 0; t < s.n_parallel; ++t) a.parallel.push_back(name(s.parallel_to[t]));
        if (s.feedback_target >= 0)
          a.feedback = AgentSpec::Feedback{name(s.feedback_target), s.feedback_probability,
                                           s.feedback_max_iterations};
        app.agents.push_back(std::move(a));
      }
      cfg.apps.push_back(std::move(app));
    }
    if (c->arrival_kind == KX_ARRIVAL_TRACE) {
      char tmpl[] = "/tmp/kxref_traceXXXXXX";
      const int fd = mkstemp(tmpl);
      if (fd < 0) throw std::runtime_error("mkstemp");
      close(fd);
      trace_path = tmpl;
      std::FILE* f = std::fopen(tmpl, "w");
      for (int64_t j = 0; j < c->n_trace; ++j) std::fprintf(f, "%.17g\n", c->trace[j]);
      std::fclose(f);
      cfg.arrival.kind = ArrivalSpec::Kind::TraceFile;
      cfg.arrival.path = trace_path;
      cfg.arrival.scale = c->trace_scale;
    } else {
      cfg.arrival.kind = ArrivalSpec::Kind::Poisson;
      cfg.arrival.rate = c->rate;
    }
    cfg.duration = c->duration;
    cfg.seed = seed;
    cfg.entry_selection = c->entry_selection == KX_ENTRY_CYCLE ? WorkloadConfig::EntrySelection::Cycle
                                                               : WorkloadConfig::EntrySelection::Weighted;
    ReferenceRates rates;
    rates.prefill_rate = prefill;
    rates.decode_rate = decode;
    const WorkloadRealization real = realize(cfg, rates, seed);
    for (const auto& inst : real.instances) {
      out->arrival.push_back(inst.arrival);
      for (const auto& call : inst.calls) {
        out->agent.push_back(std::stoi(call.agent.substr(1)));
        out->parent.push_back(call.parents.empty() ? -1 : call.parents[0]);
        out->prompt.push_back(call.prompt_tokens);
        out->target.push_back(call.target_tokens);
        out->pure.push_back(call.pure_exec);
        out->rem.push_back(call.remaining_exec);
        out->uid.push_back(call.uid);
        out->rem_map.push_back(real.remaining_by_uid.at(call.uid));
      }
      out->wf_offsets.push_back(static_cast<int64_t>(out->agent.size()));
    }
  } catch (const std::exception& e) {
    out->error = e.what();
  }
  if (!trace_path.empty()) std::remove(trace_path.c_str());
  return out;
}

// "" on success, else the exception the reference threw.
extern "C" const char* kxref_realize_error(void* h) { return static_cast<RefRealization*>(h)->error.c_str(); }

extern "C" void kxref_realize_sizes(void* h, int64_t* n_wf, int64_t* n_calls) {
  auto* r = static_cast<RefRealization*>(h);
  *n_wf = static_cast<int64_t>(r->arrival.size());
  *n_calls = static_cast<int64_t>(r->agent.size());
}

// rem_map = remaining_by_uid[uid] (must equal remaining_exec).
extern "C" void kxref_realize_copy(void* h, double* arrival, int64_t* wf_offsets, int32_t* agent,
                                   int32_t* parent, int64_t* prompt, int64_t* target, double* pure,
                                   double* rem, uint64_t* uid, double* rem_map) {
  auto* r = static_cast<RefRealization*>(h);
  auto cp = [](auto* dst, const auto& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
  };
  cp(arrival, r->arrival);
  cp(wf_offsets, r->wf_offsets);
  cp(agent, r->agent);
  cp(parent, r->parent);
  cp(prompt, r->prompt);
  cp(target, r->target);
  cp(pure, r->pure);
  cp(rem, r->rem);
  cp(uid, r->uid);
  cp(rem_map, r->rem_map);
}

extern "C" void kxref_realize_free(void* h) { delete static_cast<RefRealization*>(h); }

// ---- trace CSV + workflow reconstruction (tests of kx_trace_* / workflow) --
// read_trace (trace.cpp:111-127) of a byte buffer; WorkflowAnalyzer's
// ingest_trace + the graph's report(), topo_depth and downstream_paths per
// node; write_trace of the parsed records. Errors come back as the
// reference's exception text with a negative length.
#include <sstream>

#include "kairos/trace.hpp"
#include "kairos/workflow.hpp"

namespace {
int64_t put_text(const std::string& s, char* out, int64_t cap) {
  const int64_t n = static_cast<int64_t>(s.size());
  if (out && cap >= n) std::memcpy(out, s.data(), s.size());
  return n;
}
}  // namespace

extern "C" int64_t kxref_trace_report(const char* bytes, int64_t n, int max_loop, char* out, int64_t cap) {
  try {
    std::istringstream in(std::string(bytes, static_cast<size_t>(n)));
    const auto recs = read_trace(in);
    WorkflowAnalyzer a;
    a.ingest_trace(recs);
    const auto g = a.snapshot();
    std::string s = g->report();
    for (const auto& node : g->nodes()) {
      s += "depth " + node + " " + std::to_string(g->topo_depth(node)) + "\n";
      for (const auto& p : g->downstream_paths(node, max_loop)) {
        s += "path " + node + ":";
        for (const auto& x : p) s += " " + x;
        s += "\n";
      }
    }
    return put_text(s, out, cap);
  } catch (const std::exception& e) {
    return -put_text(e.what(), out, cap) - 1;
  }
}

extern "C" int64_t kxref_trace_write(const char* bytes, int64_t n, char* out, int64_t cap) {
  try {
    std::istringstream in(std::string(bytes, static_cast<size_t>(n)));
    std::ostringstream o;
    write_trace(o, read_trace(in));
    return put_text(o.str(), out, cap);
  } catch (const std::exception& e) {
    return -put_text(e.what(), out, cap) - 1;
  }
}

extern "C" int64_t kxref_trace_columns(const char* bytes, int64_t n, int64_t cap, double* es, double* ee,
                                       double* as, int64_t* pt, int64_t* ot) {
  std::istringstream in(std::string(bytes, static_cast<size_t>(n)));
  const auto recs = read_trace(in);
  for (size_t i = 0; i < recs.size() && static_cast<int64_t>(i) < cap; ++i) {
    es[i] = recs[i].exec_start;
    ee[i] = recs[i].exec_end;
    as[i] = recs[i].app_start;
    pt[i] = recs[i].prompt_tokens;
    ot[i] = recs[i].output_tokens;
  }
  return static_cast<int64_t>(recs.size());
}

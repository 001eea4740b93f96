// TEST INFRASTRUCTURE ONLY: the drop-in proof.
//
// Linked into oracle/_ref/libkxdropin.so (and the reference's own
// test_engine suite, oracle/_ref/test_engine_dropin) together with the
// UNMODIFIED reference sources, compiled by oracle/Makefile with one
// section per function. objcopy weakens the reference's
// Simulator::dispatch_loop (engine.cpp:220-268) and the Dispatcher's event
// methods (dispatcher.cpp:264-297) and adds kx_ref_* aliases of the
// original definitions; the strong definitions below take their place:
//
//   * under the time-slot policy the dispatch round runs on the B200 through
//     kairos_b200::DeviceScheduler (include/kairos_b200.hpp over the C ABI
//     of libkairos_b200.so): the ReadyQueue's entries are uploaded with the
//     active SchedulerPolicy's keys, one kx_tick orders them and places the
//     heads against the device-resident ledgers, and the decision log is
//     applied to the Simulator exactly as the reference loop applies its own
//     decisions (log row, overload retry, ReadyQueue::pop, admit);
//   * the Dispatcher's ledger events (finish, preemption, overload, live
//     usage, gc) go to the device-resident Dispatcher state;
//   * the other dispatch policies run the reference's own code.
//
// The reference Simulator is otherwise untouched: events, admission,
// preemption, profiling and metrics are its own code. Comparing its
// RunResult with the stock build's (tests/test_dropin_sim.py) checks the
// device path as a drop-in for the reference's in-process operator API.
#include <cstdio>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "kairos/dispatcher.hpp"
#include "kairos/engine.hpp"
#include "kairos/scheduler.hpp"
#include "kairos_b200.hpp"

extern "C" {
// aliases of the original (weakened) definitions, added by oracle/Makefile
void kx_ref_dispatch_loop(kairos::Simulator* self);
void kx_ref_on_request_finished(kairos::Dispatcher* self, int instance, uint64_t uid, double t);
void kx_ref_on_request_preempted(kairos::Dispatcher* self, int instance, uint64_t uid, double t);
void kx_ref_on_overload(kairos::Dispatcher* self, int instance);
void kx_ref_on_live_usage(kairos::Dispatcher* self, int instance, double live_kv);
void kx_ref_gc(kairos::Dispatcher* self, double now);
}

namespace {

// The device-resident Dispatcher of one reference Dispatcher object.
struct DeviceDispatcher {
  std::unique_ptr<kairos_b200::DeviceScheduler> sched;
  double last_clock = -1.0;
  uint64_t last_events = 0;
};

std::mutex g_mu;
std::map<const kairos::Dispatcher*, std::unique_ptr<DeviceDispatcher>> g_dev;

DeviceDispatcher* device_of(const kairos::Dispatcher* d) {
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_dev.find(d);
  return it == g_dev.end() ? nullptr : it->second.get();
}

int32_t scheduler_kind(const std::string& name) {
  if (name == "fcfs") return KX_SCHED_FCFS;
  if (name == "topo_depth") return KX_SCHED_TOPO;
  if (name == "oracle") return KX_SCHED_ORACLE;
  return KX_SCHED_KAIROS;
}

}  // namespace

// Ends the device state of a Dispatcher (called by ref_bridge.cpp after a
// run; a later Dispatcher at the same address starts fresh).
extern "C" void kx_dropin_release(const void* dispatcher) {
  std::lock_guard<std::mutex> lock(g_mu);
  g_dev.erase(static_cast<const kairos::Dispatcher*>(dispatcher));
}

namespace kairos {

// ---- Dispatcher events -> the device-resident ledgers / suspension --------
void Dispatcher::on_request_finished(InstanceId instance, std::uint64_t uid, double actual_end) {
  if (auto* d = device_of(this)) d->sched->on_request_finished(instance, uid, actual_end);
  else kx_ref_on_request_finished(this, instance, uid, actual_end);
}

void Dispatcher::on_request_preempted(InstanceId instance, std::uint64_t uid, double now) {
  if (auto* d = device_of(this)) d->sched->on_request_preempted(instance, uid, now);
  else kx_ref_on_request_preempted(this, instance, uid, now);
}

void Dispatcher::on_overload(InstanceId instance) {
  if (auto* d = device_of(this)) d->sched->on_overload(instance);
  else kx_ref_on_overload(this, instance);
}

void Dispatcher::on_live_usage(InstanceId instance, double live_kv) {
  if (auto* d = device_of(this)) d->sched->on_live_usage(instance, live_kv);
  else kx_ref_on_live_usage(this, instance, live_kv);
}

void Dispatcher::gc(double now) {
  if (auto* d = device_of(this)) d->sched->gc(now);
  else kx_ref_gc(this, now);
}

// ---- Simulator::dispatch_loop on the device (time-slot policy) ------------
void Simulator::dispatch_loop() {
  const DispatcherConfig& dc = dispatcher_.config();
  if (dc.policy != DispatchPolicy::TimeSlot) {
    kx_ref_dispatch_loop(this);
    return;
  }
  DeviceDispatcher* dev = device_of(&dispatcher_);
  // a Dispatcher reused by a new run (same address, clock or event count
  // went back) starts fresh
  if (dev && (clock_ < dev->last_clock || result_.total_events < dev->last_events)) {
    kx_dropin_release(&dispatcher_);
    dev = nullptr;
  }
  if (!dev) {
    kairos_b200::DispatcherConfig cfg;
    cfg.policy = KX_DISPATCH_TIME_SLOT;
    cfg.slot_len = dc.slot_len;
    cfg.resume_watermark = dc.resume_watermark;
    cfg.static_threshold = dc.static_threshold;
    cfg.default_expected_time = dc.default_expected_time;
    cfg.oracle_expected_time = dc.oracle_expected_time;
    std::vector<kairos_b200::InstanceProfile> inst;
    for (const auto& s : instances_) {
      kairos_b200::InstanceProfile p;
      p.id = s.profile.id;
      p.pool = 0;
      p.capacity_tokens = s.profile.capacity_tokens;
      p.decode_rate = s.profile.decode_rate;
      p.prefill_rate = s.profile.prefill_rate;
      p.max_batch = s.profile.max_batch;
      inst.push_back(p);
    }
    auto d = std::make_unique<DeviceDispatcher>();
    const int64_t cap = std::max<int64_t>(1 << 16, static_cast<int64_t>(calls_.size()) + 1);
    d->sched = std::make_unique<kairos_b200::DeviceScheduler>(cfg, inst, 1, cap);
    d->sched->set_scheduler(scheduler_kind(scheduler_.name()));
    std::lock_guard<std::mutex> lock(g_mu);
    dev = (g_dev[&dispatcher_] = std::move(d)).get();
  }
  dev->last_clock = clock_;
  dev->last_events = result_.total_events;
  if (queue_.empty()) return;
  kairos_b200::DeviceScheduler& s = *dev->sched;

  // The SchedulerPolicy's keys for this round (the reference consults the
  // latest table at dequeue time, priority.hpp:66-69): per agent for the
  // table policies, per request for the oracle; expected T per agent
  // (engine.cpp:177-185) or per request under oracle_expected_time.
  const std::vector<PendingRequest> q = queue_.entries();
  const std::string kind = scheduler_.name();
  std::set<AgentId> agents;
  for (const auto& r : q) agents.insert(r.agent);
  std::map<std::string, double> keys, T;
  std::map<std::string, int> depth;
  for (const auto& a : agents) {
    s.register_agent(a, 0);
    PendingRequest probe;
    probe.agent = a;
    const OrderKey k = scheduler_.order_key(probe);
    if (kind == "kairos") keys[a] = k.k0;
    if (kind == "topo_depth") depth[a] = static_cast<int>(k.k0);
    if (!dc.oracle_expected_time) T[a] = expected_exec_time(probe);
  }
  s.set_agent_keys(keys);
  s.set_topo_depths(depth);
  s.set_expected_times(T);
  std::vector<int64_t> kept;
  std::vector<double> pure;
  std::map<uint64_t, double> rem;
  for (const auto& r : q) {
    const CallRuntime& c = calls_.at(r.uid);
    kept.push_back(c.kept_tokens);
    if (dc.oracle_expected_time) pure.push_back(c.plan->pure_exec);
    if (kind == "oracle") rem[r.uid] = scheduler_.order_key(r).k0;
  }
  if (kind == "oracle") s.set_remaining(rem);
  std::vector<double> live;
  std::vector<int32_t> running, waiting;
  for (const auto& inst : instances_) {
    live.push_back(inst.live_kv);
    running.push_back(static_cast<int32_t>(inst.running.size()));
    waiting.push_back(static_cast<int32_t>(inst.waiting.size()));
  }
  s.set_live(live, running, waiting);
  s.upload(q, &kept, dc.oracle_expected_time ? &pure : nullptr);

  // One device round: ReadyQueue order + every placement of the round.
  const std::vector<kairos_b200::DecisionLogRow> rows = s.dispatch_round(clock_);

  // Apply it as the reference loop applies its decisions (engine.cpp:240-262).
  std::set<uint64_t> popped;
  std::map<uint64_t, std::size_t> index;
  for (std::size_t i = 0; i < q.size(); ++i) index[q[i].uid] = i;
  for (const auto& row : rows) {
    if (cfg_.collect_decision_log) {
      DecisionLogRow d;
      d.time = clock_;
      d.uid = row.uid;
      d.agent = row.agent;
      if (row.target) d.target = *row.target;
      d.predicted_peak = row.predicted_peak;
      d.candidate_peaks = row.candidate_peaks;
      result_.decisions.push_back(std::move(d));
    }
    if (!row.target) break;      // the head keeps its place until the next round
    if (!row.admitted) continue;  // overload: the device suspended the target, same head again
    admit(state_of(*row.target), q[index.at(row.uid)]);
    popped.insert(row.uid);
  }
  if (!popped.empty()) {  // ReadyQueue::pop of the admitted heads, the rest keep their order
    ReadyQueue rest;
    for (const auto& r : q)
      if (!popped.count(r.uid)) rest.enqueue(r);
    queue_ = std::move(rest);
  }
}

}  // namespace kairos

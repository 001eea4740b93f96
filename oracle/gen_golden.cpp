// TEST INFRASTRUCTURE ONLY. Generates the golden fixtures in tests/golden/
// by running the UNMODIFIED reference (built from /root/reference/proj by
// oracle/Makefile) through its own public API:
//   order_*.kxf     ReadyQueue::pop order / harness.cpp:92-100 comparator sort
//                   and SchedulerPolicy::order_key for all four policies
//   dispatch_*.kxf  multi-round dispatch_loop restatement over the reference's
//                   Dispatcher / ReadyQueue / SchedulerPolicy (engine.cpp:220-268)
//   dp_*.kxf        realize() -> finalize_instance uid / pure_exec / remaining
//   remaining.kxf   LatencyProfiler::record_remaining samples
//   stats.kxf       quantile_sorted / mode_estimate / median anchor distance
// Usage: gen_golden <out_dir>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "kairos/dispatcher.hpp"
#include "kairos/distribution.hpp"
#include "kairos/priority.hpp"
#include "kairos/profiler.hpp"
#include "kairos/rng.hpp"
#include "kairos/scheduler.hpp"
#include "kairos/workload.hpp"

using namespace kairos;

namespace {

// ---- KXF1 writer: named 1-D little-endian arrays --------------------------
struct Kxf {
  std::vector<std::pair<std::string, std::pair<char, std::vector<unsigned char>>>> items;
  template <typename T>
  void put(const std::string& name, char code, const std::vector<T>& v) {
    std::vector<unsigned char> bytes(v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(bytes.data(), v.data(), bytes.size());
    items.push_back({name, {code, std::move(bytes)}});
  }
  void f64(const std::string& n, const std::vector<double>& v) { put(n, 'f', v); }
  void i64(const std::string& n, const std::vector<int64_t>& v) { put(n, 'q', v); }
  void u64(const std::string& n, const std::vector<uint64_t>& v) { put(n, 'Q', v); }
  void i32(const std::string& n, const std::vector<int32_t>& v) { put(n, 'i', v); }
  void u32(const std::string& n, const std::vector<uint32_t>& v) { put(n, 'I', v); }
  void u8(const std::string& n, const std::vector<uint8_t>& v) { put(n, 'B', v); }
  void scalar_i(const std::string& n, int64_t x) { i64(n, std::vector<int64_t>{x}); }
  void scalar_f(const std::string& n, double x) { f64(n, std::vector<double>{x}); }
  void write(const std::string& path) const {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("cannot write " + path);
    std::fwrite("KXF1", 1, 4, f);
    const uint32_t count = static_cast<uint32_t>(items.size());
    std::fwrite(&count, 4, 1, f);
    for (const auto& [name, data] : items) {
      const uint32_t nl = static_cast<uint32_t>(name.size());
      std::fwrite(&nl, 4, 1, f);
      std::fwrite(name.data(), 1, nl, f);
      std::fwrite(&data.first, 1, 1, f);
      const uint64_t nb = data.second.size();
      std::fwrite(&nb, 8, 1, f);
      if (nb) std::fwrite(data.second.data(), 1, nb, f);
    }
    std::fclose(f);
  }
};

// Agent/msg interning shared by a fixture.
struct Names {
  std::vector<std::string> agents;
  std::map<std::string, int32_t> agent_idx;
  int32_t agent(const std::string& a) {
    auto it = agent_idx.find(a);
    if (it != agent_idx.end()) return it->second;
    const int32_t i = static_cast<int32_t>(agents.size());
    agents.push_back(a);
    agent_idx[a] = i;
    return i;
  }
};

// msg_key = rank of the msg_id string among the distinct ids (lexicographic,
// types.hpp:51 / SURVEY H1).
std::vector<uint64_t> msg_keys(const std::vector<PendingRequest>& q) {
  std::vector<std::string> ids;
  for (const auto& r : q) ids.push_back(r.msg_id);
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  std::vector<uint64_t> out;
  for (const auto& r : q)
    out.push_back(static_cast<uint64_t>(std::lower_bound(ids.begin(), ids.end(), r.msg_id) - ids.begin()));
  return out;
}

struct QueueFixture {
  std::vector<PendingRequest> q;
  std::vector<int32_t> pool_of;  // per request
};

void put_queue(Kxf& k, Names& names, const std::vector<PendingRequest>& q, const std::string& pre = "") {
  std::vector<int32_t> agent;
  std::vector<int64_t> prompt;
  std::vector<double> app, qe;
  std::vector<uint64_t> uid;
  for (const auto& r : q) {
    agent.push_back(names.agent(r.agent));
    prompt.push_back(r.prompt_tokens);
    app.push_back(r.app_start);
    qe.push_back(r.queue_enter);
    uid.push_back(r.uid);
  }
  k.i32(pre + "agent", agent);
  k.i64(pre + "prompt", prompt);
  k.f64(pre + "app_start", app);
  k.f64(pre + "queue_enter", qe);
  k.u64(pre + "msg_key", msg_keys(q));
  k.u64(pre + "uid", uid);
}

// Reference order of one pool's queue: ReadyQueue::pop repeatedly (small),
// or std::sort with the harness.cpp:92-100 comparator (large).
std::vector<std::size_t> reference_order(const std::vector<PendingRequest>& q,
                                         const SchedulerPolicy& s, bool use_pop) {
  auto key = [&](const PendingRequest& r) { return s.order_key(r); };
  std::vector<std::size_t> idx(q.size());
  for (std::size_t i = 0; i < q.size(); ++i) idx[i] = i;
  if (use_pop) {
    // Tag each request with its index via uid lookup (uids unique here).
    std::map<uint64_t, std::size_t> where;
    for (std::size_t i = 0; i < q.size(); ++i) where[q[i].uid] = i;
    ReadyQueue rq;
    for (const auto& r : q) rq.enqueue(r);
    std::vector<std::size_t> out;
    while (!rq.empty()) out.push_back(where.at(rq.pop(key).uid));
    return out;
  }
  std::stable_sort(idx.begin(), idx.end(), [&](std::size_t ia, std::size_t ib) {
    const auto& a = q[ia];
    const auto& b = q[ib];
    const auto ka = s.order_key(a);
    const auto kb = s.order_key(b);
    return std::tie(ka, a.app_start, a.queue_enter, a.msg_id, a.uid) <
           std::tie(kb, b.app_start, b.queue_enter, b.msg_id, b.uid);
  });
  return idx;
}

// Priority table built the reference way: W1 matrix over per-agent
// remaining samples + 1-D MDS (priority.cpp:60-112).
PriorityTable table_from_samples(const std::map<AgentId, std::vector<double>>& samples) {
  std::map<AgentId, std::vector<double>> sorted;
  for (auto [a, v] : samples) {
    std::sort(v.begin(), v.end());
    sorted[a] = v;
  }
  return mds_embed_1d(build_distance_matrix_from_samples(sorted), 1);
}

// A realize()-based queue snapshot: every call of the first
// workflows, queue_enter = app_start + sum of ancestors' pure_exec.
std::vector<PendingRequest> snapshot_queue(const WorkloadRealization& real, std::size_t n) {
  std::vector<PendingRequest> q;
  for (const auto& inst : real.instances) {
    std::vector<double> enter(inst.calls.size(), inst.arrival);
    for (const auto& c : inst.calls) {
      if (!c.parents.empty()) {
        const auto& p = inst.calls[static_cast<std::size_t>(c.parents[0])];
        enter[static_cast<std::size_t>(c.node_id)] = enter[static_cast<std::size_t>(p.node_id)] + p.pure_exec;
      }
      PendingRequest r;
      r.msg_id = inst.msg_id;
      r.agent = c.agent;
      r.prompt_tokens = c.prompt_tokens;
      r.app_start = inst.arrival;
      r.queue_enter = enter[static_cast<std::size_t>(c.node_id)];
      r.uid = c.uid;
      q.push_back(r);
      if (q.size() >= n) return q;
    }
  }
  return q;
}

void write_order_fixture(const std::string& dir, const std::string& name,
                         const std::vector<PendingRequest>& q, const std::vector<int32_t>& pool_of_req,
                         int n_pools, bool use_pop, const PriorityTable& table,
                         const std::map<AgentId, int>& depths,
                         const std::map<uint64_t, double>& remaining) {
  Names names;
  Kxf k;
  put_queue(k, names, q);
  // agent -> pool (all requests of an agent share a pool)
  std::vector<int32_t> agent_pool(names.agents.size(), 0);
  for (std::size_t i = 0; i < q.size(); ++i) agent_pool[names.agent_idx[q[i].agent]] = pool_of_req[i];
  std::vector<double> pk;
  std::vector<int32_t> depth;
  for (const auto& a : names.agents) {
    pk.push_back(table.priority_key(a));
    auto it = depths.find(a);
    depth.push_back(it == depths.end() ? 1 : it->second);
  }
  k.i32("agent_pool", agent_pool);
  k.f64("pk", pk);
  k.i32("depth", depth);
  k.scalar_i("n_pools", n_pools);
  // dense remaining table over the uid range of the queue
  uint64_t lo = UINT64_MAX, hi = 0;
  for (const auto& r : q) {
    lo = std::min(lo, r.uid);
    hi = std::max(hi, r.uid);
  }
  if (q.empty()) lo = hi = 0;
  std::vector<double> rem(hi - lo + 1, 0.0);
  std::vector<uint8_t> present(hi - lo + 1, 0);
  for (uint64_t u = lo; u <= hi; ++u) {
    auto it = remaining.find(u);
    if (it != remaining.end()) {
      rem[u - lo] = it->second;
      present[u - lo] = 1;
    }
  }
  k.scalar_i("rem_base", static_cast<int64_t>(lo));
  k.f64("rem", rem);
  k.u8("rem_present", present);

  KairosScheduler kairos;
  // Inject the table through the public rebuild path is not possible; use a
  // key lambda with the same semantics as KairosScheduler::order_key
  // (scheduler.hpp:111-113) over `table`.
  struct TableKairos : SchedulerPolicy {
    const PriorityTable* t;
    std::string name() const override { return "kairos"; }
    OrderKey order_key(const PendingRequest& r) const override {
      return {t->priority_key(r.agent), r.app_start, r.queue_enter};
    }
  } kz;
  kz.t = &table;
  FcfsScheduler fcfs;
  TopoDepthScheduler topo(depths);
  OracleScheduler oracle(&remaining);
  const SchedulerPolicy* pols[4] = {&kz, &fcfs, &topo, &oracle};
  const char* pnames[4] = {"kairos", "fcfs", "topo_depth", "oracle"};
  for (int pi = 0; pi < 4; ++pi) {
    std::vector<uint32_t> perm;
    std::vector<int64_t> offs(1, 0);
    for (int p = 0; p < n_pools; ++p) {
      std::vector<PendingRequest> sub;
      std::vector<uint32_t> back;
      for (std::size_t i = 0; i < q.size(); ++i)
        if (pool_of_req[i] == p) {
          sub.push_back(q[i]);
          back.push_back(static_cast<uint32_t>(i));
        }
      for (std::size_t j : reference_order(sub, *pols[pi], use_pop)) perm.push_back(back[j]);
      offs.push_back(static_cast<int64_t>(perm.size()));
    }
    std::vector<double> k0, k1, k2;
    for (const auto& r : q) {
      const OrderKey ok = pols[pi]->order_key(r);
      k0.push_back(ok.k0);
      k1.push_back(ok.k1);
      k2.push_back(ok.k2);
    }
    k.u32(std::string(pnames[pi]) + ".perm", perm);
    k.i64(std::string(pnames[pi]) + ".pool_offsets", offs);
    k.f64(std::string(pnames[pi]) + ".k0", k0);
    k.f64(std::string(pnames[pi]) + ".k1", k1);
    k.f64(std::string(pnames[pi]) + ".k2", k2);
  }
  k.write(dir + "/" + name);
  std::printf("  %s: %zu requests, %d pools, %zu agents\n", name.c_str(), q.size(), n_pools,
              names.agents.size());
}

PendingRequest req(const std::string& msg, const std::string& agent, double app, double qe,
                   uint64_t uid, int64_t prompt = 10) {
  PendingRequest r;
  r.msg_id = msg;
  r.agent = agent;
  r.prompt_tokens = prompt;
  r.app_start = app;
  r.queue_enter = qe;
  r.uid = uid;
  return r;
}

void gen_order(const std::string& dir) {
  // (1) tests/test_priority.cpp:179-234 cases, one pool.
  {
    std::map<AgentId, std::vector<double>> s{{"Router", {1.0}}, {"Math", {6.0}}};
    const PriorityTable t = table_from_samples(s);
    std::vector<PendingRequest> q{req("m-0", "Math", 5.0, 5.0, 1), req("m-1", "Router", 9.0, 9.0, 2),
                                  req("m-1", "Math", 7.0, 10.0, 3), req("m-0", "Math", 3.0, 11.0, 4),
                                  req("m-2", "C", 3.0, 3.0, 5), req("m-0", "A", 1.0, 2.0, 10),
                                  req("m-0", "A", 1.0, 2.0, 11), req("m-10", "A", 1.0, 2.0, 12),
                                  req("m-9", "A", 1.0, 2.0, 13)};
    write_order_fixture(dir, "order_unit.kxf", q, std::vector<int32_t>(q.size(), 0), 1, true, t,
                        {{"Router", 2}, {"Math", 1}}, {{1, 4.0}, {2, 1.0}, {3, 4.0}});
  }
  // (2) random ties / lexicographic traps / cold-start agents, 3 pools.
  {
    Rng rng(20250806);
    const int A = 12;
    std::map<AgentId, std::vector<double>> s;
    std::map<AgentId, int> depths;
    for (int a = 0; a < A - 3; ++a) {  // last 3 agents unknown to the table
      std::vector<double> v;
      const int nv = 1 + static_cast<int>(rng.next_u64() % 5);
      for (int j = 0; j < nv; ++j) v.push_back(std::floor(rng.uniform(0.0, 6.0) * 4.0) / 4.0);
      s["ag" + std::to_string(a)] = v;
      depths["ag" + std::to_string(a)] = 1 + static_cast<int>(rng.next_u64() % 4);
    }
    // two agents with identical distributions -> equal priority keys
    s["ag7"] = s["ag3"];
    const PriorityTable t = table_from_samples(s);
    std::vector<PendingRequest> q;
    std::vector<int32_t> pool;
    std::map<uint64_t, double> rem;
    for (int i = 0; i < 600; ++i) {
      const int a = static_cast<int>(rng.next_u64() % A);
      const int m = static_cast<int>(rng.next_u64() % 40);
      const double app = std::floor(rng.uniform(0.0, 5.0) * 2.0) / 2.0;  // coarse: many ties
      const double qe = app + std::floor(rng.uniform(0.0, 3.0) * 2.0) / 2.0;
      const uint64_t uid = 1000 + rng.next_u64() % 100000;
      q.push_back(req("m-" + std::to_string(m), "ag" + std::to_string(a), app, qe, uid,
                      1 + static_cast<int64_t>(rng.next_u64() % 200)));
      pool.push_back(a % 3);
      if (rng.uniform() < 0.8) rem[uid] = std::floor(rng.uniform(0.0, 8.0) * 2.0) / 2.0;
    }
    // make uids unique (ReadyQueue fixture uses uid to identify pops)
    std::set<uint64_t> seen;
    for (auto& r : q) {
      while (!seen.insert(r.uid).second) ++r.uid;
    }
    write_order_fixture(dir, "order_ties.kxf", q, pool, 3, true, t, depths, rem);
  }
  // (3) realize() snapshot, co-located QA+RG+CG, larger.
  for (uint64_t seed : {1ull, 2ull}) {
    const auto cfg = colocated_workload(400.0, 10.0, seed);
    const auto real = realize(cfg, ReferenceRates{8000.0, 50.0}, seed);
    const auto q = snapshot_queue(real, 12000);
    std::map<AgentId, std::vector<double>> samples;
    for (const auto& inst : real.instances)
      for (const auto& c : inst.calls)
        if (c.agent != "Humanities" && samples[c.agent].size() < 64) samples[c.agent].push_back(c.remaining_exec);
    samples.erase("Humanities");  // left out -> cold-start median
    const PriorityTable t = table_from_samples(samples);
    write_order_fixture(dir, "order_colocated_s" + std::to_string(seed) + ".kxf", q,
                        std::vector<int32_t>(q.size(), 0), 1, false, t, topo_depths(cfg),
                        real.remaining_by_uid);
  }
}

// ---- dispatch: multi-round dispatch_loop restatement -------------------------
struct PoolSim {
  std::vector<InstanceId> ids;
  std::vector<double> cap, k;
  std::vector<int> max_batch;
  std::vector<double> live;
  std::vector<int> running, waiting;
};

void gen_dispatch(const std::string& dir, const std::string& name, uint64_t seed, int n_inst,
                  int max_batch, double cap, int rounds, int per_round, double prompt_hi,
                  bool preload) {
  Rng rng(seed);
  DispatcherConfig dcfg;
  dcfg.policy = DispatchPolicy::TimeSlot;
  PoolSim ps;
  for (int i = 0; i < n_inst; ++i) {
    ps.ids.push_back(10 + 3 * i);  // ids not equal to indices
    ps.cap.push_back(cap * (i % 3 == 2 ? 0.8 : 1.0));
    ps.k.push_back(i % 2 ? 40.0 : 50.0);
    ps.max_batch.push_back(max_batch);
  }
  ps.live.assign(n_inst, 0.0);
  ps.running.assign(n_inst, 0);
  ps.waiting.assign(n_inst, 0);
  Dispatcher disp(dcfg, ps.ids, ps.cap, ps.k);
  FcfsScheduler sched;  // order is not under test here; FCFS keys
  auto key = [&](const PendingRequest& r) { return sched.order_key(r); };

  Names names;
  const int A = 5;
  std::vector<double> T_agent;
  for (int a = 0; a < A; ++a) {
    names.agent("d" + std::to_string(a));
    T_agent.push_back(0.3 + 1.7 * a + rng.uniform(0.0, 0.4));
  }
  Kxf k;
  k.scalar_i("n_inst", n_inst);
  k.i32("inst_id", std::vector<int32_t>(ps.ids.begin(), ps.ids.end()));
  k.f64("inst_cap", ps.cap);
  k.f64("inst_k", ps.k);
  k.i32("inst_max_batch", std::vector<int32_t>(ps.max_batch.begin(), ps.max_batch.end()));
  k.f64("agent_T", T_agent);
  k.scalar_i("rounds", rounds);

  // Preloaded ledgers: commits before round 0.
  std::vector<int64_t> pre_inst;
  std::vector<uint64_t> pre_uid;
  std::vector<double> pre_P, pre_t0, pre_T;
  if (preload) {
    for (int j = 0; j < 3 * n_inst; ++j) {
      const int i = static_cast<int>(rng.next_u64() % n_inst);
      const double P = std::floor(rng.uniform(20.0, cap * 0.2));
      const double t0 = rng.uniform(0.0, 1.0);
      const double T = rng.uniform(0.5, 6.0);
      const MemoryModel m{P, ps.k[i], t0, T};
      const uint64_t uid = 900000 + j;
      if (!disp.ledger(ps.ids[i]).try_place(m).fits) continue;
      // Dispatcher::commit uses the instance's k; book via a decision.
      DispatchDecision d;
      d.request = req("pre", "d0", 0, 0, uid, static_cast<int64_t>(P));
      d.target = ps.ids[i];
      disp.commit(d, t0, T);
      pre_inst.push_back(ps.ids[i]);
      pre_uid.push_back(uid);
      pre_P.push_back(P);
      pre_t0.push_back(t0);
      pre_T.push_back(T);
    }
  }
  k.i64("pre_inst", pre_inst);
  k.u64("pre_uid", pre_uid);
  k.f64("pre_P", pre_P);
  k.f64("pre_t0", pre_t0);
  k.f64("pre_T", pre_T);

  std::vector<PendingRequest> queue;
  uint64_t next_uid = 1;
  double now = 1.0;
  struct Running {
    InstanceId inst;
    uint64_t uid;
    double start;
    int64_t kv;
  };
  std::vector<Running> live_reqs;
  for (int r = 0; r < rounds; ++r) {
    const std::string R = "r" + std::to_string(r) + ".";
    // arrivals
    for (int j = 0; j < per_round; ++j) {
      const int a = static_cast<int>(rng.next_u64() % A);
      PendingRequest p = req("m-" + std::to_string(next_uid), "d" + std::to_string(a),
                             now - rng.uniform(0.0, 2.0), now - rng.uniform(0.0, 0.5), next_uid,
                             1 + static_cast<int64_t>(rng.next_u64() % static_cast<uint64_t>(prompt_hi)));
      ++next_uid;
      queue.push_back(p);
    }
    // engine-side live state at round start
    k.scalar_f(R + "now", now);
    k.f64(R + "live_kv", ps.live);
    k.i32(R + "running", std::vector<int32_t>(ps.running.begin(), ps.running.end()));
    k.i32(R + "waiting", std::vector<int32_t>(ps.waiting.begin(), ps.waiting.end()));
    put_queue(k, names, queue, R + "q.");
    // order (FCFS keys) and the dispatch loop, engine.cpp:220-268
    std::vector<double> dec_time, dec_peak, dec_cand;
    std::vector<uint64_t> dec_uid;
    std::vector<int32_t> dec_target, dec_admitted;
    ReadyQueue rq;
    for (const auto& p : queue) rq.enqueue(p);
    while (!rq.empty()) {
      const std::size_t idx = rq.best_index(key);
      const PendingRequest head = rq.entries()[idx];
      const double T = T_agent[static_cast<std::size_t>(names.agent(head.agent))];
      std::vector<InstanceLive> live;
      for (int i = 0; i < n_inst; ++i) {
        disp.on_live_usage(ps.ids[i], ps.live[i]);
        InstanceLive l;
        l.live_kv = ps.live[i];
        l.running = ps.running[i];
        l.waiting = ps.waiting[i];
        l.batch_full = l.running + l.waiting >= ps.max_batch[i];
        live.push_back(l);
      }
      DispatchDecision d = disp.choose(head, now, T, live);
      dec_time.push_back(now);
      dec_uid.push_back(head.uid);
      dec_target.push_back(d.target ? *d.target : -1);
      dec_peak.push_back(d.predicted_peak);
      for (double c : d.candidate_peaks) dec_cand.push_back(c);
      if (!d.target) {
        dec_admitted.push_back(0);
        break;
      }
      const int ti = static_cast<int>(std::find(ps.ids.begin(), ps.ids.end(), *d.target) - ps.ids.begin());
      if (ps.live[ti] + static_cast<double>(head.prompt_tokens) > ps.cap[ti]) {
        disp.on_overload(*d.target);
        dec_admitted.push_back(0);
        continue;
      }
      dec_admitted.push_back(1);
      PendingRequest popped = rq.pop(key);
      disp.commit(d, now, T);
      ps.live[ti] += static_cast<double>(popped.prompt_tokens);
      ps.running[ti] += 1;
      live_reqs.push_back({*d.target, popped.uid, now, popped.prompt_tokens});
    }
    disp.gc(now);
    k.f64(R + "dec_time", dec_time);
    k.u64(R + "dec_uid", dec_uid);
    k.i32(R + "dec_target", dec_target);
    k.f64(R + "dec_peak", dec_peak);
    k.f64(R + "dec_cand", dec_cand);
    k.i32(R + "dec_admitted", dec_admitted);
    // ledger state after the round (slots present in usage_ and their values)
    std::vector<int64_t> led_inst, led_slot;
    std::vector<double> led_used;
    for (int i = 0; i < n_inst; ++i) {
      const auto& L = disp.ledger(ps.ids[i]);
      for (int64_t s = -4; s < 400; ++s) {
        const double u = L.usage_in_slot(s);
        if (u != 0.0) {
          led_inst.push_back(ps.ids[i]);
          led_slot.push_back(s);
          led_used.push_back(u);
        }
      }
    }
    k.i64(R + "ledger_inst", led_inst);
    k.i64(R + "ledger_slot", led_slot);
    k.f64(R + "ledger_used", led_used);
    std::vector<uint8_t> susp;
    for (int i = 0; i < n_inst; ++i) susp.push_back(disp.suspended(ps.ids[i]) ? 1 : 0);
    k.u8(R + "suspended", susp);
    // remove dispatched from the host queue
    std::set<uint64_t> gone;
    for (std::size_t j = 0; j < dec_uid.size(); ++j)
      if (dec_admitted[j]) gone.insert(dec_uid[j]);
    std::vector<PendingRequest> rest;
    for (const auto& p : queue)
      if (!gone.count(p.uid)) rest.push_back(p);
    queue = rest;
    // time advances; some running requests finish (early or late)
    const double next_now = now + rng.uniform(0.2, 1.5);
    std::vector<int64_t> fin_inst;
    std::vector<uint64_t> fin_uid;
    std::vector<double> fin_end;
    std::vector<Running> still;
    for (const auto& lr : live_reqs) {
      if (rng.uniform() < 0.45) {
        const double end = rng.uniform(now, next_now);
        disp.on_request_finished(lr.inst, lr.uid, end);
        const int ti = static_cast<int>(std::find(ps.ids.begin(), ps.ids.end(), lr.inst) - ps.ids.begin());
        ps.live[ti] -= static_cast<double>(lr.kv);
        ps.running[ti] -= 1;
        fin_inst.push_back(lr.inst);
        fin_uid.push_back(lr.uid);
        fin_end.push_back(end);
      } else {
        still.push_back(lr);
      }
    }
    live_reqs = still;
    // token growth on the engine side
    for (int i = 0; i < n_inst; ++i) ps.live[i] += std::floor(rng.uniform(0.0, 30.0) * ps.running[i]);
    k.i64(R + "fin_inst", fin_inst);
    k.u64(R + "fin_uid", fin_uid);
    k.f64(R + "fin_end", fin_end);
    now = next_now;
  }
  k.write(dir + "/" + name);
  std::printf("  %s: %d instances, %d rounds\n", name.c_str(), n_inst, rounds);
}

// ---- dispatch under RoundRobin / StaticThreshold: waiting lists ---------------
// The dispatch_loop restatement above with the non-TimeSlot branch
// (engine.cpp:259-262) and Simulator::try_admit (engine.cpp:270-296)
// restated over the reference's own Dispatcher, ReadyQueue and
// TopoDepthScheduler (whose waiting comparator (order_key, msg_id, uid)
// differs from the queue order when depth and queue_enter tie).
void gen_dispatch_waiting(const std::string& dir, const std::string& name, uint64_t seed,
                          DispatchPolicy policy, int n_inst, int max_batch, double cap, int rounds,
                          int per_round, double prompt_hi) {
  Rng rng(seed);
  DispatcherConfig dcfg;
  dcfg.policy = policy;
  std::vector<InstanceId> ids;
  std::vector<double> caps, ks;
  for (int i = 0; i < n_inst; ++i) {
    ids.push_back(7 + 5 * i);
    caps.push_back(cap * (i % 3 == 1 ? 0.7 : 1.0));
    ks.push_back(50.0);
  }
  Dispatcher disp(dcfg, ids, caps, ks);
  Names names;
  const int A = 4;
  std::map<AgentId, int> depths;
  for (int a = 0; a < A; ++a) {
    names.agent("w" + std::to_string(a));
    if (a != 3) depths["w" + std::to_string(a)] = 1 + (a % 2);  // w3: unknown -> depth 1
  }
  TopoDepthScheduler sched(depths);
  auto key = [&](const PendingRequest& r) { return sched.order_key(r); };
  std::vector<int32_t> depth_arr;
  for (int a = 0; a < A; ++a) {
    auto it = depths.find("w" + std::to_string(a));
    depth_arr.push_back(it == depths.end() ? 1 : it->second);
  }
  // every request of every round up front: one msg-key space for all of them
  std::vector<std::vector<PendingRequest>> arrivals(rounds);
  std::vector<std::string> all_msgs;
  uint64_t next_uid = 1;
  double now = 2.0;
  std::vector<double> nows;
  for (int r = 0; r < rounds; ++r) {
    nows.push_back(now);
    for (int j = 0; j < per_round; ++j) {
      const int a = static_cast<int>(rng.next_u64() % A);
      // coarse times: queue_enter ties across apps, app_start decides the
      // queue order, msg_id the waiting order
      const std::string msg = "m-" + std::to_string(1 + rng.next_u64() % (3 * per_round));
      PendingRequest p = req(msg, "w" + std::to_string(a), now - 0.125 * double(rng.next_u64() % 16),
                             now - 0.25 * double(rng.next_u64() % 4), next_uid++,
                             1 + static_cast<int64_t>(rng.next_u64() % static_cast<uint64_t>(prompt_hi)));
      arrivals[r].push_back(p);
      all_msgs.push_back(msg);
    }
    now += rng.uniform(0.2, 1.0);
  }
  std::sort(all_msgs.begin(), all_msgs.end());
  all_msgs.erase(std::unique(all_msgs.begin(), all_msgs.end()), all_msgs.end());
  auto mkey = [&](const std::string& m) {
    return static_cast<uint64_t>(std::lower_bound(all_msgs.begin(), all_msgs.end(), m) - all_msgs.begin());
  };
  auto put_reqs = [&](Kxf& k, const std::vector<PendingRequest>& q, const std::string& pre) {
    std::vector<int32_t> agent;
    std::vector<int64_t> prompt;
    std::vector<double> app, qe;
    std::vector<uint64_t> uid, msg;
    for (const auto& r : q) {
      agent.push_back(names.agent(r.agent));
      prompt.push_back(r.prompt_tokens);
      app.push_back(r.app_start);
      qe.push_back(r.queue_enter);
      uid.push_back(r.uid);
      msg.push_back(mkey(r.msg_id));
    }
    k.i32(pre + "agent", agent);
    k.i64(pre + "prompt", prompt);
    k.f64(pre + "app_start", app);
    k.f64(pre + "queue_enter", qe);
    k.u64(pre + "msg_key", msg);
    k.u64(pre + "uid", uid);
  };

  Kxf k;
  k.scalar_i("n_inst", n_inst);
  k.scalar_i("policy", static_cast<int64_t>(policy));
  k.i32("inst_id", std::vector<int32_t>(ids.begin(), ids.end()));
  k.f64("inst_cap", caps);
  k.f64("inst_k", ks);
  k.i32("inst_max_batch", std::vector<int32_t>(n_inst, max_batch));
  k.i32("agent_depth", depth_arr);

  std::vector<double> live(n_inst, 0.0);
  std::vector<int> running(n_inst, 0);
  std::vector<std::vector<PendingRequest>> waiting(n_inst);
  struct Run {
    int inst;
    int64_t kv;
  };
  std::vector<Run> runs;
  std::vector<PendingRequest> queue;
  auto put_waiting = [&](const std::string& pre) {
    std::vector<PendingRequest> flat;
    std::vector<int32_t> pos;
    for (int i = 0; i < n_inst; ++i)
      for (const auto& r : waiting[i]) {
        flat.push_back(r);
        pos.push_back(i);
      }
    put_reqs(k, flat, pre);
    k.i32(pre + "inst", pos);
  };
  for (int r = 0; r < rounds; ++r) {
    const std::string R = "r" + std::to_string(r) + ".";
    now = nows[r];
    for (const auto& p : arrivals[r]) queue.push_back(p);
    k.scalar_f(R + "now", now);
    k.f64(R + "live_kv", live);
    k.i32(R + "running", std::vector<int32_t>(running.begin(), running.end()));
    put_waiting(R + "w.");
    put_reqs(k, queue, R + "q.");
    std::vector<uint64_t> dec_uid, adm_uid;
    std::vector<int32_t> dec_target, dec_admitted, adm_inst;
    auto try_admit = [&](int i) {  // engine.cpp:270-296
      while (!waiting[i].empty() && running[i] < max_batch) {
        std::size_t best = 0;
        for (std::size_t j = 1; j < waiting[i].size(); ++j) {
          const auto& a = waiting[i][j];
          const auto& b = waiting[i][best];
          const auto ka = key(a);
          const auto kb = key(b);
          if (std::tie(ka, a.msg_id, a.uid) < std::tie(kb, b.msg_id, b.uid)) best = j;
        }
        const PendingRequest& head = waiting[i][best];
        if (live[i] + static_cast<double>(head.prompt_tokens) > caps[i]) break;
        const PendingRequest h = head;
        waiting[i].erase(waiting[i].begin() + static_cast<std::ptrdiff_t>(best));
        live[i] += static_cast<double>(h.prompt_tokens);  // kept_tokens = 0
        running[i] += 1;
        runs.push_back({i, h.prompt_tokens});
        adm_uid.push_back(h.uid);
        adm_inst.push_back(ids[i]);
      }
    };
    ReadyQueue rq;
    for (const auto& p : queue) rq.enqueue(p);
    while (!rq.empty()) {
      const std::size_t idx = rq.best_index(key);
      const PendingRequest head = rq.entries()[idx];
      std::vector<InstanceLive> lv;
      for (int i = 0; i < n_inst; ++i) {
        disp.on_live_usage(ids[i], live[i]);
        InstanceLive l;
        l.live_kv = live[i];
        l.running = running[i];
        l.waiting = static_cast<int>(waiting[i].size());
        l.batch_full = l.running + l.waiting >= max_batch;
        lv.push_back(l);
      }
      DispatchDecision d = disp.choose(head, now, 1.0, lv);
      dec_uid.push_back(head.uid);
      dec_target.push_back(d.target ? *d.target : -1);
      dec_admitted.push_back(d.target ? 1 : 0);
      if (!d.target) break;
      const int ti = static_cast<int>(std::find(ids.begin(), ids.end(), *d.target) - ids.begin());
      PendingRequest popped = rq.pop(key);
      waiting[ti].push_back(popped);
      try_admit(ti);
    }
    for (int i = 0; i < n_inst; ++i) try_admit(i);
    disp.gc(now);
    k.u64(R + "dec_uid", dec_uid);
    k.i32(R + "dec_target", dec_target);
    k.i32(R + "dec_admitted", dec_admitted);
    k.u64(R + "adm_uid", adm_uid);
    k.i32(R + "adm_inst", adm_inst);
    k.f64(R + "end_live_kv", live);
    k.i32(R + "end_running", std::vector<int32_t>(running.begin(), running.end()));
    put_waiting(R + "end_w.");
    // the queue keeps what was not popped
    std::set<uint64_t> gone;
    for (std::size_t j = 0; j < dec_uid.size(); ++j)
      if (dec_admitted[j]) gone.insert(dec_uid[j]);
    std::vector<PendingRequest> rest;
    for (const auto& p : queue)
      if (!gone.count(p.uid)) rest.push_back(p);
    queue = rest;
    // some running requests finish before the next round (engine side)
    std::vector<Run> still;
    for (const auto& x : runs) {
      if (rng.uniform() < 0.5) {
        live[x.inst] -= static_cast<double>(x.kv);
        running[x.inst] -= 1;
      } else {
        still.push_back(x);
      }
    }
    runs = still;
  }
  k.write(dir + "/" + name);
  std::printf("  %s: %d instances, %d rounds\n", name.c_str(), n_inst, rounds);
}

// ---- K1: realize() / finalize_instance ---------------------------------------
AppSpec fan_app(int width) {
  // Parallel fan-out + choice + feedback: exercises multi-child max.
  AppSpec app;
  app.name = "fan";
  app.entry = "Planner";
  AgentSpec planner;
  planner.name = "Planner";
  planner.prompt_len = LengthSpec::uniform(50, 90);
  planner.output_len = LengthSpec::lognormal(40.0, 0.4, 200);
  for (int i = 0; i < width; ++i) planner.parallel.push_back("Worker" + std::to_string(i));
  app.agents.push_back(planner);
  for (int i = 0; i < width; ++i) {
    AgentSpec w;
    w.name = "Worker" + std::to_string(i);
    w.prompt_len = LengthSpec::uniform(60, 200);
    w.output_len = LengthSpec::lognormal(60.0 + 30.0 * i, 0.5, 800);
    if (i % 2 == 0) w.choice = {{"Judge", 0.7}, {"Writer", 0.3}};
    app.agents.push_back(w);
  }
  AgentSpec judge;
  judge.name = "Judge";
  judge.prompt_len = LengthSpec::uniform(40, 80);
  judge.output_len = LengthSpec::lognormal(20.0, 0.3, 80);
  judge.feedback = AgentSpec::Feedback{"Writer", 0.4, 2};
  AgentSpec writer;
  writer.name = "Writer";
  writer.prompt_len = LengthSpec::uniform(100, 300);
  writer.output_len = LengthSpec::lognormal(200.0, 0.4, 900);
  app.agents.push_back(judge);
  app.agents.push_back(writer);
  return app;
}

void gen_dp(const std::string& dir, const std::string& name, const WorkloadConfig& cfg,
            const ReferenceRates& rates, uint64_t seed) {
  const auto real = realize(cfg, rates, seed);
  Kxf k;
  std::vector<int64_t> off{0}, prompt, target;
  std::vector<int32_t> parent;
  std::vector<uint64_t> uid;
  std::vector<double> pure, rem, rem_map, arrival;
  std::vector<int32_t> builtin_agent;
  const char* builtin[10] = {"Router", "Math", "Humanities", "Researcher", "Writer",
                             "ProductManager", "Architect", "ProjectManager", "Engineer", "QAEngineer"};
  for (const auto& inst : real.instances) {
    arrival.push_back(inst.arrival);
    for (const auto& c : inst.calls) {
      int32_t bi = -1;
      for (int a = 0; a < 10; ++a)
        if (c.agent == builtin[a]) bi = a;
      builtin_agent.push_back(bi);
      parent.push_back(c.parents.empty() ? -1 : c.parents[0]);
      prompt.push_back(c.prompt_tokens);
      target.push_back(c.target_tokens);
      uid.push_back(c.uid);
      pure.push_back(c.pure_exec);
      rem.push_back(c.remaining_exec);
      rem_map.push_back(real.remaining_by_uid.at(c.uid));
    }
    off.push_back(static_cast<int64_t>(parent.size()));
  }
  k.i64("wf_offsets", off);
  k.i32("parent", parent);
  k.i64("prompt", prompt);
  k.i64("target", target);
  k.u64("uid", uid);
  k.f64("pure_exec", pure);
  k.f64("remaining_exec", rem);
  k.f64("remaining_by_uid", rem_map);
  k.f64("arrival", arrival);
  k.i32("builtin_agent", builtin_agent);
  k.scalar_f("prefill_rate", rates.prefill_rate);
  k.scalar_f("decode_rate", rates.decode_rate);
  k.write(dir + "/" + name);
  std::printf("  %s: %zu workflows, %zu calls\n", name.c_str(), real.instances.size(), parent.size());
}

// ---- record_remaining + distribution statistics ---------------------------
void gen_remaining(const std::string& dir) {
  Rng rng(77);
  LatencyProfiler prof;
  Kxf k;
  std::vector<int64_t> off{0};
  std::vector<double> es, ee;
  std::vector<int32_t> agent;
  Names names;
  for (int w = 0; w < 300; ++w) {
    std::vector<RequestRecord> recs;
    const int n = 1 + static_cast<int>(rng.next_u64() % 9);
    double t = rng.uniform(0.0, 100.0);
    for (int j = 0; j < n; ++j) {
      RequestRecord r;
      r.msg_id = "m-" + std::to_string(w);
      r.agent = "a" + std::to_string(rng.next_u64() % 6);
      r.exec_start = t;
      r.exec_end = t + rng.uniform(0.01, 5.0);
      t = rng.uniform() < 0.5 ? r.exec_end : t + rng.uniform(0.0, 1.0);
      recs.push_back(r);
      es.push_back(r.exec_start);
      ee.push_back(r.exec_end);
      agent.push_back(names.agent(r.agent));
    }
    off.push_back(static_cast<int64_t>(es.size()));
    prof.record_remaining(recs);
  }
  k.i64("rec_offsets", off);
  k.f64("exec_start", es);
  k.f64("exec_end", ee);
  k.i32("agent", agent);
  // per-agent sorted samples as the profiler holds them
  std::vector<int32_t> s_agent;
  std::vector<double> s_val;
  for (std::size_t a = 0; a < names.agents.size(); ++a) {
    const auto* d = prof.remaining_distribution(names.agents[a]);
    for (double v : d->dist.samples()) {
      s_agent.push_back(static_cast<int32_t>(a));
      s_val.push_back(v);
    }
  }
  k.i32("samples_agent", s_agent);
  k.f64("samples_sorted", s_val);
  k.write(dir + "/remaining.kxf");

  // distribution statistics
  Kxf st;
  std::vector<int64_t> soff{0};
  std::vector<double> vals, q50, q90, q99, mode, med_fallback, w1;
  for (int t2 = 0; t2 < 200; ++t2) {
    const int n = 1 + static_cast<int>(rng.next_u64() % 300);
    std::vector<double> v;
    for (int j = 0; j < n; ++j) v.push_back(t2 % 7 == 0 ? std::floor(rng.uniform(0, 4)) : rng.uniform(0.0, 10.0) * rng.uniform());
    std::sort(v.begin(), v.end());
    for (double x : v) vals.push_back(x);
    soff.push_back(static_cast<int64_t>(vals.size()));
    q50.push_back(quantile_sorted(v, 0.5));
    q90.push_back(quantile_sorted(v, 0.9));
    q99.push_back(quantile_sorted(v, 0.99));
    const auto me = mode_estimate(v);
    mode.push_back(me.value);
    med_fallback.push_back(me.median_fallback ? 1.0 : 0.0);
  }
  // W1 between consecutive sets
  for (std::size_t i = 0; i + 1 < soff.size() - 1; ++i) {
    std::vector<double> a(vals.begin() + soff[i], vals.begin() + soff[i + 1]);
    std::vector<double> b(vals.begin() + soff[i + 1], vals.begin() + soff[i + 2]);
    w1.push_back(wasserstein_1d(a, b));
  }
  st.i64("offsets", soff);
  st.f64("values", vals);
  st.f64("q50", q50);
  st.f64("q90", q90);
  st.f64("q99", q99);
  st.f64("mode", mode);
  st.f64("median_fallback", med_fallback);
  st.f64("w1_next", w1);
  // median anchor distance of random tables
  std::vector<int64_t> toff{0};
  std::vector<double> coords, anchors, medians;
  for (int t3 = 0; t3 < 50; ++t3) {
    PriorityTable tab;
    const int n = static_cast<int>(rng.next_u64() % 8);
    tab.anchor_coord = rng.uniform(-3.0, 3.0);
    for (int j = 0; j < n; ++j) {
      const double c = rng.uniform(-10.0, 10.0);
      tab.coord["x" + std::to_string(j)] = c;
    }
    for (const auto& [a, c] : tab.coord) coords.push_back(c);
    toff.push_back(static_cast<int64_t>(coords.size()));
    anchors.push_back(tab.anchor_coord);
    medians.push_back(tab.median_anchor_distance());
  }
  st.i64("table_offsets", toff);
  st.f64("table_coords", coords);
  st.f64("table_anchor", anchors);
  st.f64("table_median", medians);
  st.write(dir + "/stats.kxf");
  std::printf("  remaining.kxf, stats.kxf\n");
}

// ---- pairwise_sorting_accuracy (priority.cpp:165-189) -----------------------
void gen_accuracy(const std::string& dir) {
  Rng rng(99);
  Kxf k;
  std::vector<int64_t> off{0};
  std::vector<int32_t> agent;
  std::vector<double> rem, acc_cross, acc_all;
  std::vector<uint8_t> present;
  for (int t = 0; t < 40; ++t) {
    const int n = 1 + static_cast<int>(rng.next_u64() % 400);
    const int A = 1 + static_cast<int>(rng.next_u64() % 6);
    std::vector<PendingRequest> order;
    std::map<uint64_t, double> remaining;
    for (int i = 0; i < n; ++i) {
      const int a = static_cast<int>(rng.next_u64() % A);
      order.push_back(req("m-" + std::to_string(i), "a" + std::to_string(a), 0, 0, i + 1));
      const double v = (t % 3 == 0) ? std::floor(rng.uniform(0.0, 5.0)) : rng.uniform(0.0, 10.0);
      const bool has = rng.uniform() < 0.9;
      if (has) remaining[i + 1] = v;
      agent.push_back(a);
      rem.push_back(v);
      present.push_back(has ? 1 : 0);
    }
    off.push_back(static_cast<int64_t>(agent.size()));
    const auto c = pairwise_sorting_accuracy(order, remaining, PairScope::CrossAgent);
    const auto a2 = pairwise_sorting_accuracy(order, remaining, PairScope::All);
    acc_cross.push_back(c ? *c : std::nan(""));
    acc_all.push_back(a2 ? *a2 : std::nan(""));
  }
  k.i64("offsets", off);
  k.i32("agent", agent);
  k.f64("remaining", rem);
  k.u8("present", present);
  k.f64("acc_cross", acc_cross);
  k.f64("acc_all", acc_all);
  k.write(dir + "/accuracy.kxf");
  std::printf("  accuracy.kxf\n");
}

}  // namespace

// W1 distance matrix (priority.cpp:15-65): per-agent sorted sample sets of
// varied sizes (singletons, ties, a large set), the reference's
// build_distance_matrix_from_samples over them (agents named so the map
// order is the index order; the anchor {0.0} is the last label).
void gen_w1matrix(const std::string& dir) {
  Rng rng(4242);
  Kxf k;
  std::vector<int64_t> set_off{0}, case_off{0}, mat_off{0};
  std::vector<double> samples, mat;
  const int sizes[][6] = {{1, 1, 1, 0, 0, 0}, {3, 7, 1, 12, 0, 0}, {64, 200, 33, 5, 400, 17},
                          {1000, 999, 1, 2, 3, 4096}};
  for (int c = 0; c < 6; ++c) {
    std::map<AgentId, std::vector<double>> sets;
    const int na = c < 4 ? 6 : (c == 4 ? 9 : 14);
    for (int a = 0; a < na; ++a) {
      int sz = c < 4 ? sizes[c][a] : 1 + static_cast<int>(rng.next_u64() % 300);
      if (sz == 0) continue;
      std::vector<double> v;
      for (int j = 0; j < sz; ++j) {
        // mix of continuous values and heavy ties (the reference's remaining
        // times often repeat)
        const double x = (j % 3 == 0) ? std::floor(rng.uniform(0.0, 8.0)) : rng.uniform(0.0, 30.0);
        v.push_back(x);
      }
      std::sort(v.begin(), v.end());
      char name[16];
      std::snprintf(name, sizeof(name), "a%02d", a);
      sets[name] = v;
    }
    for (const auto& [nm, v] : sets) {
      samples.insert(samples.end(), v.begin(), v.end());
      set_off.push_back(static_cast<int64_t>(samples.size()));
    }
    case_off.push_back(static_cast<int64_t>(set_off.size() - 1));
    const DistanceMatrix m = build_distance_matrix_from_samples(sets);
    for (const auto& row : m.d) mat.insert(mat.end(), row.begin(), row.end());
    mat_off.push_back(static_cast<int64_t>(mat.size()));
  }
  k.i64("set_offsets", set_off);
  k.i64("case_sets", case_off);
  k.f64("samples", samples);
  k.i64("matrix_offsets", mat_off);
  k.f64("matrix", mat);
  k.write(dir + "/w1_matrix.kxf");
  std::printf("  w1_matrix.kxf\n");
}

// ---- K9: profiler ingestion -------------------------------------------------
// The reference LatencyProfiler (default ProfilerConfig: remaining window
// 4096, execution unbounded) fed workflow by workflow: after each workflow's
// record_remaining the take_newly_converged() flag, and every record also
// through record_execution. Agent 0 gets enough samples to slide its window;
// agent 3 is noisy (converges late or never).
void gen_profiler(const std::string& dir) {
  Rng rng(909);
  LatencyProfiler prof;
  const int A = 4;
  std::vector<std::string> agents;
  for (int a = 0; a < A; ++a) agents.push_back("p" + std::to_string(a));
  std::vector<int64_t> off{0};
  std::vector<int32_t> agent;
  std::vector<double> es, ee;
  std::vector<uint8_t> newly;
  const int W = 2600;
  double t = 0.0;
  for (int w = 0; w < W; ++w) {
    std::vector<RequestRecord> recs;
    const int nr = 1 + static_cast<int>(rng.next_u64() % 4);
    t += rng.uniform(0.0, 0.5);
    double cur = t;
    for (int r = 0; r < nr; ++r) {
      const int a = r == 0 ? 0 : static_cast<int>(rng.next_u64() % A);
      RequestRecord rec;
      rec.msg_id = "m-" + std::to_string(w);
      rec.agent = agents[static_cast<std::size_t>(a)];
      rec.exec_start = cur + rng.uniform(0.0, 0.2);
      const double dur = a == 3 ? rng.uniform(0.01, 30.0) : 0.5 + a + rng.uniform(0.0, 0.3 * (a + 1));
      rec.exec_end = rec.exec_start + dur;
      cur = rec.exec_end - (r % 2 ? dur * 0.5 : 0.0);  // some overlap (parallel calls)
      recs.push_back(rec);
      agent.push_back(a);
      es.push_back(rec.exec_start);
      ee.push_back(rec.exec_end);
      prof.record_execution(rec.agent, rec.exec_end - rec.exec_start);
    }
    // every fifth workflow repeats agent 0 twice more (fills its window)
    if (w % 5 == 0) {
      for (int r = 0; r < 2; ++r) {
        RequestRecord rec = recs.front();
        rec.exec_start = recs.front().exec_start + rng.uniform(0.0, 0.1);
        recs.push_back(rec);
        agent.push_back(0);
        es.push_back(rec.exec_start);
        ee.push_back(rec.exec_end);
        prof.record_execution(rec.agent, rec.exec_end - rec.exec_start);
      }
    }
    off.push_back(static_cast<int64_t>(agent.size()));
    prof.record_remaining(recs);
    newly.push_back(prof.take_newly_converged() ? 1 : 0);
  }
  Kxf k;
  k.scalar_i("n_agents", A);
  k.i64("off", off);
  k.i32("agent", agent);
  k.f64("exec_start", es);
  k.f64("exec_end", ee);
  k.u8("newly", newly);
  for (int kind = 0; kind < 2; ++kind)
    for (int a = 0; a < A; ++a) {
      const std::string pre = std::string(kind ? "rem" : "exec") + std::to_string(a) + ".";
      const EmpiricalDistribution* d =
          kind ? &prof.remaining_distribution(agents[static_cast<std::size_t>(a)])->dist
               : prof.exec_distribution(agents[static_cast<std::size_t>(a)]);
      k.f64(pre + "samples", d->samples());
      k.u64(pre + "total", {d->total_added()});
      k.u8(pre + "converged", {static_cast<uint8_t>(d->converged() ? 1 : 0)});
      k.f64(pre + "last", {d->last_checkpoint_distance()});
    }
  k.write(dir + "/profiler.kxf");
  std::printf("  profiler.kxf: %d workflows, %zu records\n", W, agent.size());
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "tests/golden";
  std::filesystem::create_directories(dir);
  std::printf("gen_golden -> %s\n", dir.c_str());
  gen_order(dir);
  gen_dispatch(dir, "dispatch_small.kxf", 11, 4, 8, 3000.0, 6, 40, 450.0, false);
  gen_dispatch(dir, "dispatch_preload.kxf", 12, 16, 6, 3000.0, 8, 120, 400.0, true);
  gen_dispatch(dir, "dispatch_overload.kxf", 13, 5, 64, 1000.0, 5, 80, 150.0, false);
  gen_dispatch_waiting(dir, "dispatch_rr.kxf", 21, DispatchPolicy::RoundRobin, 5, 4, 2000.0, 6, 30, 600.0);
  gen_dispatch_waiting(dir, "dispatch_static.kxf", 22, DispatchPolicy::StaticThreshold, 6, 4, 2000.0, 6, 40,
                       1100.0);
  gen_dp(dir, "dp_colocated.kxf", colocated_workload(3.0, 400.0, 3), ReferenceRates{8000.0, 50.0}, 3);
  gen_dp(dir, "dp_cg.kxf", cg_workload(2.0, 300.0, 11), ReferenceRates{6000.0, 40.0}, 11);
  {
    WorkloadConfig cfg;
    cfg.apps = {fan_app(6), qa_app()};
    cfg.arrival.rate = 5.0;
    cfg.duration = 200.0;
    gen_dp(dir, "dp_fanout.kxf", cfg, ReferenceRates{6000.0, 40.0}, 9);
  }
  {
    WorkloadConfig cfg;
    cfg.apps = {fan_app(40)};  // > 32 calls per workflow: the sweep path
    cfg.arrival.rate = 2.0;
    cfg.duration = 30.0;
    gen_dp(dir, "dp_wide.kxf", cfg, ReferenceRates{8000.0, 50.0}, 4);
  }
  gen_remaining(dir);
  gen_accuracy(dir);
  gen_w1matrix(dir);
  gen_profiler(dir);
  return 0;
}

// kairos_b200.hpp — C++ host adapters over the C ABI (kairos_b200.h).
//
// These classes present the reference's in-process operator API
// (/root/reference/proj/include/kairos/{scheduler,priority,dispatcher}.hpp)
// on top of the device-resident B200 path, so kairos-sim's Simulator can
// call the GPU where it calls ReadyQueue / SchedulerPolicy / Dispatcher
// today. Errors are rethrown as the reference's
// exception types. Header-only; link with libkairos_b200.so.
//
// Request types are duck-typed: any struct with the fields of
// kairos::PendingRequest (types.hpp:35-42) — msg_id, agent, prompt_tokens,
// app_start, queue_enter, uid — works, including kairos::PendingRequest.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "kairos_b200.h"

namespace kairos_b200 {

// kx status -> the reference's exception types (dispatcher.cpp:21-255,
// engine.cpp:100).
inline void check(int status) {
  if (status == KX_OK) return;
  const std::string msg = kx_last_error();
  switch (status) {
    case KX_ERR_INVALID: throw std::invalid_argument(msg);
    case KX_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// quantile_sorted (distribution.cpp:33-44); compile with -ffp-contract=off
// so the interpolation rounds like the reference build.
inline double quantile_sorted(const std::vector<double>& s, double p) {
  if (s.empty()) throw std::invalid_argument("quantile of empty sample set");
  if (p <= 0.0) return s.front();
  if (p >= 1.0) return s.back();
  const double pos = p * static_cast<double>(s.size() - 1);
  const auto lo = static_cast<std::size_t>(pos);
  const double frac = pos - static_cast<double>(lo);
  if (lo + 1 >= s.size()) return s.back();
  return s[lo] + frac * (s[lo + 1] - s[lo]);
}

// PriorityTable::priority_key for every registered agent
// (priority.cpp:114-135): anchor distance, or the cold-start median of the
// table's anchor distances for agents outside the table, 0 for no table.
inline std::vector<double> priority_keys(const std::vector<std::string>& agents,
                                         const std::map<std::string, double>& coord,
                                         double anchor_coord) {
  double median = 0.0;
  if (!coord.empty()) {
    std::vector<double> d;
    for (const auto& [a, c] : coord) d.push_back(std::abs(c - anchor_coord));
    std::sort(d.begin(), d.end());
    median = quantile_sorted(d, 0.5);
  }
  std::vector<double> out;
  out.reserve(agents.size());
  for (const auto& a : agents) {
    auto it = coord.find(a);
    out.push_back(it == coord.end() ? median : std::abs(it->second - anchor_coord));
  }
  return out;
}

// Order-preserving u64 keys for msg_id strings (lexicographic).
// Fast path for MessageIdFactory ids "<prefix><decimal counter>" with one
// shared prefix (types.hpp:46-57): the decimal string is encoded base-11
// (digit+1, 0 = end) so numeric keys compare like the strings. Otherwise the
// distinct strings are ranked.
class MsgKeyer {
 public:
  template <typename Request>
  std::vector<uint64_t> keys(const std::vector<Request>& q) const {
    std::vector<uint64_t> out(q.size());
    if (q.empty()) return out;
    const std::string prefix = common_prefix(q);
    bool fast = true;
    for (std::size_t i = 0; i < q.size() && fast; ++i) fast = encode(q[i].msg_id, prefix, &out[i]);
    if (fast) return out;
    std::vector<std::string> ids;
    ids.reserve(q.size());
    for (const auto& r : q) ids.push_back(r.msg_id);
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    for (std::size_t i = 0; i < q.size(); ++i)
      out[i] = static_cast<uint64_t>(std::lower_bound(ids.begin(), ids.end(), q[i].msg_id) - ids.begin());
    return out;
  }

 private:
  template <typename Request>
  static std::string common_prefix(const std::vector<Request>& q) {
    const std::string& s = q.front().msg_id;
    std::size_t k = 0;
    while (k < s.size() && !(s[k] >= '0' && s[k] <= '9')) ++k;
    return s.substr(0, k);
  }
  static bool encode(const std::string& s, const std::string& prefix, uint64_t* key) {
    if (s.size() <= prefix.size() || s.compare(0, prefix.size(), prefix) != 0) return false;
    const std::size_t nd = s.size() - prefix.size();
    if (nd > 18) return false;
    uint64_t k = 0;
    for (std::size_t j = 0; j < 18; ++j) {
      uint64_t dgt = 0;
      if (j < nd) {
        const char c = s[prefix.size() + j];
        if (c < '0' || c > '9') return false;
        dgt = static_cast<uint64_t>(c - '0') + 1;
      }
      k = k * 11 + dgt;
    }
    *key = k;
    return true;
  }
};

struct InstanceProfile {  // engine.hpp:25-31 + pool
  int32_t id = 0;
  int32_t pool = 0;
  double capacity_tokens = 0.0;
  double decode_rate = 50.0;
  double prefill_rate = 8000.0;
  int32_t max_batch = 64;
};

struct DispatcherConfig {  // dispatcher.hpp:112-121
  int32_t policy = KX_DISPATCH_TIME_SLOT;
  double slot_len = 0.5;
  double resume_watermark = 0.85;
  double static_threshold = 0.90;
  double default_expected_time = 1.0;
  bool oracle_expected_time = false;
};

// DecisionLogRow (engine.hpp:92-99).
struct DecisionLogRow {
  double time = 0.0;
  uint64_t uid = 0;
  std::string agent;
  std::optional<int32_t> target;
  double predicted_peak = 0.0;
  std::vector<double> candidate_peaks;
  int64_t queue_index = -1;
  bool admitted = false;
};

// One device-resident scheduling domain: P pools, each with its ready
// queue, SchedulerPolicy tables and Dispatcher (ledgers + suspension).
class DeviceScheduler {
 public:
  DeviceScheduler(const DispatcherConfig& dcfg, const std::vector<InstanceProfile>& instances,
                  int32_t n_pools = 1, int64_t queue_capacity = 1 << 20, int32_t max_agents = 4096,
                  int32_t device = 0)
      : n_pools_(n_pools), instances_(instances) {
    std::vector<kx_instance> inst;
    for (const auto& p : instances) {
      kx_instance k{};
      k.id = p.id;
      k.pool = p.pool;
      k.capacity_tokens = p.capacity_tokens;
      k.decode_rate = p.decode_rate;
      k.prefill_rate = p.prefill_rate;
      k.max_batch = p.max_batch;
      inst.push_back(k);
    }
    kx_sched_config cfg{};
    cfg.n_pools = n_pools;
    cfg.n_instances = static_cast<int32_t>(inst.size());
    cfg.instances = inst.data();
    cfg.dispatcher.policy = dcfg.policy;
    cfg.dispatcher.oracle_expected_time = dcfg.oracle_expected_time ? 1 : 0;
    cfg.dispatcher.slot_len = dcfg.slot_len;
    cfg.dispatcher.resume_watermark = dcfg.resume_watermark;
    cfg.dispatcher.static_threshold = dcfg.static_threshold;
    cfg.dispatcher.default_expected_time = dcfg.default_expected_time;
    cfg.queue_capacity = queue_capacity;
    cfg.max_agents = max_agents;
    cfg.slot_ring = 256;
    cfg.device = device;
    default_T_ = dcfg.default_expected_time;
    time_slot_ = dcfg.policy == KX_DISPATCH_TIME_SLOT;
    check(kx_sched_create(&cfg, &h_));
  }
  ~DeviceScheduler() {
    if (h_) kx_sched_destroy(h_);
  }
  DeviceScheduler(const DeviceScheduler&) = delete;
  DeviceScheduler& operator=(const DeviceScheduler&) = delete;

  // Agents must be registered with their pool before they are enqueued.
  int32_t register_agent(const std::string& agent, int32_t pool) {
    auto it = agent_idx_.find(agent);
    if (it != agent_idx_.end()) return it->second;
    const auto i = static_cast<int32_t>(agents_.size());
    agents_.push_back(agent);
    agent_pool_.push_back(pool);
    agent_idx_[agent] = i;
    tables_dirty_ = true;
    return i;
  }

  // SchedulerKind (harness.hpp:16): "kairos", "fcfs", "topo_depth", "oracle".
  void set_scheduler(int32_t kind) { check(kx_set_scheduler(h_, kind)); }

  // KairosScheduler's table (PriorityTable coord + anchor_coord).
  void set_priority_table(const std::map<std::string, double>& coord, double anchor_coord) {
    coord_ = coord;
    anchor_ = anchor_coord;
    tables_dirty_ = true;
  }
  // TopoDepthScheduler depths (unknown agent -> 1, scheduler.hpp:71-74).
  void set_topo_depths(const std::map<std::string, int>& depths) {
    depths_ = depths;
    tables_dirty_ = true;
  }
  // ProfilerSnapshot::expected_exec_time per agent (fallback default_T).
  void set_expected_times(const std::map<std::string, double>& T) {
    T_ = T;
    tables_dirty_ = true;
  }
  // Priority keys computed by the caller's own SchedulerPolicy (e.g.
  // KairosScheduler::order_key(r).k0 = PriorityTable::priority_key(agent),
  // scheduler.hpp:111-113): used instead of the coord table when non-empty.
  void set_agent_keys(const std::map<std::string, double>& pk) {
    keys_ = pk;
    tables_dirty_ = true;
  }
  // OracleScheduler's remaining_by_uid. The device table is dense over
  // [min uid, max uid]; a span far wider than the map (hashed uids) is
  // refused rather than allocated.
  void set_remaining(const std::map<uint64_t, double>& rem) {
    if (rem.empty()) {
      check(kx_set_remaining_table(h_, 0, 0, nullptr, nullptr, KX_MEM_HOST));
      return;
    }
    const uint64_t lo = rem.begin()->first, hi = rem.rbegin()->first;
    if (hi - lo >= 64 * static_cast<uint64_t>(rem.size()) + (uint64_t(1) << 24))
      throw std::invalid_argument("set_remaining: uid span too sparse for the dense device table");
    std::vector<double> v(hi - lo + 1, 0.0);
    std::vector<uint8_t> p(hi - lo + 1, 0);
    for (const auto& [u, r] : rem) {
      v[u - lo] = r;
      p[u - lo] = 1;
    }
    check(kx_set_remaining_table(h_, lo, static_cast<int64_t>(v.size()), v.data(), p.data(), KX_MEM_HOST));
  }

  // Replaces the device queue (ReadyQueue::enqueue for every request).
  // kept: retained tokens per request (admit's kv_tokens = prompt + kept,
  // engine.cpp:306); pure_exec: the oracle T per request
  // (oracle_expected_time, engine.cpp:178-180).
  template <typename Request>
  void upload(const std::vector<Request>& q, const std::vector<int64_t>* kept = nullptr,
              const std::vector<double>* pure_exec = nullptr) {
    const kx_queue_view v = view(q, kept, pure_exec);
    check(kx_queue_upload(h_, static_cast<int64_t>(q.size()), &v, KX_MEM_HOST));
    n_ = static_cast<int64_t>(q.size());
  }
  // ReadyQueue::enqueue (priority.hpp:72) of n requests behind the queued
  // ones. msg_id keys must come from the same key space as the queued ones:
  // MessageIdFactory ids with one prefix (the MsgKeyer fast path).
  template <typename Request>
  void enqueue(const std::vector<Request>& q, const std::vector<int64_t>* kept = nullptr,
               const std::vector<double>* pure_exec = nullptr) {
    const kx_queue_view v = view(q, kept, pure_exec);
    check(kx_queue_enqueue(h_, static_cast<int64_t>(q.size()), &v, KX_MEM_HOST));
    check(kx_queue_size(h_, &n_));
  }
  // ReadyQueue::pop of every request the last dispatch round admitted
  // (engine.cpp:259), keeping the rest in their relative order.
  void remove_admitted() {
    check(kx_queue_remove_admitted(h_));
    check(kx_queue_size(h_, &n_));
  }
  int64_t size() const { return n_; }

 private:
  template <typename Request>
  kx_queue_view view(const std::vector<Request>& q, const std::vector<int64_t>* kept,
                     const std::vector<double>* pure_exec) {
    flush_tables();
    const std::size_t n = q.size();
    agent_.resize(n);
    prompt_.resize(n);
    app_.resize(n);
    qe_.resize(n);
    uid_.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
      auto it = agent_idx_.find(q[i].agent);
      if (it == agent_idx_.end()) throw std::invalid_argument("unregistered agent " + q[i].agent);
      agent_[i] = it->second;
      prompt_[i] = q[i].prompt_tokens;
      app_[i] = q[i].app_start;
      qe_[i] = q[i].queue_enter;
      uid_[i] = q[i].uid;
    }
    msg_ = MsgKeyer().keys(q);
    if (kept && kept->size() != n) throw std::invalid_argument("kept: one entry per request");
    if (pure_exec && pure_exec->size() != n) throw std::invalid_argument("pure_exec: one entry per request");
    return kx_queue_view{agent_.data(), prompt_.data(), app_.data(), qe_.data(), msg_.data(), uid_.data(),
                         kept ? kept->data() : nullptr, pure_exec ? pure_exec->data() : nullptr};
  }

 public:

  // Full queue order per pool (ReadyQueue pop order): indices into the
  // uploaded vector, pool-major, with pool offsets.
  std::vector<uint32_t> order(std::vector<int64_t>* pool_offsets = nullptr) {
    check(kx_order(h_));
    std::vector<uint32_t> perm(static_cast<std::size_t>(n_));
    std::vector<int64_t> offs(static_cast<std::size_t>(n_pools_) + 1);
    check(kx_order_fetch(h_, perm.data(), offs.data(), KX_MEM_HOST));
    if (pool_offsets) *pool_offsets = offs;
    return perm;
  }

  // One dispatch round (engine.cpp:220-268 + gc): order + place. Returns the
  // decision log in pool order. Admitted rows are committed to the device
  // ledgers and flagged; they stay queued on the device until
  // remove_admitted() (or the next upload). candidate_peaks are filled for
  // the time-slot policy only (Dispatcher::choose logs none otherwise,
  // dispatcher.cpp:207-250).
  std::vector<DecisionLogRow> dispatch_round(double now) {
    check(kx_tick(h_, now));
    std::vector<int64_t> cnt(static_cast<std::size_t>(n_pools_));
    int64_t rs = 0, ps = 0;
    check(kx_dispatch_fetch(h_, cnt.data(), nullptr, nullptr, &rs, &ps));
    std::vector<kx_decision> rows(static_cast<std::size_t>(n_pools_ * rs));
    std::vector<double> cand(static_cast<std::size_t>(n_pools_ * rs * ps));
    check(kx_dispatch_fetch(h_, cnt.data(), rows.data(), cand.data(), &rs, &ps));
    std::vector<DecisionLogRow> out;
    for (int32_t p = 0; p < n_pools_; ++p) {
      int64_t ni = 0;
      for (const auto& ip : instances_) ni += ip.pool == p ? 1 : 0;
      for (int64_t r = 0; r < cnt[p]; ++r) {
        const kx_decision& d = rows[static_cast<std::size_t>(p * rs + r)];
        DecisionLogRow row;
        row.time = d.time;
        row.uid = d.uid;
        row.agent = agents_[static_cast<std::size_t>(d.agent)];
        if (d.target >= 0) row.target = d.target;
        row.predicted_peak = d.predicted_peak;
        if (time_slot_) {
          const double* c = cand.data() + (p * rs + r) * ps;
          row.candidate_peaks.assign(c, c + ni);
        }
        row.queue_index = d.queue_index;
        row.admitted = d.admitted != 0;
        out.push_back(std::move(row));
      }
    }
    return out;
  }

  // Dispatcher events (dispatcher.cpp:264-297) and live view (engine.cpp:187-202).
  void on_request_finished(int32_t instance, uint64_t uid, double actual_end) {
    check(kx_on_request_finished(h_, instance, uid, actual_end));
  }
  void on_request_preempted(int32_t instance, uint64_t uid, double now) {
    on_request_finished(instance, uid, now);
  }
  void on_overload(int32_t instance) { check(kx_on_overload(h_, instance)); }
  void on_live_usage(int32_t instance, double live_kv) { check(kx_on_live_usage(h_, instance, live_kv)); }
  void gc(double now) { check(kx_gc(h_, now)); }
  void set_live(const std::vector<double>& live_kv, const std::vector<int32_t>& running,
                const std::vector<int32_t>& waiting) {
    check(kx_instances_set_live(h_, live_kv.data(), running.data(), waiting.data()));
  }
  void commit(int32_t instance, uint64_t uid, double prompt_tokens, double decode_rate, double now,
              double expected_T) {
    check(kx_ledger_commit(h_, instance, uid, prompt_tokens, decode_rate, now, expected_T));
  }

  kx_sched* handle() const { return h_; }
  const std::vector<std::string>& agents() const { return agents_; }

 private:
  void flush_tables() {
    if (!tables_dirty_) return;
    if (agents_.empty()) throw std::invalid_argument("no agents registered");
    std::vector<double> pk = priority_keys(agents_, coord_, anchor_);
    if (!keys_.empty())
      for (std::size_t i = 0; i < agents_.size(); ++i) {
        auto k = keys_.find(agents_[i]);
        pk[i] = k == keys_.end() ? 0.0 : k->second;
      }
    std::vector<int32_t> depth;
    std::vector<double> T;
    for (const auto& a : agents_) {
      auto d = depths_.find(a);
      depth.push_back(d == depths_.end() ? 1 : d->second);
      auto t = T_.find(a);
      T.push_back(t == T_.end() ? default_T_ : t->second);
    }
    check(kx_set_agent_tables(h_, static_cast<int32_t>(agents_.size()), agent_pool_.data(), pk.data(),
                              depth.data(), T.data(), ++table_version_));
    tables_dirty_ = false;
  }

  kx_sched* h_ = nullptr;
  int32_t n_pools_ = 1;
  std::vector<InstanceProfile> instances_;
  std::vector<std::string> agents_;
  std::vector<int32_t> agent_pool_;
  std::unordered_map<std::string, int32_t> agent_idx_;
  std::map<std::string, double> coord_;
  double anchor_ = 0.0;
  std::map<std::string, int> depths_;
  std::map<std::string, double> T_;
  std::map<std::string, double> keys_;
  double default_T_ = 1.0;
  bool time_slot_ = true;
  bool tables_dirty_ = true;
  uint64_t table_version_ = 0;
  int64_t n_ = 0;
  std::vector<int32_t> agent_;
  std::vector<int64_t> prompt_;
  std::vector<double> app_, qe_;
  std::vector<uint64_t> uid_, msg_;
};

}  // namespace kairos_b200

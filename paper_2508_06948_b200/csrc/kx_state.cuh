// Device-resident state of one kx_sched handle: the ready queue (SoA), the
// per-agent tables, the per-instance live view + slot ledgers, and the
// order/dispatch workspaces. Plain structs of device pointers passed to
// kernels by value.
#pragma once

#include <stdint.h>

#include "../../include/kairos_b200.h"

namespace kx {

// PendingRequest (types.hpp:35-42) as structure-of-arrays, plus the
// per-request oracle key and dispatch flags.
struct QueueDev {
  int32_t* agent;
  int64_t* prompt;
  double* app_start;
  double* queue_enter;
  uint64_t* msg;
  uint64_t* uid;
  int64_t* kept;       // CallRuntime::kept_tokens at enqueue (0 by default)
  double* pure_exec;   // for oracle_expected_time
  double* rem;         // OracleScheduler key: remaining_by_uid[uid] or 0.0
  uint8_t* admitted;   // set by the dispatch round
};

struct AgentsDev {
  int32_t* pool;
  double* pk;          // PriorityTable::priority_key(agent)
  uint32_t* pk_rank;   // dense rank of pk among table agents
  int32_t* depth;      // TopoDepthScheduler depth
  uint32_t* depth_rank;
  double* T;           // expected_exec_time(agent)
};

// Slot ledger of one instance (dispatcher.hpp:49-85) as a dense ring of
// `ring` slots starting at base_slot, plus the active-request table.
constexpr int kActiveCap = 512;

struct InstDev {
  int32_t* id;
  int32_t* pool;
  double* cap;
  double* decode_rate;
  double* prefill_rate;
  int32_t* max_batch;
  int32_t* rank_li;     // [n_inst]: per pool, the local index of the rank-th instance in InstanceId order (H9)
  // mutable (checkpointed) state
  double* live_kv;
  int32_t* running;
  int32_t* waiting;
  uint8_t* suspended;
  int64_t* base_slot;   // lowest retained slot (gc boundary)
  int64_t* hi_slot;     // highest slot ever booked (>= base_slot - 1)
  double* usage;        // [n_inst * ring]
  uint8_t* exists;      // [n_inst * ring]: slot present in the usage_ map (plain byte stores)
  int32_t* n_active;
  uint64_t* act_uid;    // [n_inst * kActiveCap]
  double* act_P;
  double* act_k;
  double* act_t0;
  double* act_T;
  int32_t* rr_next;     // per pool: Dispatcher::rr_next_
};

struct OrderParams {
  int32_t policy;       // kx_scheduler_kind
  int32_t n_pools;
  int32_t pool_bits;
  int32_t class_bits;
  int32_t q_bits;
  int32_t key_bits;     // multiple of 8
  int32_t n_agents;
};

// Per-pool quantisation of the primary time (monotone non-decreasing).
struct PoolRange {
  uint64_t lo_bits;     // ordered bits of min
  uint64_t hi_bits;     // ordered bits of max
  double lo;
  double scale;
};

}  // namespace kx

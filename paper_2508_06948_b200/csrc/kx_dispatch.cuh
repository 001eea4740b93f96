// Host-side interface of the dispatch kernels (kx_dispatch.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "kx_state.cuh"

namespace kx {

constexpr int kMaxInstPerPool = 512;
constexpr int kDispSmemLimit = 220 * 1024;  // dynamic shared memory of the dispatch CTA
// The sequential dispatch CTAs reserve a whole SM's shared memory so no other
// kernel's CTAs (the concurrent sort) share their SM's issue slots.
constexpr int kDispSmemExclusive = 220 * 1024;

struct DispatchParams {
  int32_t oracle_T;
  int32_t ring;
  int32_t logging;
  int32_t peak_stride;
  int64_t log_cap;
  double slot_len;
  double watermark;
  double now;
};

struct TopKState;

// Resumable dispatch round (k_dispatch_warp): phase 1 walks a pool's top-K
// order prefix while the full sort runs; phase 2 continues from `start`
// over the full order when phase 1 ran out of prefix heads.
struct DispResume {
  int64_t start, nrows, nadm;
  int32_t need, pad;
};

struct DispPhase {
  int32_t phase;               // 0 full order, 1 top-K prefix, 2 continuation, 3 overlapped tick
  int32_t pad;
  const uint32_t* heads;       // [P * kTopKMax] (phase 1; phase 3 writes it)
  const TopKState* tk;         // (phase 1)
  DispResume* resume;          // [P] (phases 1, 2)
  // phase 3: like phase 1, with the prefix collected by key generation and
  // sorted in the dispatch CTA (launched after key generation)
  const uint32_t* spec_on;      // [P] speculative prefix collected
  const uint32_t* spec_count;   // [P]
  const uint32_t* cand;         // [P * kTopKMax] candidate queue indices
  const uint32_t* cand_key;     // [P * kTopKMax] their compact keys
  const uint32_t* pool_counts;  // [P] from key generation
  uint32_t* heads_out;          // [P * kTopKMax]
};

// One request in an instance's waiting list (InstanceState::waiting,
// engine.hpp:147-153): what try_admit's comparator and admit read.
struct WaitRec {
  double app_start, queue_enter;
  uint64_t msg, uid;
  int64_t prompt, kept;
  int64_t qidx;     // queue index in the round it entered
  int32_t agent;
  int32_t round;    // serial of the dispatch round it entered in
};

// Waiting-list state and policy of a round_robin / static_threshold round.
struct WaitDev {
  WaitRec* rec;           // [n_inst * cap]
  int64_t cap;
  kx_admission* adm;      // [n_pools * log_cap]
  int64_t* adm_count;     // [n_pools]
  const double* rem_table;  // OracleScheduler remaining_by_uid (dense, see kx_set_remaining_table)
  const uint8_t* rem_present;
  uint64_t rem_base;
  int64_t rem_n;
  double static_thr;
  int32_t policy;         // KX_DISPATCH_ROUND_ROBIN / KX_DISPATCH_STATIC_THRESHOLD
  int32_t sched_kind;     // order_key policy for try_admit's comparator
  int32_t round;
  int32_t pad;
};

void launch_dispatch_waiting(const QueueDev& q, const AgentsDev& a, const InstDev& in,
                             const int32_t* pool_begin, const uint32_t* perm,
                             const int64_t* pool_offsets, const DispatchParams& dp, const WaitDev& w,
                             int n_pools, int max_inst_per_pool, kx_decision* rows,
                             int64_t* row_count, int64_t* admitted_count, int* pool_status,
                             cudaStream_t st);

void configure_dispatch_kernels();
void read_dispatch_debug(unsigned long long* out);
void read_dispatch_stages(unsigned long long* out);
void read_dispatch_trace(unsigned long long* out);
void read_dispatch_pool_times(unsigned long long* out);
void read_dispatch_counts(unsigned long long* out, bool reset);
bool dispatch_can_overlap(int max_inst_per_pool, int ring);
void launch_dispatch(const QueueDev& q, const AgentsDev& a, const InstDev& in,
                     const int32_t* pool_begin, const uint32_t* perm, const int64_t* pool_offsets,
                     const DispatchParams& dp, int n_pools, int max_inst_per_pool, kx_decision* rows,
                     double* cand,
                     int64_t* row_count, int64_t* admitted_count, int* pool_status,
                     cudaStream_t st, DispPhase phase = DispPhase{});
void launch_ledger_try_place(const InstDev& in, int i, int ring, double P, double k, double t0,
                             double T, double slot_len, double* out_peak, int64_t* out_viol,
                             int* out_state, cudaStream_t st);
void launch_ledger_commit(const InstDev& in, int i, int ring, uint64_t uid, double P, double k,
                          double t0, double T, double slot_len, int* status, cudaStream_t st);
void launch_ledger_commit_batch(const InstDev& in, int n_inst, int ring, const int64_t* off,
                                const int64_t* order, const uint64_t* uid, const double* P,
                                const double* k, const double* t0, const double* T, double slot_len,
                                uint8_t* fits, int* status, cudaStream_t st);
void launch_ledger_finish(const InstDev& in, int i, int ring, uint64_t uid, double actual_end,
                          double slot_len, cudaStream_t st);
void launch_on_overload(const InstDev& in, int i, cudaStream_t st);
void launch_on_live_usage(const InstDev& in, int i, double live_kv, double watermark,
                          cudaStream_t st);
void launch_gc_all(const InstDev& in, int n_inst, int ring, double now, double slot_len,
                   cudaStream_t st);

}  // namespace kx

// Host-side interface of the replica engine (kx_engine.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "kx_dist.cuh"
#include "kx_state.cuh"

namespace kx {

constexpr int kEngineScalars = 8;
constexpr int kEngineMetrics = 16;
constexpr int kHistBins = 256;

struct EngineParams {
  int32_t n_inst, sched, dpolicy, oracle_T, ring, heap_cap, max_run, pad;
  double slot_len, watermark, static_thr, default_T, period, recompute;
  uint64_t max_events;
  // profile-based expected times (engine.cpp:177-185) and KairosScheduler
  // online rebuilds (scheduler.cpp:5-24)
  int32_t n_agents, profile_T, kairos, pad2;
  uint64_t rebuild_interval;
  int64_t mds_stride;  // doubles of rebuild scratch per replica
};

constexpr int kKairosMaxAgents = 32;
// ProfilerConfig::remaining (profiler.hpp:43): {16, 0.05, 4096}
constexpr int64_t kRemWindow = 4096;
constexpr int64_t kModeMinSamples = 16;  // mode_estimate default (distribution.hpp:33-34)

// All replicas concatenated; call / workflow indices are global.
struct EngineInputs {
  const int64_t* wf_base;    // [R+1]
  const int64_t* call_base;  // [R+1]
  const double* arrival;     // [W]
  const uint64_t* wf_msg;    // [W] lexicographic key of "m-<local index>"
  const int64_t* wf_call;    // [W+1]
  const int32_t* call_wf;    // [C]
  const int32_t* agent;      // [C]
  const int32_t* has_parent; // [C]
  const int64_t* prompt;     // [C]
  const int64_t* target;     // [C]
  const double* pure;        // [C]
  const double* rem;         // [C]
  const uint64_t* uid;       // [C]
  const int64_t* child_off;  // [C+1]
  const int32_t* child;      // [C]
  const int32_t* depth;      // [A]
  const int32_t* inst_id;    // [I]
  const double* cap;
  const double* k;
  const double* prefill;
  const int32_t* max_batch;
  // profiler layout, per (replica, agent) index r * n_agents + a
  const int32_t* agent_order;  // [A] agent indices in AgentId (name) order
  const int64_t* exec_off;     // [R*A+1] exec sample buffer (one per call of the agent)
  const int64_t* rem_off;      // [R*A+1] remaining window buffers (min(calls, 4097))
};

struct EngineState {
  // per call [C]
  int32_t* rem_parents;
  double* enqueue_time;
  double* first_enqueue;
  double* queue_seconds;
  int64_t* kept;
  int32_t* episodes;
  int32_t* preemptions;
  uint32_t* epoch;
  uint8_t* ever_preempted;
  int32_t* run_slot;
  // per workflow [W]
  int32_t* wf_remaining;
  double* wf_finish;
  int64_t* wf_tokens;
  int32_t* wf_ncalls;
  // ready queue / waiting lists: per-replica segments of the call range
  uint32_t* queue;
  uint32_t* waiting;
  int32_t* waiting_inst;
  // ledgers [R * I * ring], per instance [R * I], active tables [R * I * kActiveCap]
  double* usage;
  uint8_t* ex;
  int64_t* base;
  int64_t* hi;
  int32_t* n_active;
  uint64_t* act_uid;
  double* act_P;
  double* act_k;
  double* act_t0;
  double* act_T;
  // outputs: completion order within each replica's segment
  uint32_t* out_call;
  double* out_exec_start;
  double* out_exec_end;
  int32_t* out_inst;
  int64_t* out_wf;
  double* scalars;  // [R * kEngineScalars]
  int64_t* counts;  // [R * 4]
  // profiler (LatencyProfiler, profiler.hpp:49-88) and priority table
  int64_t* done_idx;    // [C] completion slot of each call
  double* exec_buf;     // exec samples: sorted prefix [0, ns) + pending [ns, nt)
  int64_t* exec_ns;     // [R*A] samples in the last snapshot (sorted)
  int64_t* exec_nt;     // [R*A] samples recorded
  double* exec_T;       // [R*A] cached mode_estimate of the snapshot
  uint8_t* exec_dirty;  // [R*A]
  double* rem_sorted;   // remaining-latency windows (sorted_, arrival ring, snapshot_)
  double* rem_ring;
  double* rem_snap;
  DistScal* rem_d;      // [R*A]
  double* pk;           // [R*A] current priority_key per agent
  double* mds;          // [R*mds_stride] rebuild scratch
  int64_t* rebuilds;    // [R] priority-table versions built
};

size_t engine_smem_bytes(const EngineParams& p);
void launch_replica_engine(const EngineParams& p, const EngineInputs& in, const EngineState& st,
                           int n_replicas, cudaStream_t stream);
void launch_replica_metrics(const EngineInputs& in, const EngineState& st, const int32_t* wf_rep,
                            int R, int64_t W, double warmup, double* metrics, uint32_t* hist,
                            cudaStream_t stream);

}  // namespace kx

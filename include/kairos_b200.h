/*
 * kairos_b200.h — C ABI of the B200-native Kairos scheduling hot path.
 *
 * The reference (kairos-sim, /root/reference/proj) has no FFI: its operator
 * API is in-process C++ (SURVEY §8b). Every entry point below replaces one
 * reference interface, cited as file:line relative to /root/reference/proj.
 * Conventions:
 *   - opaque handles (kx_sched*), int status codes (KX_OK == 0), and a
 *     thread-local message from kx_last_error(); no exceptions cross the ABI.
 *     Status codes mirror the reference's exception types:
 *       KX_ERR_INVALID  <- std::invalid_argument (dispatcher.cpp:21,48,129,...)
 *       KX_ERR_LOGIC    <- std::logic_error      (dispatcher.cpp:73,255)
 *       KX_ERR_RUNTIME  <- std::runtime_error    (engine.cpp:100)
 *   - caller-owned structure-of-arrays buffers with explicit lengths; `mem`
 *     says whether a pointer is host (KX_MEM_HOST) or device (KX_MEM_DEVICE).
 *   - one CUDA stream per handle (kx_sched_stream); handles are re-entrant,
 *     no global mutable state (engine.hpp:125-134 threading contract).
 *   - the product path is CUDA only: with no usable sm_100 device every call
 *     that computes fails with KX_ERR_CUDA. There is no CPU fallback.
 */
#ifndef KAIROS_B200_H_
#define KAIROS_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KX_ABI_VERSION 1

enum kx_status {
  KX_OK = 0,
  KX_ERR_INVALID = 1,   /* std::invalid_argument */
  KX_ERR_LOGIC = 2,     /* std::logic_error */
  KX_ERR_RUNTIME = 3,   /* std::runtime_error */
  KX_ERR_CUDA = 4,      /* CUDA runtime failure / no device */
  KX_ERR_CAPACITY = 5,  /* a fixed device capacity was exceeded */
  KX_ERR_LIVELOCK = 6   /* reference would spin forever */
};

enum kx_mem {
  KX_MEM_HOST = 0,
  KX_MEM_DEVICE = 1,
  /* kx_queue_upload only: pinned host memory the device can address
   * (cudaHostAlloc / cudaMallocHost / cudaHostRegister). The columns every
   * request's key needs (agent, app_start, queue_enter, pure_exec) are
   * copied; prompt_tokens, kept_tokens, msg_key and uid stay in host memory
   * and are read in place by the kernels that need them (dispatched heads,
   * exact-tuple ties, decision rows) -- a few thousand reads per tick instead
   * of 32 bytes per request over the host link. The caller keeps those arrays
   * alive and unchanged until the next upload; enqueue, remove_admitted and
   * graph capture first copy them to the device. Their values are not range
   * checked up front (the reference does not check them either). */
  KX_MEM_HOST_MAPPED = 2
};

/* SchedulerKind (harness.hpp:16) */
enum kx_scheduler_kind {
  KX_SCHED_KAIROS = 0, /* KairosScheduler   scheduler.hpp:105-133 */
  KX_SCHED_FCFS = 1,   /* FcfsScheduler     scheduler.hpp:48-54   */
  KX_SCHED_TOPO = 2,   /* TopoDepthScheduler scheduler.hpp:58-76  */
  KX_SCHED_ORACLE = 3  /* OracleScheduler   scheduler.hpp:80-93   */
};

/* DispatchPolicy (dispatcher.hpp:107) */
enum kx_dispatch_policy {
  KX_DISPATCH_TIME_SLOT = 0,
  KX_DISPATCH_ROUND_ROBIN = 1,
  KX_DISPATCH_STATIC_THRESHOLD = 2
};

/* InstanceProfile (engine.hpp:25-31) plus the pool (shared LLM) it serves. */
typedef struct kx_instance {
  int32_t id;              /* InstanceId (dispatcher.hpp:14) */
  int32_t pool;            /* 0..n_pools-1 */
  double capacity_tokens;
  double decode_rate;      /* k, tokens/s per request */
  double prefill_rate;     /* prompt tokens/s */
  int32_t max_batch;
  int32_t _pad;
} kx_instance;

/* DispatcherConfig (dispatcher.hpp:112-121) + EngineConfig fields the
 * dispatch loop reads (engine.hpp:33-41). */
typedef struct kx_dispatcher_config {
  int32_t policy;                 /* kx_dispatch_policy */
  int32_t oracle_expected_time;   /* T = pure_exec of the request */
  double slot_len;                /* 0.5 */
  double resume_watermark;        /* 0.85 */
  double static_threshold;        /* 0.90 */
  double default_expected_time;   /* 1.0 */
} kx_dispatcher_config;

typedef struct kx_sched_config {
  int32_t n_pools;                /* independent shared-LLM pools */
  int32_t n_instances;
  const kx_instance* instances;   /* host array, n_instances; pool-grouped order = Dispatcher ids_ order */
  kx_dispatcher_config dispatcher;
  int64_t queue_capacity;         /* max queued requests (all pools) */
  int32_t max_agents;             /* capacity of the per-agent tables */
  int32_t slot_ring;              /* ledger slots kept per instance (power of 2, >= 64) */
  int32_t device;                 /* CUDA device ordinal */
  int32_t log_capacity_per_pool;  /* decision-log rows per pool per round (0 = default) */
} kx_sched_config;

/* Queue contents, one element per PendingRequest (types.hpp:35-42).
 * msg_key is any u64 whose order equals the lexicographic order of msg_id
 * strings in the queue; agent is a dense agent index. */
typedef struct kx_queue_view {
  const int32_t* agent;
  const int64_t* prompt_tokens;
  const double* app_start;
  const double* queue_enter;
  const uint64_t* msg_key;
  const uint64_t* uid;
  const int64_t* kept_tokens;     /* nullable: CallRuntime::kept_tokens (engine.cpp:306-307) */
  const double* pure_exec;        /* nullable: required when oracle_expected_time */
} kx_queue_view;

/* DecisionLogRow (engine.hpp:92-99) plus bookkeeping. */
typedef struct kx_decision {
  double time;
  double predicted_peak;
  uint64_t uid;
  int64_t queue_index;            /* index into the uploaded queue */
  int32_t agent;
  int32_t target;                 /* InstanceId, -1 = none (dispatch stops) */
  int32_t pool;
  int32_t admitted;               /* 1 = popped+committed+admitted; 0 = overload retry / no target */
} kx_decision;

typedef struct kx_sched kx_sched;

int kx_abi_version(void);
const char* kx_last_error(void);
/* 1 when an sm_100-class device is visible, 0 otherwise (no error). */
int kx_device_available(void);

/* ---- handle lifecycle ------------------------------------------------- */
/* Replaces Dispatcher::Dispatcher (dispatcher.cpp:185-198) + Simulator's
 * per-instance state (engine.hpp:147-153) + ReadyQueue storage. */
int kx_sched_create(const kx_sched_config* cfg, kx_sched** out);
int kx_sched_destroy(kx_sched* s);
int kx_sched_stream(kx_sched* s, void** cuda_stream);
int kx_sched_synchronize(kx_sched* s);

/* ---- scheduler policy (scheduler.hpp:31-44) ----------------------------- */
int kx_set_scheduler(kx_sched* s, int32_t kind);
/* Per-agent tables, indexed by dense agent index:
 *   agent_pool[a]   pool whose queue/instances serve agent a
 *   priority_key[a] PriorityTable::priority_key(agent) incl. the cold-start
 *                   median (priority.cpp:114-135); Kairos only
 *   topo_depth[a]   TopoDepthScheduler::depth_of (scheduler.hpp:71-74)
 *   expected_T[a]   ProfilerSnapshot::expected_exec_time(agent, default)
 *                   (profiler.cpp:11-16, engine.cpp:177-185)
 * Any of the three value tables may be NULL (kept from the previous call). */
int kx_set_agent_tables(kx_sched* s, int32_t n_agents, const int32_t* agent_pool,
                        const double* priority_key, const int32_t* topo_depth,
                        const double* expected_T, uint64_t version);
/* OracleScheduler's remaining_by_uid (scheduler.hpp:84-89): dense over
 * [uid_base, uid_base + n); present[i] == 0 means "absent" (key 0.0). */
int kx_set_remaining_table(kx_sched* s, uint64_t uid_base, int64_t n,
                           const double* remaining, const uint8_t* present, int32_t mem);

/* ---- ready queue (priority.hpp:70-116) ----------------------------------- */
/* Replaces ReadyQueue contents with n requests (ReadyQueue::enqueue x n). */
int kx_queue_upload(kx_sched* s, int64_t n, const kx_queue_view* q, int32_t mem);
/* ReadyQueue::enqueue (priority.hpp:72) x n: appends n requests behind the
 * current ones, in the given order (push_back; the order decides exact-tuple
 * ties, priority.hpp:89-103). msg_key must rank like the keys already queued
 * (H1: one key space per queue). Invalidates the last order / dispatch round. */
int kx_queue_enqueue(kx_sched* s, int64_t n, const kx_queue_view* q, int32_t mem);
int kx_queue_size(kx_sched* s, int64_t* n);
/* Drops every request admitted by the last dispatch round (ReadyQueue::pop
 * of the placed prefix), keeping the others in their relative order. The
 * queue is double-buffered: without a captured graph the buffers swap;
 * with one, the kept prefix is copied back so the graph's addresses hold. */
int kx_queue_remove_admitted(kx_sched* s);

/* K2: per-request OrderKey (SchedulerPolicy::order_key, scheduler.hpp:17-27),
 * written in queue order. */
int kx_score(kx_sched* s, double* k0, double* k1, double* k2, int32_t mem);

/* K2+K3+K4: the full queue order under the active policy: the permutation
 * std::sort with the ReadyQueue comparator would produce (priority.hpp:89-103,
 * harness.cpp:92-100), grouped by pool. Asynchronous on the handle's stream. */
int kx_order(kx_sched* s);
/* perm[n] (queue indices, sorted), pool_offsets[n_pools + 1]. */
int kx_order_fetch(kx_sched* s, uint32_t* perm, int64_t* pool_offsets, int32_t mem);

/* K5: one dispatch round at time `now` over the last order: the placement
 * part of Simulator::dispatch_loop (engine.cpp:220-268) with
 * Dispatcher::choose/commit (dispatcher.cpp:207-262), the admission
 * bookkeeping of admit (engine.cpp:298-319), try_admit (270-296) and
 * Dispatcher::gc (engine.cpp:212). One CTA per pool. Asynchronous. */
int kx_dispatch_round(kx_sched* s, double now);
/* Copies the decision log of the last round. per_pool_count[n_pools]:
 * rows written per pool; rows[] and candidate_peaks[] are pool-major with
 * `row_stride` rows per pool and `peak_stride` peaks per row (>= max
 * instances in a pool); only the first per_pool_count[p] rows of each pool's
 * block are written. Any output pointer may be NULL. Synchronizes. */
int kx_dispatch_fetch(kx_sched* s, int64_t* per_pool_count, kx_decision* rows,
                      double* candidate_peaks, int64_t* row_stride, int64_t* peak_stride);

/* One scheduling tick: kx_order + kx_dispatch_round (asynchronous). */
int kx_tick(kx_sched* s, double now);

/* ---- waiting lists: round_robin / static_threshold (engine.cpp:259-296) ---
 * Under KX_DISPATCH_ROUND_ROBIN and KX_DISPATCH_STATIC_THRESHOLD a dispatch
 * round pops each placed head into its target instance's waiting list
 * (engine.cpp:259-262) and runs try_admit on it (engine.cpp:270-296); after
 * the loop every instance runs try_admit once more (engine.cpp:211). The
 * waiting lists are device-resident between rounds. In those rounds a
 * decision row's `admitted` = 1 means "popped into the target's waiting
 * list", predicted_peak is 0.0 and no candidate peaks are logged (the
 * reference's DispatchDecision carries none), and every admission out of a
 * waiting list is logged as a kx_admission row. */
typedef struct kx_admission {
  double time;
  uint64_t uid;
  int64_t queue_index;            /* index in this round's queue, -1 = entered an earlier round */
  int32_t instance;               /* InstanceId */
  int32_t pool;
} kx_admission;
/* Entries per instance waiting list (default 1024; grows on upload). */
int kx_waiting_reserve(kx_sched* s, int64_t per_instance);
/* Replaces every waiting list: entry j joins the list of the instance at
 * position instance_pos[j] (kx_sched_config.instances order), appended in
 * array order. Host memory only. Also sets the instances' waiting counts. */
int kx_waiting_upload(kx_sched* s, int64_t n, const int32_t* instance_pos, const kx_queue_view* q);
/* uid[] of the waiting list of the instance at position instance_pos, in
 * list order (at most cap entries copied; *n_out = list length). */
int kx_waiting_fetch(kx_sched* s, int32_t instance_pos, int64_t cap, uint64_t* uid, int64_t* n_out);
/* Admission log of the last round: per_pool_count[n_pools]; rows pool-major
 * with *row_stride rows per pool (= the decision-log capacity). */
int kx_admissions_fetch(kx_sched* s, int64_t* per_pool_count, kx_admission* rows, int64_t* row_stride);
/* Dispatcher::rr_next_ per pool (dispatcher.hpp:174): get and/or set (either may be NULL). */
int kx_rr_next(kx_sched* s, int64_t* get_per_pool, const int64_t* set_per_pool);

/* ---- instance / ledger state (dispatcher.cpp:44-123, 264-297) ---------- */
/* Engine-side live view (engine.cpp:187-202): live_kv, running, waiting,
 * indexed by position in the kx_sched_config.instances array. */
int kx_instances_set_live(kx_sched* s, const double* live_kv, const int32_t* running,
                          const int32_t* waiting);
int kx_instances_get_live(kx_sched* s, double* live_kv, int32_t* running, int32_t* waiting,
                          uint8_t* suspended);
/* SlotLedger::try_place (dispatcher.cpp:52-68) without booking. */
int kx_ledger_try_place(kx_sched* s, int32_t instance_id, double prefill_tokens,
                        double decode_rate, double t_start, double expected_duration,
                        int32_t* fits, double* predicted_peak, int64_t* violating_slot);
/* SlotLedger::commit (dispatcher.cpp:70-79); KX_ERR_LOGIC when it exceeds. */
int kx_ledger_commit(kx_sched* s, int32_t instance_id, uint64_t uid, double prefill_tokens,
                     double decode_rate, double t_start, double expected_duration);
/* Many SlotLedger::commit calls at once (e.g. preloading a pool): entry j
 * books (uid[j], P[j], k[j], t0[j], T[j]) on instance_id[j] if try_place
 * fits, in array order per instance; fits_out[j] = 1/0 (nullable). */
int kx_ledger_commit_batch(kx_sched* s, int64_t n, const int32_t* instance_id, const uint64_t* uid,
                           const double* prefill_tokens, const double* decode_rate,
                           const double* t_start, const double* expected_duration,
                           uint8_t* fits_out);
/* Dispatcher::on_request_finished / on_request_preempted (dispatcher.cpp:264-276). */
int kx_on_request_finished(kx_sched* s, int32_t instance_id, uint64_t uid, double actual_end);
/* Dispatcher::on_overload / on_live_usage / suspended (dispatcher.cpp:278-293). */
int kx_on_overload(kx_sched* s, int32_t instance_id);
int kx_on_live_usage(kx_sched* s, int32_t instance_id, double live_kv);
/* Dispatcher::gc (dispatcher.cpp:295-297). */
int kx_gc(kx_sched* s, double now);
/* Dense ledger view: usage[slot_ring] and exists[slot_ring] for slots
 * base_slot .. base_slot + slot_ring - 1; active request count. */
int kx_ledger_read(kx_sched* s, int32_t instance_id, int64_t* base_slot, double* usage,
                   uint8_t* exists, int32_t* active_requests);
/* Device-side snapshot of all mutable instance/ledger state, and restore. */
int kx_state_checkpoint(kx_sched* s);
int kx_state_restore(kx_sched* s);

/* ---- measurement ---------------------------------------------------------- */
/* Per-phase device timing with CUDA events recorded on the handle's stream
 * around every launch of a phase (score/range, keygen, each radix pass,
 * tie-fix, dispatch). Algorithmic bytes are the library's own per-phase
 * accounting. */
typedef struct kx_phase_stat {
  char name[32];
  double total_ms;
  int64_t launches;
  double alg_bytes;  /* summed over launches */
} kx_phase_stat;
int kx_profile_enable(kx_sched* s, int32_t enable);  /* also clears the stats */
int kx_profile_read(kx_sched* s, kx_phase_stat* out, int32_t cap, int32_t* n_out);
/* Kernels launched by this library (all handles) since load. */
int64_t kx_launch_count(void);

/* ---- K6: replica engine --------------------------------------------------- */
/* Simulator::run (engine.cpp:85-486) for many independent replicas at once,
 * one warp per replica: the (time, kind, seq) event order, continuous
 * batching, per-token KV growth, preempt-with-recompute and the dispatch
 * rounds of engine.cpp:204-296. Supported: FCFS / TopoDepth / Oracle
 * scheduling with TimeSlot (oracle_expected_time), RoundRobin or
 * StaticThreshold dispatch. */
typedef struct kx_engine_config {
  int32_t n_instances;
  int32_t scheduler;              /* KX_SCHED_KAIROS / FCFS / TOPO / ORACLE */
  const kx_instance* instances;   /* pool ignored */
  kx_dispatcher_config dispatcher;
  int32_t n_agents;
  int32_t slot_ring;              /* 0 = 256 */
  const int32_t* topo_depth;      /* per agent index (TopoDepthScheduler) */
  double dispatch_period;         /* engine.hpp:35 (0.1) */
  double recompute_fraction;      /* engine.hpp:36 (1.0) */
  int32_t heap_capacity;          /* 0 = 1024 pending events per replica */
  int32_t device;
  uint64_t max_events;            /* 0 = 2e8 (engine.cpp:25) */
  double warmup_seconds;          /* MetricsOptions::warmup_seconds (metrics.hpp:21-25) */
  /* KairosScheduler (scheduler.hpp:94-133): agent indices in AgentId order
   * (std::map<AgentId,...> iteration order, the W1 matrix's label order);
   * NULL = index order. Rebuild every N completed workflows (0 = 256). */
  const int32_t* agent_order;
  uint64_t kairos_rebuild_interval;
} kx_engine_config;

/* Replicas concatenated (host arrays). Replica r owns workflows
 * [wf_base[r], wf_base[r+1]) in arrival order (msg ids "m-<local index>")
 * and their calls [wf_offsets[w], wf_offsets[w+1]) in node order. */
typedef struct kx_replica_batch {
  int32_t n_replicas;
  int32_t _pad;
  const int64_t* wf_base;         /* [R+1] */
  const double* arrival;          /* [W] */
  const int64_t* wf_offsets;      /* [W+1] */
  const int32_t* agent;           /* [C] agent index */
  const int32_t* parent;          /* [C] parent node id, -1 = entry */
  const int64_t* prompt_tokens;   /* [C] */
  const int64_t* target_tokens;   /* [C] */
  const double* pure_exec;        /* [C] */
  const double* remaining;        /* [C] remaining_by_uid (Oracle key) */
  const uint64_t* uid;            /* [C] */
} kx_replica_batch;

/* RunResult (engine.hpp:101-118), host arrays allocated by the caller; any
 * pointer may be NULL. Completion-ordered arrays use each replica's own
 * segment (calls: [wf_offsets[wf_base[r]], ...), workflows: [wf_base[r], ...)). */
typedef struct kx_replica_results {
  int64_t* call_order;            /* [C] completed call (global index), completion order */
  double* exec_start;             /* [C] completion order */
  double* exec_end;               /* [C] completion order */
  int32_t* instance;              /* [C] completion order (instance index) */
  double* first_enqueue;          /* [C] by call */
  double* queue_seconds;          /* [C] by call */
  int32_t* episodes;              /* [C] by call */
  int32_t* preemptions;           /* [C] by call */
  int64_t* wf_order;              /* [W] completed workflow (global index), completion order */
  double* wf_finish;              /* [W] by workflow */
  int64_t* wf_output_tokens;      /* [W] by workflow */
  int32_t* wf_calls;              /* [W] by workflow */
  double* scalars;                /* [R*8]: preemption_events, preempted_requests, wasted_kv,
                                     completed_kv, prefill_seconds, decode_seconds, events, end_time */
  int64_t* counts;                /* [R*4]: calls done, workflows done, status, events */
  /* K7, compute_metrics (metrics.cpp:13-88) per replica, computed on the
   * device: [R*16] = instances, requests, mean / p90 / p95 / p99 token
   * latency, mean request token latency, mean queueing ratio, preemption
   * rate, preempted requests, preemption events, wasted memory fraction,
   * total queue seconds, decode time fraction, sim end time, latency count */
  double* metrics;
  uint32_t* histogram;            /* [R*256] token-latency bins: floor((log2 x + 16) * 8) */
  /* Kairos: final PriorityTable::priority_key per agent index [R*n_agents]
   * and the number of tables built per replica [R] (NULL = not wanted) */
  double* priority_keys;
  int64_t* table_versions;
} kx_replica_results;

/* aggregate_metrics (metrics.cpp:90-123) over per-replica metric rows in
 * replica order (host arithmetic on R rows of kx_replica_results.metrics). */
int kx_aggregate_metrics(int32_t n_rows, const double* rows, double* out);

int kx_replicas_run(const kx_engine_config* cfg, const kx_replica_batch* batch,
                    kx_replica_results* out, double* device_ms);

/* ---- K8: pairwise sorting accuracy ---------------------------------------- */
/* pairwise_sorting_accuracy (priority.cpp:165-189) of a schedule given in
 * schedule order: agent[i], remaining[i] (true remaining latency) and
 * present[i] (0 = uid absent from true_remaining, skipped; NULL = all).
 * scope_all = 0: cross-agent pairs (PairScope::CrossAgent), 1: all pairs.
 * Exact integer counting on the device in O(N log^2 N). *pairs = compared
 * pairs, *correct = the reference's sum of 1.0 / 0.5 terms, *accuracy =
 * correct / pairs, or NaN when pairs == 0 (the reference's nullopt). */
int kx_sorting_accuracy(int64_t n, const int32_t* agent, const double* remaining,
                        const uint8_t* present, int32_t scope_all, uint64_t* pairs,
                        double* correct, double* accuracy);

/* ---- CUDA graph of a repeated step (e.g. kx_state_restore + kx_tick) ------ */
/* Calls between begin and end are captured (asynchronous calls only: no
 * fetches, profiling off) and replayed by kx_graph_launch with one launch.
 * The captured kernels carry the queue size of the capture: after a
 * kx_queue_remove_admitted / kx_queue_enqueue that changed the size,
 * kx_graph_launch fails with KX_ERR_LOGIC (capture again). After a replay
 * the last order / dispatch round is fetchable as after the captured calls. */
int kx_graph_capture_begin(kx_sched* s);
int kx_graph_capture_end(kx_sched* s);
int kx_graph_launch(kx_sched* s);
/* Drops the captured graph (kx_queue_remove_admitted then compacts by
 * swapping the queue's double buffer instead of copying back). */
int kx_graph_release(kx_sched* s);

/* ---- priority table: W1 distance matrix ------------------------------------ */
/* Replaces build_distance_matrix_from_samples (priority.cpp:60-65) ->
 * build_matrix (priority.cpp:15-46): samples holds each agent's sorted sample
 * set back to back (offsets[0..n_agents]); out receives the (n_agents + 1)^2
 * row-major matrix whose last label is the anchor (a single sample 0.0),
 * d[i][j] = wasserstein_1d (distribution.cpp:9-31), bit-identical. Errors as
 * the reference: no agents / an empty set -> KX_ERR_INVALID. Host pointers.
 * The 1-D classical MDS of the matrix (priority.cpp:67-112) stays on the host. */
int kx_w1_matrix(int32_t n_agents, const int64_t* offsets, const double* samples, double* out);

/* ProfilerSnapshot::expected_exec_time (profiler.cpp:11-16) for n_agents
 * sorted execution-sample sets back to back (offsets[0..n_agents]): out[a] =
 * mode_estimate(set a, min_samples).value (distribution.cpp:46-86; the
 * reference's default min_samples is 16), or `fallback` for an empty set.
 * Bit-identical to the reference (glibc cbrt replayed on the device). Host
 * pointers; unsorted sets -> KX_ERR_INVALID. */
int kx_expected_exec_times(int32_t n_agents, const int64_t* offsets, const double* samples,
                           int64_t min_samples, double fallback, double* out);

/* ---- workload synthesis (host) ------------------------------------------ */
/* realize() (workload.cpp:319-372) for the built-in templates
 * (workload.cpp:462-560); app_mask selects QA/RG/CG in that order
 * (colocated_workload = all three). Agents are indexed in the order of
 * kx_builtin_agent_name(0..9). Same seed -> the reference's realization. */
enum kx_app_mask { KX_APPS_QA = 1, KX_APPS_RG = 2, KX_APPS_CG = 4 };
typedef struct kx_realization kx_realization;
const char* kx_builtin_agent_name(int32_t agent);
int kx_realize_builtin(uint32_t app_mask, double rate, double duration, uint64_t seed,
                       double prefill_rate, double decode_rate, kx_realization** out);
/* realize() (workload.cpp:319-372) for a general WorkloadConfig
 * (workload.hpp:69-83): agents are dense indices 0..n_agents-1 (the caller
 * keeps the names), AgentSpec (workload.hpp:39-52) with a choice list,
 * a parallel list and an optional feedback edge; AppSpec (workload.hpp:55-60)
 * lists its member agents (the validate() cycle check walks from them).
 * TraceFile arrivals are passed as the file's raw timestamps
 * (ingest_arrival_trace's parse is the caller's; scale_arrival_gaps and the
 * duration cut are applied here). validate()'s errors -> KX_ERR_INVALID. */
enum kx_length_kind { KX_LEN_FIXED = 0, KX_LEN_UNIFORM = 1, KX_LEN_LOGNORMAL = 2 };
typedef struct kx_length_spec {   /* LengthSpec (workload.hpp:18-33) */
  int32_t kind;                   /* kx_length_kind */
  int32_t _pad;
  double a;                       /* Fixed: value; Uniform: lo; Lognormal: mu = log(median) */
  double b;                       /* Uniform: hi; Lognormal: sigma */
  int64_t min_tokens, max_tokens;
} kx_length_spec;
typedef struct kx_agent_spec {
  kx_length_spec prompt_len, output_len;
  int32_t n_choice;               /* choice: (choice_to[j], choice_p[j]) */
  int32_t n_parallel;
  const int32_t* choice_to;
  const double* choice_p;
  const int32_t* parallel_to;
  int32_t feedback_target;        /* -1 = no feedback */
  int32_t feedback_max_iterations;
  double feedback_probability;
} kx_agent_spec;
typedef struct kx_app_spec {
  int32_t entry;                  /* agent index */
  int32_t n_members;
  const int32_t* members;         /* the app's agents */
  double weight;
} kx_app_spec;
enum kx_arrival_kind { KX_ARRIVAL_POISSON = 0, KX_ARRIVAL_TRACE = 1 };
enum kx_entry_selection { KX_ENTRY_WEIGHTED = 0, KX_ENTRY_CYCLE = 1 };
typedef struct kx_workload_config {
  int32_t n_agents;
  int32_t n_apps;
  const kx_agent_spec* agents;
  const kx_app_spec* apps;
  int32_t arrival_kind;           /* kx_arrival_kind */
  int32_t entry_selection;        /* kx_entry_selection */
  double rate;                    /* Poisson arrivals per second */
  int64_t n_trace;                /* TraceFile: raw timestamps */
  const double* trace;
  double trace_scale;             /* inter-arrival scaling factor */
  double duration;                /* arrival window, seconds */
} kx_workload_config;
int kx_realize(const kx_workload_config* config, uint64_t seed, double prefill_rate, double decode_rate,
               kx_realization** out);
int kx_realization_sizes(const kx_realization* r, int64_t* n_workflows, int64_t* n_calls);
/* Any output may be NULL; wf_offsets has n_workflows + 1 entries. */
int kx_realization_copy(const kx_realization* r, double* arrival, int32_t* app, int64_t* wf_offsets,
                        int32_t* agent, int32_t* parent, int64_t* prompt, int64_t* target,
                        double* pure_exec, double* remaining, uint64_t* uid);
void kx_realization_free(kx_realization* r);

/* ---- trace CSV I/O + workflow reconstruction ------------- */
/* read_trace (trace.cpp:111-127) of a whole CSV on the device: lines split on
 * '\n' (std::getline), the header line (kTraceHeader, trace.cpp:10-12)
 * skipped on line 1, empty lines skipped, every line parsed and validated
 * as parse_trace_line + validate (trace.cpp:14-27, 90-109). The first bad
 * line fails with KX_ERR_INVALID and the reference's message ("trace line N:
 * ..."). Numbers: correctly rounded like strtod for decimal forms with <= 19
 * significant digits and a power of ten within +-22 (every format_seconds
 * output below 1e10 s); other std::stod forms (hex, inf, nan, longer
 * significands, larger exponents) are refused, never approximated. Agents are ranked
 * in std::string order (the graph's std::map/std::set order); msg ids keep
 * an internal index. */
typedef struct kx_trace kx_trace;
int kx_trace_parse(const char* bytes, int64_t n_bytes, int32_t device, kx_trace** out);
void kx_trace_free(kx_trace* t);
int kx_trace_sizes(const kx_trace* t, int64_t* n_records, int32_t* n_agents, int64_t* n_msgs,
                   int64_t* agent_name_bytes);
/* Agent names, concatenated; offsets[n_agents + 1]. */
int kx_trace_agents(const kx_trace* t, char* names, int64_t* offsets);
/* RequestRecord fields (types.hpp) in file order; upstream = -1 when empty.
 * Any output may be NULL. */
int kx_trace_columns(const kx_trace* t, int64_t* msg, int32_t* agent, int32_t* upstream, double* exec_start,
                     double* exec_end, int64_t* prompt_tokens, int64_t* output_tokens, double* app_start);
int kx_trace_msg_id(const kx_trace* t, int64_t msg, char* buf, int64_t cap, int64_t* len);
/* Byte offset and length, in the parsed bytes, of each of msgs[0..k) (the
 * msg_id strings of WorkflowGraph diagnostics, workflow.cpp:99-108, in bulk). */
int kx_trace_msg_spans(const kx_trace* t, int64_t k, const int64_t* msgs, int64_t* off, int32_t* len);
/* write_trace (trace.cpp:44-48) of the parsed records, formatted on the
 * device (format_seconds' "%.9f" exact); out = NULL returns the size. */
int kx_trace_format(kx_trace* t, char* out, int64_t cap, int64_t* n_out);
/* WorkflowAnalyzer::ingest_trace (workflow.cpp:319-343): every msg_id group
 * folded by WorkflowGraph::ingest_instance (workflow.cpp:59-111). */
typedef struct kx_workflow_sizes {
  int64_t n_edges;        /* distinct (upstream, agent) edges */
  int64_t n_diagnostics;  /* conflicting-entry diagnostics */
  int64_t instances;      /* instances_ingested */
} kx_workflow_sizes;
int kx_workflow_reconstruct(kx_trace* t, kx_workflow_sizes* sizes);
/* Edges in (from, to) name order with their observation counts; per agent:
 * entry flag and the fan-out tallies (parallel, sequential, single
 * observations; an agent with none is no fan-out node); diagnostics in
 * ingest order (msg index, the instance's entry, the conflicting entry).
 * Any output may be NULL. */
int kx_workflow_fetch(const kx_trace* t, int32_t* edge_from, int32_t* edge_to, uint64_t* edge_count,
                      uint8_t* is_entry, uint64_t* fan_parallel, uint64_t* fan_sequential, uint64_t* fan_single,
                      int64_t* diag_msg, int32_t* diag_entry, int32_t* diag_other);

/* ---- K1: orchestrator DP ------------------------------------------------ */
/* finalize_instance (workload.cpp:292-315) for many workflow instances at
 * once: calls of workflow w are [wf_offsets[w], wf_offsets[w+1]), in node_id
 * order; parent[c] is the parent's node_id within its workflow (-1 = root).
 * Writes uid (uid_base + global call index), pure_exec and remaining_exec.
 * One warp per workflow, reverse topological. Synchronous. */
int kx_orchestrator_dp(int64_t n_workflows, const int64_t* wf_offsets, const int32_t* parent,
                       const int64_t* prompt_tokens, const int64_t* target_tokens,
                       double prefill_rate, double decode_rate, uint64_t uid_base,
                       uint64_t* uid_out, double* pure_exec_out, double* remaining_out,
                       int32_t mem);
/* ---- K9: profiler ingestion (distribution.cpp:91-123, profiler.cpp:20-50) ----
 * LatencyProfiler over dense agent indices: per agent an execution and a
 * remaining-latency EmpiricalDistribution (sorted samples, sliding window,
 * doubling-checkpoint W1 convergence), device-resident. capacity = retained
 * samples per distribution (>= window_cap + 1 where window_cap > 0; an
 * unbounded kind needs room for all its samples, else KX_ERR_CAPACITY). */
typedef struct kx_convergence_config {  /* ConvergenceConfig (distribution.hpp:36-40) */
  uint64_t min_samples;                 /* 16 */
  double relative_threshold;            /* 0.05 */
  int64_t window_cap;                   /* 0 = unbounded; remaining: 4096 */
} kx_convergence_config;
typedef struct kx_profiler kx_profiler;
int kx_profiler_create(int32_t n_agents, const kx_convergence_config* exec,
                       const kx_convergence_config* remaining, int64_t capacity, int32_t device,
                       kx_profiler** out);
int kx_profiler_destroy(kx_profiler* p);
/* record_execution (profiler.cpp:20-29) for n samples in order. */
int kx_profiler_record_execution(kx_profiler* p, int64_t n, const int32_t* agent, const double* latency);
/* record_remaining (profiler.cpp:31-50) for many completed workflows in
 * completion order (records of workflow w: [rec_offsets[w], rec_offsets[w+1])).
 * newly_converged[w] (nullable) = take_newly_converged() right after w. A
 * negative sample fails the whole batch before any sample is applied. */
int kx_profiler_record_remaining(kx_profiler* p, int64_t n_workflows, const int64_t* rec_offsets,
                                 const int32_t* agent, const double* exec_start, const double* exec_end,
                                 uint8_t* newly_converged);
/* One distribution (kind 0 execution, 1 remaining): samples() (sorted, up to
 * cap copied), size, total_added, converged, last_checkpoint_distance. */
int kx_profiler_read(kx_profiler* p, int32_t kind, int32_t agent, int64_t cap, double* samples, int64_t* n,
                     uint64_t* total_added, int32_t* converged, double* last_distance);

/* LatencyProfiler::record_remaining's arithmetic (profiler.cpp:31-50) for
 * many completed workflows: finish = max exec_end (seeded with the first
 * record), sample[r] = finish - exec_start[r]. Synchronous. */
int kx_record_remaining(int64_t n_workflows, const int64_t* rec_offsets,
                        const double* exec_start, const double* exec_end,
                        double* finish_out, double* samples_out, int32_t mem);

#ifdef __cplusplus
}
#endif

#endif /* KAIROS_B200_H_ */

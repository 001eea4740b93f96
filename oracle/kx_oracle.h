/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle of the Kairos scheduling path.
 *
 * A plain-C restatement of the reference algorithms on the hot path
 * (/root/reference/proj, cited per function in kx_oracle.c). It is the
 * checker for the CUDA kernels: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. It is pinned
 * against the reference itself through fixtures produced by
 * oracle/gen_golden.cpp (which links the unmodified reference sources) and
 * checked in tests/test_oracle_golden.py.
 */
#ifndef KX_ORACLE_H_
#define KX_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { KXO_KAIROS = 0, KXO_FCFS = 1, KXO_TOPO = 2, KXO_ORACLE = 3 };

typedef struct kxo_queue {
  int64_t n;
  const int32_t* agent;
  const int64_t* prompt;
  const double* app_start;
  const double* queue_enter;
  const uint64_t* msg_key;
  const uint64_t* uid;
  const int64_t* kept;       /* nullable */
  const double* pure_exec;   /* nullable */
} kxo_queue;

typedef struct kxo_tables {
  int32_t n_agents;
  const int32_t* pool;
  const double* pk;          /* PriorityTable::priority_key per agent */
  const int32_t* depth;      /* TopoDepthScheduler depth per agent */
  const double* T;           /* expected exec time per agent */
  uint64_t rem_base;         /* Oracle: remaining_by_uid dense over [base, base+n) */
  int64_t rem_n;
  const double* rem;
  const uint8_t* rem_present;
} kxo_tables;

typedef struct kxo_decision {
  double time;
  double predicted_peak;
  uint64_t uid;
  int64_t queue_index;
  int32_t agent;
  int32_t target;
  int32_t pool;
  int32_t admitted;
} kxo_decision;

/* distribution.cpp */
double kxo_quantile_sorted(const double* sorted, int64_t n, double p);
double kxo_histogram_mode(const double* sorted, int64_t n);
double kxo_mode_estimate(const double* sorted, int64_t n, int64_t min_samples, int* median_fallback);
double kxo_wasserstein_1d(const double* a, int64_t na, const double* b, int64_t nb);
/* priority.cpp:121-135 — coords of table agents, anchor; returns the median
 * anchor distance (0 for an empty table). */
double kxo_median_anchor_distance(const double* coords, int64_t n, double anchor);

/* scheduler.hpp order_key per policy */
void kxo_order_keys(int policy, const kxo_queue* q, const kxo_tables* t, double* k0, double* k1,
                    double* k2);
/* Full order (pool-grouped, reference comparator priority.hpp:95-98). */
int kxo_sort(int policy, const kxo_queue* q, const kxo_tables* t, int32_t n_pools, uint32_t* perm,
             int64_t* pool_offsets);

/* SlotLedger (dispatcher.cpp:44-123) */
typedef struct kxo_ledger kxo_ledger;
kxo_ledger* kxo_ledger_new(int32_t id, double slot_len, double capacity);
void kxo_ledger_free(kxo_ledger* l);
int kxo_try_place(const kxo_ledger* l, double P, double k, double t0, double T, int32_t* fits,
                  double* peak, int64_t* violating_slot);
int kxo_commit(kxo_ledger* l, uint64_t uid, double P, double k, double t0, double T);
int kxo_finish(kxo_ledger* l, uint64_t uid, double actual_end);
void kxo_gc(kxo_ledger* l, double now);
int64_t kxo_ledger_dump(const kxo_ledger* l, int64_t* slots, double* usage, int64_t cap);
int64_t kxo_ledger_active(const kxo_ledger* l);

/* One pool's Dispatcher (TimeSlot) + engine live state. */
typedef struct kxo_pool {
  int32_t n_inst;
  const int32_t* id;
  const double* cap;
  const double* k;
  const int32_t* max_batch;
  double* live_kv;
  int32_t* running;
  int32_t* waiting;
  uint8_t* suspended;
  kxo_ledger** ledgers;
  double slot_len;
  double watermark;
  int32_t oracle_T;
} kxo_pool;

/* dispatch_loop (engine.cpp:220-268), TimeSlot, over the pool's order
 * perm[0..m), then gc (engine.cpp:212). Returns rows written; *status:
 * 0 ok, 6 livelock, 5 row capacity. */
int64_t kxo_dispatch_round(kxo_pool* p, const kxo_queue* q, const kxo_tables* t,
                           const uint32_t* perm, int64_t m, double now, int32_t pool_index,
                           kxo_decision* rows, double* cand, int64_t row_cap, int32_t* status);

/* One request in an instance's waiting list (InstanceState::waiting). */
typedef struct kxo_waitrec {
  double app_start, queue_enter;
  uint64_t msg, uid;
  int64_t prompt, kept, qidx;
  int32_t agent, round;
} kxo_waitrec;

typedef struct kxo_admission {
  double time;
  uint64_t uid;
  int64_t queue_index;
  int32_t instance;
  int32_t pool;
} kxo_admission;

/* dispatch_loop (engine.cpp:220-268) under RoundRobin / StaticThreshold
 * (dispatcher.cpp:214-231): each head popped into the target's waiting list
 * (p->waiting[i] entries at wrec + i * wcap) and try_admit (engine.cpp:270-296);
 * then try_admit on every instance (engine.cpp:211) and gc. *rr_next is
 * Dispatcher::rr_next_. Returns decision rows; *status: 0 ok, 5 capacity. */
int64_t kxo_dispatch_round_waiting(kxo_pool* p, int dispatch_policy, double static_thr, int sched_policy,
                                   int64_t* rr_next, kxo_waitrec* wrec, int64_t wcap, int32_t round,
                                   const kxo_queue* q, const kxo_tables* t, const uint32_t* perm,
                                   int64_t m, double now, int32_t pool_index, kxo_decision* rows,
                                   int64_t row_cap, kxo_admission* adm, int64_t adm_cap, int64_t* n_adm,
                                   int32_t* status);

/* EmpiricalDistribution (distribution.cpp:88-123): sorted samples, sliding
 * window, doubling-checkpoint convergence. add returns -1 on a negative
 * sample (invalid_argument), 1 when this add converged it, else 0. */
typedef struct kxo_dist kxo_dist;
kxo_dist* kxo_dist_new(uint64_t min_samples, double relative_threshold, int64_t window_cap);
void kxo_dist_free(kxo_dist* d);
int kxo_dist_add(kxo_dist* d, double value);
/* sorted samples (up to cap copied); returns the size */
int64_t kxo_dist_read(const kxo_dist* d, double* out, int64_t cap, uint64_t* total_added, int32_t* converged,
                      double* last_distance);

/* pairwise_sorting_accuracy (priority.cpp:165-189), O(N^2): returns 0 and
 * sets *acc when pairs > 0, returns 1 (nullopt) otherwise. */
int kxo_pairwise_accuracy(int64_t n, const int32_t* agent, const double* rem, const uint8_t* present,
                          int32_t scope_all, double* acc, uint64_t* pairs_out);

/* finalize_instance (workload.cpp:292-315) for many workflows. */
int kxo_finalize(int64_t n_wf, const int64_t* off, const int32_t* parent, const int64_t* prompt,
                 const int64_t* target, double prefill_rate, double decode_rate, uint64_t uid_base,
                 uint64_t* uid_out, double* pure_out, double* rem_out);
/* record_remaining arithmetic (profiler.cpp:31-50). */
void kxo_record_remaining(int64_t n_wf, const int64_t* off, const double* exec_start,
                          const double* exec_end, double* finish_out, double* samples_out);

#ifdef __cplusplus
}
#endif
#endif

/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle (restatement) of the Kairos
 * scheduling path. See kx_oracle.h. Compiled with -O2 -ffp-contract=off and
 * no -march=native so every multiply-add rounds twice, as the reference's
 * build does. Paths are relative to
 * /root/reference/proj.
 */
#include "kx_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double kTimeEpsilon = 1e-9; /* workflow.hpp:34 */

/* ---- distribution.cpp ---------------------------------------------------- */

/* quantile_sorted, distribution.cpp:33-44 */
double kxo_quantile_sorted(const double* s, int64_t n, double p) {
  if (n <= 0) return NAN;
  if (p <= 0.0) return s[0];
  if (p >= 1.0) return s[n - 1];
  const double pos = p * (double)(n - 1);
  const int64_t lo = (int64_t)pos;
  const double frac = pos - (double)lo;
  if (lo + 1 >= n) return s[n - 1];
  return s[lo] + frac * (s[lo + 1] - s[lo]);
}

/* histogram_mode, distribution.cpp:46-75 */
double kxo_histogram_mode(const double* s, int64_t n) {
  const double lo = s[0], hi = s[n - 1];
  if (!(hi > lo)) return lo;
  const double nn = (double)n;
  const double iqr = kxo_quantile_sorted(s, n, 0.75) - kxo_quantile_sorted(s, n, 0.25);
  int64_t bins = 64;
  if (iqr > 0.0) {
    const double width = 2.0 * iqr / cbrt(nn);
    bins = (int64_t)(uint64_t)ceil((hi - lo) / width);
    if (bins < 1) bins = 1;
    if (bins > 4096) bins = 4096;
  }
  uint64_t* counts = (uint64_t*)calloc((size_t)bins, sizeof(uint64_t));
  const double scale = (double)bins / (hi - lo);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t idx = (uint64_t)((s[i] - lo) * scale);
    if (idx >= (uint64_t)bins) idx = (uint64_t)bins - 1;
    ++counts[idx];
  }
  int64_t best = 0;
  for (int64_t k = 1; k < bins; ++k)
    if (counts[k] > counts[best]) best = k;
  free(counts);
  return lo + ((double)best + 0.5) * (hi - lo) / (double)bins;
}

/* mode_estimate, distribution.cpp:77-86 */
double kxo_mode_estimate(const double* s, int64_t n, int64_t min_samples, int* median_fallback) {
  if (n < min_samples) {
    if (median_fallback) *median_fallback = 1;
    return kxo_quantile_sorted(s, n, 0.5);
  }
  if (median_fallback) *median_fallback = 0;
  return kxo_histogram_mode(s, n);
}

/* wasserstein_1d, distribution.cpp:9-31 */
double kxo_wasserstein_1d(const double* a, int64_t na, const double* b, int64_t nb) {
  const uint64_t total = (uint64_t)na * (uint64_t)nb;
  uint64_t cur = 0;
  int64_t i = 0, j = 0;
  double acc = 0.0;
  while (cur < total) {
    const uint64_t a_next = (uint64_t)(i + 1) * (uint64_t)nb;
    const uint64_t b_next = (uint64_t)(j + 1) * (uint64_t)na;
    const uint64_t nxt = a_next < b_next ? a_next : b_next;
    acc += (double)(nxt - cur) * fabs(a[i] - b[j]);
    if (a_next == nxt) ++i;
    if (b_next == nxt) ++j;
    cur = nxt;
  }
  return acc / (double)total;
}

static int cmp_double(const void* x, const void* y) {
  const double a = *(const double*)x, b = *(const double*)y;
  return (a > b) - (a < b);
}

/* PriorityTable::median_anchor_distance, priority.cpp:121-130 */
double kxo_median_anchor_distance(const double* coords, int64_t n, double anchor) {
  if (n <= 0) return 0.0;
  double* d = (double*)malloc((size_t)n * sizeof(double));
  for (int64_t i = 0; i < n; ++i) d[i] = fabs(coords[i] - anchor);
  qsort(d, (size_t)n, sizeof(double), cmp_double);
  const double m = kxo_quantile_sorted(d, n, 0.5);
  free(d);
  return m;
}

/* ---- scheduler.hpp order_key ---------------------------------------------- */

static double rem_of(const kxo_tables* t, uint64_t uid) {
  /* OracleScheduler::order_key, scheduler.hpp:85-89: missing uid -> 0.0 */
  if (t->rem && uid >= t->rem_base && uid - t->rem_base < (uint64_t)t->rem_n &&
      t->rem_present[uid - t->rem_base])
    return t->rem[uid - t->rem_base];
  return 0.0;
}

static void key_of(int policy, const kxo_queue* q, const kxo_tables* t, int64_t i, double* k) {
  const int32_t a = q->agent[i];
  switch (policy) {
    case KXO_KAIROS: /* scheduler.hpp:111-113 */
      k[0] = t->pk[a];
      k[1] = q->app_start[i];
      k[2] = q->queue_enter[i];
      break;
    case KXO_FCFS: /* scheduler.hpp:51-53 */
      k[0] = q->queue_enter[i];
      k[1] = q->app_start[i];
      k[2] = 0.0;
      break;
    case KXO_TOPO: /* scheduler.hpp:63-65 (unknown agent: depth 1, 71-74) */
      k[0] = (double)t->depth[a];
      k[1] = q->queue_enter[i];
      k[2] = 0.0;
      break;
    default: /* Oracle */
      k[0] = rem_of(t, q->uid[i]);
      k[1] = q->queue_enter[i];
      k[2] = 0.0;
      break;
  }
}

void kxo_order_keys(int policy, const kxo_queue* q, const kxo_tables* t, double* k0, double* k1,
                    double* k2) {
  for (int64_t i = 0; i < q->n; ++i) {
    double k[3];
    key_of(policy, q, t, i, k);
    k0[i] = k[0];
    k1[i] = k[1];
    k2[i] = k[2];
  }
}

/* ---- ReadyQueue comparator (priority.hpp:95-98) ----------------------------- */

typedef struct {
  double k[3];
  double app, qe;
  uint64_t msg, uid;
  int32_t pool;
  uint32_t idx;
} sort_rec;

#define LT3(a, b) ((a) < (b) ? -1 : ((b) < (a) ? 1 : 0))

/* std::tie(key, app_start, queue_enter, msg_id, uid) <, OrderKey operator<
 * (scheduler.hpp:21-25); equal tuples keep queue order (best_index keeps the
 * first of equal minima). Pools are independent queues. */
static int cmp_rec(const void* x, const void* y) {
  const sort_rec* a = (const sort_rec*)x;
  const sort_rec* b = (const sort_rec*)y;
  int c;
  if ((c = LT3(a->pool, b->pool))) return c;
  if (a->k[0] != b->k[0]) return a->k[0] < b->k[0] ? -1 : 1;
  if (a->k[1] != b->k[1]) return a->k[1] < b->k[1] ? -1 : 1;
  if (a->k[2] != b->k[2]) return a->k[2] < b->k[2] ? -1 : 1;
  if (a->app != b->app) return a->app < b->app ? -1 : 1;
  if (a->qe != b->qe) return a->qe < b->qe ? -1 : 1;
  if ((c = LT3(a->msg, b->msg))) return c;
  if ((c = LT3(a->uid, b->uid))) return c;
  return LT3(a->idx, b->idx);
}

int kxo_sort(int policy, const kxo_queue* q, const kxo_tables* t, int32_t n_pools, uint32_t* perm,
             int64_t* pool_offsets) {
  const int64_t n = q->n;
  sort_rec* r = (sort_rec*)malloc((size_t)(n > 0 ? n : 1) * sizeof(sort_rec));
  if (!r) return 5;
  for (int64_t p = 0; p <= n_pools; ++p) pool_offsets[p] = 0;
  for (int64_t i = 0; i < n; ++i) {
    key_of(policy, q, t, i, r[i].k);
    r[i].app = q->app_start[i];
    r[i].qe = q->queue_enter[i];
    r[i].msg = q->msg_key[i];
    r[i].uid = q->uid[i];
    r[i].pool = t->pool[q->agent[i]];
    r[i].idx = (uint32_t)i;
    pool_offsets[r[i].pool + 1] += 1;
  }
  for (int32_t p = 0; p < n_pools; ++p) pool_offsets[p + 1] += pool_offsets[p];
  qsort(r, (size_t)n, sizeof(sort_rec), cmp_rec);
  for (int64_t i = 0; i < n; ++i) perm[i] = r[i].idx;
  free(r);
  return 0;
}

/* ---- SlotLedger (dispatcher.cpp:12-123) ------------------------------------ */

typedef struct {
  uint64_t uid;
  double P, k, t0, T;
} model;

struct kxo_ledger {
  int32_t id;
  double slot_len, cap;
  int64_t n_slots, slot_cap; /* std::map<int64_t,double> as a sorted array */
  int64_t* slot;
  double* used;
  int64_t n_act, act_cap;
  model* act;
};

kxo_ledger* kxo_ledger_new(int32_t id, double slot_len, double capacity) {
  kxo_ledger* l = (kxo_ledger*)calloc(1, sizeof(kxo_ledger));
  l->id = id;
  l->slot_len = slot_len;
  l->cap = capacity;
  return l;
}

void kxo_ledger_free(kxo_ledger* l) {
  if (!l) return;
  free(l->slot);
  free(l->used);
  free(l->act);
  free(l);
}

static int64_t find_slot(const kxo_ledger* l, int64_t s) {
  int64_t lo = 0, hi = l->n_slots;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (l->slot[mid] < s) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

static double usage_in_slot(const kxo_ledger* l, int64_t s) { /* dispatcher.cpp:120-123 */
  const int64_t i = find_slot(l, s);
  return (i < l->n_slots && l->slot[i] == s) ? l->used[i] : 0.0;
}

/* span_slots, dispatcher.cpp:19-31 */
static int span(double t0, double T, double L, int64_t* first, int64_t* last) {
  if (T <= 0.0) return 0;
  *first = (int64_t)floor((t0 + kTimeEpsilon) / L);
  *last = (int64_t)floor(((t0 + T) - kTimeEpsilon) / L);
  return *last >= *first;
}

/* peak_in_slot, dispatcher.cpp:33-42 */
static double peak_in_slot(double P, double k, double t0, double T, int64_t s, double L) {
  const double slot_start = (double)s * L;
  const double slot_end = slot_start + L;
  const double t_end = t0 + T;
  if (slot_end <= t0 + kTimeEpsilon || slot_start >= t_end - kTimeEpsilon) return 0.0;
  const double eval_t = (t_end < slot_end) ? t_end : slot_end;
  return P + k * (eval_t - t0);
}

/* SlotLedger::try_place, dispatcher.cpp:52-68 */
int kxo_try_place(const kxo_ledger* l, double P, double k, double t0, double T, int32_t* fits,
                  double* peak_out, int64_t* viol) {
  int64_t first = 0, last = -1;
  span(t0, T, l->slot_len, &first, &last);
  for (int64_t s = first; s <= last; ++s) {
    const double total = usage_in_slot(l, s) + peak_in_slot(P, k, t0, T, s, l->slot_len);
    if (total > l->cap) {
      *fits = 0;
      *peak_out = 0.0;
      *viol = s;
      return 0;
    }
  }
  double peak = 0.0;
  for (int64_t i = 0; i < l->n_slots; ++i) {
    const double v = l->used[i] + peak_in_slot(P, k, t0, T, l->slot[i], l->slot_len);
    if (peak < v) peak = v; /* std::max */
  }
  for (int64_t s = first; s <= last; ++s) {
    const double v = usage_in_slot(l, s) + peak_in_slot(P, k, t0, T, s, l->slot_len);
    if (peak < v) peak = v;
  }
  *fits = 1;
  *peak_out = peak;
  *viol = 0;
  return 0;
}

static void add_to_slot(kxo_ledger* l, int64_t s, double v) { /* usage_[s] += v */
  const int64_t i = find_slot(l, s);
  if (i < l->n_slots && l->slot[i] == s) {
    l->used[i] += v;
    return;
  }
  if (l->n_slots == l->slot_cap) {
    l->slot_cap = l->slot_cap ? 2 * l->slot_cap : 64;
    l->slot = (int64_t*)realloc(l->slot, (size_t)l->slot_cap * sizeof(int64_t));
    l->used = (double*)realloc(l->used, (size_t)l->slot_cap * sizeof(double));
  }
  memmove(l->slot + i + 1, l->slot + i, (size_t)(l->n_slots - i) * sizeof(int64_t));
  memmove(l->used + i + 1, l->used + i, (size_t)(l->n_slots - i) * sizeof(double));
  l->slot[i] = s;
  l->used[i] = 0.0 + v;
  ++l->n_slots;
}

/* SlotLedger::commit, dispatcher.cpp:70-79; returns 2 (logic_error) on Exceeds */
int kxo_commit(kxo_ledger* l, uint64_t uid, double P, double k, double t0, double T) {
  int32_t fits;
  double peak;
  int64_t viol;
  kxo_try_place(l, P, k, t0, T, &fits, &peak, &viol);
  if (!fits) return 2;
  int64_t first = 0, last = -1;
  span(t0, T, l->slot_len, &first, &last);
  for (int64_t s = first; s <= last; ++s) add_to_slot(l, s, peak_in_slot(P, k, t0, T, s, l->slot_len));
  for (int64_t i = 0; i < l->n_act; ++i) { /* active_[uid] = m */
    if (l->act[i].uid == uid) {
      model m = {uid, P, k, t0, T};
      l->act[i] = m;
      return 0;
    }
  }
  if (l->n_act == l->act_cap) {
    l->act_cap = l->act_cap ? 2 * l->act_cap : 64;
    l->act = (model*)realloc(l->act, (size_t)l->act_cap * sizeof(model));
  }
  model m = {uid, P, k, t0, T};
  l->act[l->n_act++] = m;
  return 0;
}

/* SlotLedger::correct_early_finish, dispatcher.cpp:81-99; 1 = unknown uid */
int kxo_finish(kxo_ledger* l, uint64_t uid, double actual_end) {
  int64_t j = -1;
  for (int64_t i = 0; i < l->n_act; ++i)
    if (l->act[i].uid == uid) j = i;
  if (j < 0) return 1;
  model* m = &l->act[j];
  if (actual_end >= (m->t0 + m->T) - kTimeEpsilon) return 0;
  const double from = actual_end > m->t0 ? actual_end : m->t0; /* std::max(actual_end, t_start) */
  const int64_t cutoff = (int64_t)floor((from + kTimeEpsilon) / l->slot_len);
  int64_t first = 0, last = -1;
  span(m->t0, m->T, l->slot_len, &first, &last);
  for (int64_t s = first; s <= last; ++s) {
    if (s <= cutoff) continue;
    const int64_t i = find_slot(l, s);
    if (!(i < l->n_slots && l->slot[i] == s)) continue;
    l->used[i] -= peak_in_slot(m->P, m->k, m->t0, m->T, s, l->slot_len);
    if (l->used[i] < 1e-9) l->used[i] = 0.0;
  }
  m->T = from - m->t0;
  return 0;
}

/* SlotLedger::gc, dispatcher.cpp:101-118 */
void kxo_gc(kxo_ledger* l, double now) {
  const int64_t current = (int64_t)floor((now + kTimeEpsilon) / l->slot_len);
  int64_t drop = 0;
  while (drop < l->n_slots && l->slot[drop] < current) ++drop;
  if (drop) {
    memmove(l->slot, l->slot + drop, (size_t)(l->n_slots - drop) * sizeof(int64_t));
    memmove(l->used, l->used + drop, (size_t)(l->n_slots - drop) * sizeof(double));
    l->n_slots -= drop;
  }
  int64_t w = 0;
  for (int64_t i = 0; i < l->n_act; ++i)
    if (!(l->act[i].t0 + l->act[i].T <= now + kTimeEpsilon)) l->act[w++] = l->act[i];
  l->n_act = w;
}

int64_t kxo_ledger_dump(const kxo_ledger* l, int64_t* slots, double* usage, int64_t cap) {
  for (int64_t i = 0; i < l->n_slots && i < cap; ++i) {
    slots[i] = l->slot[i];
    usage[i] = l->used[i];
  }
  return l->n_slots;
}

int64_t kxo_ledger_active(const kxo_ledger* l) { return l->n_act; }

/* ---- dispatch round (engine.cpp:220-268 + dispatcher.cpp:125-262) ---------- */

int64_t kxo_dispatch_round(kxo_pool* p, const kxo_queue* q, const kxo_tables* t,
                           const uint32_t* perm, int64_t m, double now, int32_t pool_index,
                           kxo_decision* rows, double* cand, int64_t row_cap, int32_t* status) {
  const int32_t ni = p->n_inst;
  int64_t pos = 0, nrows = 0;
  int retries = 0;
  *status = 0;
  while (pos < m) {
    const uint32_t idx = perm[pos];
    const int32_t agent = q->agent[idx];
    const double P = (double)q->prompt[idx];
    /* expected_exec_time, engine.cpp:177-185 */
    const double T = p->oracle_T ? q->pure_exec[idx] : t->T[agent];
    /* collect_live, engine.cpp:187-202 (on_live_usage, dispatcher.cpp:283-289) */
    for (int32_t i = 0; i < ni; ++i)
      if (p->suspended[i] && p->live_kv[i] < p->watermark * p->cap[i]) p->suspended[i] = 0;
    /* Dispatcher::choose TimeSlot (dispatcher.cpp:235-246) -> select_instance (125-158) */
    double best_peak = INFINITY;
    int32_t best = -1, best_id = 0;
    double* crow = cand && nrows < row_cap ? cand + nrows * ni : NULL;
    for (int32_t i = 0; i < ni; ++i) {
      const int full = p->running[i] + p->waiting[i] >= p->max_batch[i];
      if (p->suspended[i] || full) {
        if (crow) crow[i] = -1.0;
        continue;
      }
      int32_t fits;
      double peak;
      int64_t viol;
      kxo_try_place(p->ledgers[i], P, p->k[i], now, T, &fits, &peak, &viol);
      if (!fits) {
        if (crow) crow[i] = -(double)viol - 1.0;
        continue;
      }
      if (crow) crow[i] = peak;
      if (peak < best_peak || (peak == best_peak && best >= 0 && p->id[i] < best_id)) {
        best_peak = peak;
        best = i;
        best_id = p->id[i];
      }
    }
    int overload = 0;
    if (best >= 0) overload = p->live_kv[best] + P > p->cap[best]; /* engine.cpp:254-255 */
    if (nrows < row_cap) {
      kxo_decision* d = &rows[nrows];
      d->time = now;
      d->predicted_peak = best >= 0 ? best_peak : 0.0;
      d->uid = q->uid[idx];
      d->queue_index = idx;
      d->agent = agent;
      d->target = best >= 0 ? best_id : -1;
      d->pool = pool_index;
      d->admitted = (best >= 0 && !overload) ? 1 : 0;
    } else {
      *status = 5;
    }
    ++nrows;
    if (best < 0) break; /* engine.cpp:247 */
    if (overload) {      /* on_overload; continue (engine.cpp:256-257) */
      p->suspended[best] = 1;
      if (++retries > ni) {
        *status = 6; /* the reference would loop forever here */
        break;
      }
      continue;
    }
    retries = 0;
    /* pop; Dispatcher::commit (dispatcher.cpp:252-262); admit (engine.cpp:298-319) */
    kxo_commit(p->ledgers[best], q->uid[idx], P, p->k[best], now, T);
    p->live_kv[best] += (double)(q->prompt[idx] + (q->kept ? q->kept[idx] : 0));
    p->running[best] += 1;
    ++pos;
  }
  /* try_admit is a no-op under TimeSlot; Dispatcher::gc(clock_) (engine.cpp:212) */
  for (int32_t i = 0; i < ni; ++i) kxo_gc(p->ledgers[i], now);
  return nrows;
}

/* ---- dispatch round, RoundRobin / StaticThreshold (engine.cpp:220-296) ------ */

/* SchedulerPolicy::order_key of a waiting entry (scheduler.hpp:48-113). */
static void wkey_of(int policy, const kxo_tables* t, const kxo_waitrec* r, double* k) {
  switch (policy) {
    case KXO_KAIROS: k[0] = t->pk[r->agent]; k[1] = r->app_start; k[2] = r->queue_enter; break;
    case KXO_FCFS: k[0] = r->queue_enter; k[1] = r->app_start; k[2] = 0.0; break;
    case KXO_TOPO: k[0] = (double)t->depth[r->agent]; k[1] = r->queue_enter; k[2] = 0.0; break;
    default: k[0] = rem_of(t, r->uid); k[1] = r->queue_enter; k[2] = 0.0; break;
  }
}

/* std::tie(key(a), a.msg_id, a.uid) < std::tie(key(b), ...) (engine.cpp:280-283) */
static int wless(int policy, const kxo_tables* t, const kxo_waitrec* a, const kxo_waitrec* b) {
  double ka[3], kb[3];
  wkey_of(policy, t, a, ka);
  wkey_of(policy, t, b, kb);
  for (int j = 0; j < 3; ++j)
    if (ka[j] != kb[j]) return ka[j] < kb[j];
  if (a->msg != b->msg) return a->msg < b->msg;
  return a->uid < b->uid;
}

typedef struct {
  kxo_pool* p;
  int sched_policy;
  const kxo_tables* t;
  kxo_waitrec* wrec;
  int64_t wcap;
  int32_t round;
  double now;
  int32_t pool_index;
  kxo_admission* adm;
  int64_t adm_cap;
  int64_t n_adm;
} wctx;

/* Simulator::try_admit (engine.cpp:270-296), admit (298-319) bookkeeping. */
static void try_admit_o(wctx* c, int32_t i) {
  kxo_pool* p = c->p;
  kxo_waitrec* L = c->wrec + (int64_t)i * c->wcap;
  while (p->waiting[i] > 0 && p->running[i] < p->max_batch[i]) {
    int64_t best = 0;
    for (int64_t j = 1; j < p->waiting[i]; ++j)
      if (wless(c->sched_policy, c->t, &L[j], &L[best])) best = j;
    const kxo_waitrec h = L[best];
    if (p->live_kv[i] + (double)h.prompt > p->cap[i]) break; /* head waits for memory */
    memmove(L + best, L + best + 1, (size_t)(p->waiting[i] - best - 1) * sizeof(kxo_waitrec));
    p->waiting[i] -= 1;
    p->live_kv[i] += (double)(h.prompt + h.kept);
    p->running[i] += 1;
    if (c->n_adm < c->adm_cap) {
      kxo_admission* a = &c->adm[c->n_adm];
      a->time = c->now;
      a->uid = h.uid;
      a->queue_index = h.round == c->round ? h.qidx : -1;
      a->instance = p->id[i];
      a->pool = c->pool_index;
    }
    c->n_adm += 1;
  }
}

int64_t kxo_dispatch_round_waiting(kxo_pool* p, int dispatch_policy, double static_thr, int sched_policy,
                                   int64_t* rr_next, kxo_waitrec* wrec, int64_t wcap, int32_t round,
                                   const kxo_queue* q, const kxo_tables* t, const uint32_t* perm,
                                   int64_t m, double now, int32_t pool_index, kxo_decision* rows,
                                   int64_t row_cap, kxo_admission* adm, int64_t adm_cap, int64_t* n_adm,
                                   int32_t* status) {
  const int32_t ni = p->n_inst;
  wctx c = {p, sched_policy, t, wrec, wcap, round, now, pool_index, adm, adm_cap, 0};
  int64_t nrows = 0;
  *status = 0;
  for (int64_t pos = 0; pos < m; ++pos) {
    const uint32_t idx = perm[pos];
    /* collect_live (engine.cpp:187-202): on_live_usage per instance */
    for (int32_t i = 0; i < ni; ++i)
      if (p->suspended[i] && p->live_kv[i] < p->watermark * p->cap[i]) p->suspended[i] = 0;
    int32_t target = -1;
    if (dispatch_policy == 1) { /* RoundRobin, dispatcher.cpp:214-218 */
      target = (int32_t)((uint64_t)*rr_next % (uint64_t)ni);
      *rr_next += 1;
    } else { /* StaticThreshold, dispatcher.cpp:219-231 */
      for (int32_t probe = 0; probe < ni; ++probe) {
        const int32_t i = (int32_t)(((uint64_t)*rr_next + (uint64_t)probe) % (uint64_t)ni);
        const int full = p->running[i] + p->waiting[i] >= p->max_batch[i];
        if (p->live_kv[i] < static_thr * p->cap[i] && !full) {
          target = i;
          *rr_next = i + 1;
          break;
        }
      }
    }
    if (nrows < row_cap) {
      kxo_decision* d = &rows[nrows];
      d->time = now;
      d->predicted_peak = 0.0;
      d->uid = q->uid[idx];
      d->queue_index = idx;
      d->agent = q->agent[idx];
      d->target = target >= 0 ? p->id[target] : -1;
      d->pool = pool_index;
      d->admitted = target >= 0 ? 1 : 0;
    }
    ++nrows;
    if (target < 0) break; /* engine.cpp:247 */
    if (p->waiting[target] >= wcap) {
      *status = 5;
      break;
    }
    /* pop; inst.waiting.push_back; try_admit (engine.cpp:259-262) */
    kxo_waitrec r;
    r.app_start = q->app_start[idx];
    r.queue_enter = q->queue_enter[idx];
    r.msg = q->msg_key[idx];
    r.uid = q->uid[idx];
    r.prompt = q->prompt[idx];
    r.kept = q->kept ? q->kept[idx] : 0;
    r.qidx = idx;
    r.agent = q->agent[idx];
    r.round = round;
    wrec[(int64_t)target * wcap + p->waiting[target]] = r;
    p->waiting[target] += 1;
    try_admit_o(&c, target);
  }
  if (*status == 0)
    for (int32_t i = 0; i < ni; ++i) try_admit_o(&c, i); /* engine.cpp:211 */
  for (int32_t i = 0; i < ni; ++i) kxo_gc(p->ledgers[i], now); /* engine.cpp:212 */
  *n_adm = c.n_adm;
  return nrows;
}

/* ---- EmpiricalDistribution (distribution.cpp:88-123) -------------------------- */

struct kxo_dist {
  uint64_t min_samples;
  double thr;
  int64_t window_cap;
  double* sorted;
  int64_t n, cap_s;
  double* fifo; /* arrival_order_ as a growable ring */
  int64_t f_head, f_n, cap_f;
  double* snap;
  int64_t snap_n;
  uint64_t total, next_cp;
  int converged;
  double last;
};

kxo_dist* kxo_dist_new(uint64_t min_samples, double relative_threshold, int64_t window_cap) {
  kxo_dist* d = (kxo_dist*)calloc(1, sizeof(kxo_dist));
  d->min_samples = min_samples;
  d->thr = relative_threshold;
  d->window_cap = window_cap;
  d->next_cp = min_samples; /* next_checkpoint_(cfg.min_samples) */
  d->last = -1.0;
  return d;
}

void kxo_dist_free(kxo_dist* d) {
  if (!d) return;
  free(d->sorted);
  free(d->fifo);
  free(d->snap);
  free(d);
}

static int64_t lower_bound_d(const double* s, int64_t n, double v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (s[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

int kxo_dist_add(kxo_dist* d, double value) {
  if (value < 0.0) return -1; /* distribution.cpp:92-94 */
  if (d->n == d->cap_s) {
    d->cap_s = d->cap_s ? 2 * d->cap_s : 64;
    d->sorted = (double*)realloc(d->sorted, (size_t)d->cap_s * sizeof(double));
  }
  const int64_t pos = lower_bound_d(d->sorted, d->n, value); /* sorted_.insert(lower_bound) */
  memmove(d->sorted + pos + 1, d->sorted + pos, (size_t)(d->n - pos) * sizeof(double));
  d->sorted[pos] = value;
  d->n += 1;
  if (d->window_cap > 0) {
    if (d->f_n == d->cap_f) { /* grow the ring, oldest first */
      const int64_t nc = d->cap_f ? 2 * d->cap_f : 64;
      double* nf = (double*)malloc((size_t)nc * sizeof(double));
      for (int64_t j = 0; j < d->f_n; ++j) nf[j] = d->fifo[(d->f_head + j) % d->cap_f];
      free(d->fifo);
      d->fifo = nf;
      d->cap_f = nc;
      d->f_head = 0;
    }
    d->fifo[(d->f_head + d->f_n) % d->cap_f] = value; /* arrival_order_.push_back */
    d->f_n += 1;
    if (d->f_n > d->window_cap) {
      const double oldest = d->fifo[d->f_head];
      d->f_head = (d->f_head + 1) % d->cap_f;
      d->f_n -= 1;
      const int64_t e = lower_bound_d(d->sorted, d->n, oldest);
      memmove(d->sorted + e, d->sorted + e + 1, (size_t)(d->n - e - 1) * sizeof(double));
      d->n -= 1;
    }
  }
  d->total += 1;
  int became = 0;
  if (d->total == d->next_cp) { /* check_convergence, distribution.cpp:113-123 */
    if (d->snap_n > 0) {
      const double w = kxo_wasserstein_1d(d->snap, d->snap_n, d->sorted, d->n);
      d->last = w;
      double s = 0.0;
      for (int64_t j = 0; j < d->n; ++j) s += d->sorted[j]; /* mean(), distribution.cpp:125-129 */
      const double t = d->thr * (s / (double)d->n);
      const double tau = t > 1e-12 ? t : 1e-12;
      if (w < tau) {
        became = !d->converged;
        d->converged = 1;
      }
    }
    d->snap = (double*)realloc(d->snap, (size_t)(d->n > 0 ? d->n : 1) * sizeof(double));
    memcpy(d->snap, d->sorted, (size_t)d->n * sizeof(double));
    d->snap_n = d->n;
    d->next_cp *= 2;
  }
  return became;
}

int64_t kxo_dist_read(const kxo_dist* d, double* out, int64_t cap, uint64_t* total_added, int32_t* converged,
                      double* last_distance) {
  if (out)
    for (int64_t j = 0; j < d->n && j < cap; ++j) out[j] = d->sorted[j];
  if (total_added) *total_added = d->total;
  if (converged) *converged = d->converged;
  if (last_distance) *last_distance = d->last;
  return d->n;
}

/* ---- pairwise_sorting_accuracy (priority.cpp:165-189) ------------------------ */
int kxo_pairwise_accuracy(int64_t n, const int32_t* agent, const double* rem, const uint8_t* present,
                          int32_t scope_all, double* acc, uint64_t* pairs_out) {
  double correct = 0.0;
  uint64_t pairs = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (present && !present[i]) continue;
    for (int64_t j = i + 1; j < n; ++j) {
      if (!scope_all && agent[i] == agent[j]) continue;
      if (present && !present[j]) continue;
      ++pairs;
      if (rem[i] < rem[j]) correct += 1.0;
      else if (rem[i] == rem[j]) correct += 0.5;
    }
  }
  *pairs_out = pairs;
  if (pairs == 0) return 1;
  *acc = correct / (double)pairs;
  return 0;
}

/* ---- finalize_instance (workload.cpp:292-315) -------------------------------- */
int kxo_finalize(int64_t n_wf, const int64_t* off, const int32_t* parent, const int64_t* prompt,
                 const int64_t* target, double prefill_rate, double decode_rate, uint64_t uid_base,
                 uint64_t* uid_out, double* pure_out, double* rem_out) {
  uint64_t next_uid = uid_base;
  for (int64_t w = 0; w < n_wf; ++w) {
    const int64_t b = off[w], n = off[w + 1] - b;
    for (int64_t c = 0; c < n; ++c) {
      if (parent[b + c] < -1 || parent[b + c] >= c) return 1;
      uid_out[b + c] = next_uid++;
      pure_out[b + c] = (double)prompt[b + c] / prefill_rate + (double)target[b + c] / decode_rate;
    }
    /* reverse sweep; children of c are the later calls whose parent is c */
    for (int64_t c = n - 1; c >= 0; --c) {
      double tail = 0.0;
      for (int64_t ch = c + 1; ch < n; ++ch)
        if (parent[b + ch] == c && tail < rem_out[b + ch]) tail = rem_out[b + ch];
      rem_out[b + c] = pure_out[b + c] + tail;
    }
  }
  return 0;
}

/* record_remaining arithmetic, profiler.cpp:31-50 */
void kxo_record_remaining(int64_t n_wf, const int64_t* off, const double* es, const double* ee,
                          double* finish_out, double* samples_out) {
  for (int64_t w = 0; w < n_wf; ++w) {
    const int64_t b = off[w], n = off[w + 1] - b;
    if (n <= 0) continue;
    double finish = ee[b];
    for (int64_t r = 0; r < n; ++r)
      if (finish < ee[b + r]) finish = ee[b + r];
    finish_out[w] = finish;
    for (int64_t r = 0; r < n; ++r) samples_out[b + r] = finish - es[b + r];
  }
}

// K6: the replica discrete-event engine, one warp per replica.
//
// Replays Simulator::run (engine.cpp:85-486) for many independent
// replicas (load-trace cells, harness.cpp:166-216) at once. Each warp owns
// one replica: its event heap lives in shared memory ordered by
// (time, kind, seq) (engine.hpp:178-184); lane 0 performs the
// sequential state changes and all lanes cooperate on the scans the
// reference does in O(N) loops (ReadyQueue::best_index, select_instance over
// instances, try_admit's waiting scan, the preemption victim arg-max).
// Scalar replica state sits in shared memory, written by lane 0 and read by
// every lane after __syncwarp, so control flow stays warp-uniform.
//
// Supported: all four scheduling policies (scheduler.hpp:48-133) with
// TimeSlot, RoundRobin and StaticThreshold dispatch, TimeSlot's expected
// time either the oracle's pure_exec or the profiler's (engine.cpp:177-185).
// The LatencyProfiler (profiler.cpp:20-50) lives in global memory per
// (replica, agent): execution samples as a sorted prefix plus the samples
// recorded since the last workflow completion (the reference's snapshot
// point, engine.cpp:423), merged at each completion, their mode
// (mode_estimate) computed lazily when a dispatch needs it; remaining-latency
// windows with doubling checkpoints (dist_add_warp, kx_dist.cuh). The
// KairosScheduler rebuild (scheduler.cpp:5-24: converged agents in AgentId
// order, W1 matrix with the anchor, classical MDS, anchor distances, median
// for the rest) runs in the warp when a workflow completion makes an agent
// converge or every rebuild_interval completions.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "kx_common.cuh"
#include "kx_engine.cuh"
#include "kx_sortlib.cuh"
#include "kx_state.cuh"

#ifndef KX_HEAP_ARITY
#define KX_HEAP_ARITY 2  // event-heap fan-out (A/B on B200: 2 beats 4, profiles/r01_engine_ab.md)
#endif
#ifndef KX_FAST_TICKS
#define KX_FAST_TICKS 1  // lane 0 runs consecutive prefill / token events without warp syncs
#endif
#ifndef KX_TOKEN_FIFO
#define KX_TOKEN_FIFO 1  // per-instance token-event FIFOs: only each FIFO's head sits in the heap
#endif
#ifndef KX_FAST_REG
#define KX_FAST_REG 1  // the fast path keeps the scalar replica state in registers
#endif
#if KX_FAST_REG && KX_HEAP_ARITY != 2
#error "KX_FAST_REG's sift is binary: build it with KX_HEAP_ARITY=2"
#endif
#ifndef KX_FLOYD
#define KX_FLOYD 0  // bottom-up sift-down (hole to a leaf, then sift up): measured slower
#endif
#ifndef KX_REPLACE_TOP
#define KX_REPLACE_TOP 1  // reuse the popped root for the handler's first push
#endif

namespace kx {

namespace {

enum : int { EV_ARRIVAL = 0, EV_PREFILL = 1, EV_TOKEN = 2, EV_DONE = 3, EV_PREEMPT = 4, EV_ROUND = 5 };

#ifndef KX_EV_ALIGN
#define KX_EV_ALIGN 16  // 16: heap moves are two 128-bit shared loads / stores
#endif
struct __align__(KX_EV_ALIGN) Ev {
  double time;
  uint64_t ks;  // kind << 56 | seq
  uint32_t call;
  int32_t inst;
  uint32_t epoch;
  uint32_t pad;
};

__device__ __forceinline__ bool ev_less(const Ev& a, const Ev& b) {
  return a.time < b.time || (a.time == b.time && a.ks < b.ks);
}

// Scalar replica state (shared memory, lane 0 writes).
struct Scal {
  double clock;
  double prefill_seconds, decode_seconds, wasted_kv, completed_kv;
  uint64_t next_seq, processed, preemption_events, preempted_requests;
  int64_t next_arrival, arrivals_remaining, queue_n, waiting_n, calls_done, wf_done;
  double next_arrival_time;  // arrival[next_arrival], cached
  int32_t heap_n, round_pending, tick_scheduled, status;
  int32_t top_free, pad;
  int64_t rr_next;
  uint64_t completed_instances;
};

struct RunSlot {  // RunningRequest (engine.hpp:137-145)
  uint32_t call;
  uint32_t epoch;
  int64_t tokens;
  int64_t kv;
  int64_t target;  // plan->target_tokens, cached for the token ticks
  double exec_start;
  int32_t phase;  // 0 prefill, 1 decode
  int32_t used;
  int32_t inst;   // owning instance (slot / max_run, kept to avoid the division)
  int32_t pad;
};

struct InstS {  // InstanceState (engine.hpp:147-153) + Dispatcher::suspended_ + profile
  double live_kv;
  double cap, k, step;  // capacity, decode rate, 1.0 / decode rate
  int32_t running;
  int32_t waiting;
  int32_t susp;
  int32_t max_batch;
  uint64_t preempted_total;
  int32_t fh, fn;  // token FIFO: ring head, entries (the head is in the heap when fn > 0)
  double act_min_end;  // min over the active table of t0 + T (gc skips the sweep above it)
};

}  // namespace

constexpr size_t kScalBytes = (sizeof(Scal) + 15) & ~size_t(15);  // heap starts 16-byte aligned

// Token FIFO entries per instance (0 = off): running requests plus room for
// stale events of preempted ones; a full FIFO falls back to the heap.
#ifndef KX_FIFO_EXTRA
#define KX_FIFO_EXTRA 8  // FIFO room beyond max_batch (tests shrink it to force the heap fallback)
#endif
__host__ __device__ inline int fifo_cap_of(int max_run) {
  return KX_TOKEN_FIFO ? (max_run + KX_FIFO_EXTRA > 1 ? max_run + KX_FIFO_EXTRA : 1) : 0;
}
__host__ __device__ inline size_t fifo_off(const EngineParams& p) {
  const size_t end = kScalBytes + sizeof(Ev) * size_t(p.heap_cap) + sizeof(InstS) * size_t(p.n_inst) +
                     sizeof(RunSlot) * size_t(p.n_inst) * size_t(p.max_run);
  return (end + 15) & ~size_t(15);
}

size_t engine_smem_bytes(const EngineParams& p) {
  return fifo_off(p) + sizeof(Ev) * size_t(p.n_inst) * size_t(fifo_cap_of(p.max_run)) + 64;
}

__global__ void __launch_bounds__(32, 16)
k_replica_engine(EngineParams P, EngineInputs I, EngineState S) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Scal& sc = *reinterpret_cast<Scal*>(smem_raw);
  Ev* heap = reinterpret_cast<Ev*>(smem_raw + kScalBytes);
  InstS* ins = reinterpret_cast<InstS*>(heap + P.heap_cap);
  RunSlot* runs = reinterpret_cast<RunSlot*>(ins + P.n_inst);
  const int fcap = fifo_cap_of(P.max_run);
  Ev* fifo = reinterpret_cast<Ev*>(smem_raw + fifo_off(P));  // [NI][fcap]

  const int r = blockIdx.x;
  const int lane = threadIdx.x;
  const int NI = P.n_inst;
  const int64_t w0 = I.wf_base[r], w1 = I.wf_base[r + 1];
  const int64_t c0 = I.call_base[r], c1 = I.call_base[r + 1];
  const int ring = P.ring;
  const int NA = P.n_agents;
  const int64_t ab = int64_t(r) * NA;  // profiler / priority-table base of this replica
  auto sync = [] { __syncwarp(); };

  // ---- init --------------------------------------------------------------
  if (lane == 0) {
    sc = Scal{};
    sc.next_seq = static_cast<uint64_t>(w1 - w0);  // arrivals took seq 0..n-1 (engine.cpp:86-89)
    sc.next_arrival = w0;
    sc.arrivals_remaining = w1 - w0;
    sc.next_arrival_time = w1 > w0 ? I.arrival[w0] : 0.0;
  }
  for (int i = lane; i < NI; i += 32) {
    ins[i] = InstS{};
    ins[i].cap = I.cap[i];
    ins[i].k = I.k[i];
    ins[i].step = __ddiv_rn(1.0, I.k[i]);
    ins[i].max_batch = I.max_batch[i];
    ins[i].act_min_end = __longlong_as_double(0x7ff0000000000000ll);  // +inf: empty table
  }
  for (int j = lane; j < NI * P.max_run; j += 32) {
    runs[j].used = 0;
    runs[j].inst = j / P.max_run;
  }
  for (int64_t c = c0 + lane; c < c1; c += 32) {
    S.first_enqueue[c] = -1.0;
    S.queue_seconds[c] = 0.0;
    S.kept[c] = 0;
    S.episodes[c] = 0;
    S.preemptions[c] = 0;
    S.epoch[c] = 0;
    S.ever_preempted[c] = 0;
    S.run_slot[c] = -1;
  }
  const int64_t lb = int64_t(r) * NI;  // ledger / instance base of this replica
  for (int64_t j = lane; j < int64_t(NI) * ring; j += 32) {
    S.usage[lb * ring + j] = 0.0;
    S.ex[lb * ring + j] = 0;
  }
  for (int i = lane; i < NI; i += 32) {
    S.base[lb + i] = 0;
    S.hi[lb + i] = -1;
    S.n_active[lb + i] = 0;
  }
  if (P.profile_T || P.kairos) {
    for (int a = lane; a < NA; a += 32) {
      S.exec_ns[ab + a] = 0;
      S.exec_nt[ab + a] = 0;
      S.exec_dirty[ab + a] = 0;
      S.exec_T[ab + a] = P.default_T;
      S.pk[ab + a] = 0.0;  // empty table: median_anchor_distance() = 0
      S.rem_d[ab + a] = DistScal{0, 0, 0, 0, uint64_t(kModeMinSamples), 0, -1.0};
    }
  }
  if (lane == 0 && P.kairos) S.rebuilds[r] = 0;
  sync();

  // ---- helpers (uniform control flow; lane 0 writes) ------------------------
  auto fail = [&](int code) {
    if (lane == 0 && sc.status == KX_OK) sc.status = code;
    sync();
  };
  // Event heap: KX_HEAP_ARITY-ary (binary), (time, kind, seq) order (engine.hpp:178-184). The
  // keys are a strict total order (seq is unique), so the pop sequence does
  // not depend on the layout: an event popped by the loop stays at the root
  // (sc.top_free) until the handler's first push overwrites it and sifts
  // down once (replace-top), or the next iteration removes it.
  auto sift_down = [&](const Ev& e) {  // lane 0: place e from the root
    int k = 0;
    const int n = sc.heap_n;
    if (KX_FLOYD && KX_HEAP_ARITY == 2) {
      // Floyd: walk the hole down the smaller-child path to a leaf (one
      // comparison per level), then sift e up from there (e is usually a
      // late event: a token tick's successor sinks to the bottom).
      while (2 * k + 1 < n) {
        int c = 2 * k + 1;
        if (c + 1 < n) {
          const double t0 = heap[c].time, t1 = heap[c + 1].time;
          if (t1 < t0 || (t1 == t0 && heap[c + 1].ks < heap[c].ks)) ++c;
        }
        heap[k] = heap[c];
        k = c;
      }
      while (k > 0) {
        const int pk = (k - 1) >> 1;
        if (!ev_less(e, heap[pk])) break;
        heap[k] = heap[pk];
        k = pk;
      }
      heap[k] = e;
      return;
    }
    while (true) {
      const int c0 = KX_HEAP_ARITY * k + 1;
      if (c0 >= n) break;
      // the smallest of the children, comparing (time, ks) only
      int c = c0;
      double bt = heap[c0].time;
      uint64_t bk = heap[c0].ks;
      const int ce = c0 + KX_HEAP_ARITY < n ? c0 + KX_HEAP_ARITY : n;
      for (int j = c0 + 1; j < ce; ++j) {
        const double t = heap[j].time;
        const uint64_t ks = heap[j].ks;
        if (t < bt || (t == bt && ks < bk)) {
          bt = t;
          bk = ks;
          c = j;
        }
      }
      if (!(bt < e.time || (bt == e.time && bk < e.ks))) break;
      heap[k] = heap[c];
      k = c;
    }
    heap[k] = e;
  };
  auto push_l0 = [&](double t, int kind, uint32_t call, int inst, uint32_t epoch) {  // lane 0
    {
      Ev e{t, (uint64_t(kind) << 56) | sc.next_seq, call, inst, epoch, 0};
      sc.next_seq += 1;
      if (KX_REPLACE_TOP && sc.top_free) {  // replace-top
        sc.top_free = 0;
        sift_down(e);
      } else if (sc.heap_n >= P.heap_cap) {
        sc.status = KX_ERR_CAPACITY;
      } else {
        int k = sc.heap_n++;
        while (k > 0) {
          const int pk = (k - 1) / KX_HEAP_ARITY;
          if (!ev_less(e, heap[pk])) break;
          heap[k] = heap[pk];
          k = pk;
        }
        heap[k] = e;
      }
    }
  };
  auto push = [&](double t, int kind, uint32_t call, int inst, uint32_t epoch) {
    if (lane == 0) push_l0(t, kind, call, inst, epoch);
    sync();
  };
  // A token tick of instance i (lane 0). Its time is >= every pending token
  // event of i (all were scheduled at earlier clocks with the same step,
  // rounding is monotone) and its seq is larger, so i's token events form a
  // FIFO; only the FIFO's head needs to be in the heap for the heap minimum
  // to be the global minimum. seq is taken here, at scheduling time.
  auto push_token_l0 = [&](int i, double t, uint32_t call, int rs, uint32_t epoch) {
    if (fcap == 0 || ins[i].fn >= fcap) {  // no FIFO room: an ordinary heap event
      push_l0(t, EV_TOKEN, call, rs, epoch);
      return;
    }
    Ev e{t, (uint64_t(EV_TOKEN) << 56) | sc.next_seq, call, rs, epoch, 1u};
    sc.next_seq += 1;
    const int n = ins[i].fn;
    int slot = ins[i].fh + n;
    if (slot >= fcap) slot -= fcap;
    fifo[i * fcap + slot] = e;
    ins[i].fn = n + 1;
    if (n == 0) {  // new head: into the heap (seq already assigned)
      if (KX_REPLACE_TOP && sc.top_free) {
        sc.top_free = 0;
        sift_down(e);
      } else if (sc.heap_n >= P.heap_cap) {
        sc.status = KX_ERR_CAPACITY;
      } else {
        int k = sc.heap_n++;
        while (k > 0) {
          const int pk = (k - 1) / KX_HEAP_ARITY;
          if (!ev_less(e, heap[pk])) break;
          heap[k] = heap[pk];
          k = pk;
        }
        heap[k] = e;
      }
    }
  };
  // The root was just taken as the current event (sc.top_free = 1): a FIFO
  // head hands its heap place to the next entry of its FIFO.
  auto take_root_l0 = [&](const Ev& ev) {
    if (ev.pad != 1u) return;
    const int i = runs[ev.inst].inst;
    int h = ins[i].fh + 1;
    if (h >= fcap) h -= fcap;
    ins[i].fh = h;
    ins[i].fn -= 1;
    if (ins[i].fn > 0) {
      sc.top_free = 0;
      sift_down(fifo[i * fcap + h]);
    }
  };
  auto pop_l0 = [&]() {  // lane 0: remove the root (deferred pop)
    sc.top_free = 0;
    const Ev last = heap[--sc.heap_n];
    if (sc.heap_n > 0) sift_down(last);
  };
  auto pop_heap = [&]() {
    if (lane == 0) pop_l0();
    sync();
  };
  auto schedule_round = [&](double t) {  // engine.cpp:79-83
    if (sc.round_pending) return;
    if (lane == 0) sc.round_pending = 1;
    sync();
    push(t, EV_ROUND, 0, -1, 0);
  };
  auto wf_of = [&](uint32_t c) { return I.call_wf[c]; };
  auto enqueue_call = [&](uint32_t c, double now) {  // engine.cpp:162-175
    if (lane == 0) {
      S.queue[c0 + sc.queue_n] = c;
      sc.queue_n += 1;
      S.enqueue_time[c] = now;
      if (S.first_enqueue[c] < 0.0) S.first_enqueue[c] = now;
    }
    sync();
  };
  // order_key (scheduler.hpp:48-93) -> tuple head (k0, k1, k2)
  auto key0 = [&](uint32_t c) -> double {
    switch (P.sched) {
      case KX_SCHED_FCFS: return S.enqueue_time[c];
      case KX_SCHED_TOPO: return static_cast<double>(I.depth[I.agent[c]]);
      case KX_SCHED_KAIROS: return S.pk[ab + I.agent[c]];  // table_.priority_key(agent)
      default: return I.rem[c];  // Oracle: remaining_by_uid holds every call
    }
  };
  auto key1 = [&](uint32_t c) -> double {  // FCFS, Kairos: app_start; Topo, Oracle: queue_enter
    return (P.sched == KX_SCHED_FCFS || P.sched == KX_SCHED_KAIROS) ? I.arrival[wf_of(c)] : S.enqueue_time[c];
  };
  const bool k2_qe = P.sched == KX_SCHED_KAIROS;  // Kairos' third key component is queue_enter
  // ReadyQueue comparator (priority.hpp:95-98): (k0, k1, k2, app, qe, msg, uid);
  // k2 is 0, or queue_enter under Kairos where k1 = app makes it the qe test
  struct Tup {
    double k0, k1, app, qe;
    uint64_t msg, uid;
  };
  auto tup = [&](uint32_t c) {
    Tup t;
    t.k0 = key0(c);
    t.k1 = key1(c);
    t.app = I.arrival[wf_of(c)];
    t.qe = S.enqueue_time[c];
    t.msg = I.wf_msg[wf_of(c)];
    t.uid = I.uid[c];
    return t;
  };
  auto tless = [](const Tup& a, const Tup& b) {
    if (a.k0 != b.k0) return a.k0 < b.k0;
    if (a.k1 != b.k1) return a.k1 < b.k1;
    if (a.app != b.app) return a.app < b.app;
    if (a.qe != b.qe) return a.qe < b.qe;
    if (a.msg != b.msg) return a.msg < b.msg;
    return a.uid < b.uid;
  };
  // try_admit comparator (engine.cpp:280-283): (k0, k1, k2, msg, uid) (H10)
  auto wless = [k2_qe](const Tup& a, const Tup& b) {
    if (a.k0 != b.k0) return a.k0 < b.k0;
    if (a.k1 != b.k1) return a.k1 < b.k1;
    if (k2_qe && a.qe != b.qe) return a.qe < b.qe;
    if (a.msg != b.msg) return a.msg < b.msg;
    return a.uid < b.uid;
  };
  auto shfl_tup = [](Tup t, int src) {
    Tup o;
    o.k0 = __shfl_sync(0xffffffffu, t.k0, src);
    o.k1 = __shfl_sync(0xffffffffu, t.k1, src);
    o.app = __shfl_sync(0xffffffffu, t.app, src);
    o.qe = __shfl_sync(0xffffffffu, t.qe, src);
    o.msg = __shfl_sync(0xffffffffu, t.msg, src);
    o.uid = __shfl_sync(0xffffffffu, t.uid, src);
    return o;
  };
  // Warp arg-min over array entries [0, n) of `arr` (queue or waiting list)
  // filtered by pred, under comparator `lt`. Returns the position or -1.
  auto warp_argmin = [&](const uint32_t* arr, int64_t n, auto pred, auto lt) -> int64_t {
    int64_t bpos = -1;
    Tup bt{};
    for (int64_t j = lane; j < n; j += 32) {
      if (!pred(j)) continue;
      const Tup t = tup(arr[j]);
      if (bpos < 0 || lt(t, bt)) {
        bt = t;
        bpos = j;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const int src = lane ^ o;
      const Tup ot = shfl_tup(bt, src);
      const int64_t op = __shfl_sync(0xffffffffu, bpos, src);
      if (op >= 0 && (bpos < 0 || lt(ot, bt))) {
        bt = ot;
        bpos = op;
      }
    }
    return bpos;
  };

  // Slot ledger of instance i (dispatcher.cpp:44-123), global memory, owned by this warp.
  auto ring_usage = [&](int i) { return S.usage + (lb + i) * ring; };
  auto ring_ex = [&](int i) { return S.ex + (lb + i) * ring; };
  // try_place, lanes over slots.
  // (first, last) = span_bounds(t0, T): the same for every instance of a
  // head, so the caller computes it once.
  auto try_place = [&](int i, double Pt, double k, double t0, double T, int64_t first, int64_t last,
                       int64_t* viol_out) -> double {
    const double t_end = __dadd_rn(t0, T);
    const int64_t base = S.base[lb + i], hi = S.hi[lb + i];
    if (last >= first && (first < base || last >= base + ring)) fail(KX_ERR_CAPACITY);
    const double* u = ring_usage(i);
    const uint8_t* ex = ring_ex(i);
    const int64_t smax = hi > last ? hi : last;
    double peak = 0.0;
    int64_t viol = INT64_MAX;
    const double cap = ins[i].cap;
    for (int64_t s = base + lane; s <= smax; s += 32) {
      const uint32_t pos = static_cast<uint32_t>(s) & (ring - 1);
      const bool in_span = s >= first && s <= last;
      const bool exists = ex[pos] != 0;
      if (!(in_span || exists)) continue;
      const double total = __dadd_rn(exists ? u[pos] : 0.0, peak_in_slot_dev(Pt, k, t0, t_end, s, P.slot_len));
      if (in_span && total > cap && s < viol) viol = s;
      peak = fmax(peak, total);
    }
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t v2 = __shfl_xor_sync(0xffffffffu, viol, o);
      viol = v2 < viol ? v2 : viol;
      peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, o));
    }
    *viol_out = viol;
    return peak;
  };
  auto commit = [&](int i, uint64_t uidv, double Pt, double k, double t0, double T) {
    int64_t first, last;
    span_bounds_dev(t0, T, P.slot_len, &first, &last);
    const double t_end = __dadd_rn(t0, T);
    double* u = ring_usage(i);
    uint8_t* ex = ring_ex(i);
    for (int64_t s = first + lane; s <= last; s += 32) {
      const uint32_t pos = static_cast<uint32_t>(s) & (ring - 1);
      u[pos] = __dadd_rn(u[pos], peak_in_slot_dev(Pt, k, t0, t_end, s, P.slot_len));
      ex[pos] = 1;
    }
    sync();
    if (lane == 0) {
      if (last >= first && last > S.hi[lb + i]) S.hi[lb + i] = last;
      const int a = S.n_active[lb + i];
      if (a >= kActiveCap) {
        sc.status = KX_ERR_CAPACITY;
      } else {
        const int64_t o = (lb + i) * kActiveCap + a;
        S.act_uid[o] = uidv;
        S.act_P[o] = Pt;
        S.act_k[o] = k;
        S.act_t0[o] = t0;
        S.act_T[o] = T;
        S.n_active[lb + i] = a + 1;
        const double e = __dadd_rn(t0, T);
        if (e < ins[i].act_min_end) ins[i].act_min_end = e;
      }
    }
    sync();
  };
  auto finish_ledger = [&](int i, uint64_t uidv, double actual_end) {  // dispatcher.cpp:81-99,264-271
    if (P.dpolicy != KX_DISPATCH_TIME_SLOT) return;
    // active_.find(uid): lanes over the table (uids are unique)
    const int a = S.n_active[lb + i];
    const int64_t o = (lb + i) * kActiveCap;
    int j = a;
    for (int j0 = 0; j0 < a && j == a; j0 += 32) {
      const uint32_t hit = __ballot_sync(0xffffffffu, j0 + lane < a && S.act_uid[o + j0 + lane] == uidv);
      if (hit) j = j0 + __ffs(hit) - 1;
    }
    if (lane == 0) {
      if (j < a) {
        const double Pt = S.act_P[o + j], k = S.act_k[o + j], t0 = S.act_t0[o + j], T = S.act_T[o + j];
        const double t_end = __dadd_rn(t0, T);
        if (!(actual_end >= __dsub_rn(t_end, kTimeEpsilon))) {
          const double from = actual_end > t0 ? actual_end : t0;
          const int64_t cutoff = static_cast<int64_t>(floor(__ddiv_rn(__dadd_rn(from, kTimeEpsilon), P.slot_len)));
          int64_t first, last;
          span_bounds_dev(t0, T, P.slot_len, &first, &last);
          double* u = ring_usage(i);
          const uint8_t* ex = ring_ex(i);
          const int64_t base = S.base[lb + i];
          for (int64_t s = first; s <= last; ++s) {
            if (s <= cutoff) continue;
            const uint32_t pos = static_cast<uint32_t>(s) & (ring - 1);
            if (s < base || s >= base + ring || !ex[pos]) continue;
            double v = __dsub_rn(u[pos], peak_in_slot_dev(Pt, k, t0, t_end, s, P.slot_len));
            if (v < 1e-9) v = 0.0;
            u[pos] = v;
          }
          S.act_T[o + j] = __dsub_rn(from, t0);
          const double e = __dadd_rn(t0, S.act_T[o + j]);
          if (e < ins[i].act_min_end) ins[i].act_min_end = e;
        }
      }
    }
    sync();
  };
  auto gc = [&](double now) {  // Dispatcher::gc (dispatcher.cpp:101-118, 295-297)
    const int64_t current = static_cast<int64_t>(floor(__ddiv_rn(__dadd_rn(now, kTimeEpsilon), P.slot_len)));
    for (int i = 0; i < NI; ++i) {
      const int64_t base = S.base[lb + i];
      if (current > base) {
        const int64_t stop = current < base + ring ? current : base + ring;
        double* u = ring_usage(i);
        uint8_t* ex = ring_ex(i);
        for (int64_t s = base + lane; s < stop; s += 32) {
          const uint32_t pos = static_cast<uint32_t>(s) & (ring - 1);
          u[pos] = 0.0;
          ex[pos] = 0;
        }
      }
      sync();
      if (lane == 0 && current > base) S.base[lb + i] = current;
      // drop elapsed models (dispatcher.cpp:110-117): lanes over the active
      // table, survivors compacted in place (the table is a set keyed by uid)
      const double lim = __dadd_rn(now, kTimeEpsilon);
      if (!(ins[i].act_min_end <= lim)) continue;  // nothing has elapsed (all lanes read the same)
      const int a = S.n_active[lb + i];
      const int64_t o = (lb + i) * kActiveCap;
      int w = 0;
      double kept_min = __longlong_as_double(0x7ff0000000000000ll);
      for (int j0 = 0; j0 < a; j0 += 32) {
        const int j = j0 + lane;
        bool keep = false;
        double at0 = 0.0, aT = 0.0;
        if (j < a) {
          at0 = S.act_t0[o + j];
          aT = S.act_T[o + j];
          keep = !(__dadd_rn(at0, aT) <= lim);
        }
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        if (keep) kept_min = fmin(kept_min, __dadd_rn(at0, aT));
        const int d = w + __popc(m & ((1u << lane) - 1u));
        const bool move = keep && d != j;  // survivors ahead of every drop stay put
        if (__any_sync(0xffffffffu, move)) {
          uint64_t au = 0;
          double aP = 0.0, ak = 0.0;
          if (move) {
            au = S.act_uid[o + j];
            aP = S.act_P[o + j];
            ak = S.act_k[o + j];
          }
          __syncwarp();  // the chunk's loads are ordered before its in-place stores
          if (move) {
            S.act_uid[o + d] = au;
            S.act_P[o + d] = aP;
            S.act_k[o + d] = ak;
            S.act_t0[o + d] = at0;
            S.act_T[o + d] = aT;
          }
        }
        w += __popc(m);
        sync();
      }
      for (int off = 16; off > 0; off >>= 1) kept_min = fmin(kept_min, __shfl_xor_sync(0xffffffffu, kept_min, off));
      if (lane == 0) {
        S.n_active[lb + i] = w;
        ins[i].act_min_end = kept_min;
      }
      sync();
    }
  };
  auto on_live_usage = [&](int i) {  // dispatcher.cpp:283-289
    if (lane == 0 && ins[i].susp && ins[i].live_kv < __dmul_rn(P.watermark, ins[i].cap)) ins[i].susp = 0;
    sync();
  };
  auto on_overload = [&](int i) {  // dispatcher.cpp:278-281
    if (P.dpolicy != KX_DISPATCH_TIME_SLOT) return;
    if (lane == 0) ins[i].susp = 1;
    sync();
  };
  auto admit = [&](int i, uint32_t c) {  // engine.cpp:298-319
    if (lane == 0) {
      S.queue_seconds[c] = __dadd_rn(S.queue_seconds[c], __dsub_rn(sc.clock, S.enqueue_time[c]));
      S.episodes[c] += 1;
      int slot = -1;
      for (int j = 0; j < P.max_run; ++j)
        if (!runs[i * P.max_run + j].used) {
          slot = j;
          break;
        }
      if (slot < 0) {
        sc.status = KX_ERR_CAPACITY;
      } else {
        RunSlot& rs = runs[i * P.max_run + slot];
        rs.used = 1;
        rs.call = c;
        rs.target = I.target[c];
        rs.tokens = S.kept[c];
        rs.kv = I.prompt[c] + S.kept[c];
        rs.phase = 0;
        rs.exec_start = sc.clock;
        S.epoch[c] += 1;
        rs.epoch = S.epoch[c];
        S.run_slot[c] = i * P.max_run + slot;
        ins[i].live_kv = __dadd_rn(ins[i].live_kv, static_cast<double>(rs.kv));
        ins[i].running += 1;
      }
    }
    sync();
    if (sc.status != KX_OK) return;
    const double dur = __ddiv_rn(static_cast<double>(I.prompt[c]), I.prefill[i]);
    if (lane == 0) sc.prefill_seconds = __dadd_rn(sc.prefill_seconds, dur);
    sync();
    // events of a running request carry its run slot (find_running is a
    // shared-memory check: slot in use, same call, same epoch)
    push(__dadd_rn(sc.clock, dur), EV_PREFILL, c, S.run_slot[c], S.epoch[c]);
  };
  auto try_admit = [&](int i) {  // engine.cpp:270-296
    while (true) {
      if (ins[i].waiting <= 0 || ins[i].running >= ins[i].max_batch) return;
      const int64_t n = sc.waiting_n;
      const int64_t pos = warp_argmin(S.waiting + c0, n, [&](int64_t j) { return S.waiting_inst[c0 + j] == i; }, wless);
      if (pos < 0) return;
      const uint32_t c = S.waiting[c0 + pos];
      if (__dadd_rn(ins[i].live_kv, static_cast<double>(I.prompt[c])) > ins[i].cap) return;
      if (lane == 0) {  // erase (order-free: the comparator is a total order)
        const int64_t last = sc.waiting_n - 1;
        S.waiting[c0 + pos] = S.waiting[c0 + last];
        S.waiting_inst[c0 + pos] = S.waiting_inst[c0 + last];
        sc.waiting_n = last;
        ins[i].waiting -= 1;
      }
      sync();
      admit(i, c);
      if (sc.status != KX_OK) return;
    }
  };
  // ---- LatencyProfiler + KairosScheduler (profiler.cpp, scheduler.cpp) ----
  // ProfilerSnapshot::expected_exec_time (profiler.cpp:11-16) of the last
  // snapshot: mode_estimate of the agent's execution samples, cached until
  // the next snapshot changes them.
  auto expected_T = [&](int a) -> double {
    const int64_t idx = ab + a;
    const int64_t ns = S.exec_ns[idx];
    if (ns == 0) return P.default_T;  // no samples in the snapshot: fallback
    if (!S.exec_dirty[idx]) return S.exec_T[idx];
    const double T = mode_estimate_warp(S.exec_buf + I.exec_off[idx], ns, kModeMinSamples);
    sync();
    if (lane == 0) {
      S.exec_T[idx] = T;
      S.exec_dirty[idx] = 0;
    }
    sync();
    return T;
  };
  // profiler_.snapshot() (profiler.cpp:86-102): the execution samples
  // recorded since the last snapshot join the sorted prefix.
  auto exec_snapshot = [&]() {
    for (int a = 0; a < NA; ++a) {
      const int64_t idx = ab + a;
      int64_t ns = S.exec_ns[idx];
      const int64_t nt = S.exec_nt[idx];
      if (ns == nt) continue;
      double* buf = S.exec_buf + I.exec_off[idx];
      for (; ns < nt; ++ns) {
        const double v = buf[ns];
        const int64_t pos = warp_lower_bound(buf, ns, v);
        warp_shift_up(buf, pos, ns);
        if (lane == 0) buf[pos] = v;
        sync();
      }
      if (lane == 0) {
        S.exec_ns[idx] = ns;
        S.exec_dirty[idx] = 1;
      }
      sync();
    }
  };
  // LatencyProfiler::record_remaining (profiler.cpp:31-50) of workflow w:
  // its records in completion order, sample = finish - exec_start.
  auto record_remaining = [&](int64_t w) -> bool {
    const int64_t cb = I.wf_call[w], ce = I.wf_call[w + 1];
    const double finish = S.wf_finish[w];  // max(arrival, exec_end...) = max exec_end
    const DistCfg cfg{uint64_t(kModeMinSamples), 0.05, kRemWindow};
    bool newly = false;
    int64_t prev = -1;
    for (int64_t k = cb; k < ce; ++k) {
      int64_t best = INT64_MAX;  // next record: smallest completion slot after prev
      for (int64_t c = cb + lane; c < ce; c += 32) {
        const int64_t j = S.done_idx[c];
        if (j > prev && j < best) best = j;
      }
      for (int o = 16; o > 0; o >>= 1) {
        const int64_t b2 = __shfl_xor_sync(0xffffffffu, best, o);
        best = b2 < best ? b2 : best;
      }
      prev = best;
      const uint32_t call = S.out_call[best];
      const int64_t idx = ab + I.agent[call];
      const int64_t off = I.rem_off[idx], cap = I.rem_off[idx + 1] - off;
      DistScal d = S.rem_d[idx];
      const double v = __dsub_rn(finish, S.out_exec_start[best]);
      if (!dist_add_warp(S.rem_sorted + off, S.rem_ring + off, S.rem_snap + off, cap, cfg, d, v, &newly)) {
        fail(KX_ERR_CAPACITY);
        return false;
      }
      sync();
      if (lane == 0) S.rem_d[idx] = d;
      sync();
    }
    return newly;
  };
  // KairosScheduler::rebuild (scheduler.cpp:14-24) -> build_matrix
  // (priority.cpp:15-46) -> mds_embed_1d (priority.cpp:102-112).
  auto rebuild = [&]() {
    double* scr = S.mds + int64_t(r) * P.mds_stride;
    int m = 0;  // converged agents with samples, in AgentId order (std::map)
    int list[kKairosMaxAgents];
    for (int k = 0; k < NA; ++k) {
      const int a = I.agent_order[k];
      const DistScal d = S.rem_d[ab + a];
      if (d.conv && d.n > 0) list[m++] = a;
    }
    if (m == 0) return;  // nothing to rank yet
    const int n = m + 1;  // + the anchor (a single sample 0.0), last label
    double* dm = scr;
    double* coords = scr + n * n;
    double* work = coords + n;
    double* anchor = work + 3 * n * n;
    if (lane == 0) *anchor = 0.0;
    sync();
    const int pairs = n * (n - 1) / 2;
    for (int p = lane; p < pairs; p += 32) {
      int i = 0, rem = p;
      while (rem >= n - 1 - i) {
        rem -= n - 1 - i;
        ++i;
      }
      const int j = i + 1 + rem;
      auto samples = [&](int x, int64_t* cnt) -> const double* {
        if (x == n - 1) {
          *cnt = 1;
          return anchor;
        }
        const int64_t idx = ab + list[x];
        *cnt = S.rem_d[idx].n;
        return S.rem_sorted + I.rem_off[idx];
      };
      int64_t na, nb;
      const double* sa = samples(i, &na);
      const double* sb = samples(j, &nb);
      const double w = w1_walk(sa, uint64_t(na), sb, uint64_t(nb));
      dm[i * n + j] = w;
      dm[j * n + i] = w;
    }
    for (int i = lane; i < n; i += 32) dm[i * n + i] = 0.0;
    sync();
    if (lane == 0) {
      mds_1d_thread(dm, n, work, coords);
      const double anchor_coord = coords[n - 1];
      // anchor distances of the table's agents; the median for the rest
      double* dist = work;  // reuse
      for (int i = 0; i < m; ++i) dist[i] = fabs(__dsub_rn(coords[i], anchor_coord));
      double* srt = work + m;
      for (int i = 0; i < m; ++i) {  // insertion sort (std::sort of values)
        const double v = dist[i];
        int j = i;
        while (j > 0 && srt[j - 1] > v) {
          srt[j] = srt[j - 1];
          --j;
        }
        srt[j] = v;
      }
      const double median = quantile_sorted_d(srt, m, 0.5);
      for (int a = 0; a < NA; ++a) S.pk[ab + a] = median;
      for (int i = 0; i < m; ++i) S.pk[ab + list[i]] = dist[i];
      S.rebuilds[r] += 1;
    }
    sync();
  };
  // Simulator::on_workflow_complete (engine.cpp:411-427), profiler part.
  auto on_workflow_complete = [&](int64_t w) {
    bool newly = false;
    if (P.kairos) newly = record_remaining(w);
    if (sc.status != KX_OK) return;
    if (P.profile_T) exec_snapshot();
    if (lane == 0) sc.completed_instances += 1;
    sync();
    if (P.kairos && (newly || sc.completed_instances % P.rebuild_interval == 0)) rebuild();
  };
  auto dispatch_loop = [&]() {  // engine.cpp:220-268
    int retries = 0;
    while (sc.queue_n > 0 && sc.status == KX_OK) {
      const int64_t qpos = warp_argmin(S.queue + c0, sc.queue_n, [](int64_t) { return true; }, tless);
      const uint32_t head = S.queue[c0 + qpos];
      const double T = P.oracle_T ? I.pure[head]
                       : (P.profile_T && sc.completed_instances > 0) ? expected_T(I.agent[head])
                                                                     : P.default_T;
      // collect_live: watermark resume, then the live view.
      for (int i = 0; i < NI; ++i) on_live_usage(i);
      int target = -1;
      if (P.dpolicy == KX_DISPATCH_ROUND_ROBIN) {
        target = static_cast<int>(sc.rr_next % NI);
        if (lane == 0) sc.rr_next += 1;
        sync();
      } else if (P.dpolicy == KX_DISPATCH_STATIC_THRESHOLD) {
        for (int probe = 0; probe < NI; ++probe) {
          const int i = static_cast<int>((sc.rr_next + probe) % NI);
          const bool full = ins[i].running + ins[i].waiting >= ins[i].max_batch;
          if (ins[i].live_kv < __dmul_rn(P.static_thr, ins[i].cap) && !full) {
            target = i;
            break;
          }
        }
        if (target >= 0) {
          if (lane == 0) sc.rr_next = target + 1;
          sync();
        }
      } else {
        double best = 0.0;
        int64_t sfirst, slast;
        span_bounds_dev(sc.clock, T, P.slot_len, &sfirst, &slast);
        for (int i = 0; i < NI; ++i) {
          const bool full = ins[i].running + ins[i].waiting >= ins[i].max_batch;
          if (ins[i].susp || full) continue;
          int64_t viol;
          const double pk = try_place(i, static_cast<double>(I.prompt[head]), ins[i].k, sc.clock, T, sfirst,
                                      slast, &viol);
          if (sc.status != KX_OK) return;
          if (viol != INT64_MAX) continue;
          if (target < 0 || pk < best || (pk == best && I.inst_id[i] < I.inst_id[target])) {
            best = pk;
            target = i;
          }
        }
      }
      if (target < 0) break;  // engine.cpp:247
      if (P.dpolicy == KX_DISPATCH_TIME_SLOT) {
        if (__dadd_rn(ins[target].live_kv, static_cast<double>(I.prompt[head])) > ins[target].cap) {
          on_overload(target);  // engine.cpp:254-258
          if (++retries > NI) {  // the reference would spin forever here
            fail(KX_ERR_LIVELOCK);
            return;
          }
          continue;
        }
        if (lane == 0) {  // ReadyQueue::pop
          const int64_t last = sc.queue_n - 1;
          S.queue[c0 + qpos] = S.queue[c0 + last];
          sc.queue_n = last;
        }
        sync();
        retries = 0;
        commit(target, I.uid[head], static_cast<double>(I.prompt[head]), ins[target].k, sc.clock, T);
        if (sc.status != KX_OK) return;
        admit(target, head);
      } else {
        if (lane == 0) {
          const int64_t last = sc.queue_n - 1;
          S.queue[c0 + qpos] = S.queue[c0 + last];
          sc.queue_n = last;
          S.waiting[c0 + sc.waiting_n] = head;
          S.waiting_inst[c0 + sc.waiting_n] = target;
          sc.waiting_n += 1;
          ins[target].waiting += 1;
        }
        sync();
        try_admit(target);
      }
    }
  };
  auto work_pending = [&]() -> bool {  // engine.cpp:488-494
    if (sc.arrivals_remaining > 0 || sc.queue_n > 0) return true;
    for (int i = 0; i < NI; ++i)
      if (ins[i].running > 0 || ins[i].waiting > 0) return true;
    return false;
  };
  auto find_running = [&](const Ev& e) -> int {  // engine.cpp:321-332
    const RunSlot& x = runs[e.inst];
    if (!x.used || x.call != e.call || x.epoch != e.epoch) return -1;
    return e.inst;
  };
  auto evict = [&](int i, int rs) {  // engine.cpp:464-486
    const uint32_t c = runs[rs].call;
    if (lane == 0) {
      runs[rs].used = 0;
      S.run_slot[c] = -1;
      ins[i].running -= 1;
      ins[i].live_kv = __dsub_rn(ins[i].live_kv, static_cast<double>(runs[rs].kv));
      ins[i].preempted_total += 1;
      sc.preemption_events += 1;
      if (!S.ever_preempted[c]) {
        S.ever_preempted[c] = 1;
        sc.preempted_requests += 1;
      }
      sc.wasted_kv = __dadd_rn(sc.wasted_kv, static_cast<double>(runs[rs].kv));
      S.preemptions[c] += 1;
      S.epoch[c] += 1;
      S.kept[c] = static_cast<int64_t>(floor(__dmul_rn(__dsub_rn(1.0, P.recompute), static_cast<double>(runs[rs].tokens))));
    }
    sync();
    finish_ledger(i, I.uid[c], sc.clock);  // on_request_preempted
    enqueue_call(c, sc.clock);
  };

  // PrefillDone / TokenTick events (engine.cpp:334-361, ~97% of all events)
  // touch only shared-memory state, so lane 0 runs them back to back without
  // warp synchronisation until the next event is of another kind or an
  // arrival comes first (arrivals win ties: kind 0).
  auto fast_ticks = [&]() {  // lane 0
    while (sc.status == KX_OK) {
      if (sc.top_free) pop_l0();
      if (sc.heap_n == 0) return;
      const int kind = static_cast<int>(heap[0].ks >> 56);
      if (kind != EV_TOKEN && kind != EV_PREFILL) return;
      if (sc.next_arrival < w1 && !(heap[0].time < sc.next_arrival_time)) return;
      const Ev ev = heap[0];
      sc.top_free = 1;
      take_root_l0(ev);
      if (ev.time < __dsub_rn(sc.clock, kTimeEpsilon)) {
        sc.status = KX_ERR_LOGIC;  // event time ran backwards
        return;
      }
      sc.clock = sc.clock > ev.time ? sc.clock : ev.time;
      sc.processed += 1;
      if (sc.processed > P.max_events) {
        sc.status = KX_ERR_RUNTIME;
        return;
      }
      const int rs = find_running(ev);
      if (rs < 0) continue;
      const double clock = sc.clock;
      const int i = runs[rs].inst;
      const double step = ins[i].step;
      if (kind == EV_PREFILL) {
        runs[rs].phase = 1;
        push_token_l0(i, __dadd_rn(clock, step), ev.call, rs, ev.epoch);
      } else {
        runs[rs].tokens += 1;
        runs[rs].kv += 1;
        ins[i].live_kv = __dadd_rn(ins[i].live_kv, 1.0);
        sc.decode_seconds = __dadd_rn(sc.decode_seconds, step);
        if (runs[rs].tokens >= runs[rs].target) push_l0(clock, EV_DONE, ev.call, rs, ev.epoch);
        else push_token_l0(i, __dadd_rn(clock, step), ev.call, rs, ev.epoch);
        if (ins[i].live_kv > ins[i].cap) push_l0(clock, EV_PREEMPT, 0, i, 0);
      }
    }
  };

  // The same fast path with the scalar state held in registers for the whole
  // run of ticks (the shared-memory copies alias the heap and run slots, so
  // the compiler would reload them after every store otherwise).
  auto fast_ticks_reg = [&]() {  // lane 0
    int heap_n = sc.heap_n, top_free = sc.top_free, status = sc.status;
    uint64_t next_seq = sc.next_seq, processed = sc.processed;
    double clk = sc.clock, dsec = sc.decode_seconds;
    const bool have_arr = sc.next_arrival < w1;
    const double t_arr = sc.next_arrival_time;
    auto sift = [&](const Ev& e) {  // binary sift-down of e from the root
      int k = 0;
      while (true) {
        int ch = 2 * k + 1;
        if (ch >= heap_n) break;
        double bt = heap[ch].time;
        uint64_t bk = heap[ch].ks;
        if (ch + 1 < heap_n) {
          const double t1 = heap[ch + 1].time;
          const uint64_t k1 = heap[ch + 1].ks;
          if (t1 < bt || (t1 == bt && k1 < bk)) {
            bt = t1;
            bk = k1;
            ++ch;
          }
        }
        if (!(bt < e.time || (bt == e.time && bk < e.ks))) break;
        heap[k] = heap[ch];
        k = ch;
      }
      heap[k] = e;
    };
    auto hpush = [&](const Ev& e) {
      if (KX_REPLACE_TOP && top_free) {
        top_free = 0;
        sift(e);
      } else if (heap_n >= P.heap_cap) {
        status = KX_ERR_CAPACITY;
      } else {
        int k = heap_n++;
        while (k > 0) {
          const int pk = (k - 1) >> 1;
          if (!ev_less(e, heap[pk])) break;
          heap[k] = heap[pk];
          k = pk;
        }
        heap[k] = e;
      }
    };
    auto push_ev = [&](double t, int kind, uint32_t call, int inst, uint32_t epoch, uint32_t fifo_flag) {
      const Ev e{t, (uint64_t(kind) << 56) | next_seq, call, inst, epoch, fifo_flag};
      next_seq += 1;
      return e;
    };
    auto push_tok = [&](int i, double t, uint32_t call, int rs, uint32_t epoch) {
      if (fcap == 0 || ins[i].fn >= fcap) {
        hpush(push_ev(t, EV_TOKEN, call, rs, epoch, 0u));
        return;
      }
      const Ev e = push_ev(t, EV_TOKEN, call, rs, epoch, 1u);
      const int n = ins[i].fn;
      int slot = ins[i].fh + n;
      if (slot >= fcap) slot -= fcap;
      fifo[i * fcap + slot] = e;
      ins[i].fn = n + 1;
      if (n == 0) hpush(e);
    };
    while (status == KX_OK) {
      if (top_free) {
        top_free = 0;
        const Ev last = heap[--heap_n];
        if (heap_n > 0) sift(last);
      }
      if (heap_n == 0) break;
      const double t0 = heap[0].time;
      const int kind = static_cast<int>(heap[0].ks >> 56);
      if (kind != EV_TOKEN && kind != EV_PREFILL) break;
      if (have_arr && !(t0 < t_arr)) break;
      const Ev ev = heap[0];
      top_free = 1;
      if (ev.pad == 1u) {  // a FIFO head: the next entry takes the root
        const int i = runs[ev.inst].inst;
        int h = ins[i].fh + 1;
        if (h >= fcap) h -= fcap;
        ins[i].fh = h;
        ins[i].fn -= 1;
        if (ins[i].fn > 0) {
          top_free = 0;
          sift(fifo[i * fcap + h]);
        }
      }
      if (ev.time < __dsub_rn(clk, kTimeEpsilon)) {
        status = KX_ERR_LOGIC;  // event time ran backwards
        break;
      }
      clk = clk > ev.time ? clk : ev.time;
      processed += 1;
      if (processed > P.max_events) {
        status = KX_ERR_RUNTIME;
        break;
      }
      const int rs = find_running(ev);
      if (rs < 0) continue;
      const int i = runs[rs].inst;
      const double step = ins[i].step;
      if (kind == EV_PREFILL) {
        runs[rs].phase = 1;
        push_tok(i, __dadd_rn(clk, step), ev.call, rs, ev.epoch);
      } else {
        const int64_t tok = runs[rs].tokens + 1;
        runs[rs].tokens = tok;
        runs[rs].kv += 1;
        const double lv = __dadd_rn(ins[i].live_kv, 1.0);
        ins[i].live_kv = lv;
        dsec = __dadd_rn(dsec, step);
        if (tok >= runs[rs].target) hpush(push_ev(clk, EV_DONE, ev.call, rs, ev.epoch, 0u));
        else push_tok(i, __dadd_rn(clk, step), ev.call, rs, ev.epoch);
        if (lv > ins[i].cap) hpush(push_ev(clk, EV_PREEMPT, 0, i, 0, 0u));
      }
    }
    sc.heap_n = heap_n;
    sc.top_free = top_free;
    sc.status = status;
    sc.next_seq = next_seq;
    sc.processed = processed;
    sc.clock = clk;
    sc.decode_seconds = dsec;
  };

  // ---- event loop (engine.cpp:85-123) ---------------------------------------
  while (sc.status == KX_OK) {
    if (KX_FAST_TICKS) {
      if (lane == 0) {
        if (KX_FAST_REG) fast_ticks_reg();
        else fast_ticks();
      }
      sync();
      if (sc.status != KX_OK) break;
    }
    if (sc.top_free) pop_heap();  // the last event's root was not reused
    // next event: heap top vs the next arrival (kind 0, seq = local index)
    const bool have_arr = sc.next_arrival < w1;
    const bool have_heap = sc.heap_n > 0;
    if (!have_arr && !have_heap) break;
    Ev ev;
    bool from_heap = have_heap;
    if (have_arr) {
      Ev a{sc.next_arrival_time, static_cast<uint64_t>(sc.next_arrival - w0), 0, -1, 0, 0};
      if (!have_heap || ev_less(a, heap[0])) {
        ev = a;
        from_heap = false;
      }
    }
    if (from_heap) {
      ev = heap[0];
      if (lane == 0) {
        sc.top_free = 1;
        take_root_l0(ev);
      }
    } else if (lane == 0) {
      sc.next_arrival += 1;
      if (sc.next_arrival < w1) sc.next_arrival_time = I.arrival[sc.next_arrival];
    }
    sync();
    if (ev.time < __dsub_rn(sc.clock, kTimeEpsilon)) {
      fail(KX_ERR_LOGIC);  // event time ran backwards
      break;
    }
    if (lane == 0) {
      sc.clock = sc.clock > ev.time ? sc.clock : ev.time;
      sc.processed += 1;
      if (sc.processed > P.max_events) sc.status = KX_ERR_RUNTIME;  // event budget (engine.cpp:99-101)
    }
    sync();
    if (sc.status != KX_OK) break;
    const int kind = static_cast<int>(ev.ks >> 56);
    const double clock = sc.clock;
    if (kind == EV_ARRIVAL) {  // engine.cpp:137-160
      const int64_t w = w0 + static_cast<int64_t>(ev.ks & ((uint64_t(1) << 56) - 1));
      const int64_t cb = I.wf_call[w], ce = I.wf_call[w + 1];
      for (int64_t c = cb + lane; c < ce; c += 32) S.rem_parents[c] = I.has_parent[c] ? 1 : 0;
      if (lane == 0) {
        S.wf_remaining[w] = static_cast<int32_t>(ce - cb);
        S.wf_finish[w] = I.arrival[w];
        S.wf_tokens[w] = 0;
        S.wf_ncalls[w] = 0;
      }
      sync();
      for (int64_t c = cb; c < ce; ++c)
        if (!I.has_parent[c]) enqueue_call(static_cast<uint32_t>(c), clock);
      if (lane == 0) sc.arrivals_remaining -= 1;
      sync();
      schedule_round(clock);
    } else if (kind == EV_PREFILL) {  // engine.cpp:334-341
      const int rs = find_running(ev);
      if (rs < 0) continue;
      if (lane == 0) runs[rs].phase = 1;
      sync();
      if (lane == 0) push_token_l0(runs[rs].inst, __dadd_rn(clock, ins[runs[rs].inst].step), ev.call, rs, ev.epoch);
      sync();
    } else if (kind == EV_TOKEN) {  // engine.cpp:343-361
      const int rs = find_running(ev);
      if (rs < 0) continue;
      const int i = runs[rs].inst;
      const double step = ins[i].step;
      if (lane == 0) {
        runs[rs].tokens += 1;
        runs[rs].kv += 1;
        ins[i].live_kv = __dadd_rn(ins[i].live_kv, 1.0);
        sc.decode_seconds = __dadd_rn(sc.decode_seconds, step);
      }
      sync();
      if (runs[rs].tokens >= runs[rs].target) push(clock, EV_DONE, ev.call, rs, ev.epoch);
      else {
        if (lane == 0) push_token_l0(i, __dadd_rn(clock, step), ev.call, rs, ev.epoch);
        sync();
      }
      if (ins[i].live_kv > ins[i].cap) push(clock, EV_PREEMPT, 0, i, 0);
    } else if (kind == EV_DONE) {  // engine.cpp:363-409
      const int rs = find_running(ev);
      if (rs < 0) continue;
      const int i = runs[rs].inst;
      const uint32_t c = ev.call;
      const int64_t w = wf_of(c);
      if (lane == 0) {
        runs[rs].used = 0;
        S.run_slot[c] = -1;
        ins[i].running -= 1;
        ins[i].live_kv = __dsub_rn(ins[i].live_kv, static_cast<double>(runs[rs].kv));
        sc.completed_kv = __dadd_rn(sc.completed_kv, static_cast<double>(runs[rs].kv));
        const int64_t j = c0 + sc.calls_done;  // completion-order call record
        S.out_call[j] = c;
        S.out_exec_start[j] = runs[rs].exec_start;
        S.out_exec_end[j] = clock;
        S.out_inst[j] = i;
        S.done_idx[c] = j;
        sc.calls_done += 1;
        if (P.profile_T) {  // record_execution (engine.cpp:389)
          const int64_t idx = ab + I.agent[c];
          S.exec_buf[I.exec_off[idx] + S.exec_nt[idx]] = __dsub_rn(clock, runs[rs].exec_start);
          S.exec_nt[idx] += 1;
        }
        S.wf_finish[w] = S.wf_finish[w] > clock ? S.wf_finish[w] : clock;
        S.wf_tokens[w] += I.target[c];
        S.wf_ncalls[w] += 1;
        S.wf_remaining[w] -= 1;
      }
      sync();
      finish_ledger(i, I.uid[c], clock);
      on_live_usage(i);
      for (int64_t j = I.child_off[c]; j < I.child_off[c + 1]; ++j) {  // children in node order
        const uint32_t ch = static_cast<uint32_t>(I.child[j]);
        if (lane == 0) S.rem_parents[ch] -= 1;
        sync();
        if (S.rem_parents[ch] == 0) enqueue_call(ch, clock);
      }
      if (S.wf_remaining[w] == 0) {  // on_workflow_complete (engine.cpp:411-427)
        if (lane == 0) {
          S.out_wf[w0 + sc.wf_done] = w;
          sc.wf_done += 1;
        }
        sync();
        on_workflow_complete(w);
        if (sc.status != KX_OK) break;
      }
      try_admit(i);
      schedule_round(clock);
    } else if (kind == EV_PREEMPT) {  // engine.cpp:436-462
      const int i = ev.inst;
      bool evicted = false;
      while (ins[i].live_kv > ins[i].cap && ins[i].running > 0 && sc.status == KX_OK) {
        // victim: max (victim_rank(agent), exec_start, uid) over running
        double br = -1.0, bs = -1.0;
        uint64_t bu = 0;
        int brs = -1;
        for (int j = lane; j < P.max_run; j += 32) {
          const RunSlot& x = runs[i * P.max_run + j];
          if (!x.used) continue;
          const double rank = P.sched == KX_SCHED_TOPO     ? static_cast<double>(I.depth[I.agent[x.call]])
                              : P.sched == KX_SCHED_KAIROS ? S.pk[ab + I.agent[x.call]]
                                                           : 0.0;
          const uint64_t u = I.uid[x.call];
          if (brs < 0 || rank > br || (rank == br && (x.exec_start > bs || (x.exec_start == bs && u > bu)))) {
            br = rank;
            bs = x.exec_start;
            bu = u;
            brs = i * P.max_run + j;
          }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double r2 = __shfl_xor_sync(0xffffffffu, br, o);
          const double s2 = __shfl_xor_sync(0xffffffffu, bs, o);
          const uint64_t u2 = __shfl_xor_sync(0xffffffffu, bu, o);
          const int k2 = __shfl_xor_sync(0xffffffffu, brs, o);
          if (k2 >= 0 && (brs < 0 || r2 > br || (r2 == br && (s2 > bs || (s2 == bs && u2 > bu))))) {
            br = r2;
            bs = s2;
            bu = u2;
            brs = k2;
          }
        }
        if (brs < 0) break;
        evict(i, brs);
        evicted = true;
      }
      if (evicted) {
        on_overload(i);
        on_live_usage(i);
        schedule_round(clock);
      }
    } else {  // EV_ROUND, engine.cpp:204-218
      if (lane == 0) {
        if (ev.call == 1) sc.tick_scheduled = 0;
        else sc.round_pending = 0;
      }
      sync();
      dispatch_loop();
      for (int i = 0; i < NI; ++i) try_admit(i);
      if (P.dpolicy == KX_DISPATCH_TIME_SLOT) gc(clock);
      if (work_pending() && !sc.tick_scheduled) {
        if (lane == 0) sc.tick_scheduled = 1;
        sync();
        push(__dadd_rn(clock, P.period), EV_ROUND, 1, -1, 0);
      }
    }
  }
  sync();
  if (lane == 0) {
    double* o = S.scalars + int64_t(r) * kEngineScalars;
    o[0] = static_cast<double>(sc.preemption_events);
    o[1] = static_cast<double>(sc.preempted_requests);
    o[2] = sc.wasted_kv;
    o[3] = sc.completed_kv;
    o[4] = sc.prefill_seconds;
    o[5] = sc.decode_seconds;
    o[6] = static_cast<double>(sc.processed);
    o[7] = sc.clock;
    int64_t* n = S.counts + int64_t(r) * 4;
    n[0] = sc.calls_done;
    n[1] = sc.wf_done;
    n[2] = sc.status;
    n[3] = static_cast<int64_t>(sc.processed);
  }
}

__global__ void gather_rep(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ rep,
                           uint32_t* __restrict__ out, int64_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += stride) out[j] = rep[idx[j]];
}

__global__ void gather_key(const uint64_t* __restrict__ k, const uint32_t* __restrict__ pos,
                           uint64_t* __restrict__ out, int64_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += stride) out[j] = k[pos[j]];
}

// ---- K7: per-replica metrics (metrics.cpp:13-88) ----------------------------
// Token latency of each completed, measured workflow; excluded slots get
// ~0 so they sort behind every valid latency of their replica.
__global__ void k_token_latency(EngineInputs I, EngineState S, const int32_t* __restrict__ wf_rep,
                                int64_t W, double warmup, uint64_t* __restrict__ key,
                                uint32_t* __restrict__ rep) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < W; j += stride) {
    const int r = wf_rep[j];
    const int64_t w0 = I.wf_base[r];
    const int64_t done = S.counts[int64_t(r) * 4 + 1];
    uint64_t k = ~0ull;
    if (j - w0 < done) {
      const int64_t w = S.out_wf[j];
      const double app = I.arrival[w];
      const int64_t tok = S.wf_tokens[w];
      if (app >= warmup && tok > 0) {
        const double lat = __ddiv_rn(__dsub_rn(S.wf_finish[w], app), static_cast<double>(tok));
        k = static_cast<uint64_t>(__double_as_longlong(lat));  // lat >= 0: raw bits are monotone
      }
    }
    key[j] = k;
    rep[j] = static_cast<uint32_t>(r);
  }
}

__device__ double quantile_sorted_dev(const uint64_t* s, int64_t n, double p) {  // distribution.cpp:33-44
  auto at = [&](int64_t i) { return __longlong_as_double(static_cast<long long>(s[i])); };
  if (p <= 0.0) return at(0);
  if (p >= 1.0) return at(n - 1);
  const double pos = __dmul_rn(p, static_cast<double>(n - 1));
  const int64_t lo = static_cast<int64_t>(pos);
  const double frac = __dsub_rn(pos, static_cast<double>(lo));
  if (lo + 1 >= n) return at(n - 1);
  return __dadd_rn(at(lo), __dmul_rn(frac, __dsub_rn(at(lo + 1), at(lo))));
}

// One thread per replica: the sequential sums in the reference's order.
__global__ void k_replica_metrics(EngineInputs I, EngineState S, int R, double warmup,
                                  const uint64_t* __restrict__ sorted_lat, double* __restrict__ metrics,
                                  uint32_t* __restrict__ hist) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int64_t w0 = I.wf_base[r];
  const int64_t c0 = I.call_base[r];
  const int64_t wf_done = S.counts[int64_t(r) * 4 + 1];
  const int64_t calls_done = S.counts[int64_t(r) * 4 + 0];
  const double* sc = S.scalars + int64_t(r) * kEngineScalars;
  double* m = metrics + int64_t(r) * kEngineMetrics;
  for (int k = 0; k < kEngineMetrics; ++k) m[k] = 0.0;
  // measured instances: completed workflows with app_start >= warmup
  int64_t measured = 0;
  for (int64_t j = 0; j < wf_done; ++j)
    if (I.arrival[S.out_wf[w0 + j]] >= warmup) ++measured;
  // token latencies, ascending (sorted on the device beforehand)
  const uint64_t* lat = sorted_lat + w0;
  int64_t n = 0;
  double sum = 0.0;
  uint32_t* h = hist + int64_t(r) * kHistBins;
  for (int b = 0; b < kHistBins; ++b) h[b] = 0;
  while (n < (I.wf_base[r + 1] - w0) && lat[n] != ~0ull) {
    const double v = __longlong_as_double(static_cast<long long>(lat[n]));
    sum = __dadd_rn(sum, v);
    const double lg = v > 0.0 ? log2(v) : -1.0e300;
    int b = static_cast<int>(floor((lg + 16.0) * 8.0));
    b = b < 0 ? 0 : (b >= kHistBins ? kHistBins - 1 : b);
    h[b] += 1;
    ++n;
  }
  m[0] = static_cast<double>(measured);
  m[15] = static_cast<double>(n);
  if (n > 0) {
    m[2] = __ddiv_rn(sum, static_cast<double>(n));
    m[3] = quantile_sorted_dev(lat, n, 0.90);
    m[4] = quantile_sorted_dev(lat, n, 0.95);
    m[5] = quantile_sorted_dev(lat, n, 0.99);
  }
  double queue_sum = 0.0, e2e_sum = 0.0, rtl_sum = 0.0;
  int64_t requests = 0;
  for (int64_t j = 0; j < calls_done; ++j) {
    const uint32_t c = S.out_call[c0 + j];
    const int32_t w = I.call_wf[c];
    if (!(I.arrival[w] >= warmup) || S.wf_remaining[w] != 0) continue;
    ++requests;
    queue_sum = __dadd_rn(queue_sum, S.queue_seconds[c]);
    const double e2e = __dsub_rn(S.out_exec_end[c0 + j], S.first_enqueue[c]);
    e2e_sum = __dadd_rn(e2e_sum, e2e);
    rtl_sum = __dadd_rn(rtl_sum, __ddiv_rn(e2e, static_cast<double>(I.target[c])));
  }
  m[1] = static_cast<double>(requests);
  m[12] = queue_sum;
  if (e2e_sum > 0.0) m[7] = __ddiv_rn(queue_sum, e2e_sum);
  if (requests > 0) {
    m[6] = __ddiv_rn(rtl_sum, static_cast<double>(requests));
    m[8] = __ddiv_rn(sc[1], static_cast<double>(calls_done));
  }
  m[9] = sc[1];
  m[10] = sc[0];
  const double kv_total = __dadd_rn(sc[2], sc[3]);
  if (kv_total > 0.0) m[11] = __ddiv_rn(sc[2], kv_total);
  const double engine_time = __dadd_rn(sc[4], sc[5]);
  if (engine_time > 0.0) m[13] = __ddiv_rn(sc[5], engine_time);
  m[14] = sc[7];
}

void launch_replica_metrics(const EngineInputs& in, const EngineState& st, const int32_t* wf_rep,
                            int R, int64_t W, double warmup, double* metrics, uint32_t* hist,
                            cudaStream_t stream) {
  uint64_t *key = nullptr, *key2 = nullptr;
  uint32_t *rep = nullptr, *rep2 = nullptr, *val = nullptr, *val2 = nullptr;
  const size_t n = static_cast<size_t>(W > 0 ? W : 1);
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&key), n * 8, stream));
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&key2), n * 8, stream));
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rep), n * 4, stream));
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rep2), n * 4, stream));
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&val), n * 4, stream));
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&val2), n * 4, stream));
  if (W > 0) {
    k_token_latency<<<static_cast<int>(std::min<int64_t>((W + 255) / 256, 4096)), 256, 0, stream>>>(
        in, st, wf_rep, W, warmup, key, rep);
    KX_CHECK_LAUNCH();
    // (1) all latencies ascending (stable), carrying their slot index
    bool alt = false;
    sort_pairs<uint64_t>(key, val, key2, val2, W, 0, 64, true, &alt, stream);
    uint64_t* k1 = alt ? key2 : key;
    uint32_t* v1 = alt ? val2 : val;
    // (2) stable by replica: gather each element's replica, sort by it
    uint64_t* kfin = alt ? key : key2;
    gather_rep<<<static_cast<int>(std::min<int64_t>((W + 255) / 256, 4096)), 256, 0, stream>>>(
        v1, rep, rep2, W);
    KX_CHECK_LAUNCH();
    int bits = 1;
    while ((1 << bits) < R) ++bits;
    bool alt2 = false;
    // values = positions in the latency-sorted order
    sort_pairs<uint32_t>(rep2, val, rep, val2, W, 0, bits, true, &alt2, stream);
    uint32_t* pos = alt2 ? val2 : val;
    gather_key<<<static_cast<int>(std::min<int64_t>((W + 255) / 256, 4096)), 256, 0, stream>>>(
        k1, pos, kfin, W);
    KX_CHECK_LAUNCH();
    k_replica_metrics<<<(R + 127) / 128, 128, 0, stream>>>(in, st, R, warmup, kfin, metrics, hist);
    KX_CHECK_LAUNCH();
  }
  KX_CUDA(cudaFreeAsync(key, stream));
  KX_CUDA(cudaFreeAsync(key2, stream));
  KX_CUDA(cudaFreeAsync(rep, stream));
  KX_CUDA(cudaFreeAsync(rep2, stream));
  KX_CUDA(cudaFreeAsync(val, stream));
  KX_CUDA(cudaFreeAsync(val2, stream));
}

void launch_replica_engine(const EngineParams& p, const EngineInputs& in, const EngineState& st,
                           int n_replicas, cudaStream_t stream) {
  const size_t smem = engine_smem_bytes(p);
  KX_CUDA(cudaFuncSetAttribute(k_replica_engine, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  k_replica_engine<<<n_replicas, 32, smem, stream>>>(p, in, st);
  KX_CHECK_LAUNCH();
}

}  // namespace kx

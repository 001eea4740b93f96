// K5: memory-aware time-slot dispatch, one CTA per pool (shared LLM).
//
// Replaces, per dispatch round, the placement part of
//   Simulator::dispatch_loop            engine.cpp:220-268
//     collect_live / on_live_usage      engine.cpp:187-202, dispatcher.cpp:283-289
//     Dispatcher::choose (TimeSlot)     dispatcher.cpp:207-247
//       select_instance / try_place     dispatcher.cpp:125-158, 52-68
//     overload check -> on_overload     engine.cpp:254-258, dispatcher.cpp:278-281
//     Dispatcher::commit / ledger       dispatcher.cpp:252-262, 70-79
//     admit (live_kv, running)          engine.cpp:298-319
//   Dispatcher::gc                      engine.cpp:212, dispatcher.cpp:101-118
//
// Walking the pool's sorted queue keeps the reference's strict sequential
// priority order (the placed requests are a prefix, engine.cpp:247). Each
// warp owns a fixed subset of the pool's instances (their ledgers and live
// state), evaluates try_place for its instances in parallel over the slot
// ring, and every warp reduces the same arg-min over (peak, InstanceId)
// (SURVEY H9), so one __syncthreads per decision suffices.
#include <cuda_runtime.h>
#include <cstdlib>
#include <cstring>
#include <stdint.h>

#include "kx_common.cuh"
#include "kx_dispatch.cuh"
#include "kx_order.cuh"
#include "kx_state.cuh"
#include "kx_tuple.cuh"

namespace kx {

namespace {

constexpr int kDispThreads = 512;
constexpr int kDispWarps = kDispThreads / 32;
constexpr int kHeadBatch = 64;

enum : uint8_t { kExcluded = 0, kExceeds = 1, kFits = 2 };

struct Eval {
  double peak;
  int64_t viol;
  uint8_t state;
};

// One instance's slot ledger (dispatcher.hpp:49-85) as a dense ring of
// `ring` slots covering [base, base + ring); ex[] marks the slots present in
// the reference's usage_ map. Each ring is owned by exactly one warp for the
// lifetime of a kernel, and is updated with plain stores only (no atomics:
// an atomic at L2 would leave the owner's L1 copy stale).
struct Ring {
  double* usage;
  uint8_t* ex;
  int64_t base;
  int64_t hi;
};

// The candidate's memory model for one head (t0 = now): span and the
// constants peak_in_slot compares against (dispatcher.cpp:19-42).
struct Span {
  int64_t first, last;
  double t0, t_end, t0e, tee;  // t0 + eps, t_end - eps
};

__device__ __forceinline__ Span make_span(double t0, double T, double slot_len) {
  Span sp;
  span_bounds_dev(t0, T, slot_len, &sp.first, &sp.last);
  sp.t0 = t0;
  sp.t_end = __dadd_rn(t0, T);
  sp.t0e = __dadd_rn(t0, kTimeEpsilon);
  sp.tee = __dsub_rn(sp.t_end, kTimeEpsilon);
  return sp;
}

// peak_in_slot (dispatcher.cpp:33-42) with the per-head constants hoisted.
__device__ __forceinline__ double pis(const Span& sp, double P, double k, int64_t slot,
                                      double slot_len) {
  const double slot_start = __dmul_rn(static_cast<double>(slot), slot_len);
  const double slot_end = __dadd_rn(slot_start, slot_len);
  if (slot_end <= sp.t0e || slot_start >= sp.tee) return 0.0;
  const double eval_t = (sp.t_end < slot_end) ? sp.t_end : slot_end;
  return __dadd_rn(P, __dmul_rn(k, __dsub_rn(eval_t, sp.t0)));
}

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
  const uint32_t hi = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(v >> 32));
  const uint32_t lo = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(v >> 32) == hi
                                                         ? static_cast<uint32_t>(v) : 0u);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
  const uint32_t hi = __reduce_min_sync(0xffffffffu, static_cast<uint32_t>(v >> 32));
  const uint32_t lo = __reduce_min_sync(0xffffffffu, static_cast<uint32_t>(v >> 32) == hi
                                                         ? static_cast<uint32_t>(v) : 0xffffffffu);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

// SlotLedger::try_place (dispatcher.cpp:52-68), one warp: lanes stride the
// retained slots; first violating span slot = warp min, peak = warp max
// (REDUX on the order-preserving bits: max/min are exact).
__device__ Eval warp_try_place(const Ring& r, int ring, double cap, double P, double k,
                               const Span& sp, double slot_len, bool* overflow) {
  const int lane = threadIdx.x & 31;
  if (sp.last >= sp.first && (sp.first < r.base || sp.last >= r.base + ring)) *overflow = true;
  const int64_t smax = r.hi > sp.last ? r.hi : sp.last;
  uint64_t peak = ordered_bits(0.0);
  uint32_t viol = 0xffffffffu;  // offset from base
  for (int64_t s = r.base + lane; s <= smax; s += 32) {
    const uint32_t pos = static_cast<uint32_t>(s) & (ring - 1);
    const bool in_span = (s >= sp.first && s <= sp.last);
    const bool exists = r.ex[pos] != 0;
    if (!(in_span || exists)) continue;
    const double used = exists ? r.usage[pos] : 0.0;
    const double total = __dadd_rn(used, pis(sp, P, k, s, slot_len));
    const uint32_t off = static_cast<uint32_t>(s - r.base);
    if (in_span && total > cap && off < viol) viol = off;
    const uint64_t tb = ordered_bits(total);
    peak = tb > peak ? tb : peak;
  }
  viol = __reduce_min_sync(0xffffffffu, viol);
  Eval e;
  if (viol != 0xffffffffu) {
    e.state = kExceeds;
    e.viol = r.base + viol;
    e.peak = 0.0;
  } else {
    e.state = kFits;
    e.viol = 0;
    e.peak = from_ordered_bits(warp_max_u64(peak));
  }
  return e;
}

// SlotLedger::commit's booking (dispatcher.cpp:75-78), one warp.
__device__ void warp_commit(Ring& r, int ring, double P, double k, const Span& sp,
                            double slot_len) {
  const int lane = threadIdx.x & 31;
  for (int64_t s = sp.first + lane; s <= sp.last; s += 32) {
    const uint32_t pos = static_cast<uint32_t>(s) & (ring - 1);
    r.usage[pos] = __dadd_rn(r.usage[pos], pis(sp, P, k, s, slot_len));
    r.ex[pos] = 1;
  }
  if (sp.last >= sp.first && sp.last > r.hi) r.hi = sp.last;
  __syncwarp();
}

// SlotLedger::gc's slot part (dispatcher.cpp:101-110), one warp.
__device__ void warp_gc_slots(Ring& r, int ring, double now, double slot_len) {
  const int lane = threadIdx.x & 31;
  const int64_t current =
      static_cast<int64_t>(floor(__ddiv_rn(__dadd_rn(now, kTimeEpsilon), slot_len)));
  if (current > r.base) {
    const int64_t stop = current < r.base + ring ? current : r.base + ring;
    for (int64_t s = r.base + lane; s < stop; s += 32) {
      const uint32_t pos = static_cast<uint32_t>(s) & (ring - 1);
      r.usage[pos] = 0.0;
      r.ex[pos] = 0;
    }
    r.base = current;
  }
  __syncwarp();
}

// active_[uid] = m (dispatcher.cpp:78), owner lane only.
__device__ void active_append(InstDev& in, int i, uint64_t uid, double P, double k, double t0,
                              double T, int* status) {
  const int a = in.n_active[i];
  if (a >= kActiveCap) {
    *status = KX_ERR_CAPACITY;
    return;
  }
  const int64_t o = int64_t(i) * kActiveCap + a;
  in.act_uid[o] = uid;
  in.act_P[o] = P;
  in.act_k[o] = k;
  in.act_t0[o] = t0;
  in.act_T[o] = T;
  in.n_active[i] = a + 1;
}

// SlotLedger::gc's active_ part (dispatcher.cpp:111-117), owner lane only.
__device__ __forceinline__ void prefetch_l2_last(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}

// Order-preserving compaction of instance i's active table, entries loaded
// kGcChunk at a time (one memory latency per chunk instead of per entry:
// this runs at the end of the dispatch round, on the tick's critical path).
constexpr int kGcChunk = 8;
__device__ void active_gc(InstDev& in, int i, double now) {
  const int a = in.n_active[i];
  const int64_t o = int64_t(i) * kActiveCap;
  const double lim = __dadd_rn(now, kTimeEpsilon);
  int w = 0;
  for (int j0 = 0; j0 < a; j0 += kGcChunk) {
    uint64_t u[kGcChunk];
    double P[kGcChunk], k[kGcChunk], t0[kGcChunk], T[kGcChunk];
#pragma unroll
    for (int c = 0; c < kGcChunk; ++c) {
      if (j0 + c < a) {
        u[c] = in.act_uid[o + j0 + c];
        P[c] = in.act_P[o + j0 + c];
        k[c] = in.act_k[o + j0 + c];
        t0[c] = in.act_t0[o + j0 + c];
        T[c] = in.act_T[o + j0 + c];
      }
    }
#pragma unroll
    for (int c = 0; c < kGcChunk; ++c) {
      if (j0 + c >= a) break;
      if (__dadd_rn(t0[c], T[c]) <= lim) continue;  // elapsed model (dispatcher.cpp:113-117)
      if (w != j0 + c) {
        in.act_uid[o + w] = u[c];
        in.act_P[o + w] = P[c];
        in.act_k[o + w] = k[c];
        in.act_t0[o + w] = t0[c];
        in.act_T[o + w] = T[c];
      }
      ++w;
    }
  }
  in.n_active[i] = w;
}

__device__ __forceinline__ Ring global_ring(const InstDev& in, int i, int ring) {
  Ring r;
  r.usage = in.usage + int64_t(i) * ring;
  r.ex = in.exists + int64_t(i) * ring;
  r.base = in.base_slot[i];
  r.hi = in.hi_slot[i];
  return r;
}

}  // namespace

// Byte offsets of the dispatch kernel's shared-memory arrays (host-computed,
// passed by value so the kernel never re-derives them).
struct DispLayout {
  uint32_t live, cap, k, snap, peak, base, hi, viol, run, wait, mb, id, susp, state;
  uint32_t h_T, h_prompt, h_kept, h_uid, h_agent, h_idx, h_first, h_last, h_tend;
  uint32_t usage, ex, total;
};

DispLayout disp_layout(int ni, int ring, bool smem_ring) {
  DispLayout L{};
  uint32_t o = 0;
  auto take = [&](size_t bytes) {
    const uint32_t at = o;
    o = static_cast<uint32_t>((o + bytes + 15) & ~size_t(15));
    return at;
  };
  L.live = take(8 * ni);
  L.cap = take(8 * ni);
  L.k = take(8 * ni);
  L.snap = take(8 * 2 * ni);
  L.peak = take(8 * 2 * ni);
  L.base = take(8 * ni);
  L.hi = take(8 * ni);
  L.viol = take(8 * 2 * ni);
  L.run = take(4 * ni);
  L.wait = take(4 * ni);
  L.mb = take(4 * ni);
  L.id = take(4 * ni);
  L.susp = take(ni);
  L.state = take(2 * ni);
  L.h_T = take(8 * kHeadBatch);
  L.h_prompt = take(8 * kHeadBatch);
  L.h_kept = take(8 * kHeadBatch);
  L.h_uid = take(8 * kHeadBatch);
  L.h_agent = take(4 * kHeadBatch);
  L.h_idx = take(4 * kHeadBatch);
  L.h_first = take(8 * kHeadBatch);
  L.h_last = take(8 * kHeadBatch);
  L.h_tend = take(8 * kHeadBatch);
  L.usage = smem_ring ? take(size_t(8) * ni * ring) : 0;
  L.ex = smem_ring ? take(size_t(ni) * ring) : 0;
  L.total = o;
  return L;
}

#define SM(type, field) reinterpret_cast<type*>(smem_raw + lay.field)

template <bool kSmemRing>
__global__ void __launch_bounds__(kDispThreads)
k_dispatch_timeslot(QueueDev q, AgentsDev ag, InstDev in, const int32_t* __restrict__ pool_begin,
                    const uint32_t* __restrict__ perm, const int64_t* __restrict__ pool_offsets,
                    DispatchParams dp, DispLayout lay, kx_decision* __restrict__ rows,
                    double* __restrict__ cand, int64_t* __restrict__ row_count,
                    int64_t* __restrict__ admitted_count, int* __restrict__ pool_status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_status;
  const int pool = blockIdx.x;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ib = pool_begin[pool];
  const int ni = pool_begin[pool + 1] - ib;
  const int ring = dp.ring;
  const double now = dp.now;

  // Stage the pool's instance state (and rings) in shared memory.
  for (int li = threadIdx.x; li < ni; li += kDispThreads) {
    const int i = ib + li;
    SM(double, live)[li] = in.live_kv[i];
    SM(double, cap)[li] = in.cap[i];
    SM(double, k)[li] = in.decode_rate[i];
    SM(int64_t, base)[li] = in.base_slot[i];
    SM(int64_t, hi)[li] = in.hi_slot[i];
    SM(int32_t, run)[li] = in.running[i];
    SM(int32_t, wait)[li] = in.waiting[i];
    SM(int32_t, mb)[li] = in.max_batch[i];
    SM(int32_t, id)[li] = in.id[i];
    SM(uint8_t, susp)[li] = in.suspended[i];
  }
  if (kSmemRing) {
    const int64_t tot = int64_t(ni) * ring;
    const double* gu = in.usage + int64_t(ib) * ring;
    const uint8_t* ge = in.exists + int64_t(ib) * ring;
    for (int64_t j = threadIdx.x; j < tot; j += kDispThreads) {
      SM(double, usage)[j] = gu[j];
      SM(uint8_t, ex)[j] = ge[j];
    }
  }
  if (threadIdx.x == 0) s_status = KX_OK;
  __syncthreads();

  auto ring_of = [&](int li) {
    Ring r;
    if (kSmemRing) {
      r.usage = SM(double, usage) + int64_t(li) * ring;
      r.ex = SM(uint8_t, ex) + int64_t(li) * ring;
    } else {
      r.usage = in.usage + int64_t(ib + li) * ring;
      r.ex = in.exists + int64_t(ib + li) * ring;
    }
    r.base = SM(int64_t, base)[li];
    r.hi = SM(int64_t, hi)[li];
    return r;
  };

  const int64_t q_end = pool_offsets[pool + 1];
  int64_t pos = pool_offsets[pool];
  int64_t hb_start = pos, hb_n = 0;
  int64_t nrows = 0, nadm = 0;
  int retries = 0;
  int par = 0;
  const double t0e = __dadd_rn(now, kTimeEpsilon);

  while (pos < q_end) {
    if (pos >= hb_start + hb_n) {  // refill the head batch (prefix of the pool's order)
      __syncthreads();
      hb_start = pos;
      hb_n = q_end - pos < kHeadBatch ? q_end - pos : kHeadBatch;
      if (threadIdx.x < hb_n) {
        const int t = threadIdx.x;
        const uint32_t idx = perm[pos + t];
        const int32_t a = q.agent[idx];
        const double T = dp.oracle_T ? q.pure_exec[idx] : ag.T[a];
        SM(uint32_t, h_idx)[t] = idx;
        SM(int32_t, h_agent)[t] = a;
        SM(int64_t, h_prompt)[t] = q.prompt[idx];
        SM(int64_t, h_kept)[t] = q.kept[idx];
        SM(uint64_t, h_uid)[t] = q.uid[idx];
        SM(double, h_T)[t] = T;
        int64_t f, l;
        span_bounds_dev(now, T, dp.slot_len, &f, &l);
        SM(int64_t, h_first)[t] = f;
        SM(int64_t, h_last)[t] = l;
        SM(double, h_tend)[t] = __dadd_rn(now, T);
      }
      __syncthreads();
    }
    const int h = static_cast<int>(pos - hb_start);
    const int64_t prompt = SM(int64_t, h_prompt)[h];
    const double P = static_cast<double>(prompt);
    const double T = SM(double, h_T)[h];
    Span sp;
    sp.first = SM(int64_t, h_first)[h];
    sp.last = SM(int64_t, h_last)[h];
    sp.t0 = now;
    sp.t_end = SM(double, h_tend)[h];
    sp.t0e = t0e;
    sp.tee = __dsub_rn(sp.t_end, kTimeEpsilon);
    bool overflow = false;

    for (int li = warp; li < ni; li += kDispWarps) {
      // collect_live: watermark resume on the freshest usage, then batch_full.
      const double live = SM(double, live)[li];
      uint8_t susp = SM(uint8_t, susp)[li];
      if (susp && live < __dmul_rn(dp.watermark, SM(double, cap)[li])) {
        susp = 0;
        __syncwarp();
        if (lane == 0) SM(uint8_t, susp)[li] = 0;
      }
      const bool full = SM(int32_t, run)[li] + SM(int32_t, wait)[li] >= SM(int32_t, mb)[li];
      Eval e;
      if (susp || full) {
        e.state = kExcluded;
        e.peak = 0.0;
        e.viol = 0;
      } else {
        e = warp_try_place(ring_of(li), ring, SM(double, cap)[li], P, SM(double, k)[li], sp,
                           dp.slot_len, &overflow);
      }
      if (lane == 0) {
        SM(double, peak)[par * ni + li] = e.peak;
        SM(int64_t, viol)[par * ni + li] = e.viol;
        SM(uint8_t, state)[par * ni + li] = e.state;
        SM(double, snap)[par * ni + li] = live;
      }
    }
    if (overflow && lane == 0) atomicExch(&s_status, KX_ERR_CAPACITY);
    __syncthreads();
    if (s_status != KX_OK) break;

    // select_instance: min (peak, InstanceId) over fitting candidates (H9).
    uint64_t bkey = ~0ull;
    uint32_t bid = 0xffffffffu;
    int bli = -1;
    for (int li = lane; li < ni; li += 32) {
      if (SM(uint8_t, state)[par * ni + li] != kFits) continue;
      const uint64_t kb = ordered_bits(SM(double, peak)[par * ni + li]);
      const uint32_t id = static_cast<uint32_t>(SM(int32_t, id)[li]) ^ 0x80000000u;
      if (bli < 0 || kb < bkey || (kb == bkey && id < bid)) {
        bkey = kb;
        bid = id;
        bli = li;
      }
    }
    const uint64_t wkey = warp_min_u64(bkey);
    const uint32_t wid = __reduce_min_sync(0xffffffffu, (bli >= 0 && bkey == wkey) ? bid : 0xffffffffu);
    const uint32_t winners = __ballot_sync(0xffffffffu, bli >= 0 && bkey == wkey && bid == wid);
    bli = winners ? __shfl_sync(0xffffffffu, bli, __ffs(winners) - 1) : -1;
    const double bpeak = bli >= 0 ? SM(double, peak)[par * ni + bli] : 0.0;
    // Overload check (engine.cpp:254-258) on the owner's live snapshot.
    const bool overload = bli >= 0 && __dadd_rn(SM(double, snap)[par * ni + bli], P) > SM(double, cap)[bli];

    if (warp == kDispWarps - 1) {  // decision log (engine.cpp:242-246)
      if (nrows < dp.log_cap) {
        const int64_t r = int64_t(pool) * dp.log_cap + nrows;
        if (lane == 0) {
          kx_decision d;
          d.time = now;
          d.predicted_peak = bli >= 0 ? bpeak : 0.0;
          d.uid = SM(uint64_t, h_uid)[h];
          d.queue_index = SM(uint32_t, h_idx)[h];
          d.agent = SM(int32_t, h_agent)[h];
          d.target = bli >= 0 ? SM(int32_t, id)[bli] : -1;
          d.pool = pool;
          d.admitted = (bli >= 0 && !overload) ? 1 : 0;
          rows[r] = d;
        }
        for (int li = lane; li < ni; li += 32) {
          const uint8_t st = SM(uint8_t, state)[par * ni + li];
          double v = -1.0;
          if (st == kFits) v = SM(double, peak)[par * ni + li];
          else if (st == kExceeds) v = __dsub_rn(-static_cast<double>(SM(int64_t, viol)[par * ni + li]), 1.0);
          cand[r * dp.peak_stride + li] = v;
        }
      }
    }
    ++nrows;
    if (bli < 0) break;  // head keeps its place until the next round (engine.cpp:247)
    const bool owner = (bli % kDispWarps) == warp;
    if (overload) {
      if (owner && lane == 0) SM(uint8_t, susp)[bli] = 1;  // Dispatcher::on_overload
      if (++retries > ni) {
        if (threadIdx.x == 0) s_status = KX_ERR_LIVELOCK;
        break;
      }
      par ^= 1;
      continue;
    }
    retries = 0;
    if (owner) {
      Ring r = ring_of(bli);
      const double k = SM(double, k)[bli];
      warp_commit(r, ring, P, k, sp, dp.slot_len);
      if (lane == 0) {
        SM(int64_t, hi)[bli] = r.hi;
        SM(double, live)[bli] = __dadd_rn(SM(double, live)[bli],
                                          static_cast<double>(prompt + SM(int64_t, h_kept)[h]));
        SM(int32_t, run)[bli] += 1;
        const uint32_t idx = SM(uint32_t, h_idx)[h];
        q.admitted[idx] = 1;
        active_append(in, ib + bli, SM(uint64_t, h_uid)[h], P, k, now, T, &s_status);
      }
      __syncwarp();
    }
    ++nadm;
    ++pos;
    par ^= 1;
  }
  __syncthreads();
  // try_admit is a no-op for TimeSlot (waiting lists stay empty); Dispatcher::gc.
  for (int li = warp; li < ni; li += kDispWarps) {
    Ring r = ring_of(li);
    warp_gc_slots(r, ring, now, dp.slot_len);
    if (lane == 0) {
      SM(int64_t, base)[li] = r.base;
      active_gc(in, ib + li, now);
    }
  }
  __syncthreads();
  for (int li = threadIdx.x; li < ni; li += kDispThreads) {
    const int i = ib + li;
    in.live_kv[i] = SM(double, live)[li];
    in.base_slot[i] = SM(int64_t, base)[li];
    in.hi_slot[i] = SM(int64_t, hi)[li];
    in.running[i] = SM(int32_t, run)[li];
    in.suspended[i] = SM(uint8_t, susp)[li];
  }
  if (kSmemRing) {
    const int64_t tot = int64_t(ni) * ring;
    double* gu = in.usage + int64_t(ib) * ring;
    uint8_t* ge = in.exists + int64_t(ib) * ring;
    for (int64_t j = threadIdx.x; j < tot; j += kDispThreads) {
      gu[j] = SM(double, usage)[j];
      ge[j] = SM(uint8_t, ex)[j];
    }
  }
  if (threadIdx.x == 0) {
    row_count[pool] = nrows;
    admitted_count[pool] = nadm;
    pool_status[pool] = s_status;
  }
}

#undef SM

// ---- K5 fast path (pools of <= 32 instances): shared definitions ----------
// The decisions of a pool form one sequential chain (each commit changes the
// ledger the next head is placed against). The batched kernel below runs
// that chain on one resolver warp with lanes = instances, assigned in
// increasing InstanceId order, so select_instance's tie rule (smaller id,
// SURVEY H9) is the lowest lane among equal peaks.
//
// try_place's slot walk (dispatcher.cpp:52-68) is split in three. With
// c = floor((now + eps) / L) every head's span is [c, last]. When
// peak_in_slot (dispatcher.cpp:33-42) is zero on every slot outside the span
// (checked per head on the two neighbouring slots each side; the reference's
// floors make it zero further out), a stored slot outside the span
// contributes exactly `used` to the predicted peak, so:
//   * stored slots below c (stale past slots before the end-of-round gc, H5)
//     are one per-instance max, fixed for the round;
//   * stored slots above the span are a per-instance suffix max over the
//     ring, refreshed for the target after each commit;
//   * the span is evaluated slot by slot with the reference's
//     used + (P + k * dt), correctly rounded; (P + k * dt) comes from a
//     per-head table built when the head batch is loaded (per lane when the
//     pool's decode rates differ).
// Heads outside that shape (T <= 0, negative prompt, a non-zero margin slot,
// spans longer than the table) take the generic slot walk. Ledger rings are
// staged transposed (usage[slot][lane]). Invariant: a slot that is not
// stored holds usage +0.0 (gc and the initial state write 0.0).
constexpr int kWHB = 32;       // head batch (lane = head while loading)
constexpr int kDtSlots = 64;   // span slots tabulated per head


// (eval_t - t0) of peak_in_slot (dispatcher.cpp:33-42) for one slot, NaN
// when the slot takes the zero branch.
__device__ __forceinline__ double slot_dt(double t0, double t0e, double t_end, double tee,
                                          int64_t slot, double slot_len) {
  const double slot_start = __dmul_rn(static_cast<double>(slot), slot_len);
  const double slot_end = __dadd_rn(slot_start, slot_len);
  if (slot_end <= t0e || slot_start >= tee) return __longlong_as_double(0x7ff8000000000000ll);
  const double eval_t = (t_end < slot_end) ? t_end : slot_end;
  return __dsub_rn(eval_t, t0);
}

__device__ __forceinline__ double pk_of(double P, double k, double dt) {
  return dt == dt ? __dadd_rn(P, __dmul_rn(k, dt)) : 0.0;
}

__device__ __forceinline__ uint64_t shfl_up_u64(uint64_t v, int d) {
  const uint32_t lo = __shfl_up_sync(0xffffffffu, static_cast<uint32_t>(v), d);
  const uint32_t hi = __shfl_up_sync(0xffffffffu, static_cast<uint32_t>(v >> 32), d);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
  const uint32_t lo = __shfl_sync(0xffffffffu, static_cast<uint32_t>(v), src);
  const uint32_t hi = __shfl_sync(0xffffffffu, static_cast<uint32_t>(v >> 32), src);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

// Head modes (per head, warp-uniform).
enum : int32_t { kModeTabPk = 0, kModeTabDt = 1, kModeGeneric = 2 };


constexpr int kHR = 64;  // head ring: two batches of kWHB


// ---- K5 batched: parallel look-ahead rows + one resolver warp ---------------
// The heads of a round are taken in
// batches of kBatchEval: each evaluator warp computes the try_place row of
// one head of the batch (lanes = instances) against the state at the start
// of the batch, all in parallel (phase A). The resolver warp then walks the
// batch in priority order (phase B). A head's row is exact except for the
// instances changed by the batch's earlier decisions (a commit, or a
// suspension on overload); those lanes re-evaluate themselves from the
// resolver's registers, all at once. select_instance is one 64-bit warp min,
// the overload check a ballot, the commit a loop in the target's own lane.
// Decision records are staged in shared memory and written to global memory
// by another warp during the next batch's phase B.
#ifndef KX_DISPATCH_TIMERS
#define KX_DISPATCH_TIMERS 0
#endif
__device__ unsigned long long g_disp_dbg[16];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr int kBatchEval = 8;
constexpr int kBatchThreads = 32 * (kBatchEval + 1);
constexpr int kStage = 64;  // staged decision records per batch buffer
constexpr int kFlushWarp = 2;
// Ledger rows of 33 words: lanes = instances read a row conflict-free, and
// lanes = slots read one instance's column conflict-free too.
constexpr int kRow = 33;

struct StageMeta {
  int32_t hs;        // head ring slot
  int32_t target;    // lane of the target, -1 none
  int32_t admitted;
  int32_t act_slot;  // active-table slot of an admission (-1 none)
};

// One instance's try_place result for a staged decision (one 16-byte store).
struct __align__(16) StageRow {
  uint32_t viol;
  uint32_t flag;
  uint64_t peak;
};

struct BatchLayout {
  uint32_t h_idx, h_agent, h_prompt, h_kept, h_uid, h_T, h_first, h_last, h_mode, tab, lane_inst,
      st_live, st_run, st_susp, st_hi, st_umax, r_viol, r_peak, r_flag, g_meta, g_row, c_key, c_idx,
      usage, ex, total;
};

BatchLayout batch_layout(int ring) {
  BatchLayout L{};
  uint32_t o = 0;
  auto take = [&](size_t bytes) {
    const uint32_t at = o;
    o = static_cast<uint32_t>((o + bytes + 15) & ~size_t(15));
    return at;
  };
  L.h_idx = take(4 * kHR);
  L.h_agent = take(4 * kHR);
  L.h_prompt = take(8 * kHR);
  L.h_kept = take(8 * kHR);
  L.h_uid = take(8 * kHR);
  L.h_T = take(8 * kHR);
  L.h_first = take(8 * kHR);
  L.h_last = take(8 * kHR);
  L.h_mode = take(4 * kHR);
  L.tab = take(size_t(8) * kHR * kDtSlots);
  L.lane_inst = take(4 * 32);
  L.st_live = take(8 * 32);
  L.st_run = take(4 * 32);
  L.st_susp = take(4 * 32);
  L.st_hi = take(4 * 32);
  L.st_umax = take(8 * 32);
  L.r_viol = take(4 * 32 * kBatchEval);
  L.r_peak = take(8 * 32 * kBatchEval);
  L.r_flag = take(4 * 32 * kBatchEval);
  L.g_meta = take(sizeof(StageMeta) * 2 * kStage);
  L.g_row = take(sizeof(StageRow) * 32 * 2 * kStage);
  L.c_key = take(size_t(8) * kTopKMax);
  L.c_idx = take(size_t(4) * kTopKMax);
  L.usage = take(size_t(8) * 32 * ring);
  L.ex = take(size_t(32) * ring);
  L.total = o;
  return L;
}

// The collected prefix of one pool in order (all threads of the CTA): a
// bitonic sort of (compact key << 32 | slot) in shared memory, then runs of
// equal compact keys re-sorted by the exact tuple (one thread per run).
// Returns false when a run is longer than kRunMax (degenerate keys): the
// caller then dispatches from the full order instead.
constexpr int kRunMax = 16;

__device__ bool sort_prefix(const QueueDev& q, int policy, const uint32_t* __restrict__ cand,
                            const uint32_t* __restrict__ ckey, int n, uint32_t* __restrict__ heads,
                            uint64_t* sk, uint32_t* so) {
  __shared__ int s_long;
  int p2 = 1;
  while (p2 < n) p2 <<= 1;
  for (int i = threadIdx.x; i < p2; i += blockDim.x)
    sk[i] = i < n ? ((static_cast<uint64_t>(__ldcg(ckey + i)) << 32) | static_cast<uint32_t>(i)) : ~0ull;
  if (threadIdx.x == 0) s_long = 0;
  __syncthreads();
  for (int kk = 2; kk <= p2; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < p2; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const uint64_t x = sk[i], y = sk[l];
          if ((x > y) == ((i & kk) == 0)) {
            sk[i] = y;
            sk[l] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) so[i] = __ldcg(cand + static_cast<uint32_t>(sk[i]));
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t k = static_cast<uint32_t>(sk[i] >> 32);
    const bool start = (i == 0 || static_cast<uint32_t>(sk[i - 1] >> 32) != k) &&
                       (i + 1 < n && static_cast<uint32_t>(sk[i + 1] >> 32) == k);
    if (!start) continue;
    int e = i + 2;
    while (e < n && e - i <= kRunMax && static_cast<uint32_t>(sk[e] >> 32) == k) ++e;
    const int len = e - i;
    if (len > kRunMax) {
      s_long = 1;
      continue;
    }
    TKey r[kRunMax];
    for (int j = 0; j < len; ++j) r[j] = load_tkey(q, policy, so[i + j]);
    for (int j = 1; j < len; ++j) {
      const TKey x = r[j];
      int m = j - 1;
      while (m >= 0 && tkey_less(q, x, r[m])) {
        r[m + 1] = r[m];
        --m;
      }
      r[m + 1] = x;
    }
    for (int j = 0; j < len; ++j) so[i + j] = r[j].idx;
  }
  __syncthreads();
  if (s_long) return false;
  for (int i = threadIdx.x; i < n; i += blockDim.x) heads[i] = so[i];
  __threadfence_block();
  __syncthreads();
  return true;
}

__device__ __forceinline__ void batch_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kBatchThreads) : "memory"); }

__global__ void __launch_bounds__(kBatchThreads)
k_dispatch_batch(QueueDev q, AgentsDev ag, InstDev in, const int32_t* __restrict__ pool_begin,
                 const uint32_t* __restrict__ perm, const int64_t* __restrict__ pool_offsets,
                 DispatchParams dp, BatchLayout lay, kx_decision* __restrict__ rows,
                 double* __restrict__ cand, int64_t* __restrict__ row_count,
                 int64_t* __restrict__ admitted_count, int* __restrict__ pool_status,
                 DispPhase ph) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int64_t s_win[3];   // staged slot window [B, top]; top after the round
  __shared__ int64_t s_next;     // first head of the next batch (resolver -> all)
  __shared__ int32_t s_stop;     // resolver: round over
  __shared__ int32_t s_ids[32];  // InstanceId per lane
  __shared__ int32_t s_nstage[2];
  __shared__ int64_t s_row0[2];  // log row of each staging buffer's first record
  const int pool = blockIdx.x;
  // phase 3 learns its heads (and the pool size) only once key generation
  // has finished, below
  int64_t pool_n = ph.phase == 3 ? 0 : pool_offsets[pool + 1] - pool_offsets[pool];
  const uint32_t* hp = ph.phase == 3 ? ph.heads_out + int64_t(pool) * kTopKMax : perm + pool_offsets[pool];
  int64_t q_end = pool_n, pos0 = 0, nrows0 = 0, nadm0 = 0;
  bool skip = false;
  if (ph.phase == 1) {
    const TopKState t = ph.tk[pool];
    if (t.defer) {  // too many ties at the boundary key: wait for the full order
      if (threadIdx.x == 0) ph.resume[pool] = DispResume{0, 0, 0, 1, 0};
      skip = true;
    }
    hp = ph.heads + int64_t(pool) * kTopKMax;
    q_end = t.empty ? 0 : (t.n_cand < kTopKMax ? t.n_cand : kTopKMax);
  } else if (ph.phase == 2) {
    const DispResume r = ph.resume[pool];
    skip = !r.need;
    pos0 = r.start;
    nrows0 = r.nrows;
    nadm0 = r.nadm;
  }
  if (skip) return;  // uniform over the CTA
  const bool dbg = KX_DISPATCH_TIMERS && blockIdx.x == 0 && threadIdx.x == 0;
  if (dbg) g_disp_dbg[0] = gtimer();
  unsigned long long acc_a = 0, acc_b = 0, tA = 0, nbat = 0, acc_fix = 0, acc_sel = 0, acc_stg = 0, acc_com = 0;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ib = pool_begin[pool];
  const int ni = pool_begin[pool + 1] - ib;
  const int ring = dp.ring;
  const int rmask = ring - 1;
#define BL(type, field) reinterpret_cast<type*>(smem_raw + lay.field)
  double* const su = BL(double, usage);
  uint8_t* const se = BL(uint8_t, ex);
  int32_t* const s_li = BL(int32_t, lane_inst);
  uint32_t* const h_idx = BL(uint32_t, h_idx);
  int32_t* const h_agent = BL(int32_t, h_agent);
  int64_t* const h_prompt = BL(int64_t, h_prompt);
  int64_t* const h_kept = BL(int64_t, h_kept);
  uint64_t* const h_uid = BL(uint64_t, h_uid);
  double* const h_T = BL(double, h_T);
  int64_t* const h_first = BL(int64_t, h_first);
  int64_t* const h_last = BL(int64_t, h_last);
  int32_t* const h_mode = BL(int32_t, h_mode);
  double* const stab = BL(double, tab);
  double* const st_live = BL(double, st_live);
  int32_t* const st_run = BL(int32_t, st_run);
  int32_t* const st_susp = BL(int32_t, st_susp);
  int32_t* const st_hi = BL(int32_t, st_hi);
  uint64_t* const st_umax = BL(uint64_t, st_umax);
  uint32_t* const r_viol = BL(uint32_t, r_viol);
  uint64_t* const r_peak = BL(uint64_t, r_peak);
  uint32_t* const r_flag = BL(uint32_t, r_flag);
  StageMeta* const g_meta = BL(StageMeta, g_meta);
  StageRow* const g_row = BL(StageRow, g_row);
#undef BL
  const uint64_t kZeroBits = 0x8000000000000000ull;  // ordered_bits(0.0)
  constexpr uint32_t kNone = 0xffffffffu;

  // Lane of each instance: rank of its InstanceId within the pool (H9).
  if (warp == 0) {
    const int32_t myid = lane < ni ? in.id[ib + lane] : 0x7fffffff;
    int rank = 0;
    for (int l = 0; l < 32; ++l) {
      const int32_t o = __shfl_sync(0xffffffffu, myid, l);
      rank += (l < ni) && (o < myid || (o == myid && l < lane));
    }
    s_li[lane] = -1;
    __syncwarp();
    if (lane < ni) s_li[rank] = lane;
    const bool a0 = lane < ni;
    const int64_t bb = a0 ? in.base_slot[ib + lane] : INT64_MAX;
    const int64_t hh = a0 ? in.hi_slot[ib + lane] : INT64_MIN;
    const uint64_t bmin = warp_min_u64(static_cast<uint64_t>(bb) ^ 0x8000000000000000ull);
    const uint64_t hmax = warp_max_u64(static_cast<uint64_t>(hh) ^ 0x8000000000000000ull);
    if (lane == 0) {
      s_win[0] = static_cast<int64_t>(bmin ^ 0x8000000000000000ull);
      s_win[1] = static_cast<int64_t>(hmax ^ 0x8000000000000000ull);
      s_stop = 0;
      s_next = pos0;
      s_nstage[0] = s_nstage[1] = 0;
    }
  }
  __syncthreads();
  // Stage the rings transposed (usage[pos][lane]): zero everywhere, then copy
  // the slot window's positions, four independent loads in flight per thread.
  const int64_t wB = s_win[0];
  const int64_t wtop = s_win[1];
  const int win = wtop < wB ? 0 : static_cast<int>(wtop - wB + 1 < ring ? wtop - wB + 1 : ring);
  for (int j = threadIdx.x; j < kRow * ring; j += kBatchThreads) {
    su[j] = 0.0;
    se[j] = 0;
  }
  __syncthreads();
  {
    const int total = win * 32;
    for (int e0 = threadIdx.x; e0 < total; e0 += 4 * kBatchThreads) {
      double u[4];
      uint8_t x[4];
      int dst[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = e0 + k * kBatchThreads;
        const int l = e & 31;
        const int li = e < total ? s_li[l] : -1;
        const int pos = static_cast<int>((wB + (e >> 5)) & rmask);
        dst[k] = li >= 0 ? pos * kRow + l : -1;
        u[k] = li >= 0 ? in.usage[int64_t(ib + li) * ring + pos] : 0.0;
        x[k] = li >= 0 ? in.exists[int64_t(ib + li) * ring + pos] : 0;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (dst[k] >= 0) {
          su[dst[k]] = u[k];
          se[dst[k]] = x[k];
        }
    }
  }
  __syncthreads();
  if (dbg) g_disp_dbg[1] = gtimer();

  // ---- per-lane instance constants (every warp) ----
  const double now = dp.now;
  const double L = dp.slot_len;
  const int li = s_li[lane];
  const bool act = li >= 0;
  const int i = ib + (act ? li : 0);
  const double cap = act ? in.cap[i] : 0.0;
  const double kr = act ? in.decode_rate[i] : 0.0;
  const int32_t mb = act ? in.max_batch[i] : 0;
  const int32_t id = act ? in.id[i] : 0x7fffffff;
  const int32_t waiting = act ? in.waiting[i] : 0;
  const double wcap = __dmul_rn(dp.watermark, cap);
  const int64_t base = act ? in.base_slot[i] : 0;
  const int64_t hi0 = act ? in.hi_slot[i] : -1;
  const double k0 = __shfl_sync(0xffffffffu, kr, 0);
  const bool k_uniform = __all_sync(0xffffffffu, !act || kr == k0);
  const int64_t B = wB;
  const int32_t lo_off = static_cast<int32_t>(base - B);
  const double t0e = __dadd_rn(now, kTimeEpsilon);
  const int64_t cslot = static_cast<int64_t>(floor(__ddiv_rn(t0e, L)));
  if (warp == 0) s_ids[lane] = id;

  // try_place of the head in ring slot hs for this lane's instance, given
  // its live state (lanes = instances). Returns the row entry.
  struct Row {
    uint32_t viol;
    uint64_t peak;
    uint32_t flag;  // bit 0 eligible, bit 1 ring overflow
  };
  auto evaluate = [&](int hs, double live_, int32_t run_, bool susp_, uint64_t umax_, int32_t hi_off_) {
    const int mode = h_mode[hs];
    const int64_t first = h_first[hs];
    const int64_t last = h_last[hs];
    const double P = static_cast<double>(h_prompt[hs]);
    const int32_t fo = static_cast<int32_t>(first - B);
    const int32_t lo = static_cast<int32_t>(last - B);
    const bool nonempty = last >= first;
    const bool sp = susp_ && !(live_ < wcap);  // collect_live's watermark resume
    const bool eligible = act && !sp && !(run_ + waiting >= mb);
    Row r{kNone, kZeroBits, 0u};
    const bool overflow = eligible && nonempty && (first < base || last >= base + ring);
    if (eligible) {
      if (mode != kModeGeneric) {
        uint64_t peak = umax_;
        uint32_t viol = kNone;
        const double* tab = stab + hs * kDtSlots;
        const int tn = lo - fo + 1;
        int p2 = static_cast<int>((B + fo) & rmask);
        if (mode == kModeTabPk) {
#pragma unroll 4
          for (int jj = 0; jj < tn; ++jj) {
            const double total = __dadd_rn(su[p2 * kRow + lane], tab[jj]);
            if (total > cap && viol == kNone) viol = static_cast<uint32_t>(fo + jj);
            const uint64_t tb = static_cast<uint64_t>(__double_as_longlong(total)) | kZeroBits;
            peak = tb > peak ? tb : peak;
            p2 = (p2 + 1) & rmask;
          }
        } else {
#pragma unroll 4
          for (int jj = 0; jj < tn; ++jj) {
            const double total = __dadd_rn(su[p2 * kRow + lane], pk_of(P, kr, tab[jj]));
            if (total > cap && viol == kNone) viol = static_cast<uint32_t>(fo + jj);
            const uint64_t tb = static_cast<uint64_t>(__double_as_longlong(total)) | kZeroBits;
            peak = tb > peak ? tb : peak;
            p2 = (p2 + 1) & rmask;
          }
        }
        r.viol = viol;
        r.peak = peak;
      } else {  // generic slot walk over the whole window
        const double te = __dadd_rn(now, h_T[hs]);
        const double tee = __dsub_rn(te, kTimeEpsilon);
        const int32_t top = hi_off_ > lo ? hi_off_ : lo;
        uint64_t peak = kZeroBits;
        uint32_t viol = kNone;
        for (int32_t o = lo_off; o <= top; ++o) {
          const int p2 = static_cast<int>((B + o) & rmask);
          const bool e = se[p2 * kRow + lane] != 0;
          const bool in_span = o >= fo && o <= lo;
          if (!(e || in_span)) continue;
          const double used = e ? su[p2 * kRow + lane] : 0.0;
          const double total = __dadd_rn(used, pk_of(P, kr, slot_dt(now, t0e, te, tee, B + o, L)));
          if (in_span && total > cap) viol = static_cast<uint32_t>(o) < viol ? static_cast<uint32_t>(o) : viol;
          const uint64_t tb = ordered_bits(total);
          peak = tb > peak ? tb : peak;
        }
        r.viol = viol;
        r.peak = peak;
      }
    }
    r.flag = (eligible ? 1u : 0u) | (overflow ? 2u : 0u);
    return r;
  };

  // ---- head ring (warp 1 loads 32-head blocks ahead of use) ----
  int64_t nx_start = pos0, nx_n = 0;
  uint32_t nx_idx = 0;
  int32_t nx_agent = 0;
  int64_t nx_prompt = 0, nx_kept = 0;
  uint64_t nx_uid = 0;
  double nx_T = 0.0;
  int stage = 0;
  int64_t loaded_end = pos0;
  auto issue_idx = [&](int64_t start) {
    nx_start = start;
    nx_n = q_end - start < kWHB ? q_end - start : kWHB;
    if (nx_n < 0) nx_n = 0;
    nx_idx = lane < nx_n ? hp[start + lane] : 0u;
    stage = 0;
  };
  auto issue_fields = [&]() {
    if (lane < nx_n) {
      nx_agent = q.agent[nx_idx];
      nx_prompt = q.prompt[nx_idx];
      nx_kept = q.kept[nx_idx];
      nx_uid = q.uid[nx_idx];
      if (dp.oracle_T) nx_T = q.pure_exec[nx_idx];
    }
    stage = 1;
  };
  auto issue_T = [&]() {
    if (!dp.oracle_T && lane < nx_n) nx_T = ag.T[nx_agent];
    stage = 2;
  };
  auto land_block = [&]() {
    if (stage < 1) issue_fields();
    if (stage < 2) issue_T();
    const int half = static_cast<int>(((nx_start - pos0) / kWHB) & 1);
    const int hb = half * kWHB;
    const int n = static_cast<int>(nx_n);
    if (lane < n) {
      const int hs = hb + lane;
      h_idx[hs] = nx_idx;
      h_agent[hs] = nx_agent;
      h_prompt[hs] = nx_prompt;
      h_kept[hs] = nx_kept;
      h_uid[hs] = nx_uid;
      h_T[hs] = nx_T;
      int64_t f, l;
      span_bounds_dev(now, nx_T, L, &f, &l);
      h_first[hs] = f;
      h_last[hs] = l;
      bool fast = nx_T > 0.0 && nx_prompt >= 0 && f == cslot && l >= f && l - f + 1 <= kDtSlots;
      if (fast) {
        const double te = __dadd_rn(now, nx_T);
        const double tee = __dsub_rn(te, kTimeEpsilon);
        const double m0 = slot_dt(now, t0e, te, tee, f - 2, L);
        const double m1 = slot_dt(now, t0e, te, tee, f - 1, L);
        const double m2 = slot_dt(now, t0e, te, tee, l + 1, L);
        const double m3 = slot_dt(now, t0e, te, tee, l + 2, L);
        fast = m0 != m0 && m1 != m1 && m2 != m2 && m3 != m3;
      }
      h_mode[hs] = fast ? (k_uniform ? kModeTabPk : kModeTabDt) : kModeGeneric;
    }
    __syncwarp();
    for (int hh = 0; hh < n; ++hh) {
      const int hs = hb + hh;
      const int mode = h_mode[hs];
      if (mode == kModeGeneric) continue;
      const double Th = h_T[hs];
      const double Ph = static_cast<double>(h_prompt[hs]);
      const double te = __dadd_rn(now, Th);
      const double tee = __dsub_rn(te, kTimeEpsilon);
      const int tn = static_cast<int>(h_last[hs] - h_first[hs] + 1);
      for (int j = lane; j < tn; j += 32) {
        const double dt = slot_dt(now, t0e, te, tee, cslot + j, L);
        stab[hs * kDtSlots + j] = mode == kModeTabPk ? pk_of(Ph, k0, dt) : dt;
      }
    }
    __syncwarp();
    loaded_end = nx_start + nx_n;
    issue_idx(loaded_end);
  };
  // Write staged decision records of buffer `buf` (one warp): decision log
  // rows + candidate peaks (engine.cpp:242-246, dispatcher.cpp:143-147),
  // admitted flags and active_ entries (dispatcher.cpp:78).
  auto flush = [&](int buf) {
    const int n = s_nstage[buf];
    const int64_t row0 = s_row0[buf];
    for (int r = 0; r < n; ++r) {
      const int g = buf * kStage + r;
      const StageMeta m = g_meta[g];
      const int64_t row = row0 + r;
      if (row < dp.log_cap) {
        const int64_t ro = int64_t(pool) * dp.log_cap + row;
        const StageRow w = g_row[g * 32 + lane];
        const uint64_t wpeak = __shfl_sync(0xffffffffu, static_cast<unsigned long long>(w.peak), m.target >= 0 ? m.target : 0);
        if (lane == 0) {
          kx_decision d;
          d.time = now;
          d.predicted_peak = m.target >= 0 ? from_ordered_bits(wpeak) : 0.0;
          d.uid = h_uid[m.hs];
          d.queue_index = h_idx[m.hs];
          d.agent = h_agent[m.hs];
          d.target = m.target >= 0 ? s_ids[m.target] : -1;
          d.pool = pool;
          d.admitted = m.admitted;
          rows[ro] = d;
        }
        if (act) {
          double c = -1.0;
          if (w.flag & 1u)
            c = w.viol == kNone ? from_ordered_bits(w.peak)
                                : __dsub_rn(-static_cast<double>(B + static_cast<int64_t>(w.viol)), 1.0);
          cand[ro * dp.peak_stride + li] = c;
        }
      }
      if (m.admitted && lane == m.target) {
        q.admitted[h_idx[m.hs]] = 1;
        if (m.act_slot >= 0) {
          const int64_t o = int64_t(i) * kActiveCap + m.act_slot;
          in.act_uid[o] = h_uid[m.hs];
          in.act_P[o] = static_cast<double>(h_prompt[m.hs]);
          in.act_k[o] = kr;
          in.act_t0[o] = now;
          in.act_T[o] = h_T[m.hs];
        }
      }
    }
  };

  // ---- phase 3: the prefix collected by key generation, sorted here ----
  if (ph.phase == 3) {
    pool_n = ph.pool_counts[pool];
    const uint32_t on = ph.spec_on[pool], cnt = ph.spec_count[pool];
    const bool ok = on && cnt > 0 && cnt <= uint32_t(kTopKMax) &&
                    sort_prefix(q, ph.pad, ph.cand + int64_t(pool) * kTopKMax,
                                ph.cand_key + int64_t(pool) * kTopKMax, static_cast<int>(cnt),
                                ph.heads_out + int64_t(pool) * kTopKMax,
                                reinterpret_cast<uint64_t*>(smem_raw + lay.c_key),
                                reinterpret_cast<uint32_t*>(smem_raw + lay.c_idx));
    q_end = ok ? cnt : 0;
  }
  if (warp == 1) {
    issue_idx(pos0);
    if (pos0 < q_end) land_block();
  }

  // ---- resolver state (warp 0, lane = instance) ----
  double live = act ? in.live_kv[i] : 0.0;
  int32_t running = act ? in.running[i] : 0;
  bool susp = act ? in.suspended[i] != 0 : false;
  int64_t hi = hi0;
  int32_t hi_off = static_cast<int32_t>(hi0 - B);
  int32_t nact = act ? in.n_active[i] : 0;
  uint64_t umax = kZeroBits;  // max stored usage over the whole ledger window
  int64_t pend_last = -1;     // slots [cslot, pend_last] booked since umax was folded
  // Bring umax up to date with the slots booked by this lane's commits.
  auto fold_pending = [&]() {
    if (pend_last >= cslot) {
      int p2 = static_cast<int>(cslot & rmask);
      for (int64_t s2 = cslot; s2 <= pend_last; ++s2) {
        const uint64_t tb = ordered_bits(su[p2 * kRow + lane]);
        umax = tb > umax ? tb : umax;
        p2 = (p2 + 1) & rmask;
      }
      pend_last = -1;
    }
  };
  if (warp == 0) {
    for (int32_t o = lo_off; o <= hi_off; ++o) {
      const int p2 = static_cast<int>((B + o) & rmask);
      if (se[p2 * kRow + lane]) {
        const uint64_t tb = ordered_bits(su[p2 * kRow + lane]);
        umax = tb > umax ? tb : umax;
      }
    }
    st_live[lane] = live;
    st_run[lane] = running;
    st_susp[lane] = susp ? 1 : 0;
    st_hi[lane] = hi_off;
    st_umax[lane] = umax;
  }
  int64_t pos = pos0;
  int64_t nrows = nrows0, nadm = nadm0;
  int retries = 0;
  bool broke = false;
  int status = KX_OK;
  int sbuf = 0;
  __syncthreads();

  while (true) {
    const int64_t b0 = s_next;
    if (s_stop || b0 >= q_end) break;
    const int kb = static_cast<int>(q_end - b0 < kBatchEval ? q_end - b0 : kBatchEval);
    // ---------------- phase A: rows of the batch's heads ----------------
    if (dbg) tA = clock64();
    if (warp >= 1 && warp - 1 < kb) {
      const int j = warp - 1;
      const int hs = static_cast<int>((b0 + j - pos0) & (kHR - 1));
      const Row r = evaluate(hs, st_live[lane], st_run[lane], st_susp[lane] != 0, st_umax[lane], st_hi[lane]);
      r_viol[j * 32 + lane] = r.viol;
      r_peak[j * 32 + lane] = r.peak;
      r_flag[j * 32 + lane] = r.flag;
    }
    batch_sync();
    if (dbg) { const uint32_t dep = *(volatile uint32_t*)&r_flag[0]; const unsigned long long t = clock64() + (dep & 0u); acc_a += t - tA; tA = t; ++nbat; }
    // ---------------- phase B: resolve the batch in order ----------------
    if (warp == 1) {
      // the next batch's heads [b0 + kb, b0 + kb + kBatchEval) must be landed
      const int64_t need_end = b0 + kb + kBatchEval;
      if (loaded_end < q_end && need_end > loaded_end) land_block();
      else if (stage == 0) issue_fields();
      else if (stage == 1) issue_T();
    } else if (warp == kFlushWarp) {
      flush(sbuf ^ 1);  // the previous batch's records
      // keep the instances' active tables in L2 for the end-of-round gc
      // (the concurrent sort streams far more than L2 holds)
      if (act) {
        const int64_t o = int64_t(i) * kActiveCap;
        const int bytes = in.n_active[i] * 8;
        for (int off = 0; off < bytes; off += 128) {
          prefetch_l2_last(reinterpret_cast<const char*>(in.act_uid + o) + off);
          prefetch_l2_last(reinterpret_cast<const char*>(in.act_P + o) + off);
          prefetch_l2_last(reinterpret_cast<const char*>(in.act_k + o) + off);
          prefetch_l2_last(reinterpret_cast<const char*>(in.act_t0 + o) + off);
          prefetch_l2_last(reinterpret_cast<const char*>(in.act_T + o) + off);
        }
      }
    } else if (warp == 0) {
      if (lane == 0) {
        s_nstage[sbuf] = 0;
        s_row0[sbuf] = nrows;
      }
      int ns = 0;
      uint32_t dirty = 0;  // lanes changed since the batch's rows were computed
      for (int j = 0; j < kb && !broke; ++j) {
        const int hs = static_cast<int>((b0 + j - pos0) & (kHR - 1));
        uint32_t viol = r_viol[j * 32 + lane];
        uint64_t peak = r_peak[j * 32 + lane];
        uint32_t flg = r_flag[j * 32 + lane];
        const int64_t prompt = h_prompt[hs];
        const double P = static_cast<double>(prompt);
        const int64_t first = h_first[hs];
        const int64_t last = h_last[hs];
        const int mode = h_mode[hs];
        const bool nonempty = last >= first;
        const int32_t fo = static_cast<int32_t>(first - B);
        const int tn = static_cast<int>(last - first + 1);
        const int pbase = static_cast<int>((B + fo) & rmask);
        const double* tab = stab + hs * kDtSlots;
        uint32_t fixm = dirty;
        while (true) {
          // collect_live (engine.cpp:187-202), every iteration: watermark resume
          if (susp && live < wcap) {
            susp = false;
            st_susp[lane] = 0;
          }
          unsigned long long tq0 = dbg ? clock64() : 0;
          if ((fixm >> lane) & 1u) {  // changed lanes re-evaluate themselves
            if (mode == kModeTabPk) {  // the common shape, inline
              const bool el = act && !susp && !(running + waiting >= mb);
              viol = kNone;
              peak = kZeroBits;
              flg = el ? 1u : 0u;
              if (el) {
                if (first < base || last >= base + ring) flg |= 2u;
                // span slots (every span starts at cslot) fold the pending
                // commits into umax on the way; the rest of them after
                // (usage and pk are >= 0: double max orders like the bits)
                const int np = pend_last >= cslot ? static_cast<int>(pend_last - cslot + 1) : 0;
                double um = __longlong_as_double(static_cast<long long>(umax & ~kZeroBits));
                double pk_max = 0.0;
                int p2 = pbase;
#pragma unroll 4
                for (int jj = 0; jj < tn; ++jj) {
                  const double u = su[p2 * kRow + lane];
                  const double total = __dadd_rn(u, tab[jj]);
                  if (total > cap && viol == kNone) viol = static_cast<uint32_t>(fo + jj);
                  pk_max = fmax(pk_max, total);
                  if (jj < np) um = fmax(um, u);
                  p2 = (p2 + 1) & rmask;
                }
                for (int jj = tn; jj < np; ++jj) {
                  um = fmax(um, su[p2 * kRow + lane]);
                  p2 = (p2 + 1) & rmask;
                }
                umax = static_cast<uint64_t>(__double_as_longlong(um)) | kZeroBits;
                pend_last = -1;
                peak = static_cast<uint64_t>(__double_as_longlong(fmax(um, pk_max))) | kZeroBits;
              }
            } else {
              fold_pending();
              const Row r = evaluate(hs, live, running, susp, umax, hi_off);
              viol = r.viol;
              peak = r.peak;
              flg = r.flag;
            }
          }
          unsigned long long tq1 = dbg ? clock64() : 0;
          if (dbg) acc_fix += tq1 - tq0;
          const bool fits = (flg & 1u) && viol == kNone;
          // select_instance: min (peak, InstanceId) (H9); lanes are in id order.
          // Min of the high words first (peaks have the top bit set, so 0
          // flags a ring overflow); the low words only on a tie there.
          const uint32_t khi = (flg & 2u) ? 0u : fits ? static_cast<uint32_t>(peak >> 32) : 0xffffffffu;
          const uint32_t ovm = __ballot_sync(0xffffffffu, fits && __dadd_rn(live, P) > cap);  // engine.cpp:254-258
          const uint32_t fullm = __ballot_sync(0xffffffffu, nact >= kActiveCap);
          const uint32_t hmin = __reduce_min_sync(0xffffffffu, khi);
          if (hmin == 0u) {
            status = KX_ERR_CAPACITY;
            broke = true;
            break;
          }
          uint32_t winners = __ballot_sync(0xffffffffu, fits && khi == hmin);
          if (winners & (winners - 1)) {
            const uint32_t klo = ((winners >> lane) & 1u) ? static_cast<uint32_t>(peak) : 0xffffffffu;
            const uint32_t lmin = __reduce_min_sync(0xffffffffu, klo);
            winners = __ballot_sync(0xffffffffu, ((winners >> lane) & 1u) && static_cast<uint32_t>(peak) == lmin);
          }
          const int bl = winners ? __ffs(winners) - 1 : -1;
          const bool overload = bl >= 0 && ((ovm >> bl) & 1u);
          unsigned long long tq2 = dbg ? clock64() + (bl & 0) : 0;
          if (dbg) acc_sel += tq2 - tq1;
          // stage the decision record (flushed by another warp later)
          if (ns == kStage) {  // buffer full: write it out here
            if (lane == 0) s_nstage[sbuf] = ns;
            __syncwarp();
            flush(sbuf);
            if (lane == 0) s_row0[sbuf] = nrows;
            ns = 0;
          }
          {
            const int g = sbuf * kStage + ns;
            if (lane == 0) g_meta[g] = StageMeta{hs, bl, (bl >= 0 && !overload) ? 1 : 0, -1};
            g_row[g * 32 + lane] = StageRow{viol, flg, peak};
          }
          unsigned long long tq3 = dbg ? clock64() : 0;
          if (dbg) acc_stg += tq3 - tq2;
          ++ns;
          ++nrows;
          if (bl < 0) {  // head keeps its place (engine.cpp:247)
            broke = true;
            break;
          }
          if (overload) {
            if (lane == bl) {  // Dispatcher::on_overload
              susp = true;
              st_susp[lane] = 1;
            }
            if (++retries > ni) {
              status = KX_ERR_LIVELOCK;
              broke = true;
              break;
            }
            dirty |= 1u << bl;
            fixm = 1u << bl;
            continue;
          }
          retries = 0;
          // Dispatcher::commit, in the target's own lane: book the span
          // slots, raise its maximum stored usage, admit (engine.cpp:298-319).
          const double T = h_T[hs];
          if (mode == kModeTabPk && tn <= 32) {
            // the common shape: lanes = span slots, one pass; the target
            // folds the booked slots into its maximum stored usage when it
            // next needs it (pend_last)
            if (lane < tn) {
              const int p2 = (pbase + lane) & rmask;
              su[p2 * kRow + bl] = __dadd_rn(su[p2 * kRow + bl], tab[lane]);
              se[p2 * kRow + bl] = 1;
            }
            if (lane == bl) pend_last = last > pend_last ? last : pend_last;
            __syncwarp();  // the target's lane reads these slots next
          } else if (lane == bl) {
            if (mode != kModeGeneric) {  // usage + pk >= 0: raw bits order
              int p2 = static_cast<int>(first & rmask);
#pragma unroll 4
              for (int s = 0; s < tn; ++s) {
                const double pk = mode == kModeTabPk ? tab[s] : pk_of(P, kr, tab[s]);
                const double nu = __dadd_rn(su[p2 * kRow + lane], pk);
                su[p2 * kRow + lane] = nu;
                se[p2 * kRow + lane] = 1;
                const uint64_t tb = static_cast<uint64_t>(__double_as_longlong(nu)) | kZeroBits;
                umax = tb > umax ? tb : umax;
                p2 = (p2 + 1) & rmask;
              }
            } else {
              const double te = __dadd_rn(now, T);
              const double tee = __dsub_rn(te, kTimeEpsilon);
              for (int64_t s = first; s <= last; ++s) {
                const int p2 = static_cast<int>(s & rmask);
                const double nu = __dadd_rn(su[p2 * kRow + lane], pk_of(P, kr, slot_dt(now, t0e, te, tee, s, L)));
                su[p2 * kRow + lane] = nu;
                se[p2 * kRow + lane] = 1;
                const uint64_t tb = ordered_bits(nu);
                umax = tb > umax ? tb : umax;
              }
            }
          }
          if (lane == bl) {
            if (nonempty && last > hi) {
              hi = last;
              hi_off = static_cast<int32_t>(last - B);
            }
            live = __dadd_rn(live, static_cast<double>(prompt + h_kept[hs]));
            running += 1;
            st_live[lane] = live;
            st_run[lane] = running;
            st_hi[lane] = hi_off;
            if (nact < kActiveCap) {  // active_[uid] = m (dispatcher.cpp:78), written at flush
              g_meta[sbuf * kStage + ns - 1].act_slot = nact;
              ++nact;
            }
          }
          if ((fullm >> bl) & 1u) {  // the target's active table was full
            status = KX_ERR_CAPACITY;
            broke = true;
            break;
          }
          if (dbg) acc_com += clock64() - tq3;
          dirty |= 1u << bl;
          ++nadm;
          ++pos;
          break;
        }
      }
      fold_pending();
      st_umax[lane] = umax;  // the next batch's evaluators read it
      if (lane == 0) {
        s_nstage[sbuf] = ns;
        s_next = pos;
        s_stop = broke ? 1 : 0;
      }
    }
    if (dbg) acc_b += clock64() - tA;
    batch_sync();
    sbuf ^= 1;
  }
  if (dbg) g_disp_dbg[2] = gtimer();

  if (warp == 0) {
    __syncwarp();
    flush(sbuf ^ 1);  // the last batch's records
    if (dbg) g_disp_dbg[13] = gtimer();
    // Phase 1 ran out of prefix heads without finishing the round: hand the
    // state to the continuation (no gc yet: the round is not over).
    const bool defer_rest = (ph.phase == 1 || ph.phase == 3) && !broke && status == KX_OK && pos >= q_end &&
                            q_end < pool_n;
    int64_t nbase = base;
    if (!defer_rest) {
      // Dispatcher::gc (engine.cpp:212): slots below the current one, elapsed models.
      if (act && cslot > base) {
        const int64_t stop = cslot < base + ring ? cslot : base + ring;
        for (int64_t s = base; s < stop; ++s) {
          const int p2 = static_cast<int>(s & rmask);
          su[p2 * kRow + lane] = 0.0;
          se[p2 * kRow + lane] = 0;
        }
        nbase = cslot;
      }
    }
    if (act) {
      in.n_active[i] = nact;
      if (dbg) g_disp_dbg[14] = gtimer();
      if (dbg) g_disp_dbg[14] = gtimer();
      if (!defer_rest) active_gc(in, i, now);
      if (dbg) g_disp_dbg[15] = gtimer();
      if (dbg) g_disp_dbg[15] = gtimer();
      in.live_kv[i] = live;
      in.base_slot[i] = nbase;
      in.hi_slot[i] = hi;
      in.running[i] = running;
      in.suspended[i] = susp ? 1 : 0;
    }
    {
      const uint64_t hm = warp_max_u64(static_cast<uint64_t>(act ? hi : INT64_MIN) ^ 0x8000000000000000ull);
      if (lane == 0) s_win[2] = static_cast<int64_t>(hm ^ 0x8000000000000000ull);
    }
    if (lane == 0) {
      if (ph.resume) ph.resume[pool] = DispResume{pos, nrows, nadm, defer_rest ? 1 : 0, 0};
      if (!defer_rest) {
        row_count[pool] = nrows;
        admitted_count[pool] = nadm;
        pool_status[pool] = status;
      }
    }
  }
  if (dbg) { g_disp_dbg[3] = gtimer(); g_disp_dbg[5] = nrows; g_disp_dbg[6] = acc_a; g_disp_dbg[7] = acc_b; g_disp_dbg[11] = nbat; g_disp_dbg[8] = acc_fix; g_disp_dbg[9] = acc_sel; g_disp_dbg[10] = acc_stg; g_disp_dbg[12] = acc_com; }
  __syncthreads();
  {
    // write back the window (booked slots only grow hi; gc only clears inside it)
    const int64_t top = s_win[2] > wtop ? s_win[2] : wtop;
    const int wn = top < wB ? 0 : static_cast<int>(top - wB + 1 < ring ? top - wB + 1 : ring);
    for (int e = threadIdx.x; e < wn * 32; e += kBatchThreads) {
      const int l = e & 31;
      const int lj = s_li[l];
      if (lj < 0) continue;
      const int p2 = static_cast<int>((wB + (e >> 5)) & rmask);
      in.usage[int64_t(ib + lj) * ring + p2] = su[p2 * kRow + l];
      in.exists[int64_t(ib + lj) * ring + p2] = se[p2 * kRow + l];
    }
  }
  if (dbg) g_disp_dbg[4] = gtimer();
}

// ---- single-instance ledger events (host-driven, tiny launches) ----------
__global__ void k_ledger_try_place(InstDev in, int i, int ring, double P, double k, double t0,
                                   double T, double slot_len, double* out_peak, int64_t* out_viol,
                                   int* out_state) {
  bool overflow = false;
  const Eval e = warp_try_place(global_ring(in, i, ring), ring, in.cap[i], P, k,
                                make_span(t0, T, slot_len), slot_len, &overflow);
  if (threadIdx.x == 0) {
    *out_peak = e.peak;
    *out_viol = e.viol;
    *out_state = overflow ? -1 : e.state;
  }
}

// SlotLedger::commit (dispatcher.cpp:70-79): re-check, then book.
__device__ bool warp_commit_checked(InstDev& in, int i, int ring, uint64_t uid, double P, double k,
                                    double t0, double T, double slot_len, int* status) {
  bool overflow = false;
  Ring r = global_ring(in, i, ring);
  const Span sp = make_span(t0, T, slot_len);
  const Eval e = warp_try_place(r, ring, in.cap[i], P, k, sp, slot_len, &overflow);
  if (overflow) {
    if ((threadIdx.x & 31) == 0) *status = KX_ERR_CAPACITY;
    return false;
  }
  if (e.state != kFits) return false;
  warp_commit(r, ring, P, k, sp, slot_len);
  if ((threadIdx.x & 31) == 0) {
    in.hi_slot[i] = r.hi;
    active_append(in, i, uid, P, k, t0, T, status);
  }
  __syncwarp();
  return true;
}

__global__ void k_ledger_commit(InstDev in, int i, int ring, uint64_t uid, double P, double k,
                                double t0, double T, double slot_len, int* status) {
  __shared__ int st;
  if (threadIdx.x == 0) st = KX_OK;
  __syncwarp();
  const bool ok = warp_commit_checked(in, i, ring, uid, P, k, t0, T, slot_len, &st);
  if (threadIdx.x == 0) *status = (st == KX_OK && !ok) ? KX_ERR_LOGIC : st;
}

// Batched commits: one warp per instance walks its entries in order.
__global__ void k_ledger_commit_batch(InstDev in, int n_inst, int ring, const int64_t* __restrict__ off,
                                      const int64_t* __restrict__ order, const uint64_t* __restrict__ uid,
                                      const double* __restrict__ P, const double* __restrict__ k,
                                      const double* __restrict__ t0, const double* __restrict__ T,
                                      double slot_len, uint8_t* __restrict__ fits, int* status) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n_inst) return;
  const int lane = threadIdx.x & 31;
  for (int64_t e = off[i]; e < off[i + 1]; ++e) {
    const int64_t j = order[e];
    const bool ok = warp_commit_checked(in, i, ring, uid[j], P[j], k[j], t0[j], T[j], slot_len, status);
    if (lane == 0) fits[j] = ok ? 1 : 0;
    __syncwarp();
  }
}

// SlotLedger::correct_early_finish (dispatcher.cpp:81-99); no-op when the
// uid is not active (Dispatcher::on_request_finished checks has_request).
__global__ void k_ledger_finish(InstDev in, int i, int ring, uint64_t uid, double actual_end,
                                double slot_len) {
  if (threadIdx.x != 0) return;
  const int a = in.n_active[i];
  const int64_t o = int64_t(i) * kActiveCap;
  int j = 0;
  for (; j < a; ++j)
    if (in.act_uid[o + j] == uid) break;
  if (j == a) return;
  const double P = in.act_P[o + j], k = in.act_k[o + j], t0 = in.act_t0[o + j], T = in.act_T[o + j];
  const double t_end = __dadd_rn(t0, T);
  if (actual_end >= __dsub_rn(t_end, kTimeEpsilon)) return;  // finished on schedule
  const double from = actual_end > t0 ? actual_end : t0;     // std::max(actual_end, t_start)
  const int64_t cutoff = static_cast<int64_t>(floor(__ddiv_rn(__dadd_rn(from, kTimeEpsilon), slot_len)));
  int64_t first, last;
  span_bounds_dev(t0, T, slot_len, &first, &last);
  double* usage = in.usage + int64_t(i) * ring;
  const uint8_t* ex = in.exists + int64_t(i) * ring;
  const int64_t base = in.base_slot[i];
  for (int64_t s = first; s <= last; ++s) {
    if (s <= cutoff) continue;
    const uint32_t pos = static_cast<uint32_t>(s) & (ring - 1);
    if (s < base || s >= base + ring || !ex[pos]) continue;  // usage_.find == end
    double v = __dsub_rn(usage[pos], peak_in_slot_dev(P, k, t0, t_end, s, slot_len));
    if (v < 1e-9) v = 0.0;  // cancel rounding residue
    usage[pos] = v;
  }
  in.act_T[o + j] = __dsub_rn(from, t0);  // truncate the stored model
}

__global__ void k_on_overload(InstDev in, int i) {
  if (threadIdx.x == 0) in.suspended[i] = 1;
}

__global__ void k_on_live_usage(InstDev in, int i, double live_kv, double watermark) {
  if (threadIdx.x == 0 && in.suspended[i] && live_kv < __dmul_rn(watermark, in.cap[i]))
    in.suspended[i] = 0;
}

__global__ void k_gc_all(InstDev in, int n_inst, int ring, double now, double slot_len) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n_inst) return;
  Ring r = global_ring(in, i, ring);
  warp_gc_slots(r, ring, now, slot_len);
  if ((threadIdx.x & 31) == 0) {
    in.base_slot[i] = r.base;
    active_gc(in, i, now);
  }
}

// ---- K5w: round_robin / static_threshold round with waiting lists --------
// One warp per pool walks the pool's order: Dispatcher::choose for RR
// (dispatcher.cpp:214-218) or StaticThreshold (219-231), the head popped into
// the target's waiting list (engine.cpp:259-262) and try_admit on it
// (engine.cpp:270-296); after the walk try_admit on every instance
// (engine.cpp:211) and Dispatcher::gc. Lane-parallel parts: the collect_live
// resume over instances, the static probe (a warp min over probe offsets),
// the waiting-list arg-min and the erase shift. try_admit keeps each list's
// arg-min position cached between a memory-blocked check and the next
// change of the list (a push compares against it; an erase drops it).
namespace {

struct WKey {
  double k0, k1, k2;
  uint64_t msg, uid;
};

__device__ __forceinline__ WKey wait_key(const WaitRec& r, const AgentsDev& a, const WaitDev& w) {
  WKey k;
  k.k2 = 0.0;
  switch (w.sched_kind) {  // SchedulerPolicy::order_key (scheduler.hpp:48-113)
    case KX_SCHED_KAIROS: k.k0 = a.pk[r.agent]; k.k1 = r.app_start; k.k2 = r.queue_enter; break;
    case KX_SCHED_FCFS: k.k0 = r.queue_enter; k.k1 = r.app_start; break;
    case KX_SCHED_TOPO: k.k0 = static_cast<double>(a.depth[r.agent]); k.k1 = r.queue_enter; break;
    default: {  // OracleScheduler: remaining_by_uid lookup, absent -> 0.0 (scheduler.hpp:85-89)
      double rem = 0.0;
      if (w.rem_table && r.uid >= w.rem_base && r.uid - w.rem_base < static_cast<uint64_t>(w.rem_n) &&
          w.rem_present[r.uid - w.rem_base])
        rem = w.rem_table[r.uid - w.rem_base];
      k.k0 = rem;
      k.k1 = r.queue_enter;
    }
  }
  k.msg = r.msg;
  k.uid = r.uid;
  return k;
}

// try_admit's comparator: std::tie(order_key, msg_id, uid) < (engine.cpp:280-283).
__device__ __forceinline__ bool wkey_less(const WKey& a, const WKey& b) {
  if (a.k0 != b.k0) return a.k0 < b.k0;
  if (a.k1 != b.k1) return a.k1 < b.k1;
  if (a.k2 != b.k2) return a.k2 < b.k2;
  if (a.msg != b.msg) return a.msg < b.msg;
  return a.uid < b.uid;
}

}  // namespace

__global__ void __launch_bounds__(32)
k_dispatch_waiting(QueueDev q, AgentsDev a, InstDev in, const int32_t* __restrict__ pool_begin,
                   const uint32_t* __restrict__ perm, const int64_t* __restrict__ pool_offsets,
                   DispatchParams dp, WaitDev w, kx_decision* __restrict__ rows,
                   int64_t* __restrict__ row_count, int64_t* __restrict__ admitted_count,
                   int* __restrict__ pool_status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int pool = blockIdx.x;
  const int lane = threadIdx.x;
  const int ib = pool_begin[pool];
  const int ni = pool_begin[pool + 1] - ib;
  double* s_live = reinterpret_cast<double*>(smem_raw);
  double* s_cap = s_live + ni;
  int32_t* s_run = reinterpret_cast<int32_t*>(s_cap + ni);
  int32_t* s_wait = s_run + ni;
  int32_t* s_mb = s_wait + ni;
  int32_t* s_id = s_mb + ni;
  int64_t* s_wmin = reinterpret_cast<int64_t*>(smem_raw + ((size_t(ni) * 32 + 15) & ~size_t(15)));
  uint8_t* s_susp = reinterpret_cast<uint8_t*>(s_wmin + ni);
  for (int li = lane; li < ni; li += 32) {
    s_live[li] = in.live_kv[ib + li];
    s_cap[li] = in.cap[ib + li];
    s_run[li] = in.running[ib + li];
    s_wait[li] = in.waiting[ib + li];
    s_mb[li] = in.max_batch[ib + li];
    s_id[li] = in.id[ib + li];
    s_susp[li] = in.suspended[ib + li];
    s_wmin[li] = -1;
  }
  __syncwarp();
  const double now = dp.now;
  int64_t rr = in.rr_next[pool];
  int64_t nrows = 0, npop = 0, nadm = 0;
  int status = ni > 0 ? KX_OK : KX_ERR_INVALID;

  // Arg-min of instance li's waiting list under wkey_less (uid is unique, so
  // the minimum is unique: list order never decides).
  auto argmin = [&](int li) -> int64_t {
    const WaitRec* L = w.rec + int64_t(ib + li) * w.cap;
    const int64_t n = s_wait[li];
    int64_t bp = -1;
    WKey bk{};
    for (int64_t j = lane; j < n; j += 32) {
      const WKey k = wait_key(L[j], a, w);
      if (bp < 0 || wkey_less(k, bk)) {
        bk = k;
        bp = j;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      WKey ok;
      ok.k0 = __shfl_xor_sync(0xffffffffu, bk.k0, o);
      ok.k1 = __shfl_xor_sync(0xffffffffu, bk.k1, o);
      ok.k2 = __shfl_xor_sync(0xffffffffu, bk.k2, o);
      ok.msg = __shfl_xor_sync(0xffffffffu, bk.msg, o);
      ok.uid = __shfl_xor_sync(0xffffffffu, bk.uid, o);
      const int64_t op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (op >= 0 && (bp < 0 || wkey_less(ok, bk))) {
        bk = ok;
        bp = op;
      }
    }
    return bp;
  };
  // Simulator::try_admit (engine.cpp:270-296) + admit's live/running update (298-319).
  auto try_admit = [&](int li) {
    WaitRec* L = w.rec + int64_t(ib + li) * w.cap;
    while (s_wait[li] > 0 && s_run[li] < s_mb[li]) {
      int64_t pos = s_wmin[li];
      if (pos < 0) pos = argmin(li);
      const WaitRec h = L[pos];
      if (__dadd_rn(s_live[li], static_cast<double>(h.prompt)) > s_cap[li]) {
        __syncwarp();
        if (lane == 0) s_wmin[li] = pos;  // strict admission order: the head waits for memory
        __syncwarp();
        return;
      }
      const int64_t n = s_wait[li];
      for (int64_t b = pos + 1; b < n; b += 32) {  // erase, keeping list order
        const int64_t j = b + lane;
        WaitRec t;
        if (j < n) t = L[j];
        __syncwarp();
        if (j < n) L[j - 1] = t;
        __syncwarp();
      }
      if (lane == 0) {
        s_wait[li] = static_cast<int32_t>(n - 1);
        s_wmin[li] = -1;
        s_live[li] = __dadd_rn(s_live[li], static_cast<double>(h.prompt + h.kept));
        s_run[li] += 1;
        if (nadm < dp.log_cap) {
          kx_admission r;
          r.time = now;
          r.uid = h.uid;
          r.queue_index = h.round == w.round ? h.qidx : -1;
          r.instance = s_id[li];
          r.pool = pool;
          w.adm[int64_t(pool) * dp.log_cap + nadm] = r;
        }
      }
      ++nadm;
      __syncwarp();
    }
  };

  const int64_t b0 = pool_offsets[pool], e0 = pool_offsets[pool + 1];
  for (int64_t pos = b0; pos < e0 && status == KX_OK; ++pos) {
    const uint32_t idx = perm[pos];
    // collect_live: Dispatcher::on_live_usage per instance (engine.cpp:191)
    for (int li = lane; li < ni; li += 32)
      if (s_susp[li] && s_live[li] < __dmul_rn(dp.watermark, s_cap[li])) s_susp[li] = 0;
    int t = -1;
    if (w.policy == KX_DISPATCH_ROUND_ROBIN) {
      t = static_cast<int>(rr % ni);
      ++rr;
    } else {  // first probe from rr_next_ below the threshold and not batch-full
      int best = INT32_MAX;
      for (int probe = lane; probe < ni; probe += 32) {
        const int i = static_cast<int>((rr + probe) % ni);
        const bool full = s_run[i] + s_wait[i] >= s_mb[i];
        if (s_live[i] < __dmul_rn(w.static_thr, s_cap[i]) && !full) best = probe < best ? probe : best;
      }
      best = __reduce_min_sync(0xffffffffu, best);
      if (best != INT32_MAX) {
        t = static_cast<int>((rr + best) % ni);
        rr = t + 1;
      }
    }
    __syncwarp();
    if (lane == 0 && nrows < dp.log_cap) {  // decision log (engine.cpp:242-246)
      kx_decision d;
      d.time = now;
      d.predicted_peak = 0.0;
      d.uid = q.uid[idx];
      d.queue_index = idx;
      d.agent = q.agent[idx];
      d.target = t >= 0 ? s_id[t] : -1;
      d.pool = pool;
      d.admitted = t >= 0 ? 1 : 0;
      rows[int64_t(pool) * dp.log_cap + nrows] = d;
    }
    ++nrows;
    if (t < 0) break;  // engine.cpp:247
    if (s_wait[t] >= w.cap) {
      status = KX_ERR_CAPACITY;
      break;
    }
    if (lane == 0) {  // ReadyQueue::pop; inst.waiting.push_back (engine.cpp:260-261)
      WaitRec r;
      r.app_start = q.app_start[idx];
      r.queue_enter = q.queue_enter[idx];
      r.msg = q.msg[idx];
      r.uid = q.uid[idx];
      r.prompt = q.prompt[idx];
      r.kept = q.kept[idx];
      r.qidx = idx;
      r.agent = q.agent[idx];
      r.round = w.round;
      WaitRec* L = w.rec + int64_t(ib + t) * w.cap;
      const int64_t n = s_wait[t];
      L[n] = r;
      q.admitted[idx] = 1;
      const int64_t m = s_wmin[t];
      if (m >= 0 && wkey_less(wait_key(r, a, w), wait_key(L[m], a, w))) s_wmin[t] = n;
      s_wait[t] = static_cast<int32_t>(n + 1);
    }
    ++npop;
    __syncwarp();
    try_admit(t);
  }
  if (status == KX_OK)
    for (int li = 0; li < ni; ++li) try_admit(li);  // engine.cpp:211
  // Dispatcher::gc (engine.cpp:212)
  for (int li = 0; li < ni; ++li) {
    Ring r = global_ring(in, ib + li, dp.ring);
    warp_gc_slots(r, dp.ring, now, dp.slot_len);
    if (lane == 0) {
      in.base_slot[ib + li] = r.base;
      active_gc(in, ib + li, now);
    }
  }
  __syncwarp();
  for (int li = lane; li < ni; li += 32) {
    in.live_kv[ib + li] = s_live[li];
    in.running[ib + li] = s_run[li];
    in.waiting[ib + li] = s_wait[li];
    in.suspended[ib + li] = s_susp[li];
  }
  if (lane == 0) {
    // only rr mod n is ever used (RR: ids_[rr % n]; static: (rr + probe) % n)
    in.rr_next[pool] = static_cast<int32_t>(ni > 0 ? rr % ni : 0);
    row_count[pool] = nrows;
    admitted_count[pool] = npop;
    w.adm_count[pool] = nadm;
    pool_status[pool] = status;
  }
}

// ---- host wrappers -------------------------------------------------------
void read_dispatch_debug(unsigned long long* out) {
  KX_CUDA(cudaMemcpyFromSymbol(out, g_disp_dbg, sizeof(unsigned long long) * 16));
}

void configure_dispatch_kernels() {
  cudaFuncAttributes attr;  // load eagerly (see configure_sort_kernels)
  KX_CUDA(cudaFuncGetAttributes(&attr, k_dispatch_batch));
  KX_CUDA(cudaFuncGetAttributes(&attr, k_gc_all));
  KX_CUDA(cudaFuncGetAttributes(&attr, k_dispatch_waiting));
  KX_CUDA(cudaFuncSetAttribute(k_dispatch_batch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kDispSmemLimit));
  KX_CUDA(cudaFuncSetAttribute(k_dispatch_timeslot<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kDispSmemLimit));
  KX_CUDA(cudaFuncSetAttribute(k_dispatch_timeslot<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kDispSmemLimit));
}

bool dispatch_can_overlap(int max_inst_per_pool, int ring) {
  return max_inst_per_pool <= 32 && batch_layout(ring).total <= static_cast<uint32_t>(kDispSmemLimit);
}

void launch_dispatch(const QueueDev& q, const AgentsDev& a, const InstDev& in,
                     const int32_t* pool_begin, const uint32_t* perm, const int64_t* pool_offsets,
                     const DispatchParams& dp, int n_pools, int max_inst_per_pool, kx_decision* rows,
                     double* cand, int64_t* row_count, int64_t* admitted_count, int* pool_status,
                     cudaStream_t st, DispPhase phase) {
  if (max_inst_per_pool <= 32) {
    const BatchLayout bl = batch_layout(dp.ring);
    if (bl.total <= static_cast<uint32_t>(kDispSmemLimit)) {
      k_dispatch_batch<<<n_pools, kBatchThreads, kDispSmemExclusive, st>>>(q, a, in, pool_begin, perm,
                                                                         pool_offsets, dp, bl, rows, cand,
                                                                         row_count, admitted_count,
                                                                         pool_status, phase);
      KX_CHECK_LAUNCH();
      return;
    }
  }
  const DispLayout with_ring = disp_layout(max_inst_per_pool, dp.ring, true);
  if (with_ring.total <= static_cast<uint32_t>(kDispSmemLimit)) {
    k_dispatch_timeslot<true><<<n_pools, kDispThreads, with_ring.total, st>>>(
        q, a, in, pool_begin, perm, pool_offsets, dp, with_ring, rows, cand, row_count,
        admitted_count, pool_status);
  } else {
    const DispLayout no_ring = disp_layout(max_inst_per_pool, dp.ring, false);
    k_dispatch_timeslot<false><<<n_pools, kDispThreads, no_ring.total, st>>>(
        q, a, in, pool_begin, perm, pool_offsets, dp, no_ring, rows, cand, row_count,
        admitted_count, pool_status);
  }
  KX_CHECK_LAUNCH();
}

size_t waiting_smem(int ni) { return ((size_t(ni) * 32 + 15) & ~size_t(15)) + size_t(ni) * 9; }

void launch_dispatch_waiting(const QueueDev& q, const AgentsDev& a, const InstDev& in,
                             const int32_t* pool_begin, const uint32_t* perm,
                             const int64_t* pool_offsets, const DispatchParams& dp, const WaitDev& w,
                             int n_pools, int max_inst_per_pool, kx_decision* rows,
                             int64_t* row_count, int64_t* admitted_count, int* pool_status,
                             cudaStream_t st) {
  k_dispatch_waiting<<<n_pools, 32, waiting_smem(max_inst_per_pool), st>>>(
      q, a, in, pool_begin, perm, pool_offsets, dp, w, rows, row_count, admitted_count, pool_status);
  KX_CHECK_LAUNCH();
}

void launch_ledger_try_place(const InstDev& in, int i, int ring, double P, double k, double t0,
                             double T, double slot_len, double* out_peak, int64_t* out_viol,
                             int* out_state, cudaStream_t st) {
  k_ledger_try_place<<<1, 32, 0, st>>>(in, i, ring, P, k, t0, T, slot_len, out_peak, out_viol,
                                       out_state);
  KX_CHECK_LAUNCH();
}

void launch_ledger_commit(const InstDev& in, int i, int ring, uint64_t uid, double P, double k,
                          double t0, double T, double slot_len, int* status, cudaStream_t st) {
  k_ledger_commit<<<1, 32, 0, st>>>(in, i, ring, uid, P, k, t0, T, slot_len, status);
  KX_CHECK_LAUNCH();
}

void launch_ledger_commit_batch(const InstDev& in, int n_inst, int ring, const int64_t* off,
                                const int64_t* order, const uint64_t* uid, const double* P,
                                const double* k, const double* t0, const double* T, double slot_len,
                                uint8_t* fits, int* status, cudaStream_t st) {
  const int threads = 128;
  const int blocks = (n_inst * 32 + threads - 1) / threads;
  k_ledger_commit_batch<<<blocks, threads, 0, st>>>(in, n_inst, ring, off, order, uid, P, k, t0, T,
                                                    slot_len, fits, status);
  KX_CHECK_LAUNCH();
}

void launch_ledger_finish(const InstDev& in, int i, int ring, uint64_t uid, double actual_end,
                          double slot_len, cudaStream_t st) {
  k_ledger_finish<<<1, 32, 0, st>>>(in, i, ring, uid, actual_end, slot_len);
  KX_CHECK_LAUNCH();
}

void launch_on_overload(const InstDev& in, int i, cudaStream_t st) {
  k_on_overload<<<1, 32, 0, st>>>(in, i);
  KX_CHECK_LAUNCH();
}

void launch_on_live_usage(const InstDev& in, int i, double live_kv, double watermark,
                          cudaStream_t st) {
  k_on_live_usage<<<1, 32, 0, st>>>(in, i, live_kv, watermark);
  KX_CHECK_LAUNCH();
}

void launch_gc_all(const InstDev& in, int n_inst, int ring, double now, double slot_len,
                   cudaStream_t st) {
  const int threads = 256;
  const int blocks = (n_inst * 32 + threads - 1) / threads;
  if (blocks > 0) k_gc_all<<<blocks, threads, 0, st>>>(in, n_inst, ring, now, slot_len);
  KX_CHECK_LAUNCH();
}

}  // namespace kx

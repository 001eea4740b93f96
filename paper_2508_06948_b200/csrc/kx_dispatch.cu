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
#include <stdint.h>

#include "kx_common.cuh"
#include "kx_dispatch.cuh"
#include "kx_order.cuh"
#include "kx_state.cuh"

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
__device__ void active_gc(InstDev& in, int i, double now) {
  int a = in.n_active[i];
  const int64_t o = int64_t(i) * kActiveCap;
  const double lim = __dadd_rn(now, kTimeEpsilon);
  for (int j = 0; j < a;) {
    if (__dadd_rn(in.act_t0[o + j], in.act_T[o + j]) <= lim) {
      --a;
      in.act_uid[o + j] = in.act_uid[o + a];
      in.act_P[o + j] = in.act_P[o + a];
      in.act_k[o + j] = in.act_k[o + a];
      in.act_t0[o + j] = in.act_t0[o + a];
      in.act_T[o + j] = in.act_T[o + a];
    } else {
      ++j;
    }
  }
  in.n_active[i] = a;
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

// ---- K5 fast path: pools of <= 32 instances ----------------------------------
// Lanes = instances, warps = interleaved slot subsets (warp w owns absolute
// slots s with s % kLaneWarps == w). Every warp keeps an identical register
// copy of each lane-instance's live state (it is updated deterministically),
// evaluates its slot subset for all instances at once, publishes per-instance
// partial (first violating slot, peak) to shared memory, and after the single
// barrier of the decision every warp combines the partials, computes the same
// arg-min (REDUX), and books the target's slots of its own subset. Ledger
// rings are staged transposed (usage[slot][instance]) so a warp's 32 lanes
// read 32 consecutive words.
constexpr int kLaneWarps = 8;
constexpr int kLaneThreads = 32 * kLaneWarps;

struct LaneLayout {
  uint32_t part_viol, part_peak, h_T, h_prompt, h_kept, h_uid, h_agent, h_idx, h_first, h_last,
      h_tend, usage, ex, total;
};

LaneLayout lane_layout(int ring) {
  LaneLayout L{};
  uint32_t o = 0;
  auto take = [&](size_t bytes) {
    const uint32_t at = o;
    o = static_cast<uint32_t>((o + bytes + 15) & ~size_t(15));
    return at;
  };
  L.part_viol = take(4 * 2 * kLaneWarps * 32);
  L.part_peak = take(8 * 2 * kLaneWarps * 32);
  L.h_T = take(8 * kHeadBatch);
  L.h_prompt = take(8 * kHeadBatch);
  L.h_kept = take(8 * kHeadBatch);
  L.h_uid = take(8 * kHeadBatch);
  L.h_agent = take(4 * kHeadBatch);
  L.h_idx = take(4 * kHeadBatch);
  L.h_first = take(8 * kHeadBatch);
  L.h_last = take(8 * kHeadBatch);
  L.h_tend = take(8 * kHeadBatch);
  L.usage = take(size_t(8) * 32 * ring);
  L.ex = take(size_t(32) * ring);
  L.total = o;
  return L;
}

#define SL(type, field) reinterpret_cast<type*>(smem_raw + lay.field)

__global__ void __launch_bounds__(kLaneThreads)
k_dispatch_lanes(QueueDev q, AgentsDev ag, InstDev in, const int32_t* __restrict__ pool_begin,
                 const uint32_t* __restrict__ perm, const int64_t* __restrict__ pool_offsets,
                 DispatchParams dp, LaneLayout lay, kx_decision* __restrict__ rows,
                 double* __restrict__ cand, int64_t* __restrict__ row_count,
                 int64_t* __restrict__ admitted_count, int* __restrict__ pool_status,
                 DispPhase ph) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_status;
  const int pool = blockIdx.x;
  // Head source: the pool's full order (phase 0), its top-K prefix (phase 1,
  // overlapping the full sort), or the full order from where phase 1
  // stopped (phase 2).
  const int64_t pool_n = pool_offsets[pool + 1] - pool_offsets[pool];
  const uint32_t* hp = perm + pool_offsets[pool];
  int64_t q_end = pool_n, pos0 = 0, nrows0 = 0, nadm0 = 0;
  if (ph.phase == 1) {
    const TopKState t = ph.tk[pool];
    if (t.defer) {  // too many ties at the boundary key: wait for the full order
      if (threadIdx.x == 0) ph.resume[pool] = DispResume{0, 0, 0, 1, 0};
      return;
    }
    hp = ph.heads + int64_t(pool) * kTopKMax;
    q_end = t.empty ? 0 : (t.n_cand < kTopKMax ? t.n_cand : kTopKMax);
  } else if (ph.phase == 2) {
    const DispResume r = ph.resume[pool];
    if (!r.need) return;
    pos0 = r.start;
    nrows0 = r.nrows;
    nadm0 = r.nadm;
  }
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ib = pool_begin[pool];
  const int ni = pool_begin[pool + 1] - ib;
  const int ring = dp.ring;
  const double now = dp.now;
  const bool act = lane < ni;
  const int i = ib + (act ? lane : 0);

  // Per-lane instance state (identical copies in every warp).
  const double cap = act ? in.cap[i] : 0.0;
  const double kr = act ? in.decode_rate[i] : 0.0;
  const int32_t mb = act ? in.max_batch[i] : 0;
  const int32_t id = act ? in.id[i] : 0x7fffffff;
  const int32_t waiting = act ? in.waiting[i] : 0;
  double live = act ? in.live_kv[i] : 0.0;
  int32_t running = act ? in.running[i] : 0;
  bool susp = act ? in.suspended[i] != 0 : false;
  int64_t base = act ? in.base_slot[i] : 0;
  int64_t hi = act ? in.hi_slot[i] : -1;
  int32_t nact = act ? in.n_active[i] : 0;  // active_ size, kept in a register
  // Common slot origin of the pool (bases are equal after any gc; the
  // per-lane base still bounds what each instance retains).
  const int64_t B = static_cast<int64_t>(warp_min_u64(act ? static_cast<uint64_t>(base) : ~0ull));

  // Stage the rings transposed: usage[pos][lane].
  double* su = SL(double, usage);
  uint8_t* se = SL(uint8_t, ex);
  for (int j = threadIdx.x; j < 32 * ring; j += kLaneThreads) {
    const int li = j % 32, pos = j / 32;
    const bool a = li < ni;
    su[j] = a ? in.usage[int64_t(ib + li) * ring + pos] : 0.0;
    se[j] = a ? in.exists[int64_t(ib + li) * ring + pos] : 0;
  }
  if (threadIdx.x == 0) s_status = KX_OK;
  __syncthreads();

  int64_t pos = pos0;
  int64_t hb_start = pos, hb_n = 0;
  int64_t nrows = nrows0, nadm = nadm0;
  int retries = 0;
  int par = 0;
  bool broke = false;
  const double t0e = __dadd_rn(now, kTimeEpsilon);
  uint32_t* pv = SL(uint32_t, part_viol);
  uint64_t* pp = SL(uint64_t, part_peak);

  while (pos < q_end) {
    if (pos >= hb_start + hb_n) {  // refill the head batch (prefix of the pool's order)
      __syncthreads();
      hb_start = pos;
      hb_n = q_end - pos < kHeadBatch ? q_end - pos : kHeadBatch;
      if (threadIdx.x < hb_n) {
        const int t = threadIdx.x;
        const uint32_t idx = hp[pos + t];
        const int32_t a = q.agent[idx];
        const double T = dp.oracle_T ? q.pure_exec[idx] : ag.T[a];
        SL(uint32_t, h_idx)[t] = idx;
        SL(int32_t, h_agent)[t] = a;
        SL(int64_t, h_prompt)[t] = q.prompt[idx];
        SL(int64_t, h_kept)[t] = q.kept[idx];
        SL(uint64_t, h_uid)[t] = q.uid[idx];
        SL(double, h_T)[t] = T;
        int64_t f, l;
        span_bounds_dev(now, T, dp.slot_len, &f, &l);
        SL(int64_t, h_first)[t] = f;
        SL(int64_t, h_last)[t] = l;
        SL(double, h_tend)[t] = __dadd_rn(now, T);
      }
      __syncthreads();
    }
    const int h = static_cast<int>(pos - hb_start);
    const int64_t prompt = SL(int64_t, h_prompt)[h];
    const double P = static_cast<double>(prompt);
    Span sp;
    sp.first = SL(int64_t, h_first)[h];
    sp.last = SL(int64_t, h_last)[h];
    sp.t0 = now;
    sp.t_end = SL(double, h_tend)[h];
    sp.t0e = t0e;
    sp.tee = __dsub_rn(sp.t_end, kTimeEpsilon);
    const bool nonempty = sp.last >= sp.first;

    // collect_live (engine.cpp:187-202): watermark resume, batch_full.
    if (susp && live < __dmul_rn(dp.watermark, cap)) susp = false;
    const bool full = running + waiting >= mb;
    const bool eligible = act && !susp && !full;
    const bool overflow = eligible && nonempty && (sp.first < base || sp.last >= base + ring);

    // Partial try_place over this warp's slots s_m = B + warp + kLaneWarps*m.
    // The instance-independent part of peak_in_slot (the in-slot test and
    // dt = eval_t - t0, dispatcher.cpp:34-41) is computed once per slot by
    // lane m and broadcast; each lane then adds its instance's P + k*dt.
    uint32_t viol = 0xffffffffu;
    uint64_t peak = 0;  // raw bits: totals are non-negative (prompt >= 0, k > 0)
    {
      // 32-bit slot offsets from the pool origin B (the ring spans < 2^31).
      const int32_t lo_off = static_cast<int32_t>(base - B);
      const int32_t first_off = static_cast<int32_t>(sp.first - B);
      const int32_t last_off = static_cast<int32_t>(sp.last - B);
      const int32_t my_top = eligible ? static_cast<int32_t>((hi > sp.last ? hi : sp.last) - B) : -1;
      const int32_t top = static_cast<int32_t>(__reduce_max_sync(0xffffffffu, static_cast<uint32_t>(my_top + 1))) - 1;
      const int32_t nslots = top >= warp ? (top - warp) / kLaneWarps + 1 : 0;
      for (int32_t m0 = 0; m0 < nslots; m0 += 32) {
        // lane j describes slot offset o_j = warp + kLaneWarps * (m0 + j)
        const int32_t oj = warp + kLaneWarps * (m0 + lane);
        const double slot_start = __dmul_rn(static_cast<double>(B + oj), dp.slot_len);
        const double slot_end = __dadd_rn(slot_start, dp.slot_len);
        const bool zero = slot_end <= sp.t0e || slot_start >= sp.tee;
        const double eval_t = (sp.t_end < slot_end) ? sp.t_end : slot_end;
        const double dtj = zero ? -1.0 : __dsub_rn(eval_t, sp.t0);  // dt >= 0 when not zero
        const int cnt = nslots - m0 < 32 ? nslots - m0 : 32;
#pragma unroll 4
        for (int j = 0; j < cnt; ++j) {
          const double dt = __shfl_sync(0xffffffffu, dtj, j);  // all lanes take part
          const int32_t o = warp + kLaneWarps * (m0 + j);
          if (!eligible || o < lo_off) continue;
          const int p2 = static_cast<int>((B + o) & (ring - 1));
          const bool in_span = o >= first_off && o <= last_off;
          const bool exists = se[p2 * 32 + lane] != 0;
          if (!(in_span || exists)) continue;
          const double used = exists ? su[p2 * 32 + lane] : 0.0;
          const double pk = dt < 0.0 ? 0.0 : __dadd_rn(P, __dmul_rn(kr, dt));
          const double total = __dadd_rn(used, pk);
          if (in_span && total > cap) viol = static_cast<uint32_t>(o) < viol ? static_cast<uint32_t>(o) : viol;
          const uint64_t tb = static_cast<uint64_t>(__double_as_longlong(total));
          peak = tb > peak ? tb : peak;
        }
      }
    }
    pv[(par * kLaneWarps + warp) * 32 + lane] = viol;
    pp[(par * kLaneWarps + warp) * 32 + lane] = peak;
    if (overflow) atomicExch(&s_status, KX_ERR_CAPACITY);
    __syncthreads();
    if (s_status != KX_OK) {
      broke = true;
      break;
    }

    // Combine the partials of all warps for this lane's instance.
#pragma unroll
    for (int w = 0; w < kLaneWarps; ++w) {
      if (w == warp) continue;
      const uint32_t v2 = pv[(par * kLaneWarps + w) * 32 + lane];
      const uint64_t p2 = pp[(par * kLaneWarps + w) * 32 + lane];
      viol = v2 < viol ? v2 : viol;
      peak = p2 > peak ? p2 : peak;
    }
    const bool fits = eligible && viol == 0xffffffffu;
    // select_instance: min (peak, InstanceId) (H9), all warps identically.
    const uint64_t key = fits ? peak : ~0ull;
    const uint64_t wkey = warp_min_u64(key);
    const uint32_t uid_ = static_cast<uint32_t>(id) ^ 0x80000000u;
    const uint32_t wid = __reduce_min_sync(0xffffffffu, (fits && key == wkey) ? uid_ : 0xffffffffu);
    const uint32_t winners = __ballot_sync(0xffffffffu, fits && key == wkey && uid_ == wid);
    const int bl = winners ? __ffs(winners) - 1 : -1;
    const double bpeak = bl >= 0 ? __longlong_as_double(static_cast<long long>(wkey)) : 0.0;
    const double blive = __shfl_sync(0xffffffffu, live, bl >= 0 ? bl : 0);
    const double bcap = __shfl_sync(0xffffffffu, cap, bl >= 0 ? bl : 0);
    const bool overload = bl >= 0 && __dadd_rn(blive, P) > bcap;  // engine.cpp:254-258
    const int32_t bid = __shfl_sync(0xffffffffu, id, bl >= 0 ? bl : 0);

    if (warp == 0) {  // decision log (engine.cpp:242-246)
      if (nrows < dp.log_cap) {
        const int64_t r = int64_t(pool) * dp.log_cap + nrows;
        if (lane == 0) {
          kx_decision d;
          d.time = now;
          d.predicted_peak = bpeak;
          d.uid = SL(uint64_t, h_uid)[h];
          d.queue_index = SL(uint32_t, h_idx)[h];
          d.agent = SL(int32_t, h_agent)[h];
          d.target = bl >= 0 ? bid : -1;
          d.pool = pool;
          d.admitted = (bl >= 0 && !overload) ? 1 : 0;
          rows[r] = d;
        }
        if (act) {
          double v = -1.0;
          if (eligible) {
            v = fits ? __longlong_as_double(static_cast<long long>(peak))
                     : __dsub_rn(-static_cast<double>(B + static_cast<int64_t>(viol)), 1.0);
          }
          cand[r * dp.peak_stride + lane] = v;
        }
      }
    }
    ++nrows;
    if (bl < 0) {  // head keeps its place (engine.cpp:247)
      broke = true;
      break;
    }
    if (overload) {
      if (lane == bl) susp = true;  // Dispatcher::on_overload
      if (++retries > ni) {
        if (threadIdx.x == 0) s_status = KX_ERR_LIVELOCK;
        broke = true;
        break;
      }
      par ^= 1;
      continue;
    }
    retries = 0;
    // Dispatcher::commit: each warp books the target's span slots it owns.
    {
      const double kt = __shfl_sync(0xffffffffu, kr, bl);
      const int64_t f0 = sp.first + ((((B + warp) - sp.first) % kLaneWarps) + kLaneWarps) % kLaneWarps;
      for (int64_t s = f0 + int64_t(lane) * kLaneWarps; s <= sp.last; s += 32 * kLaneWarps) {
        const int p2 = static_cast<int>(s & (ring - 1));
        su[p2 * 32 + bl] = __dadd_rn(su[p2 * 32 + bl], pis(sp, P, kt, s, dp.slot_len));
        se[p2 * 32 + bl] = 1;
      }
      if (lane == bl) {
        if (nonempty && sp.last > hi) hi = sp.last;
        live = __dadd_rn(live, static_cast<double>(prompt + SL(int64_t, h_kept)[h]));  // admit
        running += 1;
      }
      if (lane == bl) {
        if (nact < kActiveCap) {
          if (warp == 0) {  // active_[uid] = m (dispatcher.cpp:78): stores only
            q.admitted[SL(uint32_t, h_idx)[h]] = 1;
            const int64_t o = int64_t(i) * kActiveCap + nact;
            in.act_uid[o] = SL(uint64_t, h_uid)[h];
            in.act_P[o] = P;
            in.act_k[o] = kt;
            in.act_t0[o] = now;
            in.act_T[o] = SL(double, h_T)[h];
          }
          ++nact;
        } else if (warp == 0) {
          s_status = KX_ERR_CAPACITY;
        }
      }
    }
    ++nadm;
    ++pos;
    par ^= 1;
  }
  __syncthreads();
  // Phase 1 ran out of prefix heads without finishing the round: hand the
  // state to the continuation (no gc yet: the round is not over).
  const bool defer_rest = ph.phase == 1 && !broke && s_status == KX_OK && pos >= q_end && q_end < pool_n;
  if (!defer_rest) {
    // Dispatcher::gc (engine.cpp:212): slots below the current one, elapsed models.
    const int64_t current =
        static_cast<int64_t>(floor(__ddiv_rn(__dadd_rn(now, kTimeEpsilon), dp.slot_len)));
    if (act && current > base) {
      const int64_t stop = current < base + ring ? current : base + ring;
      for (int64_t s = base + warp; s < stop; s += kLaneWarps) {
        const int p2 = static_cast<int>(s & (ring - 1));
        su[p2 * 32 + lane] = 0.0;
        se[p2 * 32 + lane] = 0;
      }
      base = current;
    }
  }
  if (warp == 0 && act) {
    in.n_active[i] = nact;
    if (!defer_rest) active_gc(in, i, now);
  }
  __syncthreads();
  if (warp == 0 && act) {
    in.live_kv[i] = live;
    in.base_slot[i] = base;
    in.hi_slot[i] = hi;
    in.running[i] = running;
    in.suspended[i] = susp ? 1 : 0;
  }
  for (int j = threadIdx.x; j < 32 * ring; j += kLaneThreads) {
    const int li = j % 32, p2 = j / 32;
    if (li < ni) {
      in.usage[int64_t(ib + li) * ring + p2] = su[j];
      in.exists[int64_t(ib + li) * ring + p2] = se[j];
    }
  }
  if (threadIdx.x == 0) {
    if (ph.resume) ph.resume[pool] = DispResume{pos, nrows, nadm, defer_rest ? 1 : 0, 0};
    if (!defer_rest) {
      row_count[pool] = nrows;
      admitted_count[pool] = nadm;
      pool_status[pool] = s_status;
    }
  }
}

#undef SL

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

// ---- host wrappers -------------------------------------------------------
void configure_dispatch_kernels() {
  KX_CUDA(cudaFuncSetAttribute(k_dispatch_lanes, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kDispSmemLimit));
  KX_CUDA(cudaFuncSetAttribute(k_dispatch_timeslot<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kDispSmemLimit));
  KX_CUDA(cudaFuncSetAttribute(k_dispatch_timeslot<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kDispSmemLimit));
}

bool dispatch_can_overlap(int max_inst_per_pool, int ring) {
  return max_inst_per_pool <= 32 && lane_layout(ring).total <= static_cast<uint32_t>(kDispSmemLimit);
}

void launch_dispatch(const QueueDev& q, const AgentsDev& a, const InstDev& in,
                     const int32_t* pool_begin, const uint32_t* perm, const int64_t* pool_offsets,
                     const DispatchParams& dp, int n_pools, int max_inst_per_pool, kx_decision* rows,
                     double* cand, int64_t* row_count, int64_t* admitted_count, int* pool_status,
                     cudaStream_t st, DispPhase phase) {
  if (max_inst_per_pool <= 32) {
    const LaneLayout ll = lane_layout(dp.ring);
    if (ll.total <= static_cast<uint32_t>(kDispSmemLimit)) {
      k_dispatch_lanes<<<n_pools, kLaneThreads, ll.total, st>>>(q, a, in, pool_begin, perm,
                                                               pool_offsets, dp, ll, rows, cand,
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

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
#include "kx_state.cuh"

namespace kx {

namespace {

constexpr int kDispThreads = 1024;
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

// SlotLedger::try_place (dispatcher.cpp:52-68), one warp: lanes stride the
// retained slots; first violating span slot = warp min, peak = warp max.
__device__ Eval warp_try_place(const Ring& r, int ring, double cap, double P, double k, double t0,
                               double T, double slot_len, bool* overflow) {
  const int lane = threadIdx.x & 31;
  int64_t first, last;
  span_bounds_dev(t0, T, slot_len, &first, &last);
  const double t_end = __dadd_rn(t0, T);
  if (last >= first && (first < r.base || last >= r.base + ring)) *overflow = true;
  const int64_t smax = r.hi > last ? r.hi : last;
  double peak = 0.0;
  int64_t viol = INT64_MAX;
  for (int64_t s = r.base + lane; s <= smax; s += 32) {
    const uint32_t pos = static_cast<uint32_t>(s) & (ring - 1);
    const bool in_span = (s >= first && s <= last);
    const bool exists = r.ex[pos] != 0;
    if (!(in_span || exists)) continue;
    const double used = exists ? r.usage[pos] : 0.0;
    const double total = __dadd_rn(used, peak_in_slot_dev(P, k, t0, t_end, s, slot_len));
    if (in_span && total > cap && s < viol) viol = s;
    peak = fmax(peak, total);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t v2 = __shfl_xor_sync(0xffffffffu, viol, o);
    viol = v2 < viol ? v2 : viol;
    peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, o));
  }
  Eval e;
  e.state = viol != INT64_MAX ? kExceeds : kFits;
  e.peak = peak;
  e.viol = viol;
  return e;
}

// SlotLedger::commit's booking (dispatcher.cpp:75-78), one warp.
__device__ void warp_commit(Ring& r, int ring, double P, double k, double t0, double T,
                            double slot_len) {
  const int lane = threadIdx.x & 31;
  int64_t first, last;
  span_bounds_dev(t0, T, slot_len, &first, &last);
  const double t_end = __dadd_rn(t0, T);
  for (int64_t s = first + lane; s <= last; s += 32) {
    const uint32_t pos = static_cast<uint32_t>(s) & (ring - 1);
    r.usage[pos] = __dadd_rn(r.usage[pos], peak_in_slot_dev(P, k, t0, t_end, s, slot_len));
    r.ex[pos] = 1;
  }
  if (last >= first && last > r.hi) r.hi = last;
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

// Shared-memory layout of the dispatch kernel for a pool of `ni` instances.
struct DispSmem {
  double *live, *cap, *k, *snap, *peak, *h_T;
  int64_t *base, *hi, *viol, *h_prompt, *h_kept;
  uint64_t* h_uid;
  int32_t *run, *wait, *mb, *id, *h_agent;
  uint32_t* h_idx;
  uint8_t *susp, *state;
  double* usage;  // ni * ring (smem-staged rings only)
  uint8_t* ex;
};

__host__ __device__ inline size_t disp_align(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline size_t disp_smem_bytes(int ni, int ring, bool smem_ring, DispSmem* out,
                                                  unsigned char* base) {
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = disp_align(o + bytes);
    return base ? base + at : nullptr;
  };
  DispSmem d;
  d.live = reinterpret_cast<double*>(take(8 * ni));
  d.cap = reinterpret_cast<double*>(take(8 * ni));
  d.k = reinterpret_cast<double*>(take(8 * ni));
  d.snap = reinterpret_cast<double*>(take(8 * 2 * ni));
  d.peak = reinterpret_cast<double*>(take(8 * 2 * ni));
  d.base = reinterpret_cast<int64_t*>(take(8 * ni));
  d.hi = reinterpret_cast<int64_t*>(take(8 * ni));
  d.viol = reinterpret_cast<int64_t*>(take(8 * 2 * ni));
  d.run = reinterpret_cast<int32_t*>(take(4 * ni));
  d.wait = reinterpret_cast<int32_t*>(take(4 * ni));
  d.mb = reinterpret_cast<int32_t*>(take(4 * ni));
  d.id = reinterpret_cast<int32_t*>(take(4 * ni));
  d.susp = take(ni);
  d.state = take(2 * ni);
  d.h_T = reinterpret_cast<double*>(take(8 * kHeadBatch));
  d.h_prompt = reinterpret_cast<int64_t*>(take(8 * kHeadBatch));
  d.h_kept = reinterpret_cast<int64_t*>(take(8 * kHeadBatch));
  d.h_uid = reinterpret_cast<uint64_t*>(take(8 * kHeadBatch));
  d.h_agent = reinterpret_cast<int32_t*>(take(4 * kHeadBatch));
  d.h_idx = reinterpret_cast<uint32_t*>(take(4 * kHeadBatch));
  d.usage = smem_ring ? reinterpret_cast<double*>(take(size_t(8) * ni * ring)) : nullptr;
  d.ex = smem_ring ? take(size_t(ni) * ring) : nullptr;
  if (out) *out = d;
  return o;
}

}  // namespace

template <bool kSmemRing>
__global__ void __launch_bounds__(kDispThreads)
k_dispatch_timeslot(QueueDev q, AgentsDev ag, InstDev in, const int32_t* __restrict__ pool_begin,
                    const uint32_t* __restrict__ perm, const int64_t* __restrict__ pool_offsets,
                    DispatchParams dp, kx_decision* __restrict__ rows, double* __restrict__ cand,
                    int64_t* __restrict__ row_count, int64_t* __restrict__ admitted_count,
                    int* __restrict__ pool_status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_status;
  const int pool = blockIdx.x;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ib = pool_begin[pool];
  const int ni = pool_begin[pool + 1] - ib;
  const int ring = dp.ring;
  const double now = dp.now;
  DispSmem S;
  disp_smem_bytes(ni, ring, kSmemRing, &S, smem_raw);

  // Stage the pool's instance state (and rings) in shared memory.
  for (int li = threadIdx.x; li < ni; li += kDispThreads) {
    const int i = ib + li;
    S.live[li] = in.live_kv[i];
    S.cap[li] = in.cap[i];
    S.k[li] = in.decode_rate[i];
    S.base[li] = in.base_slot[i];
    S.hi[li] = in.hi_slot[i];
    S.run[li] = in.running[i];
    S.wait[li] = in.waiting[i];
    S.mb[li] = in.max_batch[i];
    S.id[li] = in.id[i];
    S.susp[li] = in.suspended[i];
  }
  if (kSmemRing) {
    const int64_t tot = int64_t(ni) * ring;
    const double* gu = in.usage + int64_t(ib) * ring;
    const uint8_t* ge = in.exists + int64_t(ib) * ring;
    for (int64_t j = threadIdx.x; j < tot; j += kDispThreads) {
      S.usage[j] = gu[j];
      S.ex[j] = ge[j];
    }
  }
  if (threadIdx.x == 0) s_status = KX_OK;
  __syncthreads();

  auto ring_of = [&](int li) {
    Ring r;
    if (kSmemRing) {
      r.usage = S.usage + int64_t(li) * ring;
      r.ex = S.ex + int64_t(li) * ring;
    } else {
      r.usage = in.usage + int64_t(ib + li) * ring;
      r.ex = in.exists + int64_t(ib + li) * ring;
    }
    r.base = S.base[li];
    r.hi = S.hi[li];
    return r;
  };

  const int64_t q_end = pool_offsets[pool + 1];
  int64_t pos = pool_offsets[pool];
  int64_t hb_start = pos, hb_n = 0;
  int64_t nrows = 0, nadm = 0;
  int retries = 0;
  int par = 0;

  while (pos < q_end) {
    if (pos >= hb_start + hb_n) {  // refill the head batch (prefix of the pool's order)
      __syncthreads();
      hb_start = pos;
      hb_n = q_end - pos < kHeadBatch ? q_end - pos : kHeadBatch;
      if (threadIdx.x < hb_n) {
        const uint32_t idx = perm[pos + threadIdx.x];
        const int32_t a = q.agent[idx];
        S.h_idx[threadIdx.x] = idx;
        S.h_agent[threadIdx.x] = a;
        S.h_prompt[threadIdx.x] = q.prompt[idx];
        S.h_kept[threadIdx.x] = q.kept[idx];
        S.h_uid[threadIdx.x] = q.uid[idx];
        S.h_T[threadIdx.x] = dp.oracle_T ? q.pure_exec[idx] : ag.T[a];
      }
      __syncthreads();
    }
    const int h = static_cast<int>(pos - hb_start);
    const int64_t prompt = S.h_prompt[h];
    const double P = static_cast<double>(prompt);
    const double T = S.h_T[h];
    bool overflow = false;

    for (int li = warp; li < ni; li += kDispWarps) {
      // collect_live: watermark resume on the freshest usage, then batch_full.
      const double live = S.live[li];
      uint8_t susp = S.susp[li];
      if (susp && live < __dmul_rn(dp.watermark, S.cap[li])) {
        susp = 0;
        __syncwarp();
        if (lane == 0) S.susp[li] = 0;
      }
      const bool full = S.run[li] + S.wait[li] >= S.mb[li];
      Eval e;
      if (susp || full) {
        e.state = kExcluded;
        e.peak = 0.0;
        e.viol = 0;
      } else {
        e = warp_try_place(ring_of(li), ring, S.cap[li], P, S.k[li], now, T, dp.slot_len, &overflow);
      }
      if (lane == 0) {
        S.peak[par * ni + li] = e.peak;
        S.viol[par * ni + li] = e.viol;
        S.state[par * ni + li] = e.state;
        S.snap[par * ni + li] = live;
      }
    }
    if (overflow && lane == 0) atomicExch(&s_status, KX_ERR_CAPACITY);
    __syncthreads();
    if (s_status != KX_OK) break;

    // select_instance: min (peak, InstanceId) over fitting candidates (H9).
    double bpeak = 0.0;
    int bid = INT32_MAX, bli = -1;
    for (int li = lane; li < ni; li += 32) {
      if (S.state[par * ni + li] != kFits) continue;
      const double pk = S.peak[par * ni + li];
      const int id = S.id[li];
      if (bli < 0 || pk < bpeak || (pk == bpeak && id < bid)) {
        bpeak = pk;
        bid = id;
        bli = li;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double p2 = __shfl_xor_sync(0xffffffffu, bpeak, o);
      const int id2 = __shfl_xor_sync(0xffffffffu, bid, o);
      const int l2 = __shfl_xor_sync(0xffffffffu, bli, o);
      if (l2 >= 0 && (bli < 0 || p2 < bpeak || (p2 == bpeak && (id2 < bid || (id2 == bid && l2 < bli))))) {
        bpeak = p2;
        bid = id2;
        bli = l2;
      }
    }
    // Overload check (engine.cpp:254-258) on the owner's live snapshot.
    const bool overload = bli >= 0 && __dadd_rn(S.snap[par * ni + bli], P) > S.cap[bli];

    if (warp == 0) {  // decision log (engine.cpp:242-246)
      if (nrows < dp.log_cap) {
        const int64_t r = int64_t(pool) * dp.log_cap + nrows;
        if (lane == 0) {
          kx_decision d;
          d.time = now;
          d.predicted_peak = bli >= 0 ? bpeak : 0.0;
          d.uid = S.h_uid[h];
          d.queue_index = S.h_idx[h];
          d.agent = S.h_agent[h];
          d.target = bli >= 0 ? bid : -1;
          d.pool = pool;
          d.admitted = (bli >= 0 && !overload) ? 1 : 0;
          rows[r] = d;
        }
        for (int li = lane; li < ni; li += 32) {
          const uint8_t st = S.state[par * ni + li];
          double v = -1.0;
          if (st == kFits) v = S.peak[par * ni + li];
          else if (st == kExceeds) v = __dsub_rn(-static_cast<double>(S.viol[par * ni + li]), 1.0);
          cand[r * dp.peak_stride + li] = v;
        }
      }
    }
    ++nrows;
    if (bli < 0) break;  // head keeps its place until the next round (engine.cpp:247)
    const bool owner = (bli % kDispWarps) == warp;
    if (overload) {
      if (owner && lane == 0) S.susp[bli] = 1;  // Dispatcher::on_overload
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
      warp_commit(r, ring, P, S.k[bli], now, T, dp.slot_len);
      if (lane == 0) {
        S.hi[bli] = r.hi;
        S.live[bli] = __dadd_rn(S.live[bli], static_cast<double>(prompt + S.h_kept[h]));
        S.run[bli] += 1;
        q.admitted[S.h_idx[h]] = 1;
        active_append(in, ib + bli, S.h_uid[h], P, S.k[bli], now, T, &s_status);
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
      S.base[li] = r.base;
      active_gc(in, ib + li, now);
    }
  }
  __syncthreads();
  for (int li = threadIdx.x; li < ni; li += kDispThreads) {
    const int i = ib + li;
    in.live_kv[i] = S.live[li];
    in.base_slot[i] = S.base[li];
    in.hi_slot[i] = S.hi[li];
    in.running[i] = S.run[li];
    in.suspended[i] = S.susp[li];
  }
  if (kSmemRing) {
    const int64_t tot = int64_t(ni) * ring;
    double* gu = in.usage + int64_t(ib) * ring;
    uint8_t* ge = in.exists + int64_t(ib) * ring;
    for (int64_t j = threadIdx.x; j < tot; j += kDispThreads) {
      gu[j] = S.usage[j];
      ge[j] = S.ex[j];
    }
  }
  if (threadIdx.x == 0) {
    row_count[pool] = nrows;
    admitted_count[pool] = nadm;
    pool_status[pool] = s_status;
  }
}

// ---- single-instance ledger events (host-driven, tiny launches) ----------
__global__ void k_ledger_try_place(InstDev in, int i, int ring, double P, double k, double t0,
                                   double T, double slot_len, double* out_peak, int64_t* out_viol,
                                   int* out_state) {
  bool overflow = false;
  const Eval e = warp_try_place(global_ring(in, i, ring), ring, in.cap[i], P, k, t0, T, slot_len,
                                &overflow);
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
  const Eval e = warp_try_place(r, ring, in.cap[i], P, k, t0, T, slot_len, &overflow);
  if (overflow) {
    if ((threadIdx.x & 31) == 0) *status = KX_ERR_CAPACITY;
    return false;
  }
  if (e.state != kFits) return false;
  warp_commit(r, ring, P, k, t0, T, slot_len);
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
  KX_CUDA(cudaFuncSetAttribute(k_dispatch_timeslot<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kDispSmemLimit));
  KX_CUDA(cudaFuncSetAttribute(k_dispatch_timeslot<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kDispSmemLimit));
}

void launch_dispatch(const QueueDev& q, const AgentsDev& a, const InstDev& in,
                     const int32_t* pool_begin, const uint32_t* perm, const int64_t* pool_offsets,
                     const DispatchParams& dp, int n_pools, int max_inst_per_pool, kx_decision* rows,
                     double* cand, int64_t* row_count, int64_t* admitted_count, int* pool_status,
                     cudaStream_t st) {
  const size_t with_ring = disp_smem_bytes(max_inst_per_pool, dp.ring, true, nullptr, nullptr);
  if (with_ring <= static_cast<size_t>(kDispSmemLimit)) {
    k_dispatch_timeslot<true><<<n_pools, kDispThreads, with_ring, st>>>(
        q, a, in, pool_begin, perm, pool_offsets, dp, rows, cand, row_count, admitted_count,
        pool_status);
  } else {
    const size_t no_ring = disp_smem_bytes(max_inst_per_pool, dp.ring, false, nullptr, nullptr);
    k_dispatch_timeslot<false><<<n_pools, kDispThreads, no_ring, st>>>(
        q, a, in, pool_begin, perm, pool_offsets, dp, rows, cand, row_count, admitted_count,
        pool_status);
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

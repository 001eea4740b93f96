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

constexpr int kDispThreads = 512;
constexpr int kDispWarps = kDispThreads / 32;

enum : uint8_t { kExcluded = 0, kExceeds = 1, kFits = 2 };

struct Eval {
  double peak;
  int64_t viol;
  uint8_t state;
};

__device__ __forceinline__ bool slot_exists(const uint32_t* ex, int64_t s, int ring) {
  const uint32_t pos = static_cast<uint32_t>(s) & (ring - 1);
  return (ex[pos >> 5] >> (pos & 31)) & 1u;
}

// SlotLedger::try_place (dispatcher.cpp:52-68) for one instance, one warp.
// Returns false (and sets *overflow) if the span leaves the slot ring.
__device__ Eval warp_try_place(const InstDev& in, int i, int ring, double P, double k, double t0,
                               double T, double slot_len, bool* overflow) {
  const int lane = threadIdx.x & 31;
  int64_t first, last;
  span_bounds_dev(t0, T, slot_len, &first, &last);
  const double t_end = __dadd_rn(t0, T);
  const double cap = in.cap[i];
  const int64_t base = in.base_slot[i];
  const int64_t hi = in.hi_slot[i];
  if (last >= first && (first < base || last >= base + ring)) *overflow = true;
  const double* usage = in.usage + int64_t(i) * ring;
  const uint32_t* ex = in.exists + int64_t(i) * (ring / 32);
  const int64_t smax = hi > last ? hi : last;
  double peak = 0.0;
  int64_t viol = INT64_MAX;
  for (int64_t s = base + lane; s <= smax; s += 32) {
    const bool in_span = (s >= first && s <= last);
    const bool exists = slot_exists(ex, s, ring);
    if (!(in_span || exists)) continue;
    const double used = exists ? usage[static_cast<uint32_t>(s) & (ring - 1)] : 0.0;
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
__device__ void warp_commit(InstDev& in, int i, int ring, uint64_t uid, double P, double k,
                            double t0, double T, double slot_len, int* status) {
  const int lane = threadIdx.x & 31;
  int64_t first, last;
  span_bounds_dev(t0, T, slot_len, &first, &last);
  const double t_end = __dadd_rn(t0, T);
  double* usage = in.usage + int64_t(i) * ring;
  uint32_t* ex = in.exists + int64_t(i) * (ring / 32);
  for (int64_t s = first + lane; s <= last; s += 32) {
    const uint32_t pos = static_cast<uint32_t>(s) & (ring - 1);
    usage[pos] = __dadd_rn(usage[pos], peak_in_slot_dev(P, k, t0, t_end, s, slot_len));
    atomicOr(&ex[pos >> 5], 1u << (pos & 31));
  }
  __syncwarp();
  if (lane == 0) {
    if (last >= first && last > in.hi_slot[i]) in.hi_slot[i] = last;
    const int a = in.n_active[i];
    if (a >= kActiveCap) {
      *status = KX_ERR_CAPACITY;
    } else {
      const int64_t o = int64_t(i) * kActiveCap + a;
      in.act_uid[o] = uid;
      in.act_P[o] = P;
      in.act_k[o] = k;
      in.act_t0[o] = t0;
      in.act_T[o] = T;
      in.n_active[i] = a + 1;
    }
  }
  __syncwarp();
}

// SlotLedger::gc (dispatcher.cpp:101-118), one warp.
__device__ void warp_gc(InstDev& in, int i, int ring, double now, double slot_len) {
  const int lane = threadIdx.x & 31;
  const int64_t current =
      static_cast<int64_t>(floor(__ddiv_rn(__dadd_rn(now, kTimeEpsilon), slot_len)));
  const int64_t base = in.base_slot[i];
  double* usage = in.usage + int64_t(i) * ring;
  uint32_t* ex = in.exists + int64_t(i) * (ring / 32);
  if (current > base) {
    const int64_t stop = current < base + ring ? current : base + ring;
    for (int64_t s = base + lane; s < stop; s += 32) {
      const uint32_t pos = static_cast<uint32_t>(s) & (ring - 1);
      usage[pos] = 0.0;
      atomicAnd(&ex[pos >> 5], ~(1u << (pos & 31)));
    }
  }
  __syncwarp();
  if (lane == 0) {
    if (current > base) in.base_slot[i] = current;
    // active_: drop fully elapsed models (t_end <= now + eps); order-free.
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
  __syncwarp();
}

}  // namespace

__global__ void __launch_bounds__(kDispThreads)
k_dispatch_timeslot(QueueDev q, AgentsDev ag, InstDev in, const int32_t* __restrict__ pool_begin,
                    const uint32_t* __restrict__ perm, const int64_t* __restrict__ pool_offsets,
                    DispatchParams dp, kx_decision* __restrict__ rows, double* __restrict__ cand,
                    int64_t* __restrict__ row_count, int64_t* __restrict__ admitted_count,
                    int* __restrict__ pool_status) {
  __shared__ double s_peak[2][kMaxInstPerPool];
  __shared__ int64_t s_viol[2][kMaxInstPerPool];
  __shared__ double s_live[2][kMaxInstPerPool];
  __shared__ uint8_t s_state[2][kMaxInstPerPool];
  __shared__ int s_status;

  const int pool = blockIdx.x;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ib = pool_begin[pool];
  const int ni = pool_begin[pool + 1] - ib;
  if (threadIdx.x == 0) s_status = KX_OK;
  __syncthreads();

  const int64_t q_end = pool_offsets[pool + 1];
  int64_t pos = pool_offsets[pool];
  int64_t nrows = 0, nadm = 0;
  int retries = 0;
  int par = 0;
  const int ring = dp.ring;
  const double now = dp.now;

  while (pos < q_end) {
    const uint32_t idx = perm[pos];
    const int32_t agent = q.agent[idx];
    const int64_t prompt = q.prompt[idx];
    const double P = static_cast<double>(prompt);
    const double T = dp.oracle_T ? q.pure_exec[idx] : ag.T[agent];
    bool overflow = false;

    for (int li = warp; li < ni; li += kDispWarps) {
      const int i = ib + li;
      // collect_live: watermark resume on the freshest usage, then batch_full.
      const double live = in.live_kv[i];
      uint8_t susp = in.suspended[i];
      if (susp && live < __dmul_rn(dp.watermark, in.cap[i])) {
        susp = 0;
        if (lane == 0) in.suspended[i] = 0;
      }
      const bool full = in.running[i] + in.waiting[i] >= in.max_batch[i];
      Eval e;
      if (susp || full) {
        e.state = kExcluded;
        e.peak = 0.0;
        e.viol = 0;
      } else {
        e = warp_try_place(in, i, ring, P, in.decode_rate[i], now, T, dp.slot_len, &overflow);
      }
      if (lane == 0) {
        s_peak[par][li] = e.peak;
        s_viol[par][li] = e.viol;
        s_state[par][li] = e.state;
        s_live[par][li] = live;
      }
    }
    if (overflow && lane == 0) atomicExch(&s_status, KX_ERR_CAPACITY);
    __syncthreads();
    if (s_status != KX_OK) break;

    // select_instance: min (peak, InstanceId) over fitting candidates.
    double bpeak = 0.0;
    int bid = INT32_MAX, bli = -1;
    for (int li = lane; li < ni; li += 32) {
      if (s_state[par][li] != kFits) continue;
      const double pk = s_peak[par][li];
      const int id = in.id[ib + li];
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

    // Overload check (engine.cpp:254-258) on the live snapshot taken by the
    // owning warp during evaluation (no second barrier needed).
    bool overload = false;
    if (bli >= 0) overload = __dadd_rn(s_live[par][bli], P) > in.cap[ib + bli];

    if (dp.logging && warp == 0) {
      if (nrows < dp.log_cap) {
        const int64_t r = int64_t(pool) * dp.log_cap + nrows;
        if (lane == 0) {
          kx_decision d;
          d.time = now;
          d.predicted_peak = bli >= 0 ? bpeak : 0.0;
          d.uid = q.uid[idx];
          d.queue_index = idx;
          d.agent = agent;
          d.target = bli >= 0 ? bid : -1;
          d.pool = pool;
          d.admitted = (bli >= 0 && !overload) ? 1 : 0;
          rows[r] = d;
        }
        for (int li = lane; li < ni; li += 32) {
          const uint8_t st = s_state[par][li];
          double v = -1.0;
          if (st == kFits) v = s_peak[par][li];
          else if (st == kExceeds) v = __dsub_rn(-static_cast<double>(s_viol[par][li]), 1.0);
          cand[r * dp.peak_stride + li] = v;
        }
      } else if (lane == 0) {
        atomicExch(&s_status, KX_ERR_CAPACITY);
      }
    }
    ++nrows;
    if (bli < 0) break;  // head keeps its place until the next round
    const int t = ib + bli;
    const bool owner = (bli % kDispWarps) == warp;
    if (overload) {
      if (owner && lane == 0) in.suspended[t] = 1;
      if (++retries > ni) {
        if (threadIdx.x == 0) s_status = KX_ERR_LIVELOCK;
        break;
      }
      par ^= 1;
      continue;
    }
    retries = 0;
    if (owner) {
      warp_commit(in, t, ring, q.uid[idx], P, in.decode_rate[t], now, T, dp.slot_len, &s_status);
      if (lane == 0) {
        in.live_kv[t] = __dadd_rn(in.live_kv[t], static_cast<double>(prompt + q.kept[idx]));
        in.running[t] += 1;
        q.admitted[idx] = 1;
      }
    }
    ++nadm;
    ++pos;
    par ^= 1;
  }
  __syncthreads();
  // try_admit is a no-op for TimeSlot (waiting lists stay empty); gc.
  for (int li = warp; li < ni; li += kDispWarps) warp_gc(in, ib + li, ring, now, dp.slot_len);
  __syncthreads();
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
  const Eval e = warp_try_place(in, i, ring, P, k, t0, T, slot_len, &overflow);
  if (threadIdx.x == 0) {
    *out_peak = e.peak;
    *out_viol = e.viol;
    *out_state = overflow ? -1 : e.state;
  }
}

__global__ void k_ledger_commit(InstDev in, int i, int ring, uint64_t uid, double P, double k,
                                double t0, double T, double slot_len, int* status) {
  bool overflow = false;
  const Eval e = warp_try_place(in, i, ring, P, k, t0, T, slot_len, &overflow);
  __shared__ int st;
  if (threadIdx.x == 0) st = KX_OK;
  __syncwarp();
  if (overflow) {
    if (threadIdx.x == 0) *status = KX_ERR_CAPACITY;
    return;
  }
  if (e.state != kFits) {
    if (threadIdx.x == 0) *status = KX_ERR_LOGIC;  // commit after Exceeds
    return;
  }
  warp_commit(in, i, ring, uid, P, k, t0, T, slot_len, &st);
  if (threadIdx.x == 0) *status = st;
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
    bool overflow = false;
    const Eval ev = warp_try_place(in, i, ring, P[j], k[j], t0[j], T[j], slot_len, &overflow);
    if (overflow) {
      if (lane == 0) atomicExch(status, KX_ERR_CAPACITY);
      return;
    }
    const bool ok = ev.state == kFits;
    if (ok) warp_commit(in, i, ring, uid[j], P[j], k[j], t0[j], T[j], slot_len, status);
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
  const uint32_t* ex = in.exists + int64_t(i) * (ring / 32);
  const int64_t base = in.base_slot[i];
  for (int64_t s = first; s <= last; ++s) {
    if (s <= cutoff) continue;
    if (s < base || s >= base + ring || !slot_exists(ex, s, ring)) continue;  // usage_.find == end
    const uint32_t pos = static_cast<uint32_t>(s) & (ring - 1);
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
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp < n_inst) warp_gc(in, warp, ring, now, slot_len);
}

// ---- host wrappers -------------------------------------------------------
void launch_dispatch(const QueueDev& q, const AgentsDev& a, const InstDev& in,
                     const int32_t* pool_begin, const uint32_t* perm, const int64_t* pool_offsets,
                     const DispatchParams& dp, int n_pools, kx_decision* rows, double* cand,
                     int64_t* row_count, int64_t* admitted_count, int* pool_status,
                     cudaStream_t st) {
  k_dispatch_timeslot<<<n_pools, kDispThreads, 0, st>>>(q, a, in, pool_begin, perm, pool_offsets,
                                                        dp, rows, cand, row_count,
                                                        admitted_count, pool_status);
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

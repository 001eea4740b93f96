// K2 (score), K3 (compact-key LSD radix sort) and K4 (exact tie-fix): the
// full ReadyQueue order of every pool in one pass over HBM.
//
// Reference semantics: the queue is ordered by
//   (order_key(r), app_start, queue_enter, msg_id, uid)      priority.hpp:97-98
// with order_key per policy (scheduler.hpp:48-113). We sort by a 32-bit
// compact key
//   [ pool | class rank | q(primary time) ]
// where `class` is the dense rank of the discrete primary component
// (Kairos priority key, Topo depth; none for FCFS/Oracle) and q is a
// monotone non-decreasing quantisation of the primary double over the
// pool's [min, max] range. The compact key therefore never orders two
// requests against the reference order; requests it cannot separate are
// adjacent after the sort and are re-sorted by the exact tuple
// (ordered-bits of the doubles, msg key, uid, queue index) in K4.
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "kx_common.cuh"
#include "kx_order.cuh"
#include "kx_sort.cuh"
#include "kx_state.cuh"
#include "kx_tuple.cuh"

namespace kx {

void read_sort_debug(unsigned long long* out64, bool reset) {
  KX_CUDA(cudaMemcpyFromSymbol(out64, g_sort_tim, sizeof(unsigned long long) * 64));
  if (reset) {
    static const unsigned long long z[64] = {};
    KX_CUDA(cudaMemcpyToSymbol(g_sort_tim, z, sizeof(z)));
  }
}

__global__ void k_scan_hist(uint32_t* __restrict__ hist, int passes) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= passes) return;
  uint32_t* h = hist + warp * kRadix;
  uint32_t carry = 0;
  for (int c = 0; c < kRadix; c += 32) {
    const uint32_t v = h[c + lane];
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    h[c + lane] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
}

namespace {

__device__ __forceinline__ uint32_t class_of(const AgentsDev& a, int policy, int32_t agent) {
  if (policy == KX_SCHED_KAIROS) return a.pk_rank[agent];
  if (policy == KX_SCHED_TOPO) return a.depth_rank[agent];
  return 0;
}

// Exact comparison record: ordered bits of the tuple after the class.
struct TRec {
  uint64_t w0, w1, w2, msg, uid;
  uint32_t idx;
};

__device__ __forceinline__ TRec load_rec(const QueueDev& q, int policy, uint32_t idx) {
  TRec r;
  const double app = q.app_start[idx];
  const double qe = q.queue_enter[idx];
  switch (policy) {
    case KX_SCHED_KAIROS:  // (pk, app, qe) then app, qe, msg, uid
      r.w0 = ordered_bits(app);
      r.w1 = ordered_bits(qe);
      r.w2 = 0;
      break;
    case KX_SCHED_ORACLE:  // (rem, qe, 0) then app, qe, msg, uid
      r.w0 = ordered_bits(q.rem[idx]);
      r.w1 = ordered_bits(qe);
      r.w2 = ordered_bits(app);
      break;
    default:  // FCFS (qe, app, 0) / Topo (depth, qe, 0): then app, qe, msg, uid
      r.w0 = ordered_bits(qe);
      r.w1 = ordered_bits(app);
      r.w2 = 0;
      break;
  }
  r.msg = q.msg[idx];
  r.uid = q.uid[idx];
  r.idx = idx;
  return r;
}

__device__ __forceinline__ bool rec_less(const TRec& a, const TRec& b) {
  if (a.w0 != b.w0) return a.w0 < b.w0;
  if (a.w1 != b.w1) return a.w1 < b.w1;
  if (a.w2 != b.w2) return a.w2 < b.w2;
  if (a.msg != b.msg) return a.msg < b.msg;
  if (a.uid != b.uid) return a.uid < b.uid;
  return a.idx < b.idx;  // identical tuples: first-enqueued wins (best_index uses strict <)
}


}  // namespace

// ---- K2: per-request OrderKey -------------------------------------------
__global__ void k_score(QueueDev q, AgentsDev a, int policy, int64_t n, double* __restrict__ k0,
                        double* __restrict__ k1, double* __restrict__ k2) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int32_t ag = q.agent[i];
    double x0, x1, x2 = 0.0;
    switch (policy) {
      case KX_SCHED_KAIROS: x0 = a.pk[ag]; x1 = q.app_start[i]; x2 = q.queue_enter[i]; break;
      case KX_SCHED_FCFS: x0 = q.queue_enter[i]; x1 = q.app_start[i]; break;
      case KX_SCHED_TOPO: x0 = static_cast<double>(a.depth[ag]); x1 = q.queue_enter[i]; break;
      default: x0 = q.rem[i]; x1 = q.queue_enter[i]; break;
    }
    k0[i] = x0;
    k1[i] = x1;
    k2[i] = x2;
  }
}

// Primary time column of the policy's order key.
__device__ __forceinline__ const double* primary_ptr(const QueueDev& q, int policy) {
  return policy == KX_SCHED_KAIROS ? q.app_start : policy == KX_SCHED_ORACLE ? q.rem : q.queue_enter;
}

// Per-order reset: header counters, the first radix pass's look-back array
// and the caller's extra buffers (OrderHooks::zero_*).
struct OrderInit {
  uint32_t* hdr;
  int hdr_words;
  uint32_t* words;
  int n_words;
  uint8_t* bytes;
  int64_t n_bytes;
  uint4* lb;
  int64_t lb_vecs;
};

// ---- sampled quantisation window ---------------------------------------
// The compact key only needs the quantisation to be monotone: any window
// [lo, hi] works (values outside clamp to the ends and tie, and ties are
// resolved by the exact tuple), the window only sets the time resolution.
// So it comes from a sample: kSampleLen contiguous requests out of every
// `stride` (all of them for small queues), per-pool min / max of the primary
// time. Validation of every request happens in k_keygen.
constexpr int kSampleLen = 64;

// Sample stride for n requests: ~256K samples (every request below that).
__host__ __device__ inline int64_t sample_stride(int64_t n) {
  const int64_t target = int64_t(1) << 18;
  return n <= target ? kSampleLen : kSampleLen * ((n + target - 1) / target);
}

// The per-order reset (OrderInit, grid-stride) and the sample, in one launch:
// the blocks fold their samples' extremes into a persistent staging array;
// the last block to finish publishes them as the pools' windows and resets
// the staging array and the block counter for the next order.
__device__ __forceinline__ void order_reset(const OrderInit& in) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nt = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = t; i < in.hdr_words; i += nt) in.hdr[i] = 0;
  for (int64_t i = t; i < in.n_words; i += nt) in.words[i] = 0;
  const int64_t vecs = in.n_bytes / 16;
  uint4* v = reinterpret_cast<uint4*>(in.bytes);
  for (int64_t i = t; i < vecs; i += nt) v[i] = make_uint4(0, 0, 0, 0);
  if (t < in.n_bytes - vecs * 16) in.bytes[vecs * 16 + t] = 0;
  for (int64_t i = t; i < in.lb_vecs; i += nt) in.lb[i] = make_uint4(0, 0, 0, 0);
}

constexpr int kSampleWins = 8;  // sample windows per block of the sample launch
__global__ void __launch_bounds__(kSampleLen * kSampleWins)
k_pool_sample(QueueDev q, AgentsDev a, OrderParams op, int64_t n, int64_t stride, int64_t windows,
              PoolRange* __restrict__ ranges, PoolRange* __restrict__ stage, uint32_t* __restrict__ done,
              OrderInit init) {
  order_reset(init);
  const int64_t wdw = int64_t(blockIdx.x) * kSampleWins + threadIdx.x / kSampleLen;
  const int64_t i = wdw < windows ? wdw * stride + threadIdx.x % kSampleLen : n;
  int32_t p = -1;
  uint64_t lo = ~0ull, hi = 0ull;
  if (i < n) {
    const int32_t ag = q.agent[i];
    const double t = primary_ptr(q, op.policy)[i];
    if (ag >= 0 && ag < op.n_agents && t == t) {
      p = a.pool[ag];
      lo = hi = ordered_bits(t);
    }
  }
  // per warp: one (pool, min, max) when its samples share a pool (pools are
  // mostly contiguous), per-sample atomics otherwise; then one atomic pair
  // per distinct pool of the block (few global atomics: the staging array
  // and the block counter are single addresses)
  constexpr int kWarps = kSampleLen * kSampleWins / 32;
  __shared__ int32_t s_wp[kWarps];
  __shared__ uint64_t s_wlo[kWarps], s_whi[kWarps];
  const int warp = threadIdx.x >> 5;
  const uint32_t valid = __ballot_sync(0xffffffffu, p >= 0);
  int32_t wp = -1;
  if (valid) {
    const int32_t p0 = __shfl_sync(0xffffffffu, p, __ffs(valid) - 1);
    if (__all_sync(0xffffffffu, p < 0 || p == p0)) {
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t l2 = __shfl_xor_sync(0xffffffffu, lo, o);
        const uint64_t h2 = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = l2 < lo ? l2 : lo;
        hi = h2 > hi ? h2 : hi;
      }
      wp = p0;
    } else if (p >= 0) {
      atomicMin(reinterpret_cast<unsigned long long*>(&stage[p].lo_bits), (unsigned long long)lo);
      atomicMax(reinterpret_cast<unsigned long long*>(&stage[p].hi_bits), (unsigned long long)hi);
    }
  }
  if ((threadIdx.x & 31) == 0) {
    s_wp[warp] = wp;
    s_wlo[warp] = lo;
    s_whi[warp] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < kWarps; ++w) {
      const int32_t pw = s_wp[w];
      if (pw < 0) continue;
      uint64_t l = s_wlo[w], h = s_whi[w];
      for (int w2 = w + 1; w2 < kWarps; ++w2)
        if (s_wp[w2] == pw) {
          l = s_wlo[w2] < l ? s_wlo[w2] : l;
          h = s_whi[w2] > h ? s_whi[w2] : h;
          s_wp[w2] = -1;
        }
      atomicMin(reinterpret_cast<unsigned long long*>(&stage[pw].lo_bits), (unsigned long long)l);
      atomicMax(reinterpret_cast<unsigned long long*>(&stage[pw].hi_bits), (unsigned long long)h);
    }
  }
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int k = threadIdx.x; k < op.n_pools; k += blockDim.x) {
    volatile PoolRange* sv = stage + k;
    ranges[k] = PoolRange{sv->lo_bits, sv->hi_bits, 0.0, 0.0};  // lo / scale: finalize_range
    sv->lo_bits = ~0ull;
    sv->hi_bits = 0ull;
  }
  if (threadIdx.x == 0) *done = 0u;
}

// The quantisation window of a pool from its sampled extremes (lo_bits /
// hi_bits, filled by k_pool_sample): lo and scale. Every reader computes it
// itself (the same correctly-rounded operations, so the same result): no
// launch of its own between the sample and key generation.
__device__ __forceinline__ PoolRange finalize_range(PoolRange r, int q_bits) {
  if (r.lo_bits > r.hi_bits) {  // empty pool
    r.lo = 0.0;
    r.scale = 0.0;
  } else {
    double lo = from_ordered_bits(r.lo_bits);
    double hi = from_ordered_bits(r.hi_bits);
    // The sampled extremes sit inside the true ones: widen by 1/64 of the
    // span each side so unsampled tails rarely clamp (clamped values only tie).
    const double m = __dmul_rn(__dsub_rn(hi, lo), 0.015625);
    lo = __dsub_rn(lo, m);
    hi = __dadd_rn(hi, m);
    const double span = __dsub_rn(hi, lo);
    const double qmax = static_cast<double>((uint64_t(1) << q_bits) - 1);
    r.lo = lo;
    // Degenerate or non-finite range: every request shares q = 0 and the
    // exact tie-fix orders them.
    r.scale = (span > 0.0 && span < 1.0e300 && isfinite(lo)) ? __ddiv_rn(qmax, span) : 0.0;
  }
  return r;
}

// Compact key of one request: [pool | class rank | q(primary time)].
// Monotone: (t - lo) and the product are correctly rounded, floor and the
// clamp are monotone, so t1 <= t2 implies q1 <= q2.
__device__ __forceinline__ uint32_t compact_key(const AgentsDev& a, const OrderParams& op,
                                                const PoolRange& r, int32_t p, int32_t ag, double t,
                                                uint32_t qmax) {
  const double x = __dmul_rn(__dsub_rn(t, r.lo), r.scale);
  uint32_t qv;
  if (!(x > 0.0)) qv = 0;
  else if (x >= static_cast<double>(qmax)) qv = qmax;
  else qv = static_cast<uint32_t>(x);
  uint32_t key = qv;
  if (op.class_bits) key |= class_of(a, op.policy, ag) << op.q_bits;
  if (op.pool_bits) key |= static_cast<uint32_t>(p) << (op.class_bits + op.q_bits);
  return key;
}

__device__ __forceinline__ uint32_t q_max(const OrderParams& op) {
  return (op.q_bits >= 32) ? 0xffffffffu : ((1u << op.q_bits) - 1u);
}

// ---- speculative dispatch-prefix bound (CTA per pool) --------------------
// The dispatch round of pool p reads at most `need` heads (free batch slots
// + 1). From the sampled requests of p (a uniform subsample of <=
// kSpecMax), take the k-th smallest compact key with k ~ 1.5 * need * the
// sampling fraction: about 1.5 * need of the pool's keys are <= it. Key
// generation then collects exactly the keys <= bound - a prefix of the
// pool's order by construction (equal keys are all in or all out) - and the
// prefix select needs no pass of its own. If the collection overflows the
// candidate buffer the pool falls back to the radix select; if it is short
// of `need`, the dispatch continues over the full order (phase 2).
constexpr int kSpecMax = 32768;
constexpr int kSpecThreads = 1024;

// Compact keys of the sampled requests (every m-th block of k_pool_sample's
// positions), appended to per-pool lists of at most kSpecMax (block-
// aggregated: a block's requests mostly share one pool). plist_count[p]
// counts every sample of p, kept or not.
__global__ void __launch_bounds__(kSampleLen)
k_sample_keys(QueueDev q, AgentsDev a, OrderParams op, int64_t n, int64_t stride, int64_t m,
              const PoolRange* __restrict__ ranges, uint32_t* __restrict__ plist,
              uint32_t* __restrict__ plist_count) {
  const int64_t i = int64_t(blockIdx.x) * m * stride + threadIdx.x;
  int32_t p = -1;
  uint32_t key = 0;
  if (i < n) {
    const int32_t ag = q.agent[i];
    const double t = primary_ptr(q, op.policy)[i];
    if (ag >= 0 && ag < op.n_agents && t == t) {
      p = a.pool[ag];
      key = compact_key(a, op, finalize_range(ranges[p], op.q_bits), p, ag, t, q_max(op));
    }
  }
  const int lane = threadIdx.x & 31;
  const uint32_t valid = __ballot_sync(0xffffffffu, p >= 0);
  const int32_t p0 = valid ? __shfl_sync(0xffffffffu, p, __ffs(valid) - 1) : -1;
  if (__all_sync(0xffffffffu, p < 0 || p == p0)) {  // one reservation per warp
    uint32_t base = 0;
    if (lane == 0 && valid) base = atomicAdd(&plist_count[p0], static_cast<uint32_t>(__popc(valid)));
    base = __shfl_sync(0xffffffffu, base, 0);
    const uint32_t slot = base + __popc(valid & lanemask_lt());
    if (p >= 0 && slot < kSpecMax) plist[int64_t(p) * kSpecMax + slot] = key;
  } else if (p >= 0) {
    const uint32_t slot = atomicAdd(&plist_count[p], 1u);
    if (slot < kSpecMax) plist[int64_t(p) * kSpecMax + slot] = key;
  }
}

__global__ void __launch_bounds__(kSpecThreads)
k_spec_bound(InstDev in, const int32_t* __restrict__ pool_begin, OrderParams op, int64_t n,
             int64_t stride, int64_t m, const uint32_t* __restrict__ plist,
             const uint32_t* __restrict__ plist_count, uint32_t max_need,
             uint32_t* __restrict__ spec_bound, uint32_t* __restrict__ spec_on,
             uint32_t* __restrict__ spec_count) {
  extern __shared__ uint32_t s_keys[];  // [kSpecMax]
  __shared__ uint32_t s_hist[kRadix];
  __shared__ uint32_t s_n;
  __shared__ uint32_t s_prefix, s_mask, s_rank, s_ok;
  const int p = blockIdx.x;
  const int tid = threadIdx.x;
  const uint32_t S = plist_count[p];
  const uint32_t Sk = S < kSpecMax ? S : kSpecMax;
  if (tid == 0) {
    s_n = Sk;
    spec_count[p] = 0;
  }
  const uint4* src = reinterpret_cast<const uint4*>(plist + int64_t(p) * kSpecMax);
  uint4* dst = reinterpret_cast<uint4*>(s_keys);
  for (uint32_t v = tid; v < (Sk + 3) / 4; v += kSpecThreads) dst[v] = src[v];
  __syncthreads();
  if (tid == 0) {
    const uint32_t Sp = s_n < kSpecMax ? s_n : kSpecMax;
    int64_t free_slots = 0;
    for (int k = pool_begin[p]; k < pool_begin[p + 1]; ++k) {
      const int64_t f = int64_t(in.max_batch[k]) - in.running[k] - in.waiting[k];
      free_slots += f > 0 ? f : 0;
    }
    int64_t need = free_slots + 1;
    need = need < int64_t(max_need) ? need : int64_t(max_need);
    // pool size estimate: the S samples cover kSampleLen / (m * stride) of the queue
    const double Np = double(S) * double(m) * double(stride) / double(kSampleLen);
    const double frac = Np > 0.0 ? double(Sp) / Np : 0.0;
    const uint32_t k = static_cast<uint32_t>(ceil(1.5 * double(need) * frac)) + 3u;
    s_ok = (Sp >= k && Sp >= 64) ? 1u : 0u;
    s_rank = k;
    s_prefix = 0;
    s_mask = 0;
  }
  __syncthreads();
  if (!s_ok) {
    if (tid == 0) spec_on[p] = 0;
    return;
  }
  const uint32_t Sp = s_n < kSpecMax ? s_n : kSpecMax;
  // k-th smallest sampled key: MSD radix select over the four bytes
  for (int d = 3; d >= 0; --d) {
    for (int j = tid; j < kRadix; j += kSpecThreads) s_hist[j] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix, mask = s_mask;
    // warp-aggregated: the high digits of one pool's keys are mostly equal
    for (uint32_t j0 = 0; j0 < Sp; j0 += kSpecThreads) {
      const uint32_t j = j0 + tid;
      const uint32_t key = j < Sp ? s_keys[j] : 0u;
      hist_add(s_hist, (key >> (8 * d)) & 0xFF, j < Sp && (key & mask) == prefix);
    }
    __syncthreads();
    if (tid < 32) {  // warp 0: bucket of the rank-th key (eight bins per lane)
      const uint32_t rank = s_rank;
      uint32_t h[8], sum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        h[j] = s_hist[tid * 8 + j];
        sum += h[j];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += y;
      }
      const uint32_t hit = __ballot_sync(0xffffffffu, incl >= rank);
      const int lane_hit = __ffs(hit) - 1;
      if (tid == lane_hit) {
        uint32_t cum = incl - sum;
        int j = 0;
        for (; j < 8; ++j) {
          if (cum + h[j] >= rank) break;
          cum += h[j];
        }
        s_prefix = prefix | (static_cast<uint32_t>(tid * 8 + j) << (8 * d));
        s_mask = mask | (0xFFu << (8 * d));
        s_rank = rank - cum;
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    spec_bound[p] = s_prefix;
    spec_on[p] = 1;
  }
}

// ---- compact key + upfront digit histograms + pool counts -------------
// 16-byte loads (four requests per thread per step), keys stored as uint4.
// The per-agent (pool, class) pairs and the per-pool window and prefix
// bound are staged in shared memory when the agent table is small.
constexpr int kKeygenAgents = 2048;

#ifndef KX_KG_MINB
#define KX_KG_MINB 8  // 32 registers: 8 CTAs per SM (measured: 0.055 vs 0.067 ms at C4 with 1)
#endif
#ifndef KX_KG_U
#define KX_KG_U 1
#endif
template <bool kSmemTables>
__global__ void __launch_bounds__(256, kSmemTables ? KX_KG_MINB : 4)
k_keygen(QueueDev q, AgentsDev a, OrderParams op, int64_t n, const PoolRange* __restrict__ ranges,
         uint32_t* __restrict__ keys, uint32_t* __restrict__ hist, uint32_t* __restrict__ pool_counts,
         int* __restrict__ error_flags, KeygenSpec spec) {
  __shared__ uint32_t sh[kRadix];
  __shared__ uint32_t s_ag[kSmemTables ? kKeygenAgents : 1];  // pool << 16 | class
  extern __shared__ __align__(16) unsigned char kg_dyn[];
  double* s_lo = reinterpret_cast<double*>(kg_dyn);                 // [P]
  double* s_scale = s_lo + op.n_pools;                              // [P]
  int64_t* s_bnd = reinterpret_cast<int64_t*>(s_scale + op.n_pools);  // [P] prefix bound, -1 off
  uint32_t* s_pool = reinterpret_cast<uint32_t*>(s_bnd + op.n_pools);  // [P] counts
  for (int i = threadIdx.x; i < kRadix; i += blockDim.x) sh[i] = 0;
  for (int i = threadIdx.x; i < op.n_pools; i += blockDim.x) {
    s_pool[i] = 0;
    const PoolRange r = finalize_range(ranges[i], op.q_bits);
    s_lo[i] = r.lo;
    s_scale[i] = r.scale;
    s_bnd[i] = (spec.bound && spec.on[i]) ? int64_t(spec.bound[i]) : int64_t(-1);
  }
  if (kSmemTables)
    for (int i = threadIdx.x; i < op.n_agents; i += blockDim.x)
      s_ag[i] = (static_cast<uint32_t>(a.pool[i]) << 16) | class_of(a, op.policy, i);
  __syncthreads();
  const uint32_t qmax = q_max(op);
  int32_t cur_pool = -1;
  uint32_t cur_cnt = 0;
  int err = 0;
  auto make_key = [&](int32_t ag, double t, int64_t idx) {
    if (ag < 0 || ag >= op.n_agents) {  // reported at order fetch; key 0 in pool 0
      err |= 1;
      ag = 0;
    }
    if (t != t) {
      err |= 2;
      t = 0.0;
    }
    int32_t p;
    uint32_t cls;
    if (kSmemTables) {
      const uint32_t pc = s_ag[ag];
      p = static_cast<int32_t>(pc >> 16);
      cls = pc & 0xFFFFu;
    } else {
      p = a.pool[ag];
      cls = class_of(a, op.policy, ag);
    }
    // monotone quantisation (see compact_key)
    const double x = __dmul_rn(__dsub_rn(t, s_lo[p]), s_scale[p]);
    uint32_t qv;
    if (!(x > 0.0)) qv = 0;
    else if (x >= static_cast<double>(qmax)) qv = qmax;
    else qv = static_cast<uint32_t>(x);
    uint32_t key = qv;
    if (op.class_bits) key |= cls << op.q_bits;
    if (op.pool_bits) key |= static_cast<uint32_t>(p) << (op.class_bits + op.q_bits);
    if (p != cur_pool) {
      if (cur_pool >= 0) atomicAdd(&s_pool[cur_pool], cur_cnt);
      cur_pool = p;
      cur_cnt = 0;
    }
    ++cur_cnt;
    if (int64_t(key) <= s_bnd[p]) {  // dispatch-prefix candidate
      const uint32_t slot = atomicAdd(&spec.count[p], 1u);
      if (slot < kTopKMax) {
        spec.cand[int64_t(p) * kTopKMax + slot] = static_cast<uint32_t>(idx);
        spec.cand_key[int64_t(p) * kTopKMax + slot] = key;
      }
    }
    return key;
  };
  const double* tp = primary_ptr(q, op.policy);
  const int4* av = reinterpret_cast<const int4*>(q.agent);
  const double2* tv = reinterpret_cast<const double2*>(tp);
  uint4* kv = reinterpret_cast<uint4*>(keys);
  const int64_t nv = n >> 2;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  constexpr int U = KX_KG_U;
  // the loop trip count is uniform over the block (hist_add is warp-collective)
  for (int64_t b0 = int64_t(blockIdx.x) * blockDim.x; b0 < nv; b0 += U * stride) {
    int4 ag[U];
    double2 t0[U], t1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = b0 + u * stride + threadIdx.x;
      if (v < nv) {
        ag[u] = av[v];
        t0[u] = tv[2 * v];
        t1[u] = tv[2 * v + 1];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = b0 + u * stride + threadIdx.x;
      const bool valid = v < nv;
      uint4 k4 = make_uint4(0, 0, 0, 0);
      if (valid) {
        k4.x = make_key(ag[u].x, t0[u].x, 4 * v);
        k4.y = make_key(ag[u].y, t0[u].y, 4 * v + 1);
        k4.z = make_key(ag[u].z, t1[u].x, 4 * v + 2);
        k4.w = make_key(ag[u].w, t1[u].y, 4 * v + 3);
        kv[v] = k4;
      }
      // the first pass's digit (spread: plain shared atomics); each radix
      // pass counts the next pass's digit as it writes its keys
      if (valid) {
        atomicAdd(&sh[digit_of(k4.x, 0)], 1u);
        atomicAdd(&sh[digit_of(k4.y, 0)], 1u);
        atomicAdd(&sh[digit_of(k4.z, 0)], 1u);
        atomicAdd(&sh[digit_of(k4.w, 0)], 1u);
      }
    }
  }
  if (blockIdx.x == 0) {
    for (int64_t base = nv << 2; base < n; base += blockDim.x) {
      const int64_t i = base + threadIdx.x;
      const bool valid = i < n;
      uint32_t key = 0;
      if (valid) {
        key = make_key(q.agent[i], tp[i], i);
        keys[i] = key;
      }
      hist_add(sh, digit_of(key, 0), valid);
    }
  }
  if (cur_pool >= 0) atomicAdd(&s_pool[cur_pool], cur_cnt);
  if (err) atomicOr(error_flags, err);
  __syncthreads();
  for (int i = threadIdx.x; i < kRadix; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
  for (int i = threadIdx.x; i < op.n_pools; i += blockDim.x)
    if (s_pool[i]) atomicAdd(&pool_counts[i], s_pool[i]);
}

// Diagnostics: globaltimer when the pool offsets (the end of key generation)
// were written, read by the dispatch probe against the dispatch kernel's start.
__device__ unsigned long long g_keys_done_ns;
void read_keys_done(unsigned long long* out) { KX_CUDA(cudaMemcpyFromSymbol(out, g_keys_done_ns, sizeof(*out))); }

__global__ void k_pool_offsets(const uint32_t* __restrict__ counts, int n_pools,
                               int64_t* __restrict__ offsets) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_keys_done_ns = t;
    int64_t acc = 0;
    for (int p = 0; p < n_pools; ++p) {
      offsets[p] = acc;
      acc += counts[p];
    }
    offsets[n_pools] = acc;
  }
}

// ---- K4: exact tie-fix ---------------------------------------------------
// Runs of equal compact keys are re-sorted by the exact tuple. Runs of up to
// kThreadRun requests (the common case: a workflow's repeated agent shares
// app_start) are sorted by the thread that finds the run start, with no
// list and no atomics; msg/uid are fetched only when the time fields tie.
// Longer runs are listed for the warp / CTA kernels below.
constexpr int kThreadRun = 16;

namespace {

}  // namespace

// Warp-aggregated list append (the long-run list of the CTA fixer).
__device__ __forceinline__ void list_append(bool want, uint32_t value, uint32_t* list,
                                            uint32_t* count, uint32_t cap, uint32_t* lens = nullptr,
                                            uint32_t len = 0) {
  const uint32_t m = __ballot_sync(0xffffffffu, want);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(count, static_cast<uint32_t>(__popc(m)));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (want) {
    const uint32_t slot = base + __popc(m & lanemask_lt());
    if (slot < cap) {
      list[slot] = value;
      if (lens) lens[slot] = len;
    }
  }
}

// One CTA per chunk of kTieChunk sorted keys: it finds the runs of equal
// compact keys that START in its chunk (a run is owned by the chunk of its
// first element; it may extend past the chunk), compacts their starts into
// shared memory and fixes them with one thread per run. Runs of up to
// kThreadRun requests (the common case: a workflow's repeated agent shares
// app_start) are re-sorted by the exact tuple in registers, msg/uid fetched
// only when the time fields tie, and written back only when their order
// changes; longer runs are listed for the CTA fixer (k_tie_fix_big).
// All key loads are issued before any use; a vector's neighbouring keys come
// from the adjacent lanes (shuffles), only the warp's edge lanes load them.
constexpr int kRunVec = 4;
constexpr int kTieChunk = 256 * kRunVec * 4;

__device__ __forceinline__ void fix_run(const QueueDev& q, int policy, uint32_t* __restrict__ perm,
                                        int64_t i, int len) {
  bool moved = false;
  if (len <= 4) {
    // the common runs (a workflow's repeated agent: 2-4 calls) in registers:
    // odd-even transposition with the exact comparator (a total order, the
    // queue index breaks every tie)
    uint32_t pv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) pv[j] = j < len ? perm[i + j] : 0u;
    TKey r0 = load_tkey(q, policy, pv[0]), r1 = load_tkey(q, policy, pv[1]);
    TKey r2 = load_tkey(q, policy, len > 2 ? pv[2] : pv[1]), r3 = load_tkey(q, policy, len > 3 ? pv[3] : pv[1]);
    auto cx = [&](TKey& a, TKey& b, bool on) {
      if (on && tkey_less(q, b, a)) {
        const TKey tk = a;
        a = b;
        b = tk;
        moved = true;
      }
    };
#pragma unroll
    for (int round = 0; round < 4; ++round) {
      if (round >= len) break;
      if ((round & 1) == 0) {
        cx(r0, r1, true);
        cx(r2, r3, len > 3);
      } else {
        cx(r1, r2, len > 2);
      }
    }
    if (moved) {
      perm[i] = r0.idx;
      perm[i + 1] = r1.idx;
      if (len > 2) perm[i + 2] = r2.idx;
      if (len > 3) perm[i + 3] = r3.idx;
    }
    return;
  }
  TKey r[kThreadRun];
  for (int j = 0; j < len; ++j) r[j] = load_tkey(q, policy, perm[i + j]);
  for (int j = 1; j < len; ++j) {  // insertion sort, exact comparator
    const TKey x = r[j];
    int m = j - 1;
    while (m >= 0 && tkey_less(q, x, r[m])) {
      r[m + 1] = r[m];
      --m;
      moved = true;
    }
    r[m + 1] = x;
  }
  if (moved)
    for (int j = 0; j < len; ++j) perm[i + j] = r[j].idx;
}

__global__ void __launch_bounds__(256)
k_tie_fix(QueueDev q, int policy, const uint32_t* __restrict__ keys, uint32_t* __restrict__ perm,
          int64_t n, uint32_t* __restrict__ big_starts, uint32_t* __restrict__ big_lens,
          uint32_t* __restrict__ n_big, uint32_t cap) {
  __shared__ __align__(16) uint32_t s_keys[kTieChunk];
  __shared__ uint16_t s_list[kTieChunk / 2];  // chunk-local run starts
  __shared__ uint32_t s_warp[8];
  __shared__ uint32_t s_total;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t cbase = int64_t(blockIdx.x) * kTieChunk;
  const int64_t nv = (n + 3) >> 2;
  const int64_t vb = cbase / 4 + threadIdx.x;
  uint32_t k[kRunVec][6];  // keys[4v - 1 .. 4v + 4]
#pragma unroll
  for (int u = 0; u < kRunVec; ++u) {
    const int64_t v = vb + u * blockDim.x;
    const int64_t b = 4 * v;
    if (v < nv && b + 3 < n) {
      const uint4 x = reinterpret_cast<const uint4*>(keys)[v];
      k[u][1] = x.x; k[u][2] = x.y; k[u][3] = x.z; k[u][4] = x.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) k[u][1 + j] = (v < nv && b + j < n) ? keys[b + j] : 0u;
    }
    k[u][0] = (lane == 0 && v < nv && b > 0) ? keys[b - 1] : 0u;
    k[u][5] = (lane == 31 && v < nv && b + 4 < n) ? keys[b + 4] : 0u;
  }
  uint32_t mask = 0;  // bit u*4+j: element 4v+j of vector u starts a run
#pragma unroll
  for (int u = 0; u < kRunVec; ++u) {
    const uint32_t prev = __shfl_up_sync(0xffffffffu, k[u][4], 1);
    const uint32_t next = __shfl_down_sync(0xffffffffu, k[u][1], 1);
    if (lane > 0) k[u][0] = prev;
    if (lane < 31) k[u][5] = next;
    reinterpret_cast<uint4*>(s_keys)[u * blockDim.x + threadIdx.x] = make_uint4(k[u][1], k[u][2], k[u][3], k[u][4]);
    const int64_t v = vb + u * blockDim.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t i = 4 * v + j;
      const bool start = v < nv && i + 1 < n && (i == 0 || k[u][j] != k[u][j + 1]) && k[u][j + 2] == k[u][j + 1];
      mask |= start ? (1u << (u * 4 + j)) : 0u;
    }
  }
  // block-wide exclusive prefix of the per-thread counts: the chunk's run list
  const uint32_t c = __popc(mask);
  uint32_t x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tot = 0;
    for (int w = 0; w < 8; ++w) {
      const uint32_t t = s_warp[w];
      s_warp[w] = tot;
      tot += t;
    }
    s_total = tot;
  }
  __syncthreads();
  uint32_t slot = s_warp[warp] + x - c;
  while (mask) {
    const int bit = __ffs(mask) - 1;
    mask &= mask - 1;
    s_list[slot++] = static_cast<uint16_t>(4 * ((bit >> 2) * blockDim.x + threadIdx.x) + (bit & 3));
  }
  __syncthreads();
  const uint32_t total = s_total;
  for (uint32_t w0 = 0; w0 < total; w0 += blockDim.x) {  // uniform trip count: list_append is warp-wide
    const uint32_t w = w0 + threadIdx.x;
    int64_t i = 0, e = 0;
    bool big = false;
    if (w < total) {
      const int li = s_list[w];
      i = cbase + li;
      const uint32_t kk = s_keys[li];
      e = i + 2;  // a run has at least two
      while (e < n && e - i <= kThreadRun && (e - cbase < kTieChunk ? s_keys[e - cbase] : keys[e]) == kk) ++e;
      if (e - i > kThreadRun) {
        while (e < n && keys[e] == kk) ++e;
        big = true;
      }
    }
    list_append(big, static_cast<uint32_t>(i), big_starts, n_big, cap, big_lens,
                static_cast<uint32_t>(e - i));
    if (w < total && !big) fix_run(q, policy, perm, i, static_cast<int>(e - i));
  }
}

// Runs longer than 32: one CTA each. Up to kBigSmem records are sorted in
// shared memory (bitonic); longer runs use a global merge sort on indices
// with the exact comparator (only for degenerate inputs).
constexpr int kBigThreads = 512;
constexpr int kBigSmem = 1024;

__global__ void __launch_bounds__(kBigThreads)
k_tie_fix_big(QueueDev q, int policy, uint32_t* __restrict__ perm, uint32_t* __restrict__ scratch,
              const uint32_t* __restrict__ starts, const uint32_t* __restrict__ lens,
              const uint32_t* __restrict__ n_big, uint32_t cap) {
  __shared__ TRec s[kBigSmem];
  const uint32_t total = min(*n_big, cap);
  for (uint32_t seg = blockIdx.x; seg < total; seg += gridDim.x) {
    const int64_t st = starts[seg];
    const int64_t len = lens[seg];
    if (len <= kBigSmem) {
      int64_t p2 = 1;
      while (p2 < len) p2 <<= 1;
      for (int64_t i = threadIdx.x; i < p2; i += blockDim.x) {
        if (i < len) {
          s[i] = load_rec(q, policy, perm[st + i]);
        } else {
          s[i].w0 = s[i].w1 = s[i].w2 = s[i].msg = s[i].uid = ~0ull;
          s[i].idx = 0xffffffffu;
        }
      }
      __syncthreads();
      for (int64_t kk = 2; kk <= p2; kk <<= 1) {
        for (int64_t j = kk >> 1; j > 0; j >>= 1) {
          for (int64_t i = threadIdx.x; i < p2; i += blockDim.x) {
            const int64_t l = i ^ j;
            if (l > i) {
              const bool up = (i & kk) == 0;
              const bool sw = up ? rec_less(s[l], s[i]) : rec_less(s[i], s[l]);
              if (sw) {
                const TRec t = s[i];
                s[i] = s[l];
                s[l] = t;
              }
            }
          }
          __syncthreads();
        }
      }
      for (int64_t i = threadIdx.x; i < len; i += blockDim.x) perm[st + i] = s[i].idx;
      __syncthreads();
    } else {
      // Bottom-up merge sort; element i of run A lands at i + |{b in B: b < a}|.
      uint32_t* src = perm + st;
      uint32_t* dst = scratch + st;
      for (int64_t w = 1; w < len; w <<= 1) {
        for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
          const int64_t run = i / (2 * w);
          const int64_t a0 = run * 2 * w;
          const int64_t b0 = a0 + w;
          const int64_t b1 = min(a0 + 2 * w, len);
          const bool inA = i < b0;
          const TRec x = load_rec(q, policy, src[i]);
          int64_t lo, hi;
          if (inA) {
            lo = b0 < len ? b0 : len;
            hi = b1 > lo ? b1 : lo;
          } else {
            lo = a0;
            hi = b0;
          }
          const int64_t base_lo = lo;
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (rec_less(load_rec(q, policy, src[mid]), x)) lo = mid + 1;
            else hi = mid;
          }
          const int64_t within = inA ? (i - a0) : (i - b0);
          dst[a0 + within + (lo - base_lo)] = src[i];
        }
        __syncthreads();
        uint32_t* t = src;
        src = dst;
        dst = t;
      }
      if (src != perm + st)
        for (int64_t i = threadIdx.x; i < len; i += blockDim.x) perm[st + i] = src[i];
      __syncthreads();
    }
  }
}

void launch_spec_bound(const QueueDev& q, const AgentsDev& a, const InstDev& in,
                       const int32_t* pool_begin, const OrderParams& op, int64_t n,
                       const OrderWorkspace& ws, TopKWork& w, cudaStream_t st) {
  const int64_t stride = sample_stride(n);
  const int64_t blocks = (n + stride - 1) / stride;
  // every m-th sample block: about kSpecMax / 2 samples per pool when the
  // pools are balanced
  const int64_t per = int64_t(kSpecMax / 2) * op.n_pools;
  const int64_t m = std::max<int64_t>(1, (blocks * kSampleLen + per - 1) / per);
  // w.plist_count was zeroed by the order's init launch (the tick's hooks)
  k_sample_keys<<<static_cast<unsigned>((blocks + m - 1) / m), kSampleLen, 0, st>>>(
      q, a, op, n, stride, m, ws.ranges, w.plist, w.plist_count);
  KX_CHECK_LAUNCH();
  k_spec_bound<<<op.n_pools, kSpecThreads, sizeof(uint32_t) * kSpecMax, st>>>(
      in, pool_begin, op, n, stride, m, w.plist, w.plist_count, w.max_need, w.spec_bound, w.spec_on,
      w.spec_count);
  KX_CHECK_LAUNCH();
}

size_t spec_list_words(int n_pools) { return size_t(n_pools) * kSpecMax; }

// ---- host orchestration --------------------------------------------------
// Warp ranking per radix pass (kx_sort.cuh kRank), chosen by measurement
// on the C4 keys: MATCH.ANY peers for the spread low digits, ballots for the
// top digit (few distinct values). With 12-key tiles the leader-broadcast
// form (2) won the low digits (profiles/r01_sort_rank.md); with 16-key tiles
// every peer reading the running count (0) does: 0001 0.464 ms for the four
// passes, 2221 0.468, 0201 0.466, 0011 0.478, 0000 0.498.
constexpr int kSortRankDefault[4] = {0, 0, 0, 1};

size_t order_lookback_bytes(int64_t cap) {  // two arrays, alternating between passes
  const int64_t tiles = (cap + kSortTile - 1) / kSortTile;
  return 2 * size_t(tiles) * kRadix * sizeof(uint32_t);
}

void launch_score(const QueueDev& q, const AgentsDev& a, int policy, int64_t n, double* k0,
                  double* k1, double* k2, int sms, cudaStream_t st) {
  if (n == 0) return;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, int64_t(sms) * 8));
  k_score<<<grid, 256, 0, st>>>(q, a, policy, n, k0, k1, k2);
  KX_CHECK_LAUNCH();
}

int keygen_grid(int64_t n, int sms) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n / 4 + 511) / 512, int64_t(sms) * 8)));
}


__global__ void __launch_bounds__(256) k_order_init(OrderInit in) { order_reset(in); }

OrderResultDev launch_order(const QueueDev& q, const AgentsDev& a, const OrderParams& op,
                            int64_t n, OrderWorkspace& ws, int sms, cudaStream_t st,
                            PhaseProfiler* prof, const OrderHooks* hooks) {
  PhaseProfiler dummy;
  PhaseProfiler& P = prof ? *prof : dummy;
  const double N = static_cast<double>(n);
  OrderResultDev res{};
  const int passes = op.key_bits / kRadixBits;
  // the per-order reset (header counters, the first radix pass's look-back
  // array, and whatever the caller's hooks add: the tick's admitted flags
  // and sample counters) runs inside the sample launch
  OrderInit in{};
  in.hdr = static_cast<uint32_t*>(ws.small_hdr);
  in.hdr_words = static_cast<int>(ws.small_hdr_bytes / 4);
  if (hooks) {
    in.words = hooks->zero_words;
    in.n_words = hooks->n_zero_words;
    in.bytes = hooks->zero_bytes;
    in.n_bytes = hooks->n_zero_bytes;
  }
  in.lb = reinterpret_cast<uint4*>(ws.lookback);
  in.lb_vecs = n > 0 ? (n + kSortTile - 1) / kSortTile * kRadix / 4 : 0;
  if (n == 0) {
    k_order_init<<<1, 256, 0, st>>>(in);
    KX_CHECK_LAUNCH();
    k_pool_offsets<<<1, 32, 0, st>>>(ws.pool_counts, op.n_pools, ws.pool_offsets);
    KX_CHECK_LAUNCH();
    if (hooks && hooks->after_keys) hooks->after_keys();
    if (hooks && hooks->before_key_overwrite) hooks->before_key_overwrite();
    res.perm = ws.vals[0];
    res.keys = ws.keys[0];
    return res;
  }
  const int grid = keygen_grid(n, sms);
  {
    // sampled window: ~256K requests (every request below that)
    const int64_t stride = sample_stride(n);
    const int64_t blocks = (n + stride - 1) / stride;  // sample windows
    P.begin("pool_sample", double(blocks) * kSampleLen * 12.0, st);
    k_pool_sample<<<static_cast<unsigned>((blocks + kSampleWins - 1) / kSampleWins), kSampleLen * kSampleWins, 0,
                    st>>>(q, a, op, n, stride, blocks, ws.ranges,
                                                                        ws.range_stage, ws.sample_done, in);
    KX_CHECK_LAUNCH();
    P.end(st);
  }
  if (hooks && hooks->before_keygen) hooks->before_keygen();
  // reads agent + primary time (12 B), writes the compact key (4 B)
  P.begin("keygen_hist", N * 16.0, st);
  {
    const size_t dyn = size_t(op.n_pools) * (8 + 8 + 8 + 4);
    const KeygenSpec sp = hooks ? hooks->spec : KeygenSpec{};
    // class ranks must fit 16 bits for the packed shared table
    if (op.n_agents <= kKeygenAgents && op.class_bits <= 16 && op.n_pools <= 65536)
      k_keygen<true><<<grid, 256, dyn, st>>>(q, a, op, n, ws.ranges, ws.keys[0], ws.hist,
                                             ws.pool_counts, ws.error_flags, sp);
    else
      k_keygen<false><<<grid, 256, dyn, st>>>(q, a, op, n, ws.ranges, ws.keys[0], ws.hist,
                                              ws.pool_counts, ws.error_flags, sp);
  }
  KX_CHECK_LAUNCH();
  P.end(st);
  // compact keys, histograms and pool counts ready (the hook's consumers do
  // not read the pool offsets, computed next)
  if (hooks && hooks->after_keys) hooks->after_keys();
  // (pass p scans its raw digit counts itself; pass p counts digit p + 1)
  k_pool_offsets<<<1, 32, 0, st>>>(ws.pool_counts, op.n_pools, ws.pool_offsets);
  KX_CHECK_LAUNCH();
  cudaStreamCaptureStatus cap_status = cudaStreamCaptureStatusNone;
  KX_CUDA(cudaStreamIsCapturing(st, &cap_status));
  const char* dump = cap_status == cudaStreamCaptureStatusNone ? getenv("KX_DUMP_KEYS") : nullptr;
  if (dump) {  // diagnostics: the compact keys, raw u32 (not while a graph is captured)
    std::vector<uint32_t> hk(static_cast<size_t>(n));
    KX_CUDA(cudaMemcpyAsync(hk.data(), ws.keys[0], size_t(n) * 4, cudaMemcpyDeviceToHost, st));
    KX_CUDA(cudaStreamSynchronize(st));
    if (FILE* f = fopen(dump, "wb")) {
      fwrite(hk.data(), 4, hk.size(), f);
      fclose(f);
    }
  }

  const int64_t tiles = (n + kSortTile - 1) / kSortTile;
  const size_t smem = sort_dyn_smem<uint32_t>();
  int cur = 0;
  for (int p = 0; p < passes; ++p) {
    uint32_t* const lb = ws.lookback + (p & 1) * size_t(tiles) * kRadix;
    uint32_t* const lb_next = p + 1 < passes ? ws.lookback + ((p + 1) & 1) * size_t(tiles) * kRadix : nullptr;
    // key (4 B) [+ index (4 B) after the first pass] in, key + index out
    P.begin("radix_pass", N * (p == 0 ? 12.0 : 16.0), st);
    {
      static const char* variants = getenv("KX_SORT_RANK");  // experiment knob, per pass
      const int v = (variants && int(strlen(variants)) > p) ? variants[p] - '0' : kSortRankDefault[p < 4 ? p : 3];
      const uint32_t* vin = p == 0 ? nullptr : ws.vals[cur];
      uint32_t* nh = p + 1 < passes ? ws.hist + (p + 1) * kRadix : nullptr;
      const unsigned g = static_cast<unsigned>(tiles);
      if (v == 1)
        k_onesweep_pass<uint32_t, 1><<<g, kSortThreads, smem, st>>>(ws.keys[cur], ws.keys[cur ^ 1], vin,
            ws.vals[cur ^ 1], n, p * kRadixBits, ws.hist + p * kRadix, lb, lb_next, ws.tile_counters + p, 1, nh, (p + 1) * kRadixBits);
      else if (v == 2)
        k_onesweep_pass<uint32_t, 2><<<g, kSortThreads, smem, st>>>(ws.keys[cur], ws.keys[cur ^ 1], vin,
            ws.vals[cur ^ 1], n, p * kRadixBits, ws.hist + p * kRadix, lb, lb_next, ws.tile_counters + p, 1, nh, (p + 1) * kRadixBits);
      else
        k_onesweep_pass<uint32_t, 0><<<g, kSortThreads, smem, st>>>(ws.keys[cur], ws.keys[cur ^ 1], vin,
            ws.vals[cur ^ 1], n, p * kRadixBits, ws.hist + p * kRadix, lb, lb_next, ws.tile_counters + p, 1, nh, (p + 1) * kRadixBits);
    }
    KX_CHECK_LAUNCH();
    P.end(st);
    cur ^= 1;
    // pass 1 overwrites keys[0]: readers of the original keys finish first
    if (p == 0 && hooks && hooks->before_key_overwrite) hooks->before_key_overwrite();
  }
  res.keys = ws.keys[cur];
  res.perm = ws.vals[cur];

  // finds the runs of equal compact keys (reads the sorted keys, 4 B) and
  // fixes the short ones; their exact tuples are gathered
  P.begin("tie_fix", N * 4.0, st);
  k_tie_fix<<<static_cast<unsigned>((n + kTieChunk - 1) / kTieChunk), 256, 0, st>>>(
      q, op.policy, res.keys, res.perm, n, ws.big_starts, ws.big_lens, ws.n_big, ws.tie_cap);
  KX_CHECK_LAUNCH();
  k_tie_fix_big<<<sms, kBigThreads, 0, st>>>(q, op.policy, res.perm, ws.vals[cur ^ 1],
                                             ws.big_starts, ws.big_lens, ws.n_big, ws.tie_cap);
  KX_CHECK_LAUNCH();
  P.end(st);
  return res;
}



// Module lazy loading (CUDA 12 default) loads a kernel at its first launch
// and may wait for the device to drain while doing so; the overlapped tick
// has CTAs that wait on other kernels, so every kernel of the tick is
// loaded up front.
template <typename F>
static void preload(F f) {
  cudaFuncAttributes attr;
  KX_CUDA(cudaFuncGetAttributes(&attr, f));
}

void configure_sort_kernels() {
  preload(k_scan_hist);
  preload(k_pool_sample);
  preload(k_sample_keys);
  preload(k_spec_bound);
  preload(k_keygen<true>);
  preload(k_keygen<false>);
  preload(k_pool_offsets);
  preload(k_tie_fix);
  preload(k_tie_fix_big);
  preload(k_order_init);
  preload(k_onesweep_pass<uint32_t, 0>);
  preload(k_onesweep_pass<uint32_t, 1>);
  preload(k_onesweep_pass<uint32_t, 2>);
  KX_CUDA(cudaFuncSetAttribute(k_spec_bound, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(sizeof(uint32_t) * kSpecMax)));
  for (auto f : {k_onesweep_pass<uint32_t, 0>, k_onesweep_pass<uint32_t, 1>, k_onesweep_pass<uint32_t, 2>})
    KX_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(sort_dyn_smem<uint32_t>())));
}

}  // namespace kx

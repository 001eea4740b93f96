// §8(f)3: profiler ingestion on the device (K9).
//
// Replaces EmpiricalDistribution::add (distribution.cpp:91-111) with its
// doubling-checkpoint convergence test (check_convergence, 113-123) behind
// LatencyProfiler::record_remaining / record_execution (profiler.cpp:20-50).
// One warp per distribution (kind x agent) applies that distribution's
// samples of a batch in arrival order; distributions are independent, so the
// batch is exact however it is split over warps. Per sample:
//   * the sorted window lives in shared memory: std::lower_bound is a
//     32-ary search (every lane probes one position per step), the insert
//     an order-preserving warp shift;
//   * with window_cap > 0 the arrival ring (std::deque) lives next to it; the
//     oldest sample is evicted with the same search + shift;
//   * at total_added == next_checkpoint: W1(snapshot, samples) with the
//     reference's integer quantile walk (kx_w1.cuh, bit-exact), the mean as
//     the reference's sequential sum, tau = max(threshold * mean, 1e-12),
//     then snapshot = samples (a warp copy to global memory).
// Distributions whose retained window does not fit shared memory run the
// same code on global memory.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kx_common.cuh"
#include "kx_profiler.cuh"
#include "../../include/kairos_b200.h"
#include "kx_w1.cuh"

namespace kx {

namespace {

// std::lower_bound over s[0, n): first position with s[pos] >= v.
__device__ __forceinline__ int64_t warp_lower_bound(const double* s, int64_t n, double v) {
  const int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = n;
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t idx = lo + lane * step;
    const uint32_t m = __ballot_sync(0xffffffffu, idx < hi && s[idx] < v);
    const int c = __popc(m);  // sampled positions below v: a prefix (sorted)
    if (c == 0) return lo;
    const int64_t nlo = lo + int64_t(c - 1) * step + 1;
    const int64_t nhi = lo + int64_t(c) * step;
    lo = nlo;
    hi = nhi < hi ? nhi : hi;
  }
  const uint32_t m = __ballot_sync(0xffffffffu, lo + lane < hi && s[lo + lane] < v);
  return lo + __popc(m);
}

// s[pos + 1 .. n] = s[pos .. n - 1] (order kept), top chunk first.
__device__ __forceinline__ void warp_shift_up(double* s, int64_t pos, int64_t n) {
  const int lane = threadIdx.x & 31;
  for (int64_t top = n; top > pos; top -= 32) {
    const int64_t idx = top - 1 - lane;
    double t = 0.0;
    if (idx >= pos) t = s[idx];
    __syncwarp();
    if (idx >= pos) s[idx + 1] = t;
    __syncwarp();
  }
}

// s[pos .. n - 2] = s[pos + 1 .. n - 1], bottom chunk first.
__device__ __forceinline__ void warp_shift_down(double* s, int64_t pos, int64_t n) {
  const int lane = threadIdx.x & 31;
  for (int64_t b = pos + 1; b < n; b += 32) {
    const int64_t idx = b + lane;
    double t = 0.0;
    if (idx < n) t = s[idx];
    __syncwarp();
    if (idx < n) s[idx - 1] = t;
    __syncwarp();
  }
}

}  // namespace

// Block = one warp = one distribution. Samples of distribution d in
// [off[d], off[d+1]) in arrival order; item[k] is the caller's index of the
// record (workflow) sample k belongs to.
template <bool kSmem>
__global__ void __launch_bounds__(32)
k_dist_ingest(DistDev dd, int32_t n_dist, const int64_t* __restrict__ off, const double* __restrict__ values,
              const int64_t* __restrict__ item, int* __restrict__ status) {
  extern __shared__ __align__(16) double dist_smem[];
  const int d = blockIdx.x;
  const int lane = threadIdx.x;
  if (d >= n_dist || off[d] == off[d + 1]) return;
  const DistCfg cfg = dd.cfg[d];
  const int64_t cap = dd.cap;
  double* gs = dd.sorted + int64_t(d) * cap;
  double* gr = dd.ring + int64_t(d) * cap;
  double* s = kSmem ? dist_smem : gs;
  double* ring = kSmem ? dist_smem + cap : gr;
  int64_t n = dd.n[d];
  const bool windowed = cfg.window_cap > 0;
  int64_t head = dd.ring_head[d];  // oldest retained sample (ring holds the n retained ones)
  if (kSmem) {
    for (int64_t j = lane; j < n; j += 32) {
      s[j] = gs[j];
      if (windowed) ring[j] = gr[(head + j) % cap];
    }
    head = 0;
    __syncwarp();
  }
  uint64_t total = dd.total[d];
  uint64_t next_cp = dd.next_cp[d];
  uint8_t conv = dd.conv[d];
  double last = dd.last_dist[d];
  int64_t conv_item = -1;
  int st = KX_OK;
  for (int64_t k = off[d]; k < off[d + 1]; ++k) {
    const double v = values[k];
    if (n + 1 > cap) {  // the retained window must fit before eviction
      st = KX_ERR_CAPACITY;
      break;
    }
    // sorted_.insert(lower_bound(value), value)
    const int64_t pos = warp_lower_bound(s, n, v);
    warp_shift_up(s, pos, n);
    if (lane == 0) s[pos] = v;
    ++n;
    if (windowed) {
      if (lane == 0) ring[(head + n - 1) % cap] = v;  // arrival_order_.push_back
      __syncwarp();
      if (uint64_t(n) > uint64_t(cfg.window_cap)) {  // evict the oldest
        const double oldest = ring[head];
        head = (head + 1) % cap;
        const int64_t ep = warp_lower_bound(s, n, oldest);
        warp_shift_down(s, ep, n);
        --n;
      }
    }
    __syncwarp();
    ++total;
    if (total == next_cp) {  // check_convergence (distribution.cpp:113-123)
      const int64_t sn = dd.snap_n[d];
      double* snap = dd.snap + int64_t(d) * cap;
      if (sn > 0) {
        double w = 0.0, sum = 0.0;
        if (lane == 0) {
          w = w1_walk(snap, uint64_t(sn), s, uint64_t(n));
          for (int64_t j = 0; j < n; ++j) sum = __dadd_rn(sum, s[j]);  // mean(): sequential
        }
        w = __shfl_sync(0xffffffffu, w, 0);
        sum = __shfl_sync(0xffffffffu, sum, 0);
        const double mean = __ddiv_rn(sum, static_cast<double>(n));
        const double t = __dmul_rn(cfg.threshold, mean);
        const double tau = t > 1e-12 ? t : 1e-12;  // std::max(t, 1e-12)
        last = w;
        if (w < tau) {
          if (!conv && conv_item < 0) conv_item = item ? item[k] : k;
          conv = 1;
        }
      }
      __syncwarp();
      for (int64_t j = lane; j < n; j += 32) snap[j] = s[j];  // snapshot_ = sorted_
      if (lane == 0) dd.snap_n[d] = n;
      __syncwarp();
      next_cp *= 2;
    }
  }
  __syncwarp();
  if (kSmem) {
    for (int64_t j = lane; j < n; j += 32) {
      gs[j] = s[j];
      if (windowed) gr[j] = ring[(head + j) % cap];
    }
    head = 0;
  }
  if (lane == 0) {
    dd.n[d] = n;
    dd.ring_head[d] = head;
    dd.total[d] = total;
    dd.next_cp[d] = next_cp;
    dd.conv[d] = conv;
    dd.last_dist[d] = last;
    dd.conv_item[d] = conv_item;
    if (st != KX_OK) atomicExch(status, st);
  }
}

size_t dist_smem_bytes(int64_t cap) { return size_t(cap) * 2 * sizeof(double); }

void launch_dist_ingest(const DistDev& dd, int32_t n_dist, const int64_t* off, const double* values,
                        const int64_t* item, int* status, cudaStream_t st) {
  if (n_dist == 0) return;
  const size_t smem = dist_smem_bytes(dd.cap);
  if (smem <= size_t(kDistSmemMax)) {
    static bool configured = false;
    if (!configured) {
      KX_CUDA(cudaFuncSetAttribute(k_dist_ingest<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kDistSmemMax));
      configured = true;
    }
    k_dist_ingest<true><<<n_dist, 32, smem, st>>>(dd, n_dist, off, values, item, status);
  } else {
    k_dist_ingest<false><<<n_dist, 32, 0, st>>>(dd, n_dist, off, values, item, status);
  }
  KX_CHECK_LAUNCH();
}

}  // namespace kx

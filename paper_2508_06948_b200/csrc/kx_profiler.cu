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

namespace kx {

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
  DistScal ds{n, head, dd.snap_n[d], dd.total[d], dd.next_cp[d], dd.conv[d], dd.last_dist[d]};
  double* snap = dd.snap + int64_t(d) * cap;
  int64_t conv_item = -1;
  int st = KX_OK;
  for (int64_t k = off[d]; k < off[d + 1]; ++k) {
    bool newly = false;
    if (!dist_add_warp(s, ring, snap, cap, cfg, ds, values[k], &newly)) {
      st = KX_ERR_CAPACITY;  // the retained window must fit before eviction
      break;
    }
    if (newly && conv_item < 0) conv_item = item ? item[k] : k;
  }
  n = ds.n;
  head = ds.head;
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
    dd.snap_n[d] = ds.snap_n;
    dd.total[d] = ds.total;
    dd.next_cp[d] = ds.next_cp;
    dd.conv[d] = static_cast<uint8_t>(ds.conv);
    dd.last_dist[d] = ds.last;
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
    static std::once_flag configured[kMaxDevices];
    once_per_device(configured, [] {
      KX_CUDA(cudaFuncSetAttribute(k_dist_ingest<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kDistSmemMax));
    });
    k_dist_ingest<true><<<n_dist, 32, smem, st>>>(dd, n_dist, off, values, item, status);
  } else {
    k_dist_ingest<false><<<n_dist, 32, 0, st>>>(dd, n_dist, off, values, item, status);
  }
  KX_CHECK_LAUNCH();
}

}  // namespace kx

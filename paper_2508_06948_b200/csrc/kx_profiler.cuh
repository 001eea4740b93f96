// Host-side interface of the profiler-ingestion kernel (kx_profiler.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "kx_dist.cuh"

namespace kx {

// EmpiricalDistribution state (distribution.hpp:72-82) of n_dist
// distributions, each with room for `cap` retained samples.
struct DistDev {
  int64_t cap;
  const DistCfg* cfg;   // [n_dist]
  double* sorted;       // [n_dist * cap] sorted_
  double* ring;         // [n_dist * cap] arrival_order_ (window_cap > 0), ring from ring_head
  double* snap;         // [n_dist * cap] snapshot_
  int64_t* n;           // sorted_.size()
  int64_t* ring_head;
  int64_t* snap_n;
  uint64_t* total;      // total_added_
  uint64_t* next_cp;    // next_checkpoint_
  uint8_t* conv;        // converged_
  double* last_dist;    // last_checkpoint_distance_
  int64_t* conv_item;   // this batch: item index whose sample converged the distribution, -1 none
};

constexpr int kDistSmemMax = 200 * 1024;

void launch_dist_ingest(const DistDev& dd, int32_t n_dist, const int64_t* off, const double* values,
                        const int64_t* item, int* status, cudaStream_t st);

}  // namespace kx

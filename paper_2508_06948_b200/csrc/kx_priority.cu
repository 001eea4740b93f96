// §8(f)2: the priority table's W1 distance matrix on the device.
//
// Replaces build_matrix (priority.cpp:15-46) behind
// build_distance_matrix_from_samples (priority.cpp:60-65): labels are the
// agents in order plus the anchor (a single sample 0.0) last, d[i][j] =
// wasserstein_1d(samples_i, samples_j) (distribution.cpp:9-31), symmetric,
// zero diagonal. One thread per pair (i < j) walks the merged quantile grid
// in the reference's exact integer steps and accumulates
// (nxt - cur) * |a[i] - b[j]| in the reference's order with correctly rounded
// multiply and add (the site is an FMA hazard), then divides by
// na * nb: bit-identical to the CPU. Classical MDS on the matrix stays on the
// host (Eigen's eigensolver is not reproducible on the device).
#include <cuda_runtime.h>
#include <stdint.h>

#include "kx_common.cuh"
#include "kx_dist.cuh"
#include "kx_w1.cuh"

namespace kx {

__global__ void k_w1_matrix(int32_t n_agents, const int64_t* __restrict__ off,
                            const double* __restrict__ samples, double* __restrict__ d) {
  const int m = n_agents + 1;  // + anchor
  const int64_t pairs = int64_t(m) * (m - 1) / 2;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const double anchor = 0.0;
  for (int64_t pid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; pid < pairs; pid += stride) {
    // pair index -> (i, j), i < j, row-major over the upper triangle
    int64_t i = 0, rem = pid;
    while (rem >= m - 1 - i) {
      rem -= m - 1 - i;
      ++i;
    }
    const int64_t j = i + 1 + rem;
    const double* a = i < n_agents ? samples + off[i] : &anchor;
    const double* b = j < n_agents ? samples + off[j] : &anchor;
    const uint64_t na = i < n_agents ? uint64_t(off[i + 1] - off[i]) : 1u;
    const uint64_t nb = j < n_agents ? uint64_t(off[j + 1] - off[j]) : 1u;
    const double w = w1_walk(a, na, b, nb);
    d[i * m + j] = w;
    d[j * m + i] = w;
  }
}

__global__ void k_zero_diag(int m, double* d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) d[int64_t(i) * m + i] = 0.0;
}

void launch_w1_matrix(int32_t n_agents, const int64_t* off, const double* samples, double* d, int sms,
                      cudaStream_t st) {
  const int m = n_agents + 1;
  const int64_t pairs = int64_t(m) * (m - 1) / 2;
  k_zero_diag<<<(m + 255) / 256, 256, 0, st>>>(m, d);
  KX_CHECK_LAUNCH();
  if (pairs == 0) return;
  const int grid = static_cast<int>(std::min<int64_t>((pairs + 127) / 128, int64_t(sms) * 16));
  k_w1_matrix<<<grid, 128, 0, st>>>(n_agents, off, samples, d);
  KX_CHECK_LAUNCH();
}

// ProfilerSnapshot::expected_exec_time (profiler.cpp:11-16) for every agent
// of a snapshot: warp per agent, mode_estimate (distribution.cpp:46-86) of
// its sorted execution samples, `fallback` for an empty set.
__global__ void __launch_bounds__(128)
k_expected_T(int32_t n_agents, const int64_t* __restrict__ off, const double* __restrict__ samples,
             int64_t min_samples, double fallback, double* __restrict__ out) {
  const int a = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (a >= n_agents) return;
  const int64_t n = off[a + 1] - off[a];
  const double T = n == 0 ? fallback : mode_estimate_warp(samples + off[a], n, min_samples);
  if ((threadIdx.x & 31) == 0) out[a] = T;
}

void launch_expected_T(int32_t n_agents, const int64_t* off, const double* samples, int64_t min_samples,
                       double fallback, double* out, cudaStream_t st) {
  if (n_agents == 0) return;
  k_expected_T<<<(n_agents + 3) / 4, 128, 0, st>>>(n_agents, off, samples, min_samples, fallback, out);
  KX_CHECK_LAUNCH();
}

}  // namespace kx

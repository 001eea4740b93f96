// K1: workflow-orchestrator remaining-latency DP, one warp per workflow.
//
//   finalize_instance        workload.cpp:292-315
//     uid = next_uid++ (call order), pure_exec = prompt/prefill + target/decode,
//     reverse sweep remaining = pure_exec + max(0, children's remaining)
//   LatencyProfiler::record_remaining's arithmetic   profiler.cpp:31-50
//     finish = max exec_end (seeded with the first record),
//     sample = finish - exec_start
//
// Every call has at most one parent with a smaller node id (calls are
// created parents-first, workload.cpp:266-283), so each workflow is a tree
// whose reverse topological order is node order reversed. Workflows of up to
// 32 calls are evaluated level by level in registers (lane = node, children
// pushed to parents with warp shuffles); longer ones by a reverse sweep.
// Only +, / and max are involved, so results are bit-identical to the
// reference (max is exact and order-free for non-NaN values).
#include <cuda_runtime.h>
#include <stdint.h>

#include "kx_common.cuh"

namespace kx {

__global__ void k_orchestrator_dp(int64_t n_wf, const int64_t* __restrict__ off,
                                  const int32_t* __restrict__ parent,
                                  const int64_t* __restrict__ prompt,
                                  const int64_t* __restrict__ target, double prefill_rate,
                                  double decode_rate, uint64_t uid_base,
                                  uint64_t* __restrict__ uid_out, double* __restrict__ pure_out,
                                  double* __restrict__ rem_out, int* __restrict__ error) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n_wf; w += warps) {
    const int64_t b = off[w];
    const int64_t n = off[w + 1] - b;
    // uid and pure_exec (workload.cpp:300-305), all calls.
    for (int64_t c = lane; c < n; c += 32) {
      const int64_t g = b + c;
      uid_out[g] = uid_base + static_cast<uint64_t>(g);
      pure_out[g] = __dadd_rn(__ddiv_rn(static_cast<double>(prompt[g]), prefill_rate),
                              __ddiv_rn(static_cast<double>(target[g]), decode_rate));
      const int32_t p = parent[g];
      if (p < -1 || p >= c) atomicOr(error, 1);  // not parents-first
    }
    if (n <= 32) {
      const bool act = lane < n;
      const int32_t par = act ? parent[b + lane] : -1;
      const double pure = act ? pure_out[b + lane] : 0.0;
      // depth by pointer jumping over the parent links
      int d = (act && par < 0) ? 0 : -1;
      for (int it = 0; it < 32; ++it) {
        const int pd = __shfl_sync(0xffffffffu, d, par >= 0 && par < 32 ? par : 0);
        if (act && d < 0 && par >= 0 && pd >= 0) d = pd + 1;
        if (__all_sync(0xffffffffu, !act || d >= 0)) break;
      }
      int dmax = d;
      for (int o = 16; o > 0; o >>= 1) dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
      double tail = 0.0, rem = 0.0;
      for (int level = dmax; level >= 0; --level) {
        if (act && d == level) rem = __dadd_rn(pure, tail);
        for (int src = 0; src < n; ++src) {
          const double v = __shfl_sync(0xffffffffu, rem, src);
          const int ps = __shfl_sync(0xffffffffu, par, src);
          const int ds = __shfl_sync(0xffffffffu, d, src);
          if (ds == level && ps == lane && tail < v) tail = v;  // std::max(tail, child)
        }
      }
      if (act) rem_out[b + lane] = rem;
    } else {
      // Reverse sweep with rem_out as the tail accumulator.
      for (int64_t c = lane; c < n; c += 32) rem_out[b + c] = 0.0;
      __syncwarp();
      if (lane == 0) {
        for (int64_t c = n - 1; c >= 0; --c) {
          const double r = __dadd_rn(pure_out[b + c], rem_out[b + c]);
          rem_out[b + c] = r;
          const int32_t p = parent[b + c];
          if (p >= 0 && p < c && rem_out[b + p] < r) rem_out[b + p] = r;
        }
      }
      __syncwarp();
    }
  }
}

__global__ void k_record_remaining(int64_t n_wf, const int64_t* __restrict__ off,
                                   const double* __restrict__ exec_start,
                                   const double* __restrict__ exec_end,
                                   double* __restrict__ finish_out, double* __restrict__ samples) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n_wf; w += warps) {
    const int64_t b = off[w];
    const int64_t n = off[w + 1] - b;
    if (n <= 0) continue;  // empty record list: nothing recorded
    double fin = exec_end[b];
    for (int64_t r = lane; r < n; r += 32) fin = fmax(fin, exec_end[b + r]);
    for (int o = 16; o > 0; o >>= 1) fin = fmax(fin, __shfl_xor_sync(0xffffffffu, fin, o));
    for (int64_t r = lane; r < n; r += 32) samples[b + r] = __dsub_rn(fin, exec_start[b + r]);
    if (lane == 0) finish_out[w] = fin;
  }
}

void launch_orchestrator_dp(int64_t n_wf, const int64_t* off, const int32_t* parent,
                            const int64_t* prompt, const int64_t* target, double prefill,
                            double decode, uint64_t uid_base, uint64_t* uid_out, double* pure_out,
                            double* rem_out, int* error, int sms, cudaStream_t st) {
  if (n_wf <= 0) return;
  const int64_t want = (n_wf * 32 + 255) / 256;
  const int grid = static_cast<int>(want < int64_t(sms) * 16 ? want : int64_t(sms) * 16);
  k_orchestrator_dp<<<grid, 256, 0, st>>>(n_wf, off, parent, prompt, target, prefill, decode,
                                          uid_base, uid_out, pure_out, rem_out, error);
  KX_CHECK_LAUNCH();
}

void launch_record_remaining(int64_t n_wf, const int64_t* off, const double* es, const double* ee,
                             double* fin, double* samples, int sms, cudaStream_t st) {
  if (n_wf <= 0) return;
  const int64_t want = (n_wf * 32 + 255) / 256;
  const int grid = static_cast<int>(want < int64_t(sms) * 16 ? want : int64_t(sms) * 16);
  k_record_remaining<<<grid, 256, 0, st>>>(n_wf, off, es, ee, fin, samples);
  KX_CHECK_LAUNCH();
}

}  // namespace kx

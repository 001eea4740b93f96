// K8: pairwise sorting accuracy (priority.cpp:165-189) in O(N log^2 N).
//
// The reference scores a schedule by walking every pair i < j (optionally
// only cross-agent pairs): +1.0 when remaining_i < remaining_j, +0.5 on a
// tie, over the number of compared pairs — O(N^2) with a map lookup per pair
// (91% of run_cell time). Those sums are exact multiples of 0.5
// (< 2^53 for any N the reference could run), so they equal integer counts:
//   correct = concordant + ties / 2,   concordant = pairs - ties - inversions
// where inversions (i < j, x_i > x_j) come from a bottom-up merge sort in
// which every element finds its rank in the sibling run by binary search,
// and ties from runs of equal values in the sorted result. Cross-agent scope
// subtracts the same counts taken within each agent: a stable partition by
// agent makes composite keys (agent, x) whose inversions are exactly the
// within-agent ones. One division at the end, as in the reference.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "../../include/kairos_b200.h"
#include "kx_common.cuh"

namespace kx {

namespace {

struct Key {
  uint32_t hi;  // agent (composite pass) or 0
  uint64_t lo;  // order-preserving bits of the remaining latency
};

__device__ __forceinline__ bool key_lt(const Key& a, const Key& b) {
  return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
}
__device__ __forceinline__ bool key_le(const Key& a, const Key& b) { return !key_lt(b, a); }

// One merge level: runs of width w in src are merged pairwise into dst.
// Left elements precede equal right ones (stable); each right element adds
// the number of strictly greater left elements to the inversion count.
__global__ void k_merge_level(const uint32_t* __restrict__ shi, const uint64_t* __restrict__ slo,
                              uint32_t* __restrict__ dhi, uint64_t* __restrict__ dlo, int64_t n,
                              int64_t w, unsigned long long* __restrict__ inversions) {
  unsigned long long local = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t a0 = (i / (2 * w)) * 2 * w;
    const int64_t b0 = a0 + w < n ? a0 + w : n;
    const int64_t b1 = a0 + 2 * w < n ? a0 + 2 * w : n;
    const Key x{shi[i], slo[i]};
    int64_t lo, hi;
    const bool left = i < b0;
    if (left) {
      lo = b0;
      hi = b1;
      while (lo < hi) {  // count right elements < x
        const int64_t m = (lo + hi) >> 1;
        if (key_lt(Key{shi[m], slo[m]}, x)) lo = m + 1;
        else hi = m;
      }
      const int64_t pos = a0 + (i - a0) + (lo - b0);
      dhi[pos] = x.hi;
      dlo[pos] = x.lo;
    } else {
      lo = a0;
      hi = b0;
      while (lo < hi) {  // count left elements <= x
        const int64_t m = (lo + hi) >> 1;
        if (key_le(Key{shi[m], slo[m]}, x)) lo = m + 1;
        else hi = m;
      }
      local += static_cast<unsigned long long>(b0 - lo);  // left elements > x
      const int64_t pos = a0 + (i - b0) + (lo - a0);
      dhi[pos] = x.hi;
      dlo[pos] = x.lo;
    }
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(inversions, local);
}

// Pairs of equal keys in a sorted array: sum over runs of C(len, 2).
__global__ void k_tie_pairs(const uint32_t* __restrict__ hi, const uint64_t* __restrict__ lo, int64_t n,
                            unsigned long long* __restrict__ ties) {
  unsigned long long local = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    // element i pairs with every earlier equal element of its run
    if (i > 0 && hi[i] == hi[i - 1] && lo[i] == lo[i - 1]) {
      int64_t s = i - 1;
      // distance to the run start, found by doubling then bisection
      int64_t step = 1;
      while (s - step >= 0 && hi[s - step] == hi[i] && lo[s - step] == lo[i]) {
        s -= step;
        step <<= 1;
      }
      while (step > 1) {
        step >>= 1;
        if (s - step >= 0 && hi[s - step] == hi[i] && lo[s - step] == lo[i]) s -= step;
      }
      local += static_cast<unsigned long long>(i - s);
    }
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(ties, local);
}

// Inversions and tie pairs of the key sequence (hi, lo) of length n.
void count_sequence(uint32_t* hi, uint64_t* lo, uint32_t* hi2, uint64_t* lo2, int64_t n,
                    unsigned long long* d_inv, unsigned long long* d_ties, int sms, cudaStream_t st) {
  uint32_t* sh = hi;
  uint64_t* sl = lo;
  uint32_t* dh = hi2;
  uint64_t* dl = lo2;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, int64_t(sms) * 8));
  for (int64_t w = 1; w < n; w <<= 1) {
    k_merge_level<<<grid, 256, 0, st>>>(sh, sl, dh, dl, n, w, d_inv);
    KX_CHECK_LAUNCH();
    std::swap(sh, dh);
    std::swap(sl, dl);
  }
  k_tie_pairs<<<grid, 256, 0, st>>>(sh, sl, n, d_ties);
  KX_CHECK_LAUNCH();
}

}  // namespace

// Host driver: schedule-ordered (agent, remaining, present) arrays on host.
void sorting_accuracy(int64_t n, const int32_t* agent, const double* remaining, const uint8_t* present,
                      int32_t scope_all, uint64_t* pairs_out, double* correct_out, int sms,
                      cudaStream_t st) {
  // Filter the comparable requests (reference skips missing remaining).
  std::vector<uint32_t> ag;
  std::vector<uint64_t> x;
  ag.reserve(static_cast<size_t>(n));
  x.reserve(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    if (present && !present[i]) continue;
    if (remaining[i] != remaining[i]) throw KxError(KX_ERR_INVALID, "NaN remaining latency");
    double v = remaining[i];
    if (v == 0.0) v = 0.0;  // -0 == +0
    uint64_t u;
    std::memcpy(&u, &v, 8);
    u = (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
    ag.push_back(static_cast<uint32_t>(agent[i]));
    x.push_back(u);
  }
  const int64_t m = static_cast<int64_t>(x.size());
  *pairs_out = 0;
  *correct_out = 0.0;
  if (m < 2) return;
  // Stable partition by agent (counting sort) for the within-agent counts.
  uint32_t amax = 0;
  for (uint32_t a : ag) amax = std::max(amax, a);
  std::vector<int64_t> cnt(static_cast<size_t>(amax) + 2, 0);
  for (uint32_t a : ag) cnt[a + 1] += 1;
  unsigned long long same_pairs = 0;
  for (size_t a = 1; a < cnt.size(); ++a) {
    const unsigned long long c = static_cast<unsigned long long>(cnt[a]);
    same_pairs += c * (c - 1) / 2;
    cnt[a] += cnt[a - 1];
  }
  std::vector<uint32_t> ph(static_cast<size_t>(m));
  std::vector<uint64_t> pl(static_cast<size_t>(m));
  for (int64_t i = 0; i < m; ++i) {
    const int64_t p = cnt[ag[i]]++;
    ph[p] = ag[i];
    pl[p] = x[i];
  }
  const size_t N = static_cast<size_t>(m);
  uint32_t *h1 = nullptr, *h2 = nullptr;
  uint64_t *l1 = nullptr, *l2 = nullptr;
  unsigned long long* d = nullptr;
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&h1), N * 4, st));
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&h2), N * 4, st));
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&l1), N * 8, st));
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&l2), N * 8, st));
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), 4 * 8, st));
  KX_CUDA(cudaMemsetAsync(d, 0, 4 * 8, st));
  // (1) whole schedule: keys (0, x)
  KX_CUDA(cudaMemsetAsync(h1, 0, N * 4, st));
  KX_CUDA(cudaMemcpyAsync(l1, x.data(), N * 8, cudaMemcpyHostToDevice, st));
  count_sequence(h1, l1, h2, l2, m, d + 0, d + 1, sms, st);
  // (2) within agents: composite keys over the agent-partitioned schedule
  if (!scope_all) {
    KX_CUDA(cudaMemcpyAsync(h1, ph.data(), N * 4, cudaMemcpyHostToDevice, st));
    KX_CUDA(cudaMemcpyAsync(l1, pl.data(), N * 8, cudaMemcpyHostToDevice, st));
    count_sequence(h1, l1, h2, l2, m, d + 2, d + 3, sms, st);
  }
  unsigned long long c[4] = {0, 0, 0, 0};
  KX_CUDA(cudaMemcpyAsync(c, d, 4 * 8, cudaMemcpyDeviceToHost, st));
  KX_CUDA(cudaFreeAsync(h1, st));
  KX_CUDA(cudaFreeAsync(h2, st));
  KX_CUDA(cudaFreeAsync(l1, st));
  KX_CUDA(cudaFreeAsync(l2, st));
  KX_CUDA(cudaFreeAsync(d, st));
  KX_CUDA(cudaStreamSynchronize(st));
  const unsigned long long all_pairs = static_cast<unsigned long long>(m) * (m - 1) / 2;
  unsigned long long pairs = all_pairs, inv = c[0], ties = c[1];
  if (!scope_all) {
    pairs -= same_pairs;
    inv -= c[2];
    ties -= c[3];
  }
  const unsigned long long conc = pairs - ties - inv;
  *pairs_out = pairs;
  // the reference's running sum of 1.0 / 0.5 terms, exactly
  *correct_out = static_cast<double>(conc) + 0.5 * static_cast<double>(ties);
}

}  // namespace kx

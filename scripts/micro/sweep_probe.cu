// Timing probe only (not product code): the K3 onesweep pass on 16M random
// (u32 key, u32 index) pairs, with the decoupled look-back on and off
// (off = wrong offsets, timing only), to bound what the look-back costs.
#include <cstdio>
#include <vector>
#include <random>
#define KX_PROBE_NO_LOOKBACK_SWITCH 1
#include "../../paper_2508_06948_b200/csrc/kx_sort.cuh"
using namespace kx;
int main() {
  const int64_t n = 16000000;
  std::vector<uint32_t> hk(n);
  std::mt19937 g(1);
  for (auto& x : hk) x = g();
  uint32_t *k0, *k1, *v1, *lb, *hist, *tc;
  cudaMalloc(&k0, n * 4); cudaMalloc(&k1, n * 4); cudaMalloc(&v1, n * 4);
  const int64_t tiles = (n + kSortTile - 1) / kSortTile;
  cudaMalloc(&lb, tiles * kRadix * 4); cudaMalloc(&hist, 4 * kRadix * 4); cudaMalloc(&tc, 64);
  cudaMemcpy(k0, hk.data(), n * 4, cudaMemcpyHostToDevice);
  std::vector<uint32_t> h(kRadix, 0);
  for (auto x : hk) h[x & 255]++;
  uint32_t acc = 0; for (auto& x : h) { uint32_t c = x; x = acc; acc += c; }
  cudaMemcpy(hist, h.data(), kRadix * 4, cudaMemcpyHostToDevice);
  const size_t smem = sort_dyn_smem<uint32_t>();
  cudaFuncSetAttribute(k_onesweep_pass<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode) {
    float best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaMemset(lb, 0, tiles * kRadix * 4); cudaMemset(tc, 0, 64);
      cudaEventRecord(a);
      k_onesweep_pass<uint32_t><<<tiles, kSortThreads, smem>>>(k0, k1, nullptr, v1, n, 0, hist, lb, nullptr, tc, 0, nullptr, 0, mode);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("onesweep pass (%s look-back): %.1f us, %.2f TB/s at 12 B/elem (pass 0)\n", mode ? "NO" : "with", best * 1e3,
           n * 12.0 / (best * 1e-3) / 1e12);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}

// Reference point only (not product code): the K3 onesweep passes
// (kx_sort.cuh, the product's kernel and tile shape) against CUB
// DeviceRadixSort::SortPairs on the same 16M random (u32 key, u32 index)
// pairs, 32 key bits, same output checked; CUDA events, best of 20.
#include <cub/cub.cuh>
#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_2508_06948_b200/csrc/kx_sort.cuh"
using namespace kx;

__global__ void k_scan4(uint32_t* hist) {  // exclusive scan of 4 x 256 bins, warp per pass
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 16000000;
  std::vector<uint32_t> hk(n);
  std::mt19937 g(1);
  for (auto& x : hk) x = g();
  if (argc > 2) {  // keys from a file (KX_DUMP_KEYS of a bench tick)
    FILE* f = fopen(argv[2], "rb");
    if (!f || fread(hk.data(), 4, n, f) != size_t(n)) { fprintf(stderr, "cannot read %s\n", argv[2]); return 1; }
    fclose(f);
  }
  uint32_t *k0, *k1, *v0, *v1, *ck, *cv, *hist, *lb, *tc;
  cudaMalloc(&k0, n * 4); cudaMalloc(&k1, n * 4); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
  cudaMalloc(&ck, n * 4); cudaMalloc(&cv, n * 4);
  const int64_t tiles = (n + kSortTile - 1) / kSortTile;
  cudaMalloc(&hist, 4 * kRadix * 4); cudaMalloc(&lb, tiles * kRadix * 4); cudaMalloc(&tc, 64);
  std::vector<uint32_t> hv(n);
  for (int64_t i = 0; i < n; ++i) hv[i] = uint32_t(i);
  uint32_t *src_k, *src_v;
  cudaMalloc(&src_k, n * 4); cudaMalloc(&src_v, n * 4);
  cudaMemcpy(src_k, hk.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(src_v, hv.data(), n * 4, cudaMemcpyHostToDevice);
  const size_t smem = sort_dyn_smem<uint32_t>();
  cudaFuncSetAttribute(k_onesweep_pass<uint32_t, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto ours = [&]() {  // histograms of the 4 digits, then 4 passes (pass 0 values implicit)
    cudaMemsetAsync(hist, 0, 4 * kRadix * 4);
    cudaMemsetAsync(tc, 0, 64);
    k_upfront_hist<uint32_t><<<148 * 8, 256>>>(src_k, n, 0, 4, hist);
    k_scan4<<<1, 128>>>(hist);
    const uint32_t* kin = src_k;
    const uint32_t* vin = nullptr;
    uint32_t* kout[2] = {k0, k1};
    uint32_t* vout[2] = {v0, v1};
    for (int p = 0; p < 4; ++p) {
      cudaMemsetAsync(lb, 0, tiles * kRadix * 4);
      k_onesweep_pass<uint32_t, 2><<<unsigned(tiles), kSortThreads, smem>>>(
          kin, kout[p & 1], vin, vout[p & 1], n, 8 * p, hist + p * kRadix, lb, nullptr, tc + p, 0, nullptr, 0);
      kin = kout[p & 1];
      vin = vout[p & 1];
    }
  };
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, src_k, ck, src_v, cv, n);
  void* t;
  cudaMalloc(&t, tmp);
  auto cubs = [&]() { cub::DeviceRadixSort::SortPairs(t, tmp, src_k, ck, src_v, cv, n, 0, 32); };
  float best[2] = {1e9f, 1e9f};
  for (int w = 0; w < 3; ++w) { ours(); cubs(); }
  for (int it = 0; it < 20; ++it) {
    for (int m = 0; m < 2; ++m) {
      cudaEventRecord(a);
      if (m == 0) ours(); else cubs();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best[m]) best[m] = ms;
    }
  }
  std::vector<uint32_t> ok(n), ov(n), cuk(n), cuv(n);
  cudaMemcpy(ok.data(), k1, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(ov.data(), v1, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(cuk.data(), ck, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(cuv.data(), cv, n * 4, cudaMemcpyDeviceToHost);
  const bool same = ok == cuk && ov == cuv;
  printf("{\"n\": %lld, \"ours_ms\": %.4f, \"cub_ms\": %.4f, \"ours_GBps_alg\": %.1f, \"cub_GBps_alg\": %.1f, "
         "\"identical\": %s, \"alg_bytes\": %.0f, \"err\": \"%s\"}\n",
         (long long)n, best[0], best[1], 60.0 * n / (best[0] * 1e-3) / 1e9, 64.0 * n / (best[1] * 1e-3) / 1e9,
         same ? "true" : "false", 60.0 * n, cudaGetErrorString(cudaGetLastError()));
  return 0;
}

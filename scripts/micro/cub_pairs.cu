// Reference point only (not product code): CUB DeviceRadixSort::SortPairs on
// 16M (u32 key, u32 value) pairs, 32 key bits, timed with CUDA events.
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <random>
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 16000000;
  std::vector<uint32_t> hk(n), hv(n);
  std::mt19937 g(1);
  for (int i = 0; i < n; ++i) { hk[i] = g(); hv[i] = i; }
  uint32_t *k0, *k1, *v0, *v1;
  cudaMalloc(&k0, n * 4); cudaMalloc(&k1, n * 4); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
  cudaMemcpy(k0, hk.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(v0, hv.data(), n * 4, cudaMemcpyHostToDevice);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, n);
  void* t; cudaMalloc(&t, tmp);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int bits : {32, 24, 16}) {
    for (int w = 0; w < 3; ++w) cub::DeviceRadixSort::SortPairs(t, tmp, k0, k1, v0, v1, n, 0, bits);
    cudaEventRecord(a);
    const int it = 20;
    for (int w = 0; w < it; ++w) cub::DeviceRadixSort::SortPairs(t, tmp, k0, k1, v0, v1, n, 0, bits);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("cub SortPairs n=%d bits=%d: %.3f ms per sort (%.1f us per 8-bit pass)\n", n, bits, ms / it, 1000 * ms / it / (bits / 8));
  }
  return 0;
}

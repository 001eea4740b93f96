// Timing probe only (not product code): host->device bandwidth of pinned
// copies, one stream vs the same bytes split over 2 / 3 streams.
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t n = 320ull << 20;
  char *h, *d;
  cudaMallocHost(&h, n);
  cudaMalloc(&d, n);
  cudaStream_t s[3];
  for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int k : {1, 2, 3, 1}) {
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaDeviceSynchronize();
      cudaEventRecord(a, s[0]);
      for (int j = 1; j < k; ++j) cudaStreamWaitEvent(s[j], a, 0);
      const size_t c = n / k;
      for (int j = 0; j < k; ++j) cudaMemcpyAsync(d + j * c, h + j * c, c, cudaMemcpyHostToDevice, s[j]);
      for (int j = 1; j < k; ++j) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s[j]);
        cudaStreamWaitEvent(s[0], e, 0);
      }
      cudaEventRecord(b, s[0]);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("%d stream(s): %.3f ms, %.1f GB/s\n", k, best, n / (best * 1e-3) / 1e9);
  }
  return 0;
}

// Timing probe only (not product code): single-warp issue rate of FP64
// DADD / DSETP+FSEL and of 32-bit ALU ops on B200 (8 independent chains).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N = 4096;
__global__ void k(double* out, long long* t, double seed) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x + i;
  unsigned u[8];
  for (int i = 0; i < 8; ++i) u[i] = threadIdx.x * 7 + i;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __dadd_rn(a[j], 1.0);
  long long t1 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = a[j] > seed ? a[j] : seed;  // DSETP + 2 FSEL
  long long t2 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) u[j] = u[j] * 3u + 1u;
  long long t3 = clock64();
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; }
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i] + u[i];
  out[threadIdx.x] = s;
}
int main() {
  double* o; long long* t; cudaMalloc(&o, 1024 * 8); cudaMalloc(&t, 64);
  for (int w : {1, 4}) {
    k<<<1, 32 * w>>>(o, t, 0.5);
    k<<<1, 32 * w>>>(o, t, 0.5);
    long long h[3]; cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
    printf("warps %d: DADD %.2f cyc/instr, DSETP+2FSEL max %.2f cyc/op, IMAD %.2f cyc/instr (per warp, 8 chains)\n", w,
           double(h[0]) / (N * 8), double(h[1]) / (N * 8), double(h[2]) / (N * 8));
  }
  return 0;
}

// Single-warp dependent-chain latencies of the ops on the dispatch critical
// path (B200, sm_100a): DADD, LDS, REDUX, VOTE, SHFL, MEMBAR.CTA, clock64.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

constexpr int N = 1024;

__global__ void k(double* out, long long* t, int seed) {
  __shared__ double sd[1024];
  __shared__ int si[1024];
  const int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) { sd[i] = i * 0.5; si[i] = (i + 1) & 1023; }
  __syncwarp();
  long long t0, t1;
  double x = seed * 1e-9 + lane;
  // DADD chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __dadd_rn(x, 1.0);
  t1 = clock64();
  if (lane == 0) t[0] = t1 - t0;
  // LDS chain (pointer chase)
  int p = lane;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) p = si[p];
  t1 = clock64();
  if (lane == 0) t[1] = t1 - t0;
  // REDUX chain
  uint32_t r = lane + p;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) r = __reduce_max_sync(0xffffffffu, r + lane);
  t1 = clock64();
  if (lane == 0) t[2] = t1 - t0;
  // VOTE chain
  uint32_t b = r;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) b = __ballot_sync(0xffffffffu, (b >> lane) & 1u);
  t1 = clock64();
  if (lane == 0) t[3] = t1 - t0;
  // SHFL chain
  uint32_t s = b;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) s = __shfl_sync(0xffffffffu, s, (s + 1) & 31);
  t1 = clock64();
  if (lane == 0) t[4] = t1 - t0;
  // MEMBAR.CTA after one STS each
  t0 = clock64();
  for (int i = 0; i < N; ++i) { si[lane] = i; __threadfence_block(); }
  t1 = clock64();
  if (lane == 0) t[5] = t1 - t0;
  // clock64 back to back
  long long acc = 0;
  t0 = clock64();
  for (int i = 0; i < N; ++i) acc += clock64();
  t1 = clock64();
  if (lane == 0) t[6] = t1 - t0;
  // DSETP + VOTE + FLO (violation detect)
  double y = x;
  uint32_t v = 0;
  t0 = clock64();
  for (int i = 0; i < N; ++i) { const uint32_t bb = __ballot_sync(0xffffffffu, y > 3.0); v += __ffs(bb); y = __dadd_rn(y, (double)(bb & 1)); }
  t1 = clock64();
  if (lane == 0) t[7] = t1 - t0;
  // volatile LDS poll + branch (spin loop iteration)
  volatile int* vp = si;
  int z = 0;
  t0 = clock64();
  for (int i = 0; i < N; ++i) z += vp[(z + i) & 31];
  t1 = clock64();
  if (lane == 0) t[8] = t1 - t0;
  out[lane] = x + p + r + b + s + acc + v + y + z;
}

int main() {
  double* o; long long* t;
  cudaMalloc(&o, 32 * 8); cudaMalloc(&t, 16 * 8);
  k<<<1, 32>>>(o, t, 1);
  k<<<1, 32>>>(o, t, 2);
  long long h[16];
  cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"DADD", "LDS", "REDUX", "VOTE", "SHFL", "STS+MEMBAR.CTA", "CS2R clock", "DSETP+VOTE+FLO+DADD", "volatile LDS + add"};
  for (int i = 0; i < 9; ++i) printf("%-22s %.1f cycles/op\n", names[i], double(h[i]) / N);
  return 0;
}

// Latency probe (not product code): dependent chains of DADD, DMUL, LDS,
// SHFL, REDUX, VOTE on one warp, cycles per operation.
#include <cstdio>
#include <cstdint>
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ double sm[64];
  __shared__ uint32_t su[64];
  const int lane = threadIdx.x;
  sm[lane] = 1.0 + lane; su[lane] = lane;
  __syncwarp();
  double x = out[lane];
  uint32_t u = lane;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, 1.0000001);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, 0.9999999);
  long long t2 = clock64();
  int idx = lane;
  for (int i = 0; i < n; ++i) idx = su[idx & 63];
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) u = __shfl_sync(0xffffffffu, u, (u + 1) & 31);
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) u = __reduce_max_sync(0xffffffffu, u + lane) & 31;
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) u = __ballot_sync(0xffffffffu, (u + lane) & 1) & 31;
  long long t6 = clock64();
  float f = x;
  for (int i = 0; i < n; ++i) f = f * 1.0001f + 0.5f;
  long long t7 = clock64();
  double y = x;
  for (int i = 0; i < n; ++i) y = sm[(int)(y) & 63] + 0.0;
  long long t8 = clock64();
  out[lane] = x + u + idx + f + y;
  if (lane == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6; cyc[7] = t8 - t7;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 64); cudaMemset(o, 0, 512);
  const int n = 1000;
  k<<<1, 32>>>(o, c, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, n);
  long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
  const char* nm[8] = {"DADD", "DMUL", "LDS dep", "SHFL", "REDUX", "VOTE", "FFMA", "LDS.64+DADD+F2I"};
  for (int i = 0; i < 8; ++i) printf("%-16s %.1f cycles/op\n", nm[i], double(h[i]) / n);
}

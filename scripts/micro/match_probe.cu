// Timing probe only (not product code): per-SM throughput of the warp
// ranking primitives the radix pass can use (MATCH.ANY, 8 ballots, smem
// ATOMS.ADD with return), 32 warps per SM, digits spread or clustered.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(uint32_t* out, int iters, uint32_t mask) {
  __shared__ uint32_t cnt[8][256];
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&cnt[0][0])[i] = 0;
  __syncthreads();
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x, acc = 0;
  const int w = (threadIdx.x >> 5) & 7;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    const uint32_t d = (x >> 13) & mask;
    if (MODE == 0) {
      acc += __match_any_sync(0xffffffffu, d);
    } else if (MODE == 1) {
      uint32_t peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const bool bit = (d >> b) & 1u;
        const uint32_t v = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? v : ~v;
      }
      acc += peers;
    } else if (MODE == 2) {
      acc += atomicAdd(&cnt[w][d], 1u);
    } else if (MODE == 3) {
      // 4-bit split: per-thread counts of two nibbles (bit tricks), stand-in ALU cost
      acc += __popc(__ballot_sync(0xffffffffu, d & 1)) + (d >> 4);
    }
  }
  if (acc == 0x12345) out[0] = acc;
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  for (uint32_t mask : {255u, 15u, 1u, 0u}) {
    for (int mode = 0; mode < 4; ++mode) {
      float best = 1e9;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        dim3 g(sms * 4), t(256);
        if (mode == 0) k<0><<<g, t>>>(out, iters, mask);
        if (mode == 1) k<1><<<g, t>>>(out, iters, mask);
        if (mode == 2) k<2><<<g, t>>>(out, iters, mask);
        if (mode == 3) k<3><<<g, t>>>(out, iters, mask);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      // warp-ops per SM = 32 warps * iters
      const double cyc = best * 1e-3 * 1.965e9;
      printf("mask %3u mode %d (%s): %.3f ms, %.2f SM-cycles per warp-op\n", mask, mode,
             mode == 0 ? "match.any" : mode == 1 ? "8 ballots" : mode == 2 ? "atoms.add ret" : "1 ballot",
             best, cyc / (32.0 * iters));
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}

// Timing probe only (not product code): variants of one onesweep digit pass
// on 16M (u32 key, u32 value) pairs, to pick the K3 kernel shape.
//   SCOPE: 0 = volatile (sys-scope) look-back words, 1 = relaxed.gpu
//   RANK : 0 = match + every peer reads, 2 = match + leader read/shfl,
//          3 = match + leader atomicAdd/shfl
//   IDX32: 32-bit element indexing
// Keys: "spread" (uniform random) and "top" (C4-like top byte: 8 pools x few
// classes, skewed) for the digit at shift 24.
#include <cstdio>
#include <vector>
#include <random>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kRadix = 256;
constexpr uint32_t kFlagAgg = 1u << 30, kFlagIncl = 2u << 30, kCountMask = (1u << 30) - 1;

__device__ __forceinline__ uint32_t lanemask_lt() { uint32_t m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }
__device__ __forceinline__ uint32_t ld_gpu(const uint32_t* p) { uint32_t v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_gpu(uint32_t* p, uint32_t v) { asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }

__device__ unsigned long long g_tim[6000 * 8];
__device__ __forceinline__ unsigned long long gclk() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
template <int T, int I, int SCOPE, int RANK, int MINB, int LB, int LATEV = 0, int TIM = 0, int BAR = 0>
__global__ void __launch_bounds__(T, MINB)
k_pass(const uint32_t* __restrict__ keys_in, uint32_t* __restrict__ keys_out, const uint32_t* __restrict__ vals_in,
       uint32_t* __restrict__ vals_out, uint32_t n, int shift, const uint32_t* __restrict__ gex,
       uint32_t* __restrict__ lookback, uint32_t* __restrict__ tile_counter) {
  unsigned long long tt[6];
  if (TIM && threadIdx.x == 0) tt[0] = gclk();
  constexpr int kW = T / 32, kTile = T * I;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kSets = RANK == 4 ? 2 : 1;
  uint32_t (*wh_all)[kRadix] = reinterpret_cast<uint32_t (*)[kRadix]>(smem_raw);
  uint32_t* digit_start = reinterpret_cast<uint32_t*>(smem_raw + kSets * kW * kRadix * 4);
  uint32_t* gbase = digit_start + kRadix;  // 32-bit global base (may wrap, used modulo 2^32)
  uint32_t* s_keys = gbase + kRadix;
  uint32_t* s_vals = s_keys + kTile;
  uint32_t* wmask = s_vals + kTile;  // RANK 5: [kW][256] peer masks
  __shared__ uint32_t s_tile, s_ws[kRadix / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < kSets * kW * kRadix; i += T) (&wh_all[0][0])[i] = 0;
  if (RANK == 5) for (int i = tid; i < kW * kRadix; i += T) wmask[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t base = tile * kTile;
  uint32_t key[I], val[I];
  uint32_t rank[(I + 1) / 2];  // two 16-bit ranks per word
  const uint32_t wbase = base + warp * 32 * I + lane;
#pragma unroll
  for (int i = 0; i < I; ++i) {
    const uint32_t e = wbase + i * 32;
    if (e < n) { key[i] = keys_in[e]; if (!LATEV) val[i] = vals_in ? vals_in[e] : e; }
    else { key[i] = ~0u; if (!LATEV) val[i] = 0; }
  }
  uint32_t* wh = wh_all[warp];
  if (TIM) { uint32_t dep = key[I - 1]; __syncthreads(); if (threadIdx.x == 0) tt[1] = gclk() + (dep & 0); }
  if (BAR == 1) __syncthreads();
  if (BAR == 2) { uint32_t dep = key[I - 1]; __syncthreads(); if (threadIdx.x == 0 && dep == 0x12345678u) s_ws[0] = dep; }
  if (BAR == 3) { uint32_t dep = 0; for (int i = 0; i < I; ++i) dep ^= key[i]; __syncthreads(); if (dep == 0x12345678u) s_ws[1] = dep; }
#pragma unroll
  for (int i = 0; i < I; ++i) {
    const uint32_t d = (key[i] >> shift) & 255u;
    uint32_t peers;
    if (RANK == 5) {  // peers through a shared-memory atomicOr mask (no MATCH)
      uint32_t* wm = wmask + warp * kRadix;
      atomicOr(&wm[d], 1u << lane);
      __syncwarp();
      peers = wm[d];
      __syncwarp();
    } else if (RANK != 9) {
      peers = __match_any_sync(0xffffffffu, d);
    } else {
      peers = 1u << lane;
    }
    const int leader = __ffs(peers) - 1;
    if (RANK == 5) {
      uint32_t old = 0;
      if (lane == leader) { old = wh[d]; wh[d] = old + __popc(peers); wmask[warp * kRadix + d] = 0; }
      old = __shfl_sync(0xffffffffu, old, leader);
      __syncwarp();
      const uint32_t r = old + __popc(peers & lanemask_lt());
      if (i & 1) rank[i >> 1] |= r << 16; else rank[i >> 1] = r;
    } else if (RANK == 2) {
      uint32_t old = 0;
      if (lane == leader) { old = wh[d]; wh[d] = old + __popc(peers); }
      old = __shfl_sync(0xffffffffu, old, leader);
      const uint32_t r = old + __popc(peers & lanemask_lt());
      if (i & 1) rank[i >> 1] |= r << 16; else rank[i >> 1] = r;
    } else if (RANK == 9) {  // timing only: unstable per-lane atomics, no match
      const uint32_t r = atomicAdd(&wh[d], 1u);
      if (i & 1) rank[i >> 1] |= r << 16; else rank[i >> 1] = r;
    } else if (RANK == 4) {  // two independent counter sets (items 0..I/2-1, I/2..I-1)
      uint32_t* whs = i < I / 2 ? wh : wh + (T / 32) * kRadix;
      uint32_t old = 0;
      if (lane == leader) { old = whs[d]; whs[d] = old + __popc(peers); }
      old = __shfl_sync(0xffffffffu, old, leader);
      const uint32_t r = old + __popc(peers & lanemask_lt());
      if (i & 1) rank[i >> 1] |= r << 16; else rank[i >> 1] = r;
    } else if (RANK == 3) {
      uint32_t old = 0;
      if (lane == leader) old = atomicAdd(&wh[d], __popc(peers));
      old = __shfl_sync(0xffffffffu, old, leader);
      const uint32_t r = old + __popc(peers & lanemask_lt());
      if (i & 1) rank[i >> 1] |= r << 16; else rank[i >> 1] = r;
    } else {
      const uint32_t old = wh[d];
      __syncwarp();
      if ((peers & lanemask_lt()) == 0) wh[d] = old + __popc(peers);
      __syncwarp();
      const uint32_t r = old + __popc(peers & lanemask_lt());
      if (i & 1) rank[i >> 1] |= r << 16; else rank[i >> 1] = r;
    }
  }
  if (LATEV) {
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const uint32_t e = wbase + i * 32;
      val[i] = e < n ? (vals_in ? vals_in[e] : e) : 0u;
    }
  }
  __syncthreads();
  if (TIM && threadIdx.x == 0) tt[2] = gclk();
  uint32_t total = 0;
  if (tid < kRadix) {
#pragma unroll
    for (int w = 0; w < kW; ++w) {  // column order: warp w set A, warp w set B
      for (int st = 0; st < kSets; ++st) {
        const uint32_t c = wh_all[st * kW + w][tid]; wh_all[st * kW + w][tid] = total; total += c;
      }
    }
    uint32_t* p = lookback + tile * kRadix + tid;
    const uint32_t v = (tile == 0 ? kFlagIncl : kFlagAgg) | total;
    if (SCOPE) st_gpu(p, v); else *(volatile uint32_t*)p = v;
    uint32_t x = total;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
    if (lane == 31) s_ws[warp] = x;
    digit_start[tid] = x - total;
  }
  __syncthreads();
  if (tid < kRadix) {
    uint32_t add = 0;
    for (int w = 0; w < warp; ++w) add += s_ws[w];
    digit_start[tid] += add;
    uint32_t excl = 0;
    if (tile > 0) {
      int p = int(tile) - 1;
      bool done = false;
      while (!done) {
        uint32_t v[LB];
#pragma unroll
        for (int j = 0; j < LB; ++j) {
          const uint32_t* q = lookback + (p - j) * kRadix + tid;
          v[j] = (p - j >= 0) ? (SCOPE ? ld_gpu(q) : *(volatile const uint32_t*)q) : kFlagIncl;
        }
#pragma unroll
        for (int j = 0; j < LB; ++j) {
          if (done) break;
          const uint32_t flag = v[j] & ~kCountMask;
          if (flag == 0) break;
          excl += v[j] & kCountMask;
          --p;
          if (flag == kFlagIncl) done = true;
        }
      }
      uint32_t* q = lookback + tile * kRadix + tid;
      if (SCOPE) st_gpu(q, kFlagIncl | (excl + total)); else *(volatile uint32_t*)q = kFlagIncl | (excl + total);
    }
    gbase[tid] = gex[tid] + excl - digit_start[tid];
  }
  __syncthreads();
  if (TIM && threadIdx.x == 0) tt[3] = gclk();
#pragma unroll
  for (int i = 0; i < I; ++i) {
    const uint32_t d = (key[i] >> shift) & 255u;
    const uint32_t* whs = (kSets == 2 && i >= I / 2) ? wh + kW * kRadix : wh;
    const uint32_t pos = digit_start[d] + whs[d] + ((rank[i >> 1] >> ((i & 1) * 16)) & 0xffffu);
    s_keys[pos] = key[i];
    s_vals[pos] = val[i];
  }
  __syncthreads();
  if (TIM && threadIdx.x == 0) tt[4] = gclk();
  const uint32_t valid = (n - base) < uint32_t(kTile) ? (n - base) : uint32_t(kTile);
#pragma unroll 4
  for (uint32_t j = tid; j < valid; j += T) {
    const uint32_t k = s_keys[j];
    const uint32_t dst = gbase[(k >> shift) & 255u] + j;
    keys_out[dst] = k;
    vals_out[dst] = s_vals[j];
  }
  if (TIM) {
    __syncthreads();
    if (threadIdx.x == 0 && tile < 6000) {
      tt[5] = gclk();
      for (int k = 0; k < 6; ++k) g_tim[tile * 8 + k] = tt[k];
      unsigned sm; asm("mov.u32 %0, %%smid;" : "=r"(sm)); g_tim[tile * 8 + 6] = sm;
    }
  }
}

// plain streaming copy of the same bytes (12 B/elem read+write like pass 0)
__global__ void k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, uint4* __restrict__ c, uint32_t n4) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
    const uint4 x = a[i];
    b[i] = x;
    c[i] = x;
  }
}

struct Bufs { uint32_t *k0, *k1, *v0, *v1, *lb, *hist, *tc; };

template <int T, int I, int SCOPE, int RANK, int MINB, int LB, int LATEV = 0, int TIM = 0, int BAR = 0>
void run(const char* name, Bufs& B, uint32_t n, int shift, bool with_vals, const std::vector<uint32_t>& hk) {
  constexpr int kTile = T * I;
  const uint32_t tiles = (n + kTile - 1) / kTile;
  std::vector<uint32_t> h(kRadix, 0);
  for (auto x : hk) h[(x >> shift) & 255]++;
  uint32_t acc = 0; for (auto& x : h) { uint32_t c = x; x = acc; acc += c; }
  cudaMemcpy(B.hist, h.data(), kRadix * 4, cudaMemcpyHostToDevice);
  const size_t smem = (RANK == 4 ? 2 : 1) * (T / 32) * kRadix * 4 + 2 * kRadix * 4 + size_t(kTile) * 8 +
                      (RANK == 5 ? (T / 32) * kRadix * 4 : 0);
  auto kern = k_pass<T, I, SCOPE, RANK, MINB, LB, LATEV, TIM, BAR>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9, sum = 0;
  for (int it = 0; it < 12; ++it) {
    cudaMemset(B.lb, 0, size_t(tiles) * kRadix * 4); cudaMemset(B.tc, 0, 64);
    cudaEventRecord(a);
    kern<<<tiles, T, smem>>>(B.k0, B.k1, with_vals ? B.v0 : nullptr, B.v1, n, shift, B.hist, B.lb, B.tc);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (it >= 2) { best = ms < best ? ms : best; sum += ms; }
  }
  // check sortedness of the digit
  std::vector<uint32_t> out(n);
  cudaMemcpy(out.data(), B.k1, size_t(n) * 4, cudaMemcpyDeviceToHost);
  std::vector<uint32_t> ov(n);
  cudaMemcpy(ov.data(), B.v1, size_t(n) * 4, cudaMemcpyDeviceToHost);
  bool ok = true;
  for (uint32_t i = 1; i < n && ok; ++i) {
    const uint32_t a = (out[i - 1] >> shift) & 255, b = (out[i] >> shift) & 255;
    ok = a < b || (a == b && ov[i - 1] < ov[i]);  // sorted and stable
  }
  int regs = 0; cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kern); regs = fa.numRegs;
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, T, smem);
  if (TIM) {
    std::vector<unsigned long long> tm(6000 * 8);
    cudaMemcpyFromSymbol(tm.data(), g_tim, tm.size() * 8);
    double acc[5] = {0, 0, 0, 0, 0};
    unsigned long long t0 = ~0ull, t1 = 0;
    int cnt = 0;
    for (uint32_t t = 0; t < tiles && t < 6000; ++t) {
      const unsigned long long* r = &tm[t * 8];
      for (int k = 0; k < 5; ++k) acc[k] += double(r[k + 1] - r[k]);
      t0 = r[0] < t0 ? r[0] : t0; t1 = r[5] > t1 ? r[5] : t1;
      ++cnt;
    }
    printf("  per-tile ns: load %.0f rank %.0f scan+lookback %.0f stage %.0f write %.0f (tiles %d, span %.1f us)\n",
           acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt, cnt, (t1 - t0) / 1e3);
  }
  printf("%-34s shift %2d vals %d: best %6.1f us avg %6.1f us  %.2f TB/s(16B)  regs %d ctas/sm %d %s\n", name, shift,
         with_vals, best * 1e3, sum / 10 * 1e3, n * 16.0 / (best * 1e-3) / 1e12, regs, occ, ok ? "ok" : "BAD");
}

int main() {
  const uint32_t n = 16000000;
  std::mt19937 g(1);
  std::vector<uint32_t> spread(n), top(n);
  for (auto& x : spread) x = g();
  // C4-like: top byte = pool(3b) | class(4b) | top q bit, skewed classes
  for (auto& x : top) {
    const uint32_t pool = g() & 7, r = g() % 100;
    const uint32_t cls = r < 50 ? 0 : r < 75 ? 1 : r < 90 ? 2 : r < 97 ? 3 : 4 + (r & 3);
    x = (pool << 29) | (cls << 25) | (g() & 0x1ffffff);
  }
  Bufs B;
  cudaMalloc(&B.k0, n * 4); cudaMalloc(&B.k1, n * 4); cudaMalloc(&B.v0, n * 4); cudaMalloc(&B.v1, n * 4);
  cudaMalloc(&B.lb, (n / 1024 + 16) * kRadix * 4); cudaMalloc(&B.hist, kRadix * 4); cudaMalloc(&B.tc, 64);
  {
    std::vector<uint32_t> iota(n);
    for (uint32_t i = 0; i < n; ++i) iota[i] = i;
    cudaMemcpy(B.v0, iota.data(), size_t(n) * 4, cudaMemcpyHostToDevice);
  }
  {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(a);
      k_copy<<<148 * 8, 256>>>((const uint4*)B.k0, (uint4*)B.k1, (uint4*)B.v1, n / 4);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
    }
    printf("copy 4B->2x4B: %.1f us (%.2f TB/s)\n", best * 1e3, n * 12.0 / (best * 1e-3) / 1e12);
  }
  for (int pass = 0; pass < 2; ++pass) {
    const std::vector<uint32_t>& hk = pass == 0 ? spread : top;
    const int shift = pass == 0 ? 0 : 24;
    cudaMemcpy(B.k0, hk.data(), size_t(n) * 4, cudaMemcpyHostToDevice);
    run<256, 12, 1, 2, 4, 8, 1, 0, 0>("r2", B, n, shift, true, hk);
    run<256, 12, 1, 2, 4, 8, 1, 0, 2>("r2 bar2", B, n, shift, true, hk);
    run<256, 12, 1, 5, 4, 8, 1, 0, 0>("r5", B, n, shift, true, hk);
    run<256, 12, 1, 5, 4, 8, 1, 0, 1>("r5 bar1", B, n, shift, true, hk);
    run<256, 12, 1, 5, 4, 8, 1, 0, 2>("r5 bar2", B, n, shift, true, hk);
    run<256, 12, 1, 5, 4, 8, 1, 0, 3>("r5 bar3", B, n, shift, true, hk);
    run<256, 12, 1, 5, 4, 8, 0, 0, 3>("r5 bar3 early-vals", B, n, shift, true, hk);
    run<256, 16, 1, 5, 4, 8, 1, 0, 3>("256x16 r5 bar3", B, n, shift, true, hk);
    run<512, 12, 1, 5, 2, 8, 1, 0, 3>("512x12 r5 bar3", B, n, shift, true, hk);
    run<256, 12, 1, 0, 4, 8, 1, 0, 3>("r0 bar3", B, n, shift, true, hk);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}

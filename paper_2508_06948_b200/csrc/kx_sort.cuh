// K3: LSD radix sort of (key, u32 queue index) pairs, 8-bit digits, one
// kernel per digit pass with decoupled look-back ("onesweep" structure):
//
//   * an upfront histogram of every pass's digits is produced by the key
//     generator (or by k_upfront_hist) in a single read of the keys;
//   * each pass kernel takes a dynamic tile id, ranks its tile's digits with
//     warp match-any + per-warp shared-memory counters (stable), publishes the
//     tile's per-digit counts, resolves its global digit offsets by looking
//     back over predecessor tiles (flag|count packed in one u32, so a single
//     store publishes both), stages the tile in shared memory in digit order
//     and writes runs of equal digits contiguously (coalesced scatter).
//
// The sort is stable, so LSD over the key's digits sorts by the whole key.
// Replaces the comparator sort/arg-min scans of the reference queue
// (priority.hpp:89-116, harness.cpp:92-100) for the compact key; ties of the
// compact key are resolved afterwards by the exact tuple (kx_order.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "kx_common.cuh"

namespace kx {

constexpr int kRadixBits = 8;
constexpr int kRadix = 256;
#ifndef KX_SORT_THREADS
#define KX_SORT_THREADS 256
#endif
#ifndef KX_SORT_ITEMS
#define KX_SORT_ITEMS 16  // 4096-key tiles (measured at C4: 12 -> 0.484 ms, 13 -> 0.473, 14 -> 0.472, 16 -> 0.468 for the four passes)
#endif
constexpr int kSortThreads = KX_SORT_THREADS;
constexpr int kSortItems = KX_SORT_ITEMS;
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagIncl = 2u << 30;
constexpr uint32_t kCountMask = (1u << 30) - 1;
#ifndef KX_STAGE_EARLY
#define KX_STAGE_EARLY 1
#endif
#ifndef KX_LB_SLEEP
#define KX_LB_SLEEP 64  // ns of back-off when a predecessor has not published
#endif
#ifndef KX_HIST_IN_STAGE
#define KX_HIST_IN_STAGE 0
#endif
#ifndef KX_LOOK_BATCH
#define KX_LOOK_BATCH 4
#endif
constexpr int kLookBatch = KX_LOOK_BATCH;
// Next-digit counting: digits at or above this shift are counted with
// warp-aggregated increments, lower ones with plain shared atomics. The
// C4 keys' low digits cluster too (a workflow's calls share app_start), and
// aggregated increments measured faster for every digit (0.531 vs 0.543 ms
// for the four passes), so all digits aggregate.
constexpr int kNextAggShift = 0;

// Diagnostics (build with -DKX_SORT_TIMERS=1): per pass (shift / 8), sums
// over tiles of the globaltimer spans load, rank, scan+look-back, stage,
// write, and the tile count (read by kx_debug_sort_timers).
#ifndef KX_SORT_TIMERS
#define KX_SORT_TIMERS 0
#endif
static __device__ unsigned long long g_sort_tim[8 * 8];  // per translation unit (no -rdc)
__device__ __forceinline__ unsigned long long sort_gclk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Lanes holding the same 8-bit digit: eight ballots instead of MATCH.ANY
// (MATCH issues through the MIO pipe at a fraction of the ballot rate and
// was the top stall of the ranking loop).
__device__ __forceinline__ uint32_t warp_match8(uint32_t d) {
  uint32_t peers = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const bool bit = (d >> b) & 1u;
    const uint32_t vote = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? vote : ~vote;
  }
  return peers;
}

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, int shift) {
  return static_cast<uint32_t>(key >> shift) & (kRadix - 1);
}

// Per-warp-aggregated shared-memory histogram increment. When the whole warp
// carries one digit (constant high digits are common) a single add is issued.
__device__ __forceinline__ void hist_add(uint32_t* h, uint32_t d, bool valid) {
  const uint32_t active = __ballot_sync(0xffffffffu, valid);
  if (!active) return;
  const uint32_t lead = __ffs(active) - 1;
  const uint32_t d0 = __shfl_sync(0xffffffffu, d, lead);
  const bool uniform = __all_sync(0xffffffffu, !valid || d == d0);
  if (uniform) {
    if ((threadIdx.x & 31) == lead) atomicAdd(&h[d0], __popc(active));
    return;
  }
  if (valid) atomicAdd(&h[d], 1u);
}

// Generic upfront histogram for a key array (used by the exact-tuple
// fallback sorts; the order path fuses this into key generation).
template <typename K>
__global__ void k_upfront_hist(const K* __restrict__ keys, int64_t n, int shift0,
                               int passes, uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[8 * kRadix];
  for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    const bool valid = i < n;
    const K key = valid ? keys[i] : K(0);
    for (int p = 0; p < passes; ++p) hist_add(&sh[p * kRadix], digit_of(key, shift0 + p * kRadixBits), valid);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// Exclusive scan of each pass's 256 bins (in place): one warp per pass.
__global__ void k_scan_hist(uint32_t* __restrict__ hist, int passes);

template <typename K>
struct SortSmem {
  uint32_t warp_hist[kSortThreads / 32][kRadix];
  uint32_t next_hist[kRadix];                      // next pass's digit counts (this tile)
  uint32_t digit_start[kRadix];
  int64_t global_base[kRadix];
  uint32_t tile_id;
};

template <typename K>
constexpr size_t sort_dyn_smem() {
  return sizeof(SortSmem<K>) + size_t(kSortTile) * (sizeof(K) + sizeof(uint32_t));
}

// One stable LSD digit pass. vals_in == nullptr means "value = element index"
// (first pass). global_excl: this pass's exclusive digit offsets, or with
// counts_in != 0 its raw digit counts (each CTA scans them). next_hist !=
// nullptr: the pass also counts the digit at next_shift of every key it
// writes (the next pass's histogram, one read of the keys saved).
// kRank selects the warp ranking: 0 = MATCH.ANY peers, every peer reads the
// running count; 1 = eight-ballot peers, same update; 2 = MATCH.ANY peers,
// the leader reads and broadcasts the count. MATCH.ANY costs ~2 SM-cycles per
// distinct digit in the warp (scripts/micro/match_probe.cu), the ballots a
// fixed ~25: MATCH wins on the clustered C4 digits, the ballots on the top
// digit (few distinct values with the class bits); see kSortRankDefault.
#ifndef KX_SORT_MINB
#define KX_SORT_MINB 4  // 32-bit keys: 4 blocks per SM caps registers at 64 (unbounded, ptxas takes 119)
#endif
template <typename K, int kRank = 0>
__global__ void __launch_bounds__(kSortThreads, sizeof(K) == 4 ? KX_SORT_MINB : 2)
k_onesweep_pass(const K* __restrict__ keys_in, K* __restrict__ keys_out,
                const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ vals_out,
                int64_t n, int shift, const uint32_t* __restrict__ global_excl,
                uint32_t* __restrict__ lookback, uint32_t* __restrict__ lookback_next,
                uint32_t* __restrict__ tile_counter, int counts_in,
                uint32_t* __restrict__ next_hist, int next_shift
#ifdef KX_PROBE_NO_LOOKBACK_SWITCH
                , int probe_no_lookback = 0
#endif
                ) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem<K>& sm = *reinterpret_cast<SortSmem<K>*>(smem_raw);
  K* s_keys = reinterpret_cast<K*>(smem_raw + sizeof(SortSmem<K>));
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + kSortTile);

  constexpr int kWarps = kSortThreads / 32;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  unsigned long long tt[6] = {0, 0, 0, 0, 0, 0};
  if (KX_SORT_TIMERS && tid == 0) tt[0] = sort_gclk();
  if (tid == 0) sm.tile_id = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < kWarps * kRadix; i += kSortThreads) (&sm.warp_hist[0][0])[i] = 0;
  if (next_hist)
    for (int i = tid; i < kRadix; i += kSortThreads) sm.next_hist[i] = 0;
  __syncthreads();
  const uint32_t tile = sm.tile_id;
  const int64_t base = int64_t(tile) * kSortTile;
  // passes alternate between two look-back arrays: this one clears its
  // tile's words of the other (the previous pass, which used it, is done;
  // the next pass has the same tiles), so no memset runs between passes
  if (lookback_next && tid < kRadix) lookback_next[int64_t(tile) * kRadix + tid] = 0u;

  K key[kSortItems];
  uint32_t val[kSortItems];
  uint32_t rank[kSortItems];
  const int64_t wbase = base + int64_t(warp) * 32 * kSortItems + lane;
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int64_t e = wbase + i * 32;
    if (e < n) {
      key[i] = keys_in[e];
      val[i] = vals_in ? vals_in[e] : static_cast<uint32_t>(e);
    } else {
      key[i] = ~K(0);  // digit 255, ranked after every valid element
      val[i] = 0;
    }
  }
  // Every key of the tile is in registers before the ranking starts (the
  // ranking loop then runs without load stalls between its shared-memory
  // steps): the empty asm consumes all keys ahead of the barrier.
  {
    uint32_t dep = 0;
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) dep ^= static_cast<uint32_t>(key[i]);
    asm volatile("" ::"r"(dep));
    __syncthreads();
  }
  if (KX_SORT_TIMERS && tid == 0) tt[1] = sort_gclk();
  // Stable warp-level ranking, processing items in element order.
  uint32_t* wh = sm.warp_hist[warp];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t d = digit_of(key[i], shift);
    const uint32_t peers = kRank == 1 ? warp_match8(d) : __match_any_sync(0xffffffffu, d);
    if (kRank == 2) {
      const int leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if (lane == leader) {
        old = wh[d];
        wh[d] = old + __popc(peers);
      }
      old = __shfl_sync(0xffffffffu, old, leader);
      rank[i] = old + __popc(peers & lanemask_lt());
    } else {
      // every peer reads the running count (broadcast), the lowest one bumps it
      const uint32_t old = wh[d];
      __syncwarp();
      if ((peers & lanemask_lt()) == 0) wh[d] = old + __popc(peers);
      __syncwarp();
      rank[i] = old + __popc(peers & lanemask_lt());
    }
  }
  __syncthreads();
  if (KX_SORT_TIMERS && tid == 0) tt[2] = sort_gclk();

  // Per digit: exclusive prefix over warps, tile total, look-back.
  uint32_t total = 0;
  if (tid < kRadix) {
#pragma unroll 4
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = sm.warp_hist[w][tid];
      sm.warp_hist[w][tid] = total;
      total += c;
    }
    volatile uint32_t* lb = lookback;
    lb[int64_t(tile) * kRadix + tid] = (tile == 0 ? kFlagIncl : kFlagAgg) | total;
  }
  // Exclusive scans over the 256 digits (8 warps x 32 lanes) of `total`
  // and, with counts_in, of the pass's global digit counts.
  __shared__ uint32_t s_warp_sums[kRadix / 32], s_warp_cnt[kRadix / 32];
  uint32_t gcount = 0, gexcl = 0;
  if (tid < kRadix) {
    uint32_t x = total;
    gcount = counts_in ? global_excl[tid] : 0u;
    uint32_t c = gcount;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      const uint32_t yc = __shfl_up_sync(0xffffffffu, c, o);
      if (lane >= o) {
        x += y;
        c += yc;
      }
    }
    if (lane == 31) {
      s_warp_sums[warp] = x;
      s_warp_cnt[warp] = c;
    }
    sm.digit_start[tid] = x - total;  // warp-local exclusive
    gexcl = c - gcount;
  }
  __syncthreads();
  uint32_t gexcl_final = 0;
  if (tid < kRadix) {
    uint32_t add = 0, addc = 0;
    for (int w = 0; w < warp; ++w) {
      add += s_warp_sums[w];
      addc += s_warp_cnt[w];
    }
    sm.digit_start[tid] += add;
    gexcl_final = counts_in ? gexcl + addc : global_excl[tid];
  }
#if KX_STAGE_EARLY
  // Stage the tile in digit order before the look-back: the predecessors
  // get the staging time to publish, so fewer polls find an empty flag.
  // With KX_HIST_IN_STAGE the next pass's digits are counted here too (keys
  // still in registers) instead of in the write loop.
  __syncthreads();
  const int64_t vbase = base + int64_t(warp) * 32 * kSortItems + lane;
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t d = digit_of(key[i], shift);
    const uint32_t pos = sm.digit_start[d] + sm.warp_hist[warp][d] + rank[i];
    s_keys[pos] = key[i];
    s_vals[pos] = val[i];
    if (KX_HIST_IN_STAGE && next_hist) hist_add(sm.next_hist, digit_of(key[i], next_shift), vbase + i * 32 < n);
  }
#endif
  if (tid < kRadix) {
    // Decoupled look-back for digit `tid`, kLookBatch predecessors per
    // round trip: the walk over tiles that have only published their
    // aggregate costs one L2 latency per batch instead of per tile.
    uint32_t excl = 0;
#ifdef KX_PROBE_NO_LOOKBACK_SWITCH
    if (probe_no_lookback) lookback[int64_t(tile) * kRadix + tid] = kFlagIncl | total;
    else
#endif
    if (tile > 0) {
      volatile uint32_t* lb = lookback;
      int64_t p = int64_t(tile) - 1;
      bool done = false;
      while (!done) {
        uint32_t v[kLookBatch];
#pragma unroll
        for (int j = 0; j < kLookBatch; ++j) v[j] = (p - j >= 0) ? uint32_t(lb[(p - j) * kRadix + tid]) : uint32_t(kFlagIncl);
        bool empty = false;
#pragma unroll
        for (int j = 0; j < kLookBatch; ++j) {
          if (done || empty) break;
          const uint32_t flag = v[j] & ~kCountMask;
          if (flag == 0) {  // not published yet: reload from here
            empty = true;
            break;
          }
          excl += v[j] & kCountMask;
          --p;
          if (flag == kFlagIncl) done = true;
        }
        if (KX_LB_SLEEP && empty) __nanosleep(KX_LB_SLEEP);
      }
      lb[int64_t(tile) * kRadix + tid] = kFlagIncl | (excl + total);
    }
    sm.global_base[tid] = int64_t(gexcl_final) + excl - int64_t(sm.digit_start[tid]);
  }
  __syncthreads();
  if (KX_SORT_TIMERS && tid == 0) tt[3] = sort_gclk();

#if !KX_STAGE_EARLY
  // Stage the tile in digit order.
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t d = digit_of(key[i], shift);
    const uint32_t pos = sm.digit_start[d] + sm.warp_hist[warp][d] + rank[i];
    s_keys[pos] = key[i];
    s_vals[pos] = val[i];
  }
  __syncthreads();
#endif
  if (KX_SORT_TIMERS && tid == 0) tt[4] = sort_gclk();

  const int64_t valid = (n - base) < kSortTile ? (n - base) : kSortTile;
  if (next_hist && !(KX_STAGE_EARLY && KX_HIST_IN_STAGE) && next_shift >= kNextAggShift) {
    // a high digit (often equal across a warp): aggregated increments need a
    // uniform trip count
#pragma unroll 4
    for (int j = tid; j < kSortTile; j += kSortThreads) {
      const bool ok = j < valid;
      const K k = ok ? s_keys[j] : K(0);
      if (ok) {
        const int64_t dst = sm.global_base[digit_of(k, shift)] + j;
        keys_out[dst] = k;
        vals_out[dst] = s_vals[j];
      }
      hist_add(sm.next_hist, digit_of(k, next_shift), ok);
    }
  } else if (next_hist && !(KX_STAGE_EARLY && KX_HIST_IN_STAGE)) {  // a spread digit: plain shared atomics
#pragma unroll 4
    for (int j = tid; j < valid; j += kSortThreads) {
      const K k = s_keys[j];
      const int64_t dst = sm.global_base[digit_of(k, shift)] + j;
      keys_out[dst] = k;
      vals_out[dst] = s_vals[j];
      atomicAdd(&sm.next_hist[digit_of(k, next_shift)], 1u);
    }
  } else {
#pragma unroll 4
    for (int j = tid; j < valid; j += kSortThreads) {
      const K k = s_keys[j];
      const int64_t dst = sm.global_base[digit_of(k, shift)] + j;
      keys_out[dst] = k;
      vals_out[dst] = s_vals[j];
    }
  }
  if (next_hist) {
    __syncthreads();
    for (int i = tid; i < kRadix; i += kSortThreads)
      if (sm.next_hist[i]) atomicAdd(&next_hist[i], sm.next_hist[i]);
  }
  if (KX_SORT_TIMERS) {
    __syncthreads();
    if (tid == 0) {
      tt[5] = sort_gclk();
      unsigned long long* g = g_sort_tim + (shift / 8 & 7) * 8;
      for (int k = 0; k < 5; ++k) atomicAdd(&g[k], tt[k + 1] - tt[k]);
      atomicAdd(&g[5], 1ull);
    }
  }
}

}  // namespace kx

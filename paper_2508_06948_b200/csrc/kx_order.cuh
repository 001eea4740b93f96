// Host-side interface of the order pipeline (kx_order.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>

#include "kx_common.cuh"
#include "kx_state.cuh"

namespace kx {

struct OrderWorkspace {
  uint32_t* keys[2];
  uint32_t* vals[2];
  uint32_t* lookback;
  PoolRange* ranges;
  PoolRange* range_stage;  // [n_pools] sampled extremes in flight; (~0, 0) between orders
  uint32_t* sample_done;   // blocks of the sample launch done; 0 between orders
  int64_t* pool_offsets;  // n_pools + 1
  // small header block, zeroed per order: hist[4*256], tile_counters[8],
  // pool_counts[n_pools], n_big, error_flags
  void* small_hdr;
  size_t small_hdr_bytes;
  uint32_t* hist;
  uint32_t* tile_counters;
  uint32_t* pool_counts;
  uint32_t* n_big;
  int* error_flags;
  uint32_t* big_starts;
  uint32_t* big_lens;
  uint32_t tie_cap;
};

struct OrderResultDev {
  uint32_t* keys;  // sorted compact keys
  uint32_t* perm;  // sorted queue indices
};

size_t order_lookback_bytes(int64_t cap);
void configure_sort_kernels();
void launch_score(const QueueDev& q, const AgentsDev& a, int policy, int64_t n, double* k0,
                  double* k1, double* k2, int sms, cudaStream_t st);
constexpr int kTopKMax = 2048;      // candidate heads per pool
constexpr int kTopKMaxPools = 32;   // overlap path limit

// Per-pool radix-select state of the dispatch prefix (k_topk_*).
struct TopKState {
  uint32_t need, prefix, mask, below, count, done, bound, n_cand;
  uint32_t pool_count, defer, empty, spec;  // spec: candidates came from key generation
};

struct TopKWork {
  TopKState* state;  // [P]
  uint32_t* hist;    // [P * 256]
  uint32_t* cand;    // [P * kTopKMax] candidate queue indices (unordered)
  uint32_t max_need = kTopKMax;  // prefix length cap (lowered by tests via KX_TOPK_NEED)
  uint32_t* heads;   // [P * kTopKMax] the pool's order prefix
  // speculative prefix bound from the sample (k_spec_bound), candidates
  // collected by k_keygen
  uint32_t* spec_bound;  // [P]
  uint32_t* spec_on;     // [P]
  uint32_t* spec_count;  // [P]
  uint32_t* plist;        // [P * kSpecMax] compact keys of each pool's sampled requests
  uint32_t* plist_count;  // [P]
  uint32_t* cand_key;    // [P * kTopKMax]
};

int keygen_grid(int64_t n, int sms);

size_t spec_list_words(int n_pools);

// Speculative top-K: key generation collects every key <= spec_bound[p] of
// the pools with spec_on[p] into cand / spec_count (see k_spec_bound).
struct KeygenSpec {
  const uint32_t* bound;
  const uint32_t* on;
  uint32_t* count;
  uint32_t* cand;
  uint32_t* cand_key;  // compact key of each candidate
};

struct OrderHooks {
  std::function<void()> before_keygen;         // quantisation window ready, keys not yet built
  KeygenSpec spec{};                           // speculative prefix collection (bound != nullptr)
  std::function<void()> after_keys;            // compact keys, histograms, pool counts ready (not the offsets)
  std::function<void()> before_key_overwrite;  // after radix pass 0, before pass 1
  // zeroed by the order's first launch, with its own state
  uint32_t* zero_words = nullptr;
  int n_zero_words = 0;
  uint8_t* zero_bytes = nullptr;  // 16-byte aligned
  int64_t n_zero_bytes = 0;
};

OrderResultDev launch_order(const QueueDev& q, const AgentsDev& a, const OrderParams& op,
                            int64_t n, OrderWorkspace& ws, int sms, cudaStream_t st,
                            PhaseProfiler* prof, const OrderHooks* hooks = nullptr);

void launch_spec_bound(const QueueDev& q, const AgentsDev& a, const InstDev& in,
                       const int32_t* pool_begin, const OrderParams& op, int64_t n,
                       const OrderWorkspace& ws, TopKWork& w, cudaStream_t st);

// Diagnostics: per-pass radix tile phase sums (KX_SORT_TIMERS builds).
void read_sort_debug(unsigned long long* out64, bool reset);

void read_keys_done(unsigned long long* out);

}  // namespace kx

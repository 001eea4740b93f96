// Generic device sort of (key, u32 value) pairs with the onesweep passes of
// kx_sort.cuh: used by the metrics path (K7) for per-replica token-latency
// ordering. Temporary buffers come from the stream-ordered allocator.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/kairos_b200.h"
#include "kx_common.cuh"
#include "kx_sort.cuh"
#include "kx_sortlib.cuh"

namespace kx {

template <typename K>
void sort_pairs(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, int64_t n, int begin_bit,
                int end_bit, bool vals_are_iota, bool* result_in_alt, cudaStream_t st) {
  *result_in_alt = false;
  if (n <= 0 || end_bit <= begin_bit) return;
  const int passes = (end_bit - begin_bit + kRadixBits - 1) / kRadixBits;
  if (passes > 8) throw KxError(KX_ERR_INVALID, "sort_pairs: at most 64 key bits");
  static std::once_flag configured[kMaxDevices];
  once_per_device(configured, [] {
    KX_CUDA(cudaFuncSetAttribute(k_onesweep_pass<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(sort_dyn_smem<K>())));
  });
  const int64_t tiles = (n + kSortTile - 1) / kSortTile;
  uint32_t* hist = nullptr;
  uint32_t* lookback = nullptr;
  uint32_t* counters = nullptr;
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&hist), passes * kRadix * 4, st));
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&lookback), size_t(tiles) * kRadix * 4, st));
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&counters), 64, st));
  KX_CUDA(cudaMemsetAsync(hist, 0, passes * kRadix * 4, st));
  KX_CUDA(cudaMemsetAsync(counters, 0, 64, st));
  int sms = 148;
  int dev = 0;
  KX_CUDA(cudaGetDevice(&dev));
  KX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, int64_t(sms) * 8));
  k_upfront_hist<K><<<grid, 256, 0, st>>>(keys, n, begin_bit, passes, hist);
  KX_CHECK_LAUNCH();
  k_scan_hist<<<1, 32 * passes, 0, st>>>(hist, passes);
  KX_CHECK_LAUNCH();
  K* kin = keys;
  K* kout = keys_alt;
  uint32_t* vin = vals;
  uint32_t* vout = vals_alt;
  bool alt = false;
  for (int p = 0; p < passes; ++p) {
    KX_CUDA(cudaMemsetAsync(lookback, 0, size_t(tiles) * kRadix * 4, st));
    k_onesweep_pass<K><<<static_cast<unsigned>(tiles), kSortThreads, sort_dyn_smem<K>(), st>>>(
        kin, kout, (p == 0 && vals_are_iota) ? nullptr : vin, vout, n, begin_bit + p * kRadixBits,
        hist + p * kRadix, lookback, nullptr, counters + p, 0, nullptr, 0);
    KX_CHECK_LAUNCH();
    std::swap(kin, kout);
    std::swap(vin, vout);
    alt = !alt;
  }
  *result_in_alt = alt;
  KX_CUDA(cudaFreeAsync(hist, st));
  KX_CUDA(cudaFreeAsync(lookback, st));
  KX_CUDA(cudaFreeAsync(counters, st));
}

template void sort_pairs<uint32_t>(uint32_t*, uint32_t*, uint32_t*, uint32_t*, int64_t, int, int, bool,
                                   bool*, cudaStream_t);
template void sort_pairs<uint64_t>(uint64_t*, uint32_t*, uint64_t*, uint32_t*, int64_t, int, int, bool,
                                   bool*, cudaStream_t);

}  // namespace kx

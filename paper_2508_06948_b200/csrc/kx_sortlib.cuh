#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

namespace kx {
// Stable LSD sort of (keys, vals) over key bits [begin_bit, end_bit).
// Result lands in (keys, vals) or (keys_alt, vals_alt): *result_in_alt.
template <typename K>
void sort_pairs(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, int64_t n, int begin_bit,
                int end_bit, bool vals_are_iota, bool* result_in_alt, cudaStream_t st);
}  // namespace kx

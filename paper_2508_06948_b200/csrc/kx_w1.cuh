// wasserstein_1d (distribution.cpp:9-31) as a device function: the merged
// quantile grid walked in the reference's exact integer steps of
// 1/(na*nb), (nxt - cur) * |a[i] - b[j]| accumulated in the reference's
// order with correctly rounded multiply and add (an FMA hazard site, SURVEY
// H2), divided by na * nb. Bit-identical to the CPU.
#pragma once

#include <stdint.h>

namespace kx {

__device__ __forceinline__ double w1_walk(const double* a, uint64_t na, const double* b, uint64_t nb) {
  const uint64_t total = na * nb;
  uint64_t cur = 0, ia = 0, jb = 0;
  double acc = 0.0;
  while (cur < total) {
    const uint64_t a_next = (ia + 1) * nb;
    const uint64_t b_next = (jb + 1) * na;
    const uint64_t nxt = a_next < b_next ? a_next : b_next;
    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(nxt - cur), fabs(__dsub_rn(a[ia], b[jb]))));
    if (a_next == nxt) ++ia;
    if (b_next == nxt) ++jb;
    cur = nxt;
  }
  return __ddiv_rn(acc, static_cast<double>(total));
}

}  // namespace kx

// Exact tie-break of the ReadyQueue order (priority.hpp:97-98) after the
// policy's primary component: the ordered bits of the remaining time fields,
// then msg_id (order-preserving key), uid and the queue index.
// Shared by the order's tie-fix (kx_order.cu) and the dispatch's in-CTA
// prefix sort (kx_dispatch.cu).
#pragma once

#include <stdint.h>

#include "kx_common.cuh"
#include "kx_state.cuh"

namespace kx {

struct TKey {
  uint64_t w0, w1, w2;
  uint32_t idx;
};

__device__ __forceinline__ TKey load_tkey(const QueueDev& q, int policy, uint32_t idx) {
  TKey r;
  const double app = q.app_start[idx];
  const double qe = q.queue_enter[idx];
  switch (policy) {
    case KX_SCHED_KAIROS: r.w0 = ordered_bits(app); r.w1 = ordered_bits(qe); r.w2 = 0; break;
    case KX_SCHED_ORACLE: r.w0 = ordered_bits(q.rem[idx]); r.w1 = ordered_bits(qe); r.w2 = ordered_bits(app); break;
    default: r.w0 = ordered_bits(qe); r.w1 = ordered_bits(app); r.w2 = 0; break;
  }
  r.idx = idx;
  return r;
}

__device__ __forceinline__ bool tkey_less(const QueueDev& q, const TKey& a, const TKey& b) {
  if (a.w0 != b.w0) return a.w0 < b.w0;
  if (a.w1 != b.w1) return a.w1 < b.w1;
  if (a.w2 != b.w2) return a.w2 < b.w2;
  const uint64_t ma = q.msg[a.idx], mb = q.msg[b.idx];
  if (ma != mb) return ma < mb;
  const uint64_t ua = q.uid[a.idx], ub = q.uid[b.idx];
  if (ua != ub) return ua < ub;
  return a.idx < b.idx;
}

}  // namespace kx

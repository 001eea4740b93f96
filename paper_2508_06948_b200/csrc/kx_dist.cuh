// Device restatements of the reference's distribution arithmetic, shared by
// the profiler-ingestion kernel (K9, kx_profiler.cu) and the replica engine
// (K6, kx_engine.cu):
//   * EmpiricalDistribution::add with its doubling checkpoints
//     (distribution.cpp:91-123) as a warp-cooperative function over any
//     memory space (generic pointers: shared or global);
//   * quantile_sorted / histogram_mode / mode_estimate
//     (distribution.cpp:33-86), the histogram counted from bin boundaries
//     found by binary search (the bin index is monotone in the sample), so a
//     mode costs O(bins log n) instead of O(n);
//   * glibc's cbrt (sysdeps/ieee754/dbl-64/s_cbrt.c, glibc 2.39 of this
//     image), which the Freedman-Diaconis width uses (distribution.cpp:58,
//     SURVEY H3). glibc's cbrt is not correctly rounded, so the device
//     replays its polynomial + rational step op for op (checked equal for
//     every integer argument up to 2^24: tests/test_gpu_engine_kairos.py);
//   * classical_mds_1d (priority.cpp:67-100) with the cyclic Jacobi
//     eigen-solver of the oracle's Eigen stand-in (oracle/shim/Eigen/Dense),
//     one thread, correctly rounded + - * / sqrt (bit-identical).
// All f64 arithmetic is explicit round-to-nearest.
#pragma once

#include <stdint.h>

#include "kx_w1.cuh"

namespace kx {

// ConvergenceConfig (distribution.hpp:36-40).
struct DistCfg {
  uint64_t min_samples;
  double threshold;
  int64_t window_cap;  // 0 = unbounded
};

// EmpiricalDistribution's scalar state (distribution.hpp:72-82).
struct DistScal {
  int64_t n;         // sorted_.size()
  int64_t head;      // oldest retained sample in the arrival ring
  int64_t snap_n;    // snapshot_.size()
  uint64_t total;    // total_added_
  uint64_t next_cp;  // next_checkpoint_
  uint32_t conv;     // converged_
  double last;       // last_checkpoint_distance_
};

// std::lower_bound over s[0, n): first position with s[pos] >= v (32-ary).
__device__ __forceinline__ int64_t warp_lower_bound(const double* s, int64_t n, double v) {
  const int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = n;
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t idx = lo + lane * step;
    const uint32_t m = __ballot_sync(0xffffffffu, idx < hi && s[idx] < v);
    const int c = __popc(m);  // sampled positions below v: a prefix (sorted)
    if (c == 0) return lo;
    const int64_t nlo = lo + int64_t(c - 1) * step + 1;
    const int64_t nhi = lo + int64_t(c) * step;
    lo = nlo;
    hi = nhi < hi ? nhi : hi;
  }
  const uint32_t m = __ballot_sync(0xffffffffu, lo + lane < hi && s[lo + lane] < v);
  return lo + __popc(m);
}

// s[pos + 1 .. n] = s[pos .. n - 1] (order kept), top chunk first; four
// chunks in flight per step so the loads of a global-memory shift overlap.
__device__ __forceinline__ void warp_shift_up(double* s, int64_t pos, int64_t n) {
  const int lane = threadIdx.x & 31;
  for (int64_t top = n; top > pos; top -= 128) {
    double t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t idx = top - 1 - lane - 32 * u;
      t[u] = idx >= pos ? s[idx] : 0.0;
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t idx = top - 1 - lane - 32 * u;
      if (idx >= pos) s[idx + 1] = t[u];
    }
    __syncwarp();
  }
}

// s[pos .. n - 2] = s[pos + 1 .. n - 1], bottom chunk first.
__device__ __forceinline__ void warp_shift_down(double* s, int64_t pos, int64_t n) {
  const int lane = threadIdx.x & 31;
  for (int64_t b = pos + 1; b < n; b += 128) {
    double t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t idx = b + lane + 32 * u;
      t[u] = idx < n ? s[idx] : 0.0;
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t idx = b + lane + 32 * u;
      if (idx < n) s[idx - 1] = t[u];
    }
    __syncwarp();
  }
}

// EmpiricalDistribution::add (distribution.cpp:91-111) + check_convergence
// (113-123), all lanes of the warp. s / ring / snap hold `cap` doubles each;
// the ring keeps the n retained samples from d.head. Returns false when the
// retained window would not fit (capacity error); *newly is set when this
// sample made the distribution converge.
__device__ __forceinline__ bool dist_add_warp(double* s, double* ring, double* snap, int64_t cap,
                                              const DistCfg& cfg, DistScal& d, double v, bool* newly) {
  const int lane = threadIdx.x & 31;
  if (d.n + 1 > cap) return false;
  // sorted_.insert(lower_bound(value), value)
  const int64_t pos = warp_lower_bound(s, d.n, v);
  warp_shift_up(s, pos, d.n);
  if (lane == 0) s[pos] = v;
  d.n += 1;
  if (cfg.window_cap > 0) {
    if (lane == 0) ring[(d.head + d.n - 1) % cap] = v;  // arrival_order_.push_back
    __syncwarp();
    if (uint64_t(d.n) > uint64_t(cfg.window_cap)) {  // evict the oldest
      const double oldest = ring[d.head];
      d.head = (d.head + 1) % cap;
      const int64_t ep = warp_lower_bound(s, d.n, oldest);
      warp_shift_down(s, ep, d.n);
      d.n -= 1;
    }
  }
  __syncwarp();
  d.total += 1;
  if (d.total == d.next_cp) {  // check_convergence
    if (d.snap_n > 0) {
      double w = 0.0, sum = 0.0;
      if (lane == 0) {
        w = w1_walk(snap, uint64_t(d.snap_n), s, uint64_t(d.n));
        for (int64_t j = 0; j < d.n; ++j) sum = __dadd_rn(sum, s[j]);  // mean(): sequential
      }
      w = __shfl_sync(0xffffffffu, w, 0);
      sum = __shfl_sync(0xffffffffu, sum, 0);
      const double mean = __ddiv_rn(sum, static_cast<double>(d.n));
      const double t = __dmul_rn(cfg.threshold, mean);
      const double tau = t > 1e-12 ? t : 1e-12;  // std::max(t, 1e-12)
      d.last = w;
      if (w < tau) {
        if (!d.conv) *newly = true;
        d.conv = 1;
      }
    }
    __syncwarp();
    for (int64_t j = lane; j < d.n; j += 32) snap[j] = s[j];  // snapshot_ = sorted_
    d.snap_n = d.n;
    __syncwarp();
    d.next_cp *= 2;
  }
  return true;
}

// quantile_sorted (distribution.cpp:33-44), n >= 1.
__device__ __forceinline__ double quantile_sorted_d(const double* s, int64_t n, double p) {
  if (p <= 0.0) return s[0];
  if (p >= 1.0) return s[n - 1];
  const double pos = __dmul_rn(p, static_cast<double>(n - 1));
  const int64_t lo = static_cast<int64_t>(pos);
  const double frac = __dsub_rn(pos, static_cast<double>(lo));
  if (lo + 1 >= n) return s[n - 1];
  return __dadd_rn(s[lo], __dmul_rn(frac, __dsub_rn(s[lo + 1], s[lo])));
}

// glibc 2.39 __cbrt (sysdeps/ieee754/dbl-64/s_cbrt.c), finite x.
__device__ __forceinline__ double cbrt_glibc(double x) {
  const double kFactor[5] = {1.0 / 1.5874010519681994748, 1.0 / 1.2599210498948731648, 1.0,
                             1.2599210498948731648, 1.5874010519681994748};
  int xe = 0;
  const double xm = frexp(fabs(x), &xe);
  if (xe == 0 && x == 0.0) return __dadd_rn(x, x);
  double u = __dsub_rn(0.784932344976639262, __dmul_rn(0.145263899385486377, xm));
  u = __dadd_rn(-1.83469277483613086, __dmul_rn(u, xm));
  u = __dadd_rn(2.44693122563534430, __dmul_rn(u, xm));
  u = __dadd_rn(-2.11499494167371287, __dmul_rn(u, xm));
  u = __dadd_rn(1.50819193781584896, __dmul_rn(u, xm));
  u = __dadd_rn(0.354895765043919860, __dmul_rn(u, xm));
  const double t2 = __dmul_rn(__dmul_rn(u, u), u);
  const double num = __dmul_rn(u, __dadd_rn(t2, __dmul_rn(2.0, xm)));
  const double ym = __dmul_rn(__ddiv_rn(num, __dadd_rn(__dmul_rn(2.0, t2), xm)), kFactor[2 + xe % 3]);
  return ldexp(ym, xe / 3);
}

// mode_estimate(sorted, 16).value (distribution.cpp:46-86), all lanes; n >= 1.
// Bin index (x - lo) * scale truncated is monotone in x, so the count of
// bin b is the distance between the first samples of bins b and b + 1: each
// lane binary-searches the boundaries of its bins.
__device__ __forceinline__ double mode_estimate_warp(const double* s, int64_t n, int64_t min_samples) {
  const int lane = threadIdx.x & 31;
  if (n < min_samples) return quantile_sorted_d(s, n, 0.5);
  const double lo = s[0], hi = s[n - 1];
  if (!(hi > lo)) return lo;
  const double nd = static_cast<double>(n);
  const double iqr = __dsub_rn(quantile_sorted_d(s, n, 0.75), quantile_sorted_d(s, n, 0.25));
  int64_t bins = 64;
  if (iqr > 0.0) {
    const double width = __ddiv_rn(__dmul_rn(2.0, iqr), cbrt_glibc(nd));
    const double b = ceil(__ddiv_rn(__dsub_rn(hi, lo), width));
    bins = b >= 4096.0 ? 4096 : (b <= 1.0 ? 1 : static_cast<int64_t>(b));
  }
  const double range = __dsub_rn(hi, lo);
  const double scale = __ddiv_rn(static_cast<double>(bins), range);
  // first position whose bin index exceeds b  (= count of samples in bins <= b)
  auto upto = [&](int64_t b) -> int64_t {
    if (b >= bins - 1) return n;
    const double lim = static_cast<double>(b + 1);
    int64_t l = 0, h = n;
    while (l < h) {
      const int64_t m = (l + h) >> 1;
      if (__dmul_rn(__dsub_rn(s[m], lo), scale) < lim) l = m + 1;
      else h = m;
    }
    return l;
  };
  int64_t best_c = -1, best_b = 0, carry = 0;
  for (int64_t b0 = 0; b0 < bins; b0 += 32) {
    const int64_t b = b0 + lane;
    const int64_t e = b < bins ? upto(b) : n;
    int64_t prev = __shfl_up_sync(0xffffffffu, e, 1);
    if (lane == 0) prev = carry;
    const int64_t c = b < bins ? e - prev : -1;
    if (c > best_c) {  // lanes visit ascending bins: strict > keeps the lowest
      best_c = c;
      best_b = b;
    }
    carry = __shfl_sync(0xffffffffu, e, 31);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t c2 = __shfl_xor_sync(0xffffffffu, best_c, o);
    const int64_t b2 = __shfl_xor_sync(0xffffffffu, best_b, o);
    if (c2 > best_c || (c2 == best_c && b2 < best_b)) {
      best_c = c2;
      best_b = b2;
    }
  }
  return __dadd_rn(lo, __ddiv_rn(__dmul_rn(__dadd_rn(static_cast<double>(best_b), 0.5), range),
                                 static_cast<double>(bins)));
}

// classical_mds_1d (priority.cpp:67-100) for an n x n distance matrix d
// (row-major), one thread. Scratch: 3 n^2 doubles. coords[n] out.
__device__ inline void mds_1d_thread(const double* d, int n, double* scratch, double* coords) {
  double* a = scratch;          // b, then the Jacobi iterate
  double* t = scratch + n * n;  // product temporaries
  double* v = t + n * n;        // eigenvectors
  const double inv_n = __ddiv_rn(1.0, static_cast<double>(n));
  // x = -0.5 * centering (element-wise), centering = I - 1/n
  auto cen = [&](int i, int j) { return __dsub_rn(i == j ? 1.0 : 0.0, inv_n); };
  // t = x * sq   (sq = d .* d), Eigen-shim product order: m(i,j) += x(i,k) * y(k,j)
  for (int i = 0; i < n * n; ++i) t[i] = 0.0;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      const double xik = __dmul_rn(-0.5, cen(i, k));
      for (int j = 0; j < n; ++j) {
        const double sq = __dmul_rn(d[k * n + j], d[k * n + j]);
        t[i * n + j] = __dadd_rn(t[i * n + j], __dmul_rn(xik, sq));
      }
    }
  // a = t * centering
  for (int i = 0; i < n * n; ++i) a[i] = 0.0;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      const double xik = t[i * n + k];
      for (int j = 0; j < n; ++j) a[i * n + j] = __dadd_rn(a[i * n + j], __dmul_rn(xik, cen(k, j)));
    }
  // cyclic Jacobi (oracle/shim/Eigen/Dense SelfAdjointEigenSolver)
  for (int i = 0; i < n * n; ++i) v[i] = (i / n == i % n) ? 1.0 : 0.0;
  double total = 0.0;
  for (int p = 0; p < n; ++p)
    for (int q = 0; q < n; ++q) total = __dadd_rn(total, __dmul_rn(a[p * n + q], a[p * n + q]));
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off = __dadd_rn(off, __dmul_rn(a[p * n + q], a[p * n + q]));
    if (off <= __dmul_rn(1e-30, total) || off < 1e-300) break;
    for (int p = 0; p < n; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[p * n + q];
        if (fabs(apq) < 1e-300) continue;
        const double theta = __ddiv_rn(__dsub_rn(a[q * n + q], a[p * n + p]), __dmul_rn(2.0, apq));
        const double tt = __ddiv_rn(theta >= 0.0 ? 1.0 : -1.0,
                                    __dadd_rn(fabs(theta), __dsqrt_rn(__dadd_rn(__dmul_rn(theta, theta), 1.0))));
        const double c = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__dmul_rn(tt, tt), 1.0)));
        const double sn = __dmul_rn(tt, c);
        for (int k = 0; k < n; ++k) {
          const double akp = a[k * n + p], akq = a[k * n + q];
          a[k * n + p] = __dsub_rn(__dmul_rn(c, akp), __dmul_rn(sn, akq));
          a[k * n + q] = __dadd_rn(__dmul_rn(sn, akp), __dmul_rn(c, akq));
        }
        for (int k = 0; k < n; ++k) {
          const double apk = a[p * n + k], aqk = a[q * n + k];
          a[p * n + k] = __dsub_rn(__dmul_rn(c, apk), __dmul_rn(sn, aqk));
          a[q * n + k] = __dadd_rn(__dmul_rn(sn, apk), __dmul_rn(c, aqk));
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = v[k * n + p], vkq = v[k * n + q];
          v[k * n + p] = __dsub_rn(__dmul_rn(c, vkp), __dmul_rn(sn, vkq));
          v[k * n + q] = __dadd_rn(__dmul_rn(sn, vkp), __dmul_rn(c, vkq));
        }
      }
    }
  }
  // stable ascending sort by diagonal: the last entry is the highest index
  // among the maximal diagonal values
  int src = 0;
  for (int j = 1; j < n; ++j)
    if (!(a[j * n + j] < a[src * n + src])) src = j;
  const double lambda = a[src * n + src];
  if (lambda <= 1e-15) {
    for (int i = 0; i < n; ++i) coords[i] = 0.0;
    return;
  }
  const double scale = __dsqrt_rn(lambda);
  for (int i = 0; i < n; ++i) coords[i] = __dmul_rn(scale, v[i * n + src]);
}

}  // namespace kx

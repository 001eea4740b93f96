// Shared device helpers for the B200 (sm_100a) Kairos scheduling path.
//
// FP64 parity rule: every multiply-add site the
// reference evaluates as two rounded operations is written here with the
// explicit round-to-nearest intrinsics (__dmul_rn / __dadd_rn / __dsub_rn),
// and the library is additionally compiled with --fmad=false, so no FMA
// contraction can change a result bit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace kx {

constexpr double kTimeEpsilon = 1e-9;  // workflow.hpp:34

struct KxError : std::runtime_error {
  int code;
  KxError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define KX_CUDA(call)                                                           \
  do {                                                                          \
    cudaError_t kx_e_ = (call);                                                 \
    if (kx_e_ != cudaSuccess)                                                   \
      throw ::kx::KxError(4, std::string(#call) + ": " + cudaGetErrorString(kx_e_)); \
  } while (0)

extern std::atomic<long long> g_kx_launches;  // diagnostics: kernels launched

// Runs `f` once per CUDA device of the calling thread's current context,
// race-free across threads (kernel attributes and occupancy are per device;
// handles on several devices and threads share no other state).
constexpr int kMaxDevices = 64;
template <typename F>
void once_per_device(std::once_flag (&flags)[kMaxDevices], F&& f) {
  int dev = 0;
  KX_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) throw KxError(4, "device ordinal out of range");
  std::call_once(flags[dev], f);
}

#define KX_CHECK_LAUNCH()                                  \
  do {                                                     \
    ::kx::g_kx_launches.fetch_add(1, std::memory_order_relaxed); \
    KX_CUDA(cudaGetLastError());                           \
  } while (0)

// Per-phase CUDA-event timing on the launching stream (bench / ncu
// cross-check). Events are recorded only when enabled.
struct PhaseProfiler {
  struct Mark {
    int phase;
    cudaEvent_t a, b;
  };
  struct Phase {
    std::string name;
    double ms = 0.0;
    long long launches = 0;
    double bytes = 0.0;
  };
  bool enabled = false;
  std::vector<Phase> phases;
  std::vector<Mark> pending;
  std::vector<cudaEvent_t> pool;
  int open_phase = -1;
  cudaEvent_t open_ev = nullptr;

  cudaEvent_t take() {
    if (pool.empty()) {
      cudaEvent_t e;
      KX_CUDA(cudaEventCreate(&e));
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  int phase_id(const char* name, double bytes) {
    for (size_t i = 0; i < phases.size(); ++i)
      if (phases[i].name == name) {
        phases[i].bytes += bytes;
        phases[i].launches += 1;
        return static_cast<int>(i);
      }
    Phase p;
    p.name = name;
    p.bytes = bytes;
    p.launches = 1;
    phases.push_back(p);
    return static_cast<int>(phases.size() - 1);
  }
  void begin(const char* name, double alg_bytes, cudaStream_t st) {
    if (!enabled) return;
    open_phase = phase_id(name, alg_bytes);
    open_ev = take();
    KX_CUDA(cudaEventRecord(open_ev, st));
  }
  void end(cudaStream_t st) {
    if (!enabled || open_phase < 0) return;
    cudaEvent_t e = take();
    KX_CUDA(cudaEventRecord(e, st));
    pending.push_back({open_phase, open_ev, e});
    open_phase = -1;
    if (pending.size() > 2048) drain();
  }
  void drain() {
    for (auto& m : pending) {
      KX_CUDA(cudaEventSynchronize(m.b));
      float ms = 0.f;
      KX_CUDA(cudaEventElapsedTime(&ms, m.a, m.b));
      phases[m.phase].ms += ms;
      pool.push_back(m.a);
      pool.push_back(m.b);
    }
    pending.clear();
  }
  void reset() {
    drain();
    phases.clear();
  }
  ~PhaseProfiler() {
    for (auto& m : pending) {
      cudaEventDestroy(m.a);
      cudaEventDestroy(m.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

__host__ __device__ inline int ceil_log2_u64(uint64_t v) {
  int b = 0;
  while ((uint64_t(1) << b) < v) ++b;
  return b;
}

// Order-preserving map from a (non-NaN) double to u64: a < b (as doubles)
// iff map(a) < map(b); -0.0 is canonicalised to +0.0 first.
__device__ __forceinline__ uint64_t ordered_bits(double x) {
  if (x == 0.0) x = 0.0;
  uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_ordered_bits(uint64_t u) {
  u = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
  return __longlong_as_double(static_cast<long long>(u));
}

// peak_in_slot (dispatcher.cpp:33-42), bit-exact: no contraction.
__device__ __forceinline__ double peak_in_slot_dev(double P, double k, double t0,
                                                   double t_end, int64_t slot,
                                                   double slot_len) {
  const double slot_start = __dmul_rn(static_cast<double>(slot), slot_len);
  const double slot_end = __dadd_rn(slot_start, slot_len);
  if (slot_end <= __dadd_rn(t0, kTimeEpsilon) ||
      slot_start >= __dsub_rn(t_end, kTimeEpsilon)) {
    return 0.0;
  }
  const double eval_t = (t_end < slot_end) ? t_end : slot_end;  // std::min(slot_end, t_end)
  return __dadd_rn(P, __dmul_rn(k, __dsub_rn(eval_t, t0)));
}

// span_slots bounds (dispatcher.cpp:19-31): first/last inclusive; empty when
// expected_duration <= 0 (returns last < first).
__device__ __forceinline__ void span_bounds_dev(double t0, double T, double slot_len,
                                                int64_t* first, int64_t* last) {
  if (T <= 0.0) {
    *first = 0;
    *last = -1;
    return;
  }
  const double t_end = __dadd_rn(t0, T);
  *first = static_cast<int64_t>(floor(__ddiv_rn(__dadd_rn(t0, kTimeEpsilon), slot_len)));
  *last = static_cast<int64_t>(floor(__ddiv_rn(__dsub_rn(t_end, kTimeEpsilon), slot_len)));
}

}  // namespace kx

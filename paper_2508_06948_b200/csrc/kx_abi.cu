// extern "C" implementation of include/kairos_b200.h: handle lifecycle,
// device allocation, uploads, and the launches of K1-K5. Host code here is
// plumbing only; every computation runs in the CUDA kernels.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <numeric>
#include <cmath>
#include <cstring>
#include <memory>
#include <type_traits>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/kairos_b200.h"
#include "kx_common.cuh"
#include "kx_dispatch.cuh"
#include "kx_engine.cuh"
#include "kx_order.cuh"
#include "kx_profiler.cuh"
#include "kx_state.cuh"

namespace kx {
void launch_expected_T(int32_t n_agents, const int64_t* off, const double* samples, int64_t min_samples,
                       double fallback, double* out, cudaStream_t st);
void launch_w1_matrix(int32_t n_agents, const int64_t* off, const double* samples, double* d, int sms,
                      cudaStream_t st);
std::atomic<long long> g_kx_launches{0};
void sorting_accuracy(int64_t n, const int32_t* agent, const double* remaining, const uint8_t* present,
                      int32_t scope_all, uint64_t* pairs_out, double* correct_out, int sms,
                      cudaStream_t st);

void launch_orchestrator_dp(int64_t n_wf, const int64_t* off, const int32_t* parent,
                            const int64_t* prompt, const int64_t* target, double prefill,
                            double decode, uint64_t uid_base, uint64_t* uid_out, double* pure_out,
                            double* rem_out, int* error, int sms, cudaStream_t st);
void launch_record_remaining(int64_t n_wf, const int64_t* off, const double* es, const double* ee,
                             double* fin, double* samples, int sms, cudaStream_t st);

// ---- small utility kernels ---------------------------------------------
__global__ void k_fill_rem(QueueDev q, int64_t n, const double* __restrict__ table,
                           const uint8_t* __restrict__ present, uint64_t base, int64_t tn) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    double r = 0.0;  // OracleScheduler: absent uid -> 0.0 (scheduler.hpp:86-87)
    if (table) {
      const uint64_t u = q.uid[i];
      if (u >= base && u - base < static_cast<uint64_t>(tn) && present[u - base]) r = table[u - base];
    }
    q.rem[i] = r;
  }
}

__global__ void k_validate_queue(QueueDev q, int64_t n, int n_agents, int need_pure, int check_tokens,
                                 int* __restrict__ err) {
  int e = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int32_t a = q.agent[i];
    if (a < 0 || a >= n_agents) e |= 1;
    const double x = q.app_start[i], y = q.queue_enter[i];
    if (x != x || y != y) e |= 2;
    if (need_pure && !(q.pure_exec[i] >= 0.0)) e |= 8;
    if (check_tokens && (q.prompt[i] < 0 || q.kept[i] < 0)) e |= 8;
  }
  if (e) atomicOr(err, e);
}

__global__ void k_flag_count(const uint8_t* __restrict__ flags, int64_t n, int chunk,
                             uint32_t* __restrict__ keep_counts) {
  const int64_t b = int64_t(blockIdx.x) * chunk;
  const int64_t e = min(b + chunk, n);
  uint32_t c = 0;
  for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) c += flags[i] ? 0u : 1u;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ uint32_t s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    keep_counts[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024)
k_scan_counts(uint32_t* __restrict__ c, int64_t m, int64_t* __restrict__ total) {
  // Exclusive scan of m chunk counts in place, one CTA: each thread sums a
  // contiguous run, a block scan of the run sums, then the runs are written.
  __shared__ uint64_t wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t per = (m + blockDim.x - 1) / blockDim.x;
  const int64_t b = int64_t(tid) * per, e = min(b + per, m);
  uint64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += c[i];
  uint64_t x = s;  // inclusive warp scan
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    uint64_t w = lane < nw ? wsum[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) wsum[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  uint64_t acc = x - s + (warp > 0 ? wsum[warp - 1] : 0);
  for (int64_t i = b; i < e; ++i) {
    const uint32_t v = c[i];
    c[i] = static_cast<uint32_t>(acc);
    acc += v;
  }
  if (tid == blockDim.x - 1) *total = static_cast<int64_t>(wsum[(blockDim.x >> 5) - 1]);
}

// All queue columns of a chunk in one pass (ReadyQueue::pop of the placed
// requests keeps the rest in order): flags read once, every kept request's
// columns moved to its compacted position in `dst`.
__global__ void __launch_bounds__(256)
k_compact_queue(QueueDev src, QueueDev dst, int64_t n, int chunk, const uint32_t* __restrict__ offs) {
  __shared__ uint32_t wcnt[2][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = int64_t(blockIdx.x) * chunk;
  const int64_t e = min(b + chunk, n);
  uint32_t out = offs[blockIdx.x];
  int buf = 0;
  for (int64_t i0 = b; i0 < e; i0 += 256) {
    const int64_t i = i0 + threadIdx.x;
    const bool keep = i < e && !src.admitted[i];
    const uint32_t m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wcnt[buf][warp] = __popc(m);
    __syncthreads();
    uint32_t excl = 0, total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t x = wcnt[buf][w];
      excl += w < warp ? x : 0u;
      total += x;
    }
    if (keep) {
      const int64_t d = int64_t(out) + excl + __popc(m & ((1u << lane) - 1u));
      dst.agent[d] = src.agent[i];
      dst.prompt[d] = src.prompt[i];
      dst.app_start[d] = src.app_start[i];
      dst.queue_enter[d] = src.queue_enter[i];
      dst.msg[d] = src.msg[i];
      dst.uid[d] = src.uid[i];
      dst.kept[d] = src.kept[i];
      dst.pure_exec[d] = src.pure_exec[i];
      dst.rem[d] = src.rem[i];
    }
    out += total;
    buf ^= 1;
  }
}

}  // namespace kx

using namespace kx;

namespace {

thread_local std::string g_last_error;

template <typename F>
int guard(F&& f) {
  try {
    f();
    g_last_error.clear();
    return KX_OK;
  } catch (const KxError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return KX_ERR_INVALID;
  } catch (const std::logic_error& e) {
    g_last_error = e.what();
    return KX_ERR_LOGIC;
  } catch (const std::bad_alloc& e) {
    g_last_error = "out of host memory";
    return KX_ERR_CAPACITY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return KX_ERR_RUNTIME;
  }
}

[[noreturn]] void fail(int code, const std::string& m) { throw KxError(code, m); }

}  // namespace

// kx_last_error's message for entry points defined in other translation
// units (kx_workload.cpp).
namespace kx {
void set_last_error(const char* m) { g_last_error = m ? m : ""; }
}  // namespace kx

namespace {

void require(bool ok, const std::string& m) {
  if (!ok) throw std::invalid_argument(m);
}

int sm_count(int dev) {
  int n = 0;
  KX_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

void ensure_device(int dev) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count <= dev)
    fail(KX_ERR_CUDA, "no CUDA device available (the kairos_b200 path has no CPU fallback)");
  cudaDeviceProp p{};
  KX_CUDA(cudaGetDeviceProperties(&p, dev));
  if (p.major < 10)
    fail(KX_ERR_CUDA, "kairos_b200 is built for sm_100a (B200); found sm_" +
                          std::to_string(p.major) + std::to_string(p.minor));
  KX_CUDA(cudaSetDevice(dev));
}

// Device bump allocation inside one cudaMalloc'ed blob.
struct Blob {
  char* base = nullptr;
  size_t size = 0;
};

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

struct Layout {
  size_t off = 0;
  template <typename T>
  size_t take(size_t count) {
    const size_t o = off;
    off = align_up(off + count * sizeof(T));
    return o;
  }
};

}  // namespace

struct kx_sched {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  kx_dispatcher_config dcfg{};
  int n_pools = 0;
  int n_inst = 0;
  int ring = 256;
  int max_inst_per_pool = 0;
  int64_t cap = 0;
  int64_t n = 0;
  int32_t max_agents = 0;
  int32_t n_agents = 0;
  int32_t sched_kind = KX_SCHED_KAIROS;
  int32_t n_pk_classes = 1;
  int32_t n_depth_classes = 1;
  std::vector<kx_instance> inst_host;
  std::vector<int32_t> pool_begin_host;

  QueueDev q{};
  QueueDev q_dev{};  // the queue blob's own columns (q differs while mapped)
  bool q_mapped = false;
  AgentsDev a{};
  InstDev in{};
  int32_t* pool_begin = nullptr;
  Blob queue_blob, agent_blob, inst_const_blob, inst_mut_blob, inst_ckpt_blob, ws_blob, log_blob;
  Blob queue_alt_blob;  // compaction target of kx_queue_remove_admitted (allocated on first use)
  char* fetch_pinned = nullptr;  // pinned staging of kx_dispatch_fetch (allocated on first use)
  size_t fetch_pinned_size = 0;
  bool have_ckpt = false;

  OrderWorkspace ws{};
  OrderResultDev order{};
  bool order_valid = false;
  int64_t order_n = 0;

  double* rem_table = nullptr;
  uint8_t* rem_present = nullptr;
  uint64_t rem_base = 0;
  int64_t rem_n = 0;

  int64_t log_cap = 0;
  kx_decision* rows = nullptr;
  double* cand = nullptr;
  int64_t* row_count = nullptr;
  int64_t* admitted_count = nullptr;
  int* pool_status = nullptr;
  bool dispatch_valid = false;

  // scratch
  int* err_flag = nullptr;
  double* scratch_d = nullptr;
  int64_t* scratch_i = nullptr;
  int* scratch_s = nullptr;
  uint32_t* compact_counts = nullptr;
  int64_t* compact_total = nullptr;

  PhaseProfiler prof;

  // Sort/dispatch overlap (tick): top-K order prefix + dispatch phase 1 on
  // `side` while the full sort runs on `stream`.
  bool overlap = false;
  cudaStream_t side = nullptr;
  cudaGraph_t graph = nullptr;          // captured step (kx_graph_*)
  cudaGraphExec_t graph_exec = nullptr;
  // what the captured calls were recorded against (launch-time checks) and
  // the handle state they leave behind (restored after each replay)
  int64_t graph_n = 0;
  const char* graph_queue_base = nullptr;
  bool graph_order_valid = false, graph_dispatch_valid = false;
  OrderResultDev graph_order{};
  cudaEvent_t ev_keys = nullptr, ev_released = nullptr, ev_disp = nullptr;
  Blob topk_blob;
  TopKWork topk{};
  DispResume* resume = nullptr;

  // waiting lists (round_robin / static_threshold rounds)
  WaitRec* wrec = nullptr;       // [n_inst * wcap]
  int64_t wcap = 0;
  kx_admission* adm = nullptr;   // [n_pools * log_cap]
  int64_t* adm_count = nullptr;  // [n_pools]
  int32_t round = 0;
  WaitRec* wckpt = nullptr;      // checkpoint copy
  int64_t wckpt_cap = 0;
};

namespace {

void alloc_blob(Blob& b, size_t bytes) {
  b.size = std::max<size_t>(bytes, 256);
  KX_CUDA(cudaMalloc(reinterpret_cast<void**>(&b.base), b.size));
  KX_CUDA(cudaMemset(b.base, 0, b.size));
  // legacy-stream work is not ordered before the handle's non-blocking streams
  KX_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
}

void free_blob(Blob& b) {
  if (b.base) cudaFree(b.base);
  b.base = nullptr;
}

template <typename T>
T* at(const Blob& b, size_t off) {
  return reinterpret_cast<T*>(b.base + off);
}

constexpr int64_t kCompactChunk = 8192;

void check_err_flag(kx_sched* s, const char* what) {
  int h = 0;
  KX_CUDA(cudaMemcpyAsync(&h, s->err_flag, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
  KX_CUDA(cudaStreamSynchronize(s->stream));
  if (h & 1) fail(KX_ERR_INVALID, std::string(what) + ": agent index outside the agent table");
  if (h & 2) fail(KX_ERR_INVALID, std::string(what) + ": NaN time value");
  if (h & 4) fail(KX_ERR_INVALID, std::string(what) + ": parent link is not parents-first");
  if (h & 8) fail(KX_ERR_INVALID, std::string(what) + ": negative token count or pure_exec");
}

void create_impl(const kx_sched_config* cfg, kx_sched** out) {
  require(cfg && out, "null argument");
  require(cfg->n_pools >= 1 && cfg->n_pools <= 1024, "n_pools must be in [1, 1024]");
  require(cfg->n_instances >= 1 && cfg->instances, "dispatcher needs matching instance lists");
  require(cfg->queue_capacity >= 1 && cfg->queue_capacity < (int64_t(1) << 30),
          "queue_capacity must be in [1, 2^30)");
  const int ring = cfg->slot_ring ? cfg->slot_ring : 256;
  require(ring >= 64 && (ring & (ring - 1)) == 0, "slot_ring must be a power of two >= 64");
  const auto& dc = cfg->dispatcher;
  require(dc.slot_len > 0.0, "slot_len must be positive");
  require(dc.policy >= 0 && dc.policy <= 2, "unknown dispatcher policy");
  require(cfg->max_agents >= 1, "max_agents must be positive");

  std::vector<int32_t> pool_begin(cfg->n_pools + 1, 0);
  int prev_pool = -1;
  std::vector<int32_t> ids;
  for (int i = 0; i < cfg->n_instances; ++i) {
    const kx_instance& p = cfg->instances[i];
    require(p.pool >= 0 && p.pool < cfg->n_pools, "instance pool out of range");
    require(p.pool >= prev_pool, "instances must be grouped by pool (non-decreasing pool)");
    require(p.capacity_tokens > 0.0 && p.decode_rate > 0.0 && p.prefill_rate > 0.0 &&
                p.max_batch >= 1,
            "instance profile fields must be positive");
    prev_pool = p.pool;
    pool_begin[p.pool + 1] += 1;
    ids.push_back(p.id);
  }
  std::sort(ids.begin(), ids.end());
  require(std::adjacent_find(ids.begin(), ids.end()) == ids.end(), "duplicate instance id");
  int max_pp = 0;
  for (int p = 0; p < cfg->n_pools; ++p) {
    require(pool_begin[p + 1] >= 1, "every pool needs at least one instance");
    max_pp = std::max(max_pp, pool_begin[p + 1]);
    pool_begin[p + 1] += pool_begin[p];
  }
  require(max_pp <= kMaxInstPerPool, "too many instances in one pool (max 512)");

  ensure_device(cfg->device);
  auto s = std::make_unique<kx_sched>();
  s->device = cfg->device;
  s->sms = sm_count(cfg->device);
  KX_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  s->dcfg = dc;
  s->n_pools = cfg->n_pools;
  s->n_inst = cfg->n_instances;
  s->ring = ring;
  s->max_inst_per_pool = max_pp;
  s->cap = cfg->queue_capacity;
  s->max_agents = cfg->max_agents;
  s->inst_host.assign(cfg->instances, cfg->instances + cfg->n_instances);
  s->pool_begin_host = pool_begin;
  configure_sort_kernels();
  configure_dispatch_kernels();

  // queue SoA
  {
    const size_t N = static_cast<size_t>(s->cap);
    Layout L;
    const size_t o_agent = L.take<int32_t>(N), o_prompt = L.take<int64_t>(N),
                 o_app = L.take<double>(N), o_qe = L.take<double>(N), o_msg = L.take<uint64_t>(N),
                 o_uid = L.take<uint64_t>(N), o_kept = L.take<int64_t>(N),
                 o_pure = L.take<double>(N), o_rem = L.take<double>(N),
                 o_adm = L.take<uint8_t>(N);
    alloc_blob(s->queue_blob, L.off);
    auto& b = s->queue_blob;
    s->q = QueueDev{at<int32_t>(b, o_agent), at<int64_t>(b, o_prompt), at<double>(b, o_app),
                    at<double>(b, o_qe),     at<uint64_t>(b, o_msg),   at<uint64_t>(b, o_uid),
                    at<int64_t>(b, o_kept),  at<double>(b, o_pure),    at<double>(b, o_rem),
                    at<uint8_t>(b, o_adm)};
    s->q_dev = s->q;
    s->q_mapped = false;
  }
  // agent tables
  {
    const size_t A = static_cast<size_t>(s->max_agents);
    Layout L;
    const size_t o_pool = L.take<int32_t>(A), o_pk = L.take<double>(A),
                 o_pkr = L.take<uint32_t>(A), o_d = L.take<int32_t>(A),
                 o_dr = L.take<uint32_t>(A), o_T = L.take<double>(A);
    alloc_blob(s->agent_blob, L.off);
    auto& b = s->agent_blob;
    s->a = AgentsDev{at<int32_t>(b, o_pool), at<double>(b, o_pk), at<uint32_t>(b, o_pkr),
                     at<int32_t>(b, o_d),    at<uint32_t>(b, o_dr), at<double>(b, o_T)};
  }
  // instances: constant part
  {
    const size_t I = static_cast<size_t>(s->n_inst);
    Layout L;
    const size_t o_id = L.take<int32_t>(I), o_pool = L.take<int32_t>(I), o_cap = L.take<double>(I),
                 o_k = L.take<double>(I), o_pf = L.take<double>(I), o_mb = L.take<int32_t>(I),
                 o_pb = L.take<int32_t>(s->n_pools + 1), o_rk = L.take<int32_t>(I);
    alloc_blob(s->inst_const_blob, L.off);
    auto& b = s->inst_const_blob;
    s->in.id = at<int32_t>(b, o_id);
    s->in.pool = at<int32_t>(b, o_pool);
    s->in.cap = at<double>(b, o_cap);
    s->in.decode_rate = at<double>(b, o_k);
    s->in.prefill_rate = at<double>(b, o_pf);
    s->in.max_batch = at<int32_t>(b, o_mb);
    s->in.rank_li = at<int32_t>(b, o_rk);
    s->pool_begin = at<int32_t>(b, o_pb);
    std::vector<int32_t> vid(I), vpool(I), vmb(I);
    std::vector<double> vcap(I), vk(I), vpf(I);
    for (size_t i = 0; i < I; ++i) {
      vid[i] = s->inst_host[i].id;
      vpool[i] = s->inst_host[i].pool;
      vmb[i] = s->inst_host[i].max_batch;
      vcap[i] = s->inst_host[i].capacity_tokens;
      vk[i] = s->inst_host[i].decode_rate;
      vpf[i] = s->inst_host[i].prefill_rate;
    }
    KX_CUDA(cudaMemcpy(s->in.id, vid.data(), I * 4, cudaMemcpyHostToDevice));
    KX_CUDA(cudaMemcpy(s->in.pool, vpool.data(), I * 4, cudaMemcpyHostToDevice));
    KX_CUDA(cudaMemcpy(s->in.max_batch, vmb.data(), I * 4, cudaMemcpyHostToDevice));
    KX_CUDA(cudaMemcpy(s->in.cap, vcap.data(), I * 8, cudaMemcpyHostToDevice));
    KX_CUDA(cudaMemcpy(s->in.decode_rate, vk.data(), I * 8, cudaMemcpyHostToDevice));
    KX_CUDA(cudaMemcpy(s->in.prefill_rate, vpf.data(), I * 8, cudaMemcpyHostToDevice));
    KX_CUDA(cudaMemcpy(s->pool_begin, pool_begin.data(), (s->n_pools + 1) * 4,
                       cudaMemcpyHostToDevice));
    // the instances of each pool in InstanceId order (select_instance's tie
    // rule): local index by rank, ties by position
    std::vector<int32_t> vrank(I);
    for (int p = 0; p < s->n_pools; ++p) {
      const int ib = pool_begin[p], ni = pool_begin[p + 1] - ib;
      std::vector<int32_t> l(ni);
      std::iota(l.begin(), l.end(), 0);
      std::stable_sort(l.begin(), l.end(), [&](int32_t x, int32_t y) { return vid[ib + x] < vid[ib + y]; });
      for (int r = 0; r < ni; ++r) vrank[ib + r] = l[r];
    }
    KX_CUDA(cudaMemcpy(s->in.rank_li, vrank.data(), I * 4, cudaMemcpyHostToDevice));
  }
  // instances: mutable part (one blob so checkpoint/restore is one copy)
  {
    const size_t I = static_cast<size_t>(s->n_inst);
    const size_t R = static_cast<size_t>(ring);
    Layout L;
    const size_t o_live = L.take<double>(I), o_run = L.take<int32_t>(I),
                 o_wait = L.take<int32_t>(I), o_susp = L.take<uint8_t>(I),
                 o_base = L.take<int64_t>(I), o_hi = L.take<int64_t>(I),
                 o_usage = L.take<double>(I * R), o_ex = L.take<uint8_t>(I * R),
                 o_na = L.take<int32_t>(I), o_au = L.take<uint64_t>(I * kActiveCap),
                 o_ap = L.take<double>(I * kActiveCap), o_ak = L.take<double>(I * kActiveCap),
                 o_at = L.take<double>(I * kActiveCap), o_aT = L.take<double>(I * kActiveCap),
                 o_rr = L.take<int32_t>(s->n_pools);
    alloc_blob(s->inst_mut_blob, L.off);
    auto& b = s->inst_mut_blob;
    s->in.live_kv = at<double>(b, o_live);
    s->in.running = at<int32_t>(b, o_run);
    s->in.waiting = at<int32_t>(b, o_wait);
    s->in.suspended = at<uint8_t>(b, o_susp);
    s->in.base_slot = at<int64_t>(b, o_base);
    s->in.hi_slot = at<int64_t>(b, o_hi);
    s->in.usage = at<double>(b, o_usage);
    s->in.exists = at<uint8_t>(b, o_ex);
    s->in.n_active = at<int32_t>(b, o_na);
    s->in.act_uid = at<uint64_t>(b, o_au);
    s->in.act_P = at<double>(b, o_ap);
    s->in.act_k = at<double>(b, o_ak);
    s->in.act_t0 = at<double>(b, o_at);
    s->in.act_T = at<double>(b, o_aT);
    s->in.rr_next = at<int32_t>(b, o_rr);
    std::vector<int64_t> minus1(I, -1);  // hi_slot: nothing booked yet
    KX_CUDA(cudaMemcpy(s->in.hi_slot, minus1.data(), I * 8, cudaMemcpyHostToDevice));
    KX_CUDA(cudaStreamSynchronize(cudaStreamLegacy));  // the DMAs have landed before s->stream uses them
  }
  // order workspace + scratch
  {
    const size_t N = static_cast<size_t>(s->cap);
    const size_t P = static_cast<size_t>(s->n_pools);
    const size_t tie_cap = N / 2 + 1;
    Layout L;
    const size_t o_k0 = L.take<uint32_t>(N), o_k1 = L.take<uint32_t>(N),
                 o_v0 = L.take<uint32_t>(N), o_v1 = L.take<uint32_t>(N);
    const size_t lb_bytes = order_lookback_bytes(s->cap);
    const size_t o_lb = L.take<char>(lb_bytes);
    const size_t o_rng = L.take<PoolRange>(P), o_poff = L.take<int64_t>(P + 1),
                 o_rst = L.take<PoolRange>(P), o_sdone = L.take<uint32_t>(1);
    // header block
    Layout H;
    const size_t h_hist = H.take<uint32_t>(4 * 256), h_tiles = H.take<uint32_t>(8),
                 h_pc = H.take<uint32_t>(P), h_nb = H.take<uint32_t>(1),
                 h_err = H.take<int>(1);
    const size_t o_hdr = L.take<char>(H.off);
    const size_t o_bs = L.take<uint32_t>(tie_cap),
                 o_bl = L.take<uint32_t>(tie_cap);
    const size_t o_errf = L.take<int>(1), o_sd = L.take<double>(4), o_si = L.take<int64_t>(4),
                 o_ss2 = L.take<int>(4);
    const int64_t nchunks = (s->cap + kCompactChunk - 1) / kCompactChunk;
    const size_t o_cc = L.take<uint32_t>(nchunks + 1), o_ct = L.take<int64_t>(1);
    alloc_blob(s->ws_blob, L.off);
    auto& b = s->ws_blob;
    s->ws.keys[0] = at<uint32_t>(b, o_k0);
    s->ws.keys[1] = at<uint32_t>(b, o_k1);
    s->ws.vals[0] = at<uint32_t>(b, o_v0);
    s->ws.vals[1] = at<uint32_t>(b, o_v1);
    s->ws.lookback = at<uint32_t>(b, o_lb);
    s->ws.ranges = at<PoolRange>(b, o_rng);
    s->ws.range_stage = at<PoolRange>(b, o_rst);
    s->ws.sample_done = at<uint32_t>(b, o_sdone);  // zeroed with the blob
    {
      const std::vector<PoolRange> empty(P, PoolRange{~0ull, 0ull, 0.0, 0.0});
      KX_CUDA(cudaMemcpy(s->ws.range_stage, empty.data(), P * sizeof(PoolRange), cudaMemcpyHostToDevice));
      KX_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    }
    s->ws.pool_offsets = at<int64_t>(b, o_poff);
    s->ws.small_hdr = b.base + o_hdr;
    s->ws.small_hdr_bytes = H.off;
    char* hdr = b.base + o_hdr;
    s->ws.hist = reinterpret_cast<uint32_t*>(hdr + h_hist);
    s->ws.tile_counters = reinterpret_cast<uint32_t*>(hdr + h_tiles);
    s->ws.pool_counts = reinterpret_cast<uint32_t*>(hdr + h_pc);
    s->ws.n_big = reinterpret_cast<uint32_t*>(hdr + h_nb);
    s->ws.error_flags = reinterpret_cast<int*>(hdr + h_err);
    s->ws.big_starts = at<uint32_t>(b, o_bs);
    s->ws.big_lens = at<uint32_t>(b, o_bl);
    s->ws.tie_cap = static_cast<uint32_t>(tie_cap);
    s->err_flag = at<int>(b, o_errf);
    s->scratch_d = at<double>(b, o_sd);
    s->scratch_i = at<int64_t>(b, o_si);
    s->scratch_s = at<int>(b, o_ss2);
    s->compact_counts = at<uint32_t>(b, o_cc);
    s->compact_total = at<int64_t>(b, o_ct);
  }
  // overlap workspace
  if (s->n_pools <= kTopKMaxPools && dispatch_can_overlap(max_pp, ring) && !getenv("KX_NO_OVERLAP")) {
    const size_t P = static_cast<size_t>(s->n_pools);
    Layout L;
    const size_t o_st = L.take<TopKState>(P), o_h = L.take<uint32_t>(P * 256),
                 o_c = L.take<uint32_t>(P * kTopKMax), o_hd = L.take<uint32_t>(P * kTopKMax),
                 o_r = L.take<DispResume>(P), o_sb = L.take<uint32_t>(P), o_so = L.take<uint32_t>(P),
                 o_sc = L.take<uint32_t>(P);
    const size_t o_sk = L.take<uint32_t>(spec_list_words(s->n_pools)), o_sp = L.take<uint32_t>(P),
                 o_ck = L.take<uint32_t>(P * kTopKMax);
    alloc_blob(s->topk_blob, L.off);
    auto& b = s->topk_blob;
    s->topk.state = at<TopKState>(b, o_st);
    s->topk.hist = at<uint32_t>(b, o_h);
    s->topk.cand = at<uint32_t>(b, o_c);
    s->topk.heads = at<uint32_t>(b, o_hd);
    s->resume = at<DispResume>(b, o_r);
    s->topk.spec_bound = at<uint32_t>(b, o_sb);
    s->topk.spec_on = at<uint32_t>(b, o_so);
    s->topk.spec_count = at<uint32_t>(b, o_sc);
    s->topk.plist = at<uint32_t>(b, o_sk);
    s->topk.plist_count = at<uint32_t>(b, o_sp);
    s->topk.cand_key = at<uint32_t>(b, o_ck);
    if (const char* e = getenv("KX_TOPK_NEED"))  // test knob: force short prefixes
      s->topk.max_need = static_cast<uint32_t>(std::clamp(atoi(e), 1, kTopKMax));
    // The prefix select + dispatch chain is the tick's critical path: its
    // stream outranks the full sort's for SM slots.
    int prio_lo = 0, prio_hi = 0;
    KX_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    KX_CUDA(cudaStreamCreateWithPriority(&s->side, cudaStreamNonBlocking, prio_hi));
    KX_CUDA(cudaEventCreateWithFlags(&s->ev_keys, cudaEventDisableTiming));
    KX_CUDA(cudaEventCreateWithFlags(&s->ev_released, cudaEventDisableTiming));
    KX_CUDA(cudaEventCreateWithFlags(&s->ev_disp, cudaEventDisableTiming));
    s->overlap = true;
  }
  // decision log
  {
    int64_t per_pool = cfg->log_capacity_per_pool;
    if (per_pool <= 0) {
      int64_t mb_sum_max = 0;
      for (int p = 0; p < s->n_pools; ++p) {
        int64_t mb = 0;
        for (int i = pool_begin[p]; i < pool_begin[p + 1]; ++i) mb += s->inst_host[i].max_batch;
        mb_sum_max = std::max(mb_sum_max, mb);
      }
      per_pool = std::max<int64_t>(4096, 2 * mb_sum_max + 16 * max_pp);
    }
    s->log_cap = per_pool;
    const size_t P = static_cast<size_t>(s->n_pools);
    Layout L;
    const size_t o_rows = L.take<kx_decision>(P * per_pool),
                 o_cand = L.take<double>(P * per_pool * max_pp), o_rc = L.take<int64_t>(P),
                 o_ac = L.take<int64_t>(P), o_ps = L.take<int>(P);
    alloc_blob(s->log_blob, L.off);
    auto& b = s->log_blob;
    s->rows = at<kx_decision>(b, o_rows);
    s->cand = at<double>(b, o_cand);
    s->row_count = at<int64_t>(b, o_rc);
    s->admitted_count = at<int64_t>(b, o_ac);
    s->pool_status = at<int>(b, o_ps);
  }
  KX_CUDA(cudaDeviceSynchronize());
  *out = s.release();
}

void destroy_impl(kx_sched* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  free_blob(s->queue_blob);
  free_blob(s->queue_alt_blob);
  if (s->fetch_pinned) cudaFreeHost(s->fetch_pinned);
  free_blob(s->agent_blob);
  free_blob(s->inst_const_blob);
  free_blob(s->inst_mut_blob);
  free_blob(s->inst_ckpt_blob);
  free_blob(s->ws_blob);
  free_blob(s->log_blob);
  if (s->side) {
    cudaStreamSynchronize(s->side);
    cudaStreamDestroy(s->side);
  }
  free_blob(s->topk_blob);
  for (cudaEvent_t e : {s->ev_keys, s->ev_released, s->ev_disp})
    if (e) cudaEventDestroy(e);
  if (s->graph_exec) cudaGraphExecDestroy(s->graph_exec);
  if (s->graph) cudaGraphDestroy(s->graph);
  if (s->wrec) cudaFree(s->wrec);
  if (s->wckpt) cudaFree(s->wckpt);
  if (s->adm) cudaFree(s->adm);
  if (s->adm_count) cudaFree(s->adm_count);
  if (s->rem_table) cudaFree(s->rem_table);
  if (s->rem_present) cudaFree(s->rem_present);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

cudaMemcpyKind kind_in(int32_t mem) {
  return mem == KX_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
}
cudaMemcpyKind kind_out(int32_t mem) {
  return mem == KX_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
}

void refresh_rem(kx_sched* s) {
  if (s->n == 0) return;
  const int grid = static_cast<int>(std::min<int64_t>((s->n + 255) / 256, int64_t(s->sms) * 8));
  k_fill_rem<<<grid, 256, 0, s->stream>>>(s->q, s->n, s->rem_table, s->rem_present, s->rem_base,
                                          s->rem_n);
  KX_CHECK_LAUNCH();
}

std::vector<uint32_t> dense_rank(const std::vector<double>& v) {
  std::vector<double> d(v);
  for (double x : d) require(x == x, "NaN in agent table");
  std::sort(d.begin(), d.end());
  d.erase(std::unique(d.begin(), d.end(), [](double a, double b) { return a == b; }), d.end());
  std::vector<uint32_t> r(v.size());
  for (size_t i = 0; i < v.size(); ++i)
    r[i] = static_cast<uint32_t>(std::lower_bound(d.begin(), d.end(), v[i]) - d.begin());
  return r;
}

// Dense rank of each agent's value among the agents of its own pool: the
// compact key compares classes only within a pool (the pool id is its top
// field), so per-pool ranks need the fewest class bits and leave the most
// bits for the quantised time.
std::vector<uint32_t> pool_dense_rank(const std::vector<double>& v, const int32_t* pool, int n_pools) {
  std::vector<uint32_t> r(v.size(), 0);
  for (int p = 0; p < n_pools; ++p) {
    std::vector<double> sub;
    std::vector<size_t> idx;
    for (size_t i = 0; i < v.size(); ++i)
      if (pool[i] == p) {
        sub.push_back(v[i]);
        idx.push_back(i);
      }
    if (sub.empty()) continue;
    const auto rr = dense_rank(sub);
    for (size_t j = 0; j < idx.size(); ++j) r[idx[j]] = rr[j];
  }
  return r;
}

OrderParams order_params(const kx_sched* s) {
  OrderParams op{};
  op.policy = s->sched_kind;
  op.n_pools = s->n_pools;
  op.n_agents = s->n_agents;
  op.pool_bits = ceil_log2_u64(static_cast<uint64_t>(s->n_pools));
  int classes = 1;
  if (s->sched_kind == KX_SCHED_KAIROS) classes = s->n_pk_classes;
  if (s->sched_kind == KX_SCHED_TOPO) classes = s->n_depth_classes;
  op.class_bits = ceil_log2_u64(static_cast<uint64_t>(std::max(classes, 1)));
  const int need_q = std::min(32, ceil_log2_u64(static_cast<uint64_t>(std::max<int64_t>(s->n, 2))) + 8);
  int kb = op.pool_bits + op.class_bits + need_q;
  kb = std::min(32, (kb + 7) / 8 * 8);
  if (op.pool_bits + op.class_bits > 26)
    fail(KX_ERR_CAPACITY, "pool x class key space exceeds 26 bits");
  op.key_bits = kb;
  op.q_bits = kb - op.pool_bits - op.class_bits;
  return op;
}

void order_impl(kx_sched* s) {
  require(s->n_agents > 0 || s->n == 0, "agent tables not set");
  const OrderParams op = order_params(s);
  s->order = launch_order(s->q, s->a, op, s->n, s->ws, s->sms, s->stream, &s->prof);
  s->order_valid = true;
  s->order_n = s->n;
  s->dispatch_valid = false;
}

DispatchParams dispatch_params(const kx_sched* s, double now) {
  DispatchParams dp{};
  dp.oracle_T = s->dcfg.oracle_expected_time;
  dp.ring = s->ring;
  dp.logging = 1;
  dp.peak_stride = s->max_inst_per_pool;
  dp.log_cap = s->log_cap;
  dp.slot_len = s->dcfg.slot_len;
  dp.watermark = s->dcfg.resume_watermark;
  dp.now = now;
  return dp;
}

void dispatch_checks(const kx_sched* s) {
  require(s->n_agents > 0 || s->n == 0, "agent tables not set");
}

// Waiting-list storage: `per_inst` entries per instance (contents kept).
void ensure_waiting(kx_sched* s, int64_t per_inst) {
  if (!s->adm) {
    const size_t P = static_cast<size_t>(s->n_pools);
    KX_CUDA(cudaMalloc(reinterpret_cast<void**>(&s->adm), std::max<size_t>(1, P * s->log_cap) * sizeof(kx_admission)));
    KX_CUDA(cudaMalloc(reinterpret_cast<void**>(&s->adm_count), std::max<size_t>(1, P) * 8));
    KX_CUDA(cudaMemsetAsync(s->adm_count, 0, std::max<size_t>(1, P) * 8, s->stream));
  }
  if (per_inst <= s->wcap) return;
  const size_t I = static_cast<size_t>(s->n_inst);
  WaitRec* nr = nullptr;
  KX_CUDA(cudaMalloc(reinterpret_cast<void**>(&nr), std::max<size_t>(1, I * per_inst) * sizeof(WaitRec)));
  if (s->wrec) {
    KX_CUDA(cudaStreamSynchronize(s->stream));
    KX_CUDA(cudaMemcpy2D(nr, per_inst * sizeof(WaitRec), s->wrec, s->wcap * sizeof(WaitRec),
                         s->wcap * sizeof(WaitRec), I, cudaMemcpyDeviceToDevice));
    KX_CUDA(cudaFree(s->wrec));
  }
  s->wrec = nr;
  s->wcap = per_inst;
}

WaitDev waiting_dev(kx_sched* s) {
  WaitDev w{};
  w.rec = s->wrec;
  w.cap = s->wcap;
  w.adm = s->adm;
  w.adm_count = s->adm_count;
  w.rem_table = s->rem_table;
  w.rem_present = s->rem_present;
  w.rem_base = s->rem_base;
  w.rem_n = s->rem_table ? s->rem_n : 0;
  w.static_thr = s->dcfg.static_threshold;
  w.policy = s->dcfg.policy;
  w.sched_kind = s->sched_kind;
  w.round = s->round;
  return w;
}

void dispatch_impl(kx_sched* s, double now) {
  if (!s->order_valid || s->order_n != s->n)
    throw std::logic_error("dispatch round needs a current queue order (call kx_order first)");
  dispatch_checks(s);
  if (s->n > 0) KX_CUDA(cudaMemsetAsync(s->q.admitted, 0, static_cast<size_t>(s->n), s->stream));
  const DispatchParams dp = dispatch_params(s, now);
  if (s->dcfg.policy != KX_DISPATCH_TIME_SLOT) {  // round_robin / static_threshold
    ensure_waiting(s, 1024);
    ++s->round;
    s->prof.begin("dispatch", 0.0, s->stream);
    launch_dispatch_waiting(s->q, s->a, s->in, s->pool_begin, s->order.perm, s->ws.pool_offsets, dp,
                            waiting_dev(s), s->n_pools, s->max_inst_per_pool, s->rows, s->row_count,
                            s->admitted_count, s->pool_status, s->stream);
    s->prof.end(s->stream);
    s->dispatch_valid = true;
    return;
  }
  s->prof.begin("dispatch", 0.0, s->stream);
  launch_dispatch(s->q, s->a, s->in, s->pool_begin, s->order.perm, s->ws.pool_offsets, dp,
                  s->n_pools, s->max_inst_per_pool, s->rows, s->cand, s->row_count, s->admitted_count, s->pool_status,
                  s->stream);
  s->prof.end(s->stream);
  s->dispatch_valid = true;
}

// One scheduling tick = order + dispatch round. With the overlap workspace
// the round starts before the full sort ends: once the compact keys exist,
// the side stream selects each pool's top-K order prefix (radix select on
// the keys, exact sort of the few candidates) and runs the dispatch round
// over it (phase 1) while the main stream sorts; a pool whose round needs
// more heads than its prefix resumes over the full order (phase 2). The
// decisions are identical to order + dispatch_round: the prefix is exactly
// the head of the pool's order, and the round state carries over.
void tick_impl(kx_sched* s, double now) {
  if (!s->overlap || s->n == 0 || s->dcfg.policy != KX_DISPATCH_TIME_SLOT) {
    order_impl(s);
    dispatch_impl(s, now);
    return;
  }
  require(s->n_agents > 0, "agent tables not set");
  dispatch_checks(s);
  const OrderParams op = order_params(s);
  if (op.pool_bits > 8) {  // pools beyond the first radix digit: no prefix select
    order_impl(s);
    dispatch_impl(s, now);
    return;
  }
  const DispatchParams dp = dispatch_params(s, now);
  // Key generation also collects each pool's order prefix (every key below a
  // bound taken from the sample); right after it, the dispatch CTAs (high
  // priority stream) sort their prefix and run the round while the main
  // stream sorts the whole queue. A round that outlasts its prefix resumes
  // over the full order (phase 2).
  OrderHooks hooks;
  hooks.zero_bytes = s->q.admitted;
  hooks.n_zero_bytes = s->n;
  hooks.zero_words = s->topk.plist_count;  // k_sample_keys' per-pool counters
  hooks.n_zero_words = s->n_pools;
  hooks.before_keygen = [&] {
    launch_spec_bound(s->q, s->a, s->in, s->pool_begin, op, s->n, s->ws, s->topk, s->stream);
  };
  hooks.spec = KeygenSpec{s->topk.spec_bound, s->topk.spec_on, s->topk.spec_count, s->topk.cand,
                          s->topk.cand_key};
  hooks.after_keys = [&] {
    KX_CUDA(cudaEventRecord(s->ev_keys, s->stream));
    KX_CUDA(cudaStreamWaitEvent(s->side, s->ev_keys, 0));
    DispPhase ph{};
    ph.phase = 3;
    ph.pad = op.policy;
    ph.resume = s->resume;
    ph.spec_on = s->topk.spec_on;
    ph.spec_count = s->topk.spec_count;
    ph.cand = s->topk.cand;
    ph.cand_key = s->topk.cand_key;
    ph.pool_counts = s->ws.pool_counts;
    ph.heads_out = s->topk.heads;
    s->prof.begin("dispatch_prefix", 0.0, s->side);
    launch_dispatch(s->q, s->a, s->in, s->pool_begin, nullptr, s->ws.pool_offsets, dp, s->n_pools,
                    s->max_inst_per_pool, s->rows, s->cand, s->row_count, s->admitted_count,
                    s->pool_status, s->side, ph);
    s->prof.end(s->side);
    KX_CUDA(cudaEventRecord(s->ev_disp, s->side));
  };
  // the dispatch CTAs hold one SM per pool while the sort runs: size the
  // sort's grid-stride launches for the rest (no partial second wave)
  const int sort_sms = std::max(1, s->sms - s->n_pools);
  s->order = launch_order(s->q, s->a, op, s->n, s->ws, sort_sms, s->stream, &s->prof, &hooks);
  s->order_valid = true;
  s->order_n = s->n;
  KX_CUDA(cudaStreamWaitEvent(s->stream, s->ev_disp, 0));
  s->prof.begin("dispatch_rest", 0.0, s->stream);
  launch_dispatch(s->q, s->a, s->in, s->pool_begin, s->order.perm, s->ws.pool_offsets, dp, s->n_pools,
                  s->max_inst_per_pool, s->rows, s->cand, s->row_count, s->admitted_count,
                  s->pool_status, s->stream, DispPhase{2, 0, nullptr, nullptr, s->resume});
  s->prof.end(s->stream);
  s->dispatch_valid = true;
}

int instance_index(const kx_sched* s, int32_t id) {
  for (int i = 0; i < s->n_inst; ++i)
    if (s->inst_host[i].id == id) return i;
  throw std::invalid_argument("unknown instance id");
}

}  // namespace

namespace {

// Order-preserving key of "m-<n>" (see MsgKeyer in kairos_b200.hpp).
uint64_t msg_key_of(uint64_t n) {
  char d[24];
  int nd = 0;
  do {
    d[nd++] = static_cast<char>(n % 10);
    n /= 10;
  } while (n);
  uint64_t k = 0;
  for (int j = 0; j < 18; ++j) k = k * 11 + (j < nd ? static_cast<uint64_t>(d[nd - 1 - j]) + 1 : 0);
  return k;
}

struct DevArena {
  std::vector<void*> ptrs;
  template <typename T>
  T* alloc(size_t n) {
    void* p = nullptr;
    KX_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  template <typename T>
  T* upload(const T* h, size_t n) {
    T* d = alloc<T>(n);
    if (n) {
      // a pageable cudaMemcpy may return before its DMA lands, and the
      // kernels run on non-blocking streams: wait for the legacy stream
      KX_CUDA(cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice));
      KX_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    }
    return d;
  }
  ~DevArena() {
    for (void* p : ptrs) cudaFree(p);
  }
};

void replicas_run_impl(const kx_engine_config* cfg, const kx_replica_batch* b, kx_replica_results* out,
                       double* device_ms) {
  require(cfg && b && out, "null argument");
  require(cfg->n_instances >= 1 && cfg->n_instances <= 32 && cfg->instances,
          "engine supports 1..32 instances per replica");
  require(cfg->scheduler >= KX_SCHED_KAIROS && cfg->scheduler <= KX_SCHED_ORACLE, "unknown scheduler");
  const auto& dc = cfg->dispatcher;
  require(dc.policy >= 0 && dc.policy <= 2, "unknown dispatcher policy");
  const bool kairos = cfg->scheduler == KX_SCHED_KAIROS;
  // expected_exec_time only feeds TimeSlot's try_place (dispatcher.cpp:207-250)
  const bool profile_T = dc.policy == KX_DISPATCH_TIME_SLOT && !dc.oracle_expected_time;
  require(!kairos || cfg->n_agents <= kKairosMaxAgents, "kairos replica engine supports up to 32 agents");
  require(dc.slot_len > 0.0, "slot_len must be positive");
  require(b->n_replicas >= 1, "no replicas");
  require(cfg->n_agents >= 1, "n_agents must be positive");
  const int R = b->n_replicas;
  const int64_t W = b->wf_base[R];
  require(b->wf_base[0] == 0 && W >= 0, "wf_base must start at 0");
  const int64_t C = b->wf_offsets[W];
  require(b->wf_offsets[0] == 0 && C >= 0 && C < (int64_t(1) << 31), "bad wf_offsets");
  int max_run = 1;
  for (int i = 0; i < cfg->n_instances; ++i) {
    const kx_instance& p = cfg->instances[i];
    require(p.capacity_tokens > 0 && p.decode_rate > 0 && p.prefill_rate > 0 && p.max_batch >= 1,
            "instance profile fields must be positive");
    max_run = std::max(max_run, p.max_batch);
  }
  require(max_run <= 1024, "max_batch above 1024");
  // Host-side derived arrays: call -> workflow, children CSR, msg keys.
  std::vector<int64_t> call_base(R + 1);
  std::vector<int32_t> call_wf(C), has_parent(C), child(C);
  std::vector<int64_t> child_off(C + 1, 0);
  std::vector<uint64_t> wf_msg(W);
  for (int r = 0; r < R; ++r) {
    require(b->wf_base[r + 1] >= b->wf_base[r], "wf_base must be non-decreasing");
    call_base[r] = b->wf_offsets[b->wf_base[r]];
    for (int64_t w = b->wf_base[r]; w < b->wf_base[r + 1]; ++w) {
      wf_msg[w] = msg_key_of(static_cast<uint64_t>(w - b->wf_base[r]));
      if (w > b->wf_base[r]) require(b->arrival[w] >= b->arrival[w - 1], "arrivals must be sorted");
    }
  }
  call_base[R] = C;
  double maxpeak = 0.0, maxcap = 0.0;
  for (int i = 0; i < cfg->n_instances; ++i) maxcap = std::max(maxcap, cfg->instances[i].capacity_tokens);
  for (int64_t w = 0; w < W; ++w) {
    require(b->wf_offsets[w + 1] >= b->wf_offsets[w], "wf_offsets must be non-decreasing");
    for (int64_t c = b->wf_offsets[w]; c < b->wf_offsets[w + 1]; ++c) {
      const int32_t p = b->parent[c];
      require(p >= -1 && p < c - b->wf_offsets[w], "parent link is not parents-first");
      require(b->agent[c] >= 0 && b->agent[c] < cfg->n_agents, "agent index outside the agent table");
      require(b->prompt_tokens[c] >= 0 && b->target_tokens[c] >= 1, "token counts out of range");
      call_wf[c] = static_cast<int32_t>(w);
      has_parent[c] = p >= 0;
      if (p >= 0) child_off[b->wf_offsets[w] + p + 1] += 1;
      maxpeak = std::max(maxpeak, static_cast<double>(b->prompt_tokens[c] + b->target_tokens[c]));
    }
  }
  // Simulator's constructor check (engine.cpp:55-71).
  require(maxpeak <= maxcap, "instance capacity below largest single-request peak");
  for (int64_t c = 0; c < C; ++c) child_off[c + 1] += child_off[c];
  {
    std::vector<int64_t> cur(child_off.begin(), child_off.end() - 1);
    for (int64_t c = 0; c < C; ++c) {  // node order within each parent's list
      const int64_t w = call_wf[c];
      const int32_t p = b->parent[c];
      if (p >= 0) child[cur[b->wf_offsets[w] + p]++] = static_cast<int32_t>(c);
    }
  }
  ensure_device(cfg->device);
  DevArena A;
  const int NI = cfg->n_instances;
  std::vector<int32_t> iid(NI), imb(NI);
  std::vector<double> icap(NI), ik(NI), ipf(NI);
  for (int i = 0; i < NI; ++i) {
    iid[i] = cfg->instances[i].id;
    imb[i] = cfg->instances[i].max_batch;
    icap[i] = cfg->instances[i].capacity_tokens;
    ik[i] = cfg->instances[i].decode_rate;
    ipf[i] = cfg->instances[i].prefill_rate;
  }
  std::vector<int32_t> depth(cfg->n_agents, 1);
  if (cfg->topo_depth) depth.assign(cfg->topo_depth, cfg->topo_depth + cfg->n_agents);
  EngineInputs in{};
  in.wf_base = A.upload(b->wf_base, R + 1);
  in.call_base = A.upload(call_base.data(), R + 1);
  in.arrival = A.upload(b->arrival, W);
  in.wf_msg = A.upload(wf_msg.data(), W);
  in.wf_call = A.upload(b->wf_offsets, W + 1);
  in.call_wf = A.upload(call_wf.data(), C);
  in.agent = A.upload(b->agent, C);
  in.has_parent = A.upload(has_parent.data(), C);
  in.prompt = A.upload(b->prompt_tokens, C);
  in.target = A.upload(b->target_tokens, C);
  in.pure = A.upload(b->pure_exec, C);
  in.rem = A.upload(b->remaining, C);
  in.uid = A.upload(b->uid, C);
  in.child_off = A.upload(child_off.data(), C + 1);
  in.child = A.upload(child.data(), C);
  in.depth = A.upload(depth.data(), depth.size());
  in.inst_id = A.upload(iid.data(), NI);
  in.cap = A.upload(icap.data(), NI);
  in.k = A.upload(ik.data(), NI);
  in.prefill = A.upload(ipf.data(), NI);
  in.max_batch = A.upload(imb.data(), NI);
  // Profiler layout per (replica, agent): one exec slot per call of the
  // agent (each call completes once), a remaining window of min(calls, 4097).
  const int NA = cfg->n_agents;
  std::vector<int64_t> exec_off(size_t(R) * NA + 1, 0), rem_off(size_t(R) * NA + 1, 0);
  std::vector<int32_t> agent_order(NA);
  for (int a = 0; a < NA; ++a) agent_order[a] = cfg->agent_order ? cfg->agent_order[a] : a;
  {
    std::vector<uint8_t> seen(NA, 0);
    for (int a = 0; a < NA; ++a) {
      require(agent_order[a] >= 0 && agent_order[a] < NA && !seen[agent_order[a]],
              "agent_order must be a permutation of the agent indices");
      seen[agent_order[a]] = 1;
    }
  }
  if (kairos || profile_T) {
    for (int r = 0; r < R; ++r)
      for (int64_t c = call_base[r]; c < call_base[r + 1]; ++c) exec_off[size_t(r) * NA + b->agent[c] + 1] += 1;
    for (size_t k = 1; k < exec_off.size(); ++k) {
      rem_off[k] = rem_off[k - 1] + std::min<int64_t>(exec_off[k], kRemWindow + 1);
      exec_off[k] += exec_off[k - 1];
    }
  }
  const int64_t exec_total = profile_T ? exec_off.back() : 0;
  const int64_t rem_total = kairos ? rem_off.back() : 0;
  in.agent_order = A.upload(agent_order.data(), NA);
  in.exec_off = A.upload(exec_off.data(), exec_off.size());
  in.rem_off = A.upload(rem_off.data(), rem_off.size());
  const int ring = cfg->slot_ring ? cfg->slot_ring : 256;
  require(ring >= 64 && (ring & (ring - 1)) == 0, "slot_ring must be a power of two >= 64");
  EngineState st{};
  st.rem_parents = A.alloc<int32_t>(C);
  st.enqueue_time = A.alloc<double>(C);
  st.first_enqueue = A.alloc<double>(C);
  st.queue_seconds = A.alloc<double>(C);
  st.kept = A.alloc<int64_t>(C);
  st.episodes = A.alloc<int32_t>(C);
  st.preemptions = A.alloc<int32_t>(C);
  st.epoch = A.alloc<uint32_t>(C);
  st.ever_preempted = A.alloc<uint8_t>(C);
  st.run_slot = A.alloc<int32_t>(C);
  st.wf_remaining = A.alloc<int32_t>(W);
  st.wf_finish = A.alloc<double>(W);
  st.wf_tokens = A.alloc<int64_t>(W);
  st.wf_ncalls = A.alloc<int32_t>(W);
  st.queue = A.alloc<uint32_t>(C);
  st.waiting = A.alloc<uint32_t>(C);
  st.waiting_inst = A.alloc<int32_t>(C);
  const size_t RI = size_t(R) * NI;
  st.usage = A.alloc<double>(RI * ring);
  st.ex = A.alloc<uint8_t>(RI * ring);
  st.base = A.alloc<int64_t>(RI);
  st.hi = A.alloc<int64_t>(RI);
  st.n_active = A.alloc<int32_t>(RI);
  st.act_uid = A.alloc<uint64_t>(RI * kActiveCap);
  st.act_P = A.alloc<double>(RI * kActiveCap);
  st.act_k = A.alloc<double>(RI * kActiveCap);
  st.act_t0 = A.alloc<double>(RI * kActiveCap);
  st.act_T = A.alloc<double>(RI * kActiveCap);
  st.out_call = A.alloc<uint32_t>(C);
  st.out_exec_start = A.alloc<double>(C);
  st.out_exec_end = A.alloc<double>(C);
  st.out_inst = A.alloc<int32_t>(C);
  st.out_wf = A.alloc<int64_t>(W);
  st.scalars = A.alloc<double>(size_t(R) * kEngineScalars);
  st.counts = A.alloc<int64_t>(size_t(R) * 4);
  const size_t RA = size_t(R) * NA;
  st.done_idx = A.alloc<int64_t>(C);
  st.exec_buf = A.alloc<double>(size_t(exec_total));
  st.exec_ns = A.alloc<int64_t>(RA);
  st.exec_nt = A.alloc<int64_t>(RA);
  st.exec_T = A.alloc<double>(RA);
  st.exec_dirty = A.alloc<uint8_t>(RA);
  st.rem_sorted = A.alloc<double>(size_t(rem_total));
  st.rem_ring = A.alloc<double>(size_t(rem_total));
  st.rem_snap = A.alloc<double>(size_t(rem_total));
  st.rem_d = A.alloc<DistScal>(RA);
  st.pk = A.alloc<double>(RA);
  const int64_t mds_n = NA + 1;
  const int64_t mds_stride = kairos ? 4 * mds_n * mds_n + mds_n + 8 : 0;
  st.mds = A.alloc<double>(size_t(R) * size_t(mds_stride));
  st.rebuilds = A.alloc<int64_t>(size_t(R));
  EngineParams prm{};
  prm.n_agents = NA;
  prm.profile_T = profile_T;
  prm.kairos = kairos;
  prm.rebuild_interval = cfg->kairos_rebuild_interval ? cfg->kairos_rebuild_interval : 256;
  prm.mds_stride = mds_stride;
  prm.n_inst = NI;
  prm.sched = cfg->scheduler;
  prm.dpolicy = dc.policy;
  prm.oracle_T = dc.oracle_expected_time;
  prm.ring = ring;
  // Pending events: at most one per running request, the stale ones of
  // preempted episodes, two dispatch rounds and the preempt checks.
  prm.heap_cap = cfg->heap_capacity ? cfg->heap_capacity
                                    : std::max(128, 2 * cfg->n_instances * max_run + 64);
  prm.max_run = max_run;
  prm.slot_len = dc.slot_len;
  prm.watermark = dc.resume_watermark;
  prm.static_thr = dc.static_threshold;
  prm.default_T = dc.default_expected_time;
  prm.period = cfg->dispatch_period > 0.0 ? cfg->dispatch_period : 0.1;
  prm.recompute = cfg->recompute_fraction;
  prm.max_events = cfg->max_events ? cfg->max_events : 200000000ull;
  require(engine_smem_bytes(prm) <= 200 * 1024, "heap_capacity x instances x max_batch exceeds shared memory");
  cudaStream_t stm = nullptr;
  KX_CUDA(cudaStreamCreateWithFlags(&stm, cudaStreamNonBlocking));
  struct SG {
    cudaStream_t s;
    ~SG() { cudaStreamDestroy(s); }
  } sg{stm};
  cudaEvent_t e0, e1;
  KX_CUDA(cudaEventCreate(&e0));
  KX_CUDA(cudaEventCreate(&e1));
  KX_CUDA(cudaEventRecord(e0, stm));
  launch_replica_engine(prm, in, st, R, stm);
  double* d_metrics = A.alloc<double>(size_t(R) * kEngineMetrics);
  uint32_t* d_hist = A.alloc<uint32_t>(size_t(R) * kHistBins);
  {
    std::vector<int32_t> wf_rep(W);
    for (int r = 0; r < R; ++r)
      for (int64_t w = b->wf_base[r]; w < b->wf_base[r + 1]; ++w) wf_rep[w] = r;
    const int32_t* d_rep = A.upload(wf_rep.data(), W);
    launch_replica_metrics(in, st, d_rep, R, W, cfg->warmup_seconds, d_metrics, d_hist, stm);
  }
  KX_CUDA(cudaEventRecord(e1, stm));
  KX_CUDA(cudaStreamSynchronize(stm));
  float ms = 0.f;
  KX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (device_ms) *device_ms = ms;
  std::vector<int64_t> counts(size_t(R) * 4);
  KX_CUDA(cudaMemcpy(counts.data(), st.counts, counts.size() * 8, cudaMemcpyDeviceToHost));
  auto down = [&](auto* h, const auto* d, size_t n) {
    if (h && n) KX_CUDA(cudaMemcpy(h, d, n * sizeof(*h), cudaMemcpyDeviceToHost));
  };
  if (out->call_order) {
    std::vector<uint32_t> oc(C);
    down(oc.data(), st.out_call, C);
    for (int64_t j = 0; j < C; ++j) out->call_order[j] = oc[j];
  }
  down(out->exec_start, st.out_exec_start, C);
  down(out->exec_end, st.out_exec_end, C);
  down(out->instance, st.out_inst, C);
  down(out->first_enqueue, st.first_enqueue, C);
  down(out->queue_seconds, st.queue_seconds, C);
  down(out->episodes, st.episodes, C);
  down(out->preemptions, st.preemptions, C);
  down(out->wf_order, st.out_wf, W);
  down(out->wf_finish, st.wf_finish, W);
  down(out->wf_output_tokens, st.wf_tokens, W);
  down(out->wf_calls, st.wf_ncalls, W);
  down(out->scalars, st.scalars, size_t(R) * kEngineScalars);
  if (out->counts) std::memcpy(out->counts, counts.data(), counts.size() * 8);
  down(out->metrics, d_metrics, size_t(R) * kEngineMetrics);
  down(out->histogram, d_hist, size_t(R) * kHistBins);
  if (kairos) {
    down(out->priority_keys, st.pk, RA);
    down(out->table_versions, st.rebuilds, size_t(R));
  } else {
    if (out->priority_keys) std::fill(out->priority_keys, out->priority_keys + RA, 0.0);
    if (out->table_versions) std::fill(out->table_versions, out->table_versions + R, int64_t(0));
  }
  for (int r = 0; r < R; ++r) {
    const int64_t status = counts[size_t(r) * 4 + 2];
    if (status == KX_ERR_CAPACITY) fail(KX_ERR_CAPACITY, "replica " + std::to_string(r) + ": event heap / run slots / ledger ring capacity exceeded");
    if (status == KX_ERR_RUNTIME) throw std::runtime_error("replica " + std::to_string(r) + ": event budget exhausted; simulation stuck?");
    if (status == KX_ERR_LOGIC) throw std::logic_error("replica " + std::to_string(r) + ": event time ran backwards");
    if (status == KX_ERR_LIVELOCK) fail(KX_ERR_LIVELOCK, "replica " + std::to_string(r) + ": overload/resume livelock");
    if (status != KX_OK) fail(static_cast<int>(status), "replica " + std::to_string(r) + " failed");
  }
}

}  // namespace

// ===========================================================================
// LatencyProfiler state on the device (K9, kx_profiler.cu): per agent an
// execution and a remaining-latency EmpiricalDistribution.
struct kx_profiler {
  int device = 0;
  cudaStream_t stream = nullptr;
  int32_t n_agents = 0;
  int64_t cap = 0;
  kx_convergence_config cfg[2]{};
  DistDev dd{};
  DistCfg* d_cfg = nullptr;
  void* blob = nullptr;
  int* status = nullptr;
};

namespace {

// Applies a batch grouped by distribution: off[n_dist + 1], values and item
// (the caller's record index of each value) in per-distribution arrival
// order. Returns conv_item per distribution.
std::vector<int64_t> profiler_ingest(kx_profiler* p, const std::vector<int64_t>& off,
                                     const std::vector<double>& values, const std::vector<int64_t>& item) {
  const int32_t nd = 2 * p->n_agents;
  const size_t nv = values.size();
  int64_t* d_off = nullptr;
  double* d_v = nullptr;
  int64_t* d_it = nullptr;
  cudaStream_t st = p->stream;
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_off), off.size() * 8, st));
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_v), std::max<size_t>(nv, 1) * 8, st));
  KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_it), std::max<size_t>(nv, 1) * 8, st));
  KX_CUDA(cudaMemcpyAsync(d_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice, st));
  if (nv) {
    KX_CUDA(cudaMemcpyAsync(d_v, values.data(), nv * 8, cudaMemcpyHostToDevice, st));
    KX_CUDA(cudaMemcpyAsync(d_it, item.data(), nv * 8, cudaMemcpyHostToDevice, st));
  }
  KX_CUDA(cudaMemsetAsync(p->status, 0, sizeof(int), st));
  KX_CUDA(cudaMemsetAsync(p->dd.conv_item, 0xff, size_t(nd) * 8, st));  // -1: untouched this batch
  launch_dist_ingest(p->dd, nd, d_off, d_v, d_it, p->status, st);
  std::vector<int64_t> conv(static_cast<size_t>(nd));
  int status = 0;
  KX_CUDA(cudaMemcpyAsync(conv.data(), p->dd.conv_item, size_t(nd) * 8, cudaMemcpyDeviceToHost, st));
  KX_CUDA(cudaMemcpyAsync(&status, p->status, sizeof(int), cudaMemcpyDeviceToHost, st));
  KX_CUDA(cudaFreeAsync(d_off, st));
  KX_CUDA(cudaFreeAsync(d_v, st));
  KX_CUDA(cudaFreeAsync(d_it, st));
  KX_CUDA(cudaStreamSynchronize(st));
  if (status == KX_ERR_CAPACITY)
    fail(KX_ERR_CAPACITY, "profiler distribution exceeds its sample capacity (raise capacity)");
  if (status != KX_OK) fail(status, "profiler ingestion failed");
  return conv;
}

}  // namespace

extern "C" {

int kx_abi_version(void) { return KX_ABI_VERSION; }

const char* kx_last_error(void) { return g_last_error.c_str(); }

int kx_device_available(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return 0;
  }
  cudaDeviceProp p{};
  if (cudaGetDeviceProperties(&p, 0) != cudaSuccess) return 0;
  return p.major >= 10 ? 1 : 0;
}

int kx_sched_create(const kx_sched_config* cfg, kx_sched** out) {
  return guard([&] { create_impl(cfg, out); });
}

int kx_sched_destroy(kx_sched* s) {
  return guard([&] { destroy_impl(s); });
}

int kx_sched_stream(kx_sched* s, void** cuda_stream) {
  return guard([&] {
    require(s && cuda_stream, "null argument");
    *cuda_stream = s->stream;
  });
}

int kx_sched_synchronize(kx_sched* s) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    KX_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int kx_set_scheduler(kx_sched* s, int32_t kind) {
  return guard([&] {
    require(s, "null handle");
    require(kind >= 0 && kind <= 3, "unknown scheduler");
    s->sched_kind = kind;
    s->order_valid = false;
  });
}

int kx_set_agent_tables(kx_sched* s, int32_t n_agents, const int32_t* agent_pool,
                        const double* priority_key, const int32_t* topo_depth,
                        const double* expected_T, uint64_t version) {
  (void)version;
  return guard([&] {
    require(s, "null handle");
    require(n_agents >= 1 && n_agents <= s->max_agents, "n_agents outside [1, max_agents]");
    require(agent_pool != nullptr, "agent_pool is required");
    KX_CUDA(cudaSetDevice(s->device));
    for (int i = 0; i < n_agents; ++i)
      require(agent_pool[i] >= 0 && agent_pool[i] < s->n_pools, "agent pool out of range");
    const size_t A = static_cast<size_t>(n_agents);
    KX_CUDA(cudaMemcpyAsync(s->a.pool, agent_pool, A * 4, cudaMemcpyHostToDevice, s->stream));
    if (priority_key) {
      const std::vector<double> pk(priority_key, priority_key + A);
      for (double x : pk) require(x == x, "NaN in agent table");
      const auto r = pool_dense_rank(pk, agent_pool, s->n_pools);
      s->n_pk_classes = 1 + static_cast<int32_t>(*std::max_element(r.begin(), r.end()));
      KX_CUDA(cudaMemcpyAsync(s->a.pk, priority_key, A * 8, cudaMemcpyHostToDevice, s->stream));
      KX_CUDA(cudaMemcpyAsync(s->a.pk_rank, r.data(), A * 4, cudaMemcpyHostToDevice, s->stream));
      KX_CUDA(cudaStreamSynchronize(s->stream));  // r is a temporary
    } else if (s->n_agents != n_agents) {
      s->n_pk_classes = 1;
      KX_CUDA(cudaMemsetAsync(s->a.pk, 0, A * 8, s->stream));
      KX_CUDA(cudaMemsetAsync(s->a.pk_rank, 0, A * 4, s->stream));
    }
    if (topo_depth) {
      std::vector<double> d(A);
      for (size_t i = 0; i < A; ++i) d[i] = static_cast<double>(topo_depth[i]);
      const auto r = pool_dense_rank(d, agent_pool, s->n_pools);
      s->n_depth_classes = 1 + static_cast<int32_t>(*std::max_element(r.begin(), r.end()));
      KX_CUDA(cudaMemcpyAsync(s->a.depth, topo_depth, A * 4, cudaMemcpyHostToDevice, s->stream));
      KX_CUDA(cudaMemcpyAsync(s->a.depth_rank, r.data(), A * 4, cudaMemcpyHostToDevice, s->stream));
      KX_CUDA(cudaStreamSynchronize(s->stream));
    } else if (s->n_agents != n_agents) {
      s->n_depth_classes = 1;
      std::vector<int32_t> ones(A, 1);
      std::vector<uint32_t> zeros(A, 0);
      KX_CUDA(cudaMemcpyAsync(s->a.depth, ones.data(), A * 4, cudaMemcpyHostToDevice, s->stream));
      KX_CUDA(cudaMemcpyAsync(s->a.depth_rank, zeros.data(), A * 4, cudaMemcpyHostToDevice, s->stream));
      KX_CUDA(cudaStreamSynchronize(s->stream));
    }
    if (expected_T) {
      for (size_t i = 0; i < A; ++i)
        require(expected_T[i] >= 0.0, "expected execution time must be non-negative");
      KX_CUDA(cudaMemcpyAsync(s->a.T, expected_T, A * 8, cudaMemcpyHostToDevice, s->stream));
    } else if (s->n_agents != n_agents) {
      std::vector<double> dflt(A, s->dcfg.default_expected_time);
      KX_CUDA(cudaMemcpyAsync(s->a.T, dflt.data(), A * 8, cudaMemcpyHostToDevice, s->stream));
      KX_CUDA(cudaStreamSynchronize(s->stream));
    }
    KX_CUDA(cudaStreamSynchronize(s->stream));
    s->n_agents = n_agents;
    s->order_valid = false;
  });
}

int kx_set_remaining_table(kx_sched* s, uint64_t uid_base, int64_t n, const double* remaining,
                           const uint8_t* present, int32_t mem) {
  return guard([&] {
    require(s, "null handle");
    require(n >= 0, "negative table size");
    require(n == 0 || (remaining && present), "null table");
    KX_CUDA(cudaSetDevice(s->device));
    if (s->rem_table) cudaFree(s->rem_table);
    if (s->rem_present) cudaFree(s->rem_present);
    s->rem_table = nullptr;
    s->rem_present = nullptr;
    s->rem_n = n;
    s->rem_base = uid_base;
    if (n > 0) {
      KX_CUDA(cudaMalloc(reinterpret_cast<void**>(&s->rem_table), size_t(n) * 8));
      KX_CUDA(cudaMalloc(reinterpret_cast<void**>(&s->rem_present), size_t(n)));
      KX_CUDA(cudaMemcpyAsync(s->rem_table, remaining, size_t(n) * 8, kind_in(mem), s->stream));
      KX_CUDA(cudaMemcpyAsync(s->rem_present, present, size_t(n), kind_in(mem), s->stream));
    }
    refresh_rem(s);
    KX_CUDA(cudaStreamSynchronize(s->stream));
    s->order_valid = false;
  });
}

// Writes n requests at queue positions [at, at + n) (SoA columns), checks
// them and refreshes the Oracle key column.
// Copies the columns a mapped upload left in host memory into the queue
// blob (before anything that rewrites or appends to the queue, or captures
// its addresses in a graph).
static void unmap_queue(kx_sched* s) {
  if (!s->q_mapped) return;
  const size_t N = static_cast<size_t>(s->n);
  if (N) {
    KX_CUDA(cudaMemcpyAsync(s->q_dev.prompt, s->q.prompt, N * 8, cudaMemcpyDefault, s->stream));
    KX_CUDA(cudaMemcpyAsync(s->q_dev.msg, s->q.msg, N * 8, cudaMemcpyDefault, s->stream));
    KX_CUDA(cudaMemcpyAsync(s->q_dev.uid, s->q.uid, N * 8, cudaMemcpyDefault, s->stream));
    if (s->q.kept != s->q_dev.kept)
      KX_CUDA(cudaMemcpyAsync(s->q_dev.kept, s->q.kept, N * 8, cudaMemcpyDefault, s->stream));
  }
  s->q = s->q_dev;
  s->q_mapped = false;
  s->order_valid = false;  // order/dispatch results stay readable only through the copied columns
  s->dispatch_valid = false;
}

static void* device_view(const void* host) {
  void* d = nullptr;
  KX_CUDA(cudaHostGetDevicePointer(&d, const_cast<void*>(host), 0));
  return d;
}

static void queue_write(kx_sched* s, int64_t at, int64_t n, const kx_queue_view* v, int32_t mem, const char* who) {
  require(s && v, "null argument");
  require(n >= 0 && at >= 0 && at + n <= s->cap, "queue size exceeds queue_capacity");
  KX_CUDA(cudaSetDevice(s->device));
  const bool mapped = mem == KX_MEM_HOST_MAPPED && at == 0;
  if (at > 0) unmap_queue(s);
  else if (s->q_mapped) {
    s->q = s->q_dev;
    s->q_mapped = false;
  }
  const size_t N = static_cast<size_t>(n), A = static_cast<size_t>(at);
  if (n > 0) {
    require(v->agent && v->prompt_tokens && v->app_start && v->queue_enter && v->msg_key && v->uid,
            "queue view is missing a required array");
    if (s->dcfg.oracle_expected_time)
      require(v->pure_exec != nullptr, "oracle_expected_time needs pure_exec");
    const cudaMemcpyKind k = mem == KX_MEM_HOST_MAPPED ? cudaMemcpyHostToDevice : kind_in(mem);
    KX_CUDA(cudaMemcpyAsync(s->q.agent + A, v->agent, N * 4, k, s->stream));
    KX_CUDA(cudaMemcpyAsync(s->q.app_start + A, v->app_start, N * 8, k, s->stream));
    KX_CUDA(cudaMemcpyAsync(s->q.queue_enter + A, v->queue_enter, N * 8, k, s->stream));
    if (v->pure_exec) KX_CUDA(cudaMemcpyAsync(s->q.pure_exec + A, v->pure_exec, N * 8, k, s->stream));
    if (mapped) {  // read in place by the kernels that need them
      s->q.prompt = static_cast<int64_t*>(device_view(v->prompt_tokens));
      s->q.msg = static_cast<uint64_t*>(device_view(v->msg_key));
      s->q.uid = static_cast<uint64_t*>(device_view(v->uid));
      if (v->kept_tokens) s->q.kept = static_cast<int64_t*>(device_view(v->kept_tokens));
      else KX_CUDA(cudaMemsetAsync(s->q.kept, 0, N * 8, s->stream));
      s->q_mapped = true;
    } else {
      KX_CUDA(cudaMemcpyAsync(s->q.prompt + A, v->prompt_tokens, N * 8, k, s->stream));
      KX_CUDA(cudaMemcpyAsync(s->q.msg + A, v->msg_key, N * 8, k, s->stream));
      KX_CUDA(cudaMemcpyAsync(s->q.uid + A, v->uid, N * 8, k, s->stream));
      if (v->kept_tokens)
        KX_CUDA(cudaMemcpyAsync(s->q.kept + A, v->kept_tokens, N * 8, k, s->stream));
      else
        KX_CUDA(cudaMemsetAsync(s->q.kept + A, 0, N * 8, s->stream));
    }
    KX_CUDA(cudaMemsetAsync(s->err_flag, 0, sizeof(int), s->stream));
    QueueDev part = s->q;
    part.agent += A;
    part.prompt += A;
    part.app_start += A;
    part.queue_enter += A;
    part.msg += A;
    part.uid += A;
    part.kept += A;
    part.pure_exec += A;
    part.rem += A;
    part.admitted += A;
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, int64_t(s->sms) * 8));
    k_validate_queue<<<grid, 256, 0, s->stream>>>(part, n, std::max(s->n_agents, 0),
                                                  s->dcfg.oracle_expected_time ? 1 : 0, mapped ? 0 : 1,
                                                  s->err_flag);
    KX_CHECK_LAUNCH();
  }
  s->n = at + n;
  refresh_rem(s);
  s->order_valid = false;
  s->dispatch_valid = false;
  if (n > 0) check_err_flag(s, who);
}

int kx_queue_upload(kx_sched* s, int64_t n, const kx_queue_view* v, int32_t mem) {
  return guard([&] { queue_write(s, 0, n, v, mem, "kx_queue_upload"); });
}

int kx_queue_enqueue(kx_sched* s, int64_t n, const kx_queue_view* v, int32_t mem) {
  return guard([&] {
    require(s, "null handle");
    queue_write(s, s->n, n, v, mem, "kx_queue_enqueue");
  });
}

int kx_queue_size(kx_sched* s, int64_t* n) {
  return guard([&] {
    require(s && n, "null argument");
    *n = s->n;
  });
}

int kx_queue_remove_admitted(kx_sched* s) {
  return guard([&] {
    require(s, "null handle");
    if (!s->dispatch_valid) throw std::logic_error("no dispatch round to apply");
    KX_CUDA(cudaSetDevice(s->device));
    if (s->q_mapped) {  // the compaction rewrites every column in the queue blob
      const bool dv = s->dispatch_valid, ov = s->order_valid;
      unmap_queue(s);
      s->dispatch_valid = dv;
      s->order_valid = ov;
    }
    const int64_t n = s->n;
    if (n == 0) return;
    const int64_t chunks = (n + kCompactChunk - 1) / kCompactChunk;
    k_flag_count<<<static_cast<unsigned>(chunks), 256, 0, s->stream>>>(
        s->q.admitted, n, static_cast<int>(kCompactChunk), s->compact_counts);
    KX_CHECK_LAUNCH();
    k_scan_counts<<<1, 1024, 0, s->stream>>>(s->compact_counts, chunks, s->compact_total);
    KX_CHECK_LAUNCH();
    // All columns in one pass into the alternate queue blob (same layout),
    // then each column's kept prefix back: the queue's addresses stay fixed,
    // so captured graphs remain valid.
    if (!s->queue_alt_blob.base) alloc_blob(s->queue_alt_blob, s->queue_blob.size);
    auto alt = [&](auto* col) {
      using T = std::remove_pointer_t<decltype(col)>;
      return reinterpret_cast<T*>(s->queue_alt_blob.base + (reinterpret_cast<char*>(col) - s->queue_blob.base));
    };
    QueueDev qa{alt(s->q.agent), alt(s->q.prompt), alt(s->q.app_start), alt(s->q.queue_enter), alt(s->q.msg),
                alt(s->q.uid),   alt(s->q.kept),   alt(s->q.pure_exec), alt(s->q.rem),         alt(s->q.admitted)};
    k_compact_queue<<<static_cast<unsigned>(chunks), 256, 0, s->stream>>>(s->q, qa, n,
                                                                          static_cast<int>(kCompactChunk),
                                                                          s->compact_counts);
    KX_CHECK_LAUNCH();
    int64_t total = 0;
    KX_CUDA(cudaMemcpyAsync(&total, s->compact_total, 8, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
    const size_t T = static_cast<size_t>(total);
    if (!s->graph_exec) {  // no captured graph holds the queue's addresses: swap the blobs
      std::swap(s->queue_blob, s->queue_alt_blob);
      s->q = qa;
      s->n = total;
      s->order_valid = false;
      s->dispatch_valid = false;
      return;
    }
    auto back = [&](auto* col) {
      using E = std::remove_pointer_t<decltype(col)>;
      if (T) KX_CUDA(cudaMemcpyAsync(col, alt(col), T * sizeof(E), cudaMemcpyDeviceToDevice, s->stream));
    };
    back(s->q.agent);
    back(s->q.prompt);
    back(s->q.app_start);
    back(s->q.queue_enter);
    back(s->q.msg);
    back(s->q.uid);
    back(s->q.kept);
    back(s->q.pure_exec);
    back(s->q.rem);
    s->n = total;
    s->order_valid = false;
    s->dispatch_valid = false;
  });
}

int kx_score(kx_sched* s, double* k0, double* k1, double* k2, int32_t mem) {
  return guard([&] {
    require(s && k0 && k1 && k2, "null argument");
    require(s->n_agents > 0 || s->n == 0, "agent tables not set");
    KX_CUDA(cudaSetDevice(s->device));
    const size_t N = static_cast<size_t>(s->n);
    if (N == 0) return;
    if (mem == KX_MEM_DEVICE) {
      launch_score(s->q, s->a, s->sched_kind, s->n, k0, k1, k2, s->sms, s->stream);
      KX_CUDA(cudaStreamSynchronize(s->stream));
      return;
    }
    double* d = nullptr;
    KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), N * 24, s->stream));
    launch_score(s->q, s->a, s->sched_kind, s->n, d, d + N, d + 2 * N, s->sms, s->stream);
    KX_CUDA(cudaMemcpyAsync(k0, d, N * 8, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaMemcpyAsync(k1, d + N, N * 8, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaMemcpyAsync(k2, d + 2 * N, N * 8, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaFreeAsync(d, s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int kx_order(kx_sched* s) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    order_impl(s);
  });
}

int kx_order_fetch(kx_sched* s, uint32_t* perm, int64_t* pool_offsets, int32_t mem) {
  return guard([&] {
    require(s, "null handle");
    if (!s->order_valid) throw std::logic_error("no current order (call kx_order)");
    KX_CUDA(cudaSetDevice(s->device));
    const cudaMemcpyKind k = kind_out(mem);
    if (perm && s->n > 0)
      KX_CUDA(cudaMemcpyAsync(perm, s->order.perm, size_t(s->n) * 4, k, s->stream));
    if (pool_offsets)
      KX_CUDA(cudaMemcpyAsync(pool_offsets, s->ws.pool_offsets, size_t(s->n_pools + 1) * 8, k,
                              s->stream));
    int flags = 0;
    KX_CUDA(cudaMemcpyAsync(&flags, s->ws.error_flags, 4, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
    if (flags) fail(KX_ERR_INVALID, "queue holds an invalid agent index or NaN key");
  });
}

int kx_dispatch_round(kx_sched* s, double now) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    dispatch_impl(s, now);
  });
}

int kx_tick(kx_sched* s, double now) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    tick_impl(s, now);
  });
}

int kx_dispatch_fetch(kx_sched* s, int64_t* per_pool_count, kx_decision* rows,
                      double* candidate_peaks, int64_t* row_stride, int64_t* peak_stride) {
  return guard([&] {
    require(s, "null handle");
    if (!s->dispatch_valid) throw std::logic_error("no dispatch round to fetch");
    KX_CUDA(cudaSetDevice(s->device));
    const size_t P = static_cast<size_t>(s->n_pools);
    std::vector<int64_t> cnt(P);
    std::vector<int> status(P);
    KX_CUDA(cudaMemcpyAsync(cnt.data(), s->row_count, P * 8, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaMemcpyAsync(status.data(), s->pool_status, P * 4, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
    if (row_stride) *row_stride = s->log_cap;
    if (peak_stride) *peak_stride = s->max_inst_per_pool;
    for (size_t p = 0; p < P; ++p) {
      if (status[p] == KX_ERR_LIVELOCK)
        fail(KX_ERR_LIVELOCK, "pool " + std::to_string(p) +
                                  ": overload/resume livelock (reference would spin forever)");
      if (status[p] == KX_ERR_CAPACITY)
        fail(KX_ERR_CAPACITY, "pool " + std::to_string(p) +
                                  ": slot ring, active-request table or waiting-list capacity exceeded");
      if (status[p] != KX_OK) fail(status[p], "pool " + std::to_string(p) + ": dispatch failed");
      if (cnt[p] > s->log_cap && (rows || candidate_peaks))
        fail(KX_ERR_CAPACITY, "decision log truncated (raise log_capacity_per_pool)");
    }
    if (per_pool_count) std::memcpy(per_pool_count, cnt.data(), P * 8);
    // Only each pool's filled rows travel (the layout keeps the log stride),
    // through a pinned staging buffer, then one host copy per block.
    const size_t w = static_cast<size_t>(s->max_inst_per_pool);
    size_t need = 0;
    for (size_t p = 0; p < P; ++p) {
      const size_t n = static_cast<size_t>(std::min<int64_t>(cnt[p], s->log_cap));
      need += (rows ? n * sizeof(kx_decision) : 0) + (candidate_peaks ? n * w * sizeof(double) : 0);
    }
    if (need > s->fetch_pinned_size) {
      if (s->fetch_pinned) cudaFreeHost(s->fetch_pinned);
      s->fetch_pinned = nullptr;
      s->fetch_pinned_size = 0;
      const size_t full = P * static_cast<size_t>(s->log_cap) * (sizeof(kx_decision) + w * sizeof(double));
      KX_CUDA(cudaMallocHost(reinterpret_cast<void**>(&s->fetch_pinned), full));
      s->fetch_pinned_size = full;
    }
    struct Piece {
      char* dst;
      size_t off, bytes;
    };
    std::vector<Piece> pieces;
    size_t off = 0;
    for (size_t p = 0; p < P; ++p) {
      const size_t n = static_cast<size_t>(std::min<int64_t>(cnt[p], s->log_cap));
      if (n == 0) continue;
      const size_t r0 = p * static_cast<size_t>(s->log_cap);
      if (rows) {
        const size_t b = n * sizeof(kx_decision);
        KX_CUDA(cudaMemcpyAsync(s->fetch_pinned + off, s->rows + r0, b, cudaMemcpyDeviceToHost, s->stream));
        pieces.push_back({reinterpret_cast<char*>(rows + r0), off, b});
        off += b;
      }
      if (candidate_peaks) {
        const size_t b = n * w * sizeof(double);
        KX_CUDA(cudaMemcpyAsync(s->fetch_pinned + off, s->cand + r0 * w, b, cudaMemcpyDeviceToHost, s->stream));
        pieces.push_back({reinterpret_cast<char*>(candidate_peaks + r0 * w), off, b});
        off += b;
      }
    }
    KX_CUDA(cudaStreamSynchronize(s->stream));
    for (const Piece& pc : pieces) std::memcpy(pc.dst, s->fetch_pinned + pc.off, pc.bytes);
  });
}

int kx_waiting_reserve(kx_sched* s, int64_t per_instance) {
  return guard([&] {
    require(s, "null handle");
    require(per_instance >= 0, "negative waiting-list capacity");
    KX_CUDA(cudaSetDevice(s->device));
    ensure_waiting(s, per_instance);
  });
}

int kx_waiting_upload(kx_sched* s, int64_t n, const int32_t* instance_pos, const kx_queue_view* v) {
  return guard([&] {
    require(s, "null handle");
    require(n >= 0, "negative count");
    KX_CUDA(cudaSetDevice(s->device));
    std::vector<int32_t> cnt(static_cast<size_t>(s->n_inst), 0);
    if (n > 0) {
      require(instance_pos && v && v->agent && v->prompt_tokens && v->app_start && v->queue_enter &&
                  v->msg_key && v->uid,
              "waiting view is missing a required array");
      for (int64_t j = 0; j < n; ++j) {
        require(instance_pos[j] >= 0 && instance_pos[j] < s->n_inst, "instance position out of range");
        require(v->agent[j] >= 0 && v->agent[j] < std::max(s->n_agents, 1), "agent index out of range");
        require(v->app_start[j] == v->app_start[j] && v->queue_enter[j] == v->queue_enter[j], "NaN time");
        ++cnt[static_cast<size_t>(instance_pos[j])];
      }
    }
    const int64_t need = cnt.empty() ? 0 : *std::max_element(cnt.begin(), cnt.end());
    ensure_waiting(s, std::max<int64_t>(need, 1024));
    const size_t I = static_cast<size_t>(s->n_inst);
    std::vector<WaitRec> h(I * static_cast<size_t>(s->wcap));
    std::vector<int32_t> fill(I, 0);
    for (int64_t j = 0; j < n; ++j) {
      const size_t i = static_cast<size_t>(instance_pos[j]);
      WaitRec r{};
      r.app_start = v->app_start[j];
      r.queue_enter = v->queue_enter[j];
      r.msg = v->msg_key[j];
      r.uid = v->uid[j];
      r.prompt = v->prompt_tokens[j];
      r.kept = v->kept_tokens ? v->kept_tokens[j] : 0;
      r.qidx = -1;
      r.agent = v->agent[j];
      r.round = -1;  // not from a dispatch round
      h[i * static_cast<size_t>(s->wcap) + static_cast<size_t>(fill[i]++)] = r;
    }
    KX_CUDA(cudaMemcpyAsync(s->wrec, h.data(), h.size() * sizeof(WaitRec), cudaMemcpyHostToDevice, s->stream));
    KX_CUDA(cudaMemcpyAsync(s->in.waiting, cnt.data(), I * 4, cudaMemcpyHostToDevice, s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int kx_waiting_fetch(kx_sched* s, int32_t instance_pos, int64_t cap, uint64_t* uid, int64_t* n_out) {
  return guard([&] {
    require(s, "null handle");
    require(instance_pos >= 0 && instance_pos < s->n_inst, "instance position out of range");
    KX_CUDA(cudaSetDevice(s->device));
    int32_t n = 0;
    KX_CUDA(cudaMemcpyAsync(&n, s->in.waiting + instance_pos, 4, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
    if (n_out) *n_out = n;
    const int64_t m = std::min<int64_t>(n, cap);
    if (!uid || m <= 0) return;
    require(s->wrec != nullptr && n <= s->wcap, "waiting list storage missing");
    std::vector<WaitRec> h(static_cast<size_t>(m));
    KX_CUDA(cudaMemcpyAsync(h.data(), s->wrec + int64_t(instance_pos) * s->wcap, size_t(m) * sizeof(WaitRec),
                            cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
    for (int64_t j = 0; j < m; ++j) uid[j] = h[static_cast<size_t>(j)].uid;
  });
}

int kx_admissions_fetch(kx_sched* s, int64_t* per_pool_count, kx_admission* rows, int64_t* row_stride) {
  return guard([&] {
    require(s, "null handle");
    if (!s->dispatch_valid) throw std::logic_error("no dispatch round to fetch");
    KX_CUDA(cudaSetDevice(s->device));
    const size_t P = static_cast<size_t>(s->n_pools);
    if (row_stride) *row_stride = s->log_cap;
    std::vector<int64_t> cnt(P, 0);
    if (s->adm_count && s->dcfg.policy != KX_DISPATCH_TIME_SLOT) {
      KX_CUDA(cudaMemcpyAsync(cnt.data(), s->adm_count, P * 8, cudaMemcpyDeviceToHost, s->stream));
      KX_CUDA(cudaStreamSynchronize(s->stream));
    }
    for (size_t p = 0; p < P; ++p)
      if (cnt[p] > s->log_cap && rows)
        fail(KX_ERR_CAPACITY, "admission log truncated (raise log_capacity_per_pool)");
    if (per_pool_count) std::memcpy(per_pool_count, cnt.data(), P * 8);
    if (rows && s->adm)
      KX_CUDA(cudaMemcpyAsync(rows, s->adm, P * s->log_cap * sizeof(kx_admission), cudaMemcpyDeviceToHost,
                              s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int kx_rr_next(kx_sched* s, int64_t* get_per_pool, const int64_t* set_per_pool) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    const size_t P = static_cast<size_t>(s->n_pools);
    std::vector<int32_t> v(P);
    if (get_per_pool) {
      KX_CUDA(cudaMemcpyAsync(v.data(), s->in.rr_next, P * 4, cudaMemcpyDeviceToHost, s->stream));
      KX_CUDA(cudaStreamSynchronize(s->stream));
      for (size_t p = 0; p < P; ++p) get_per_pool[p] = v[p];
    }
    if (set_per_pool) {
      for (size_t p = 0; p < P; ++p) {
        const int64_t np = s->pool_begin_host[p + 1] - s->pool_begin_host[p];
        require(set_per_pool[p] >= 0, "negative rr_next");
        v[p] = static_cast<int32_t>(np > 0 ? set_per_pool[p] % np : 0);
      }
      KX_CUDA(cudaMemcpyAsync(s->in.rr_next, v.data(), P * 4, cudaMemcpyHostToDevice, s->stream));
      KX_CUDA(cudaStreamSynchronize(s->stream));
    }
  });
}

int kx_instances_set_live(kx_sched* s, const double* live_kv, const int32_t* running,
                          const int32_t* waiting) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    const size_t I = static_cast<size_t>(s->n_inst);
    if (live_kv) KX_CUDA(cudaMemcpyAsync(s->in.live_kv, live_kv, I * 8, cudaMemcpyHostToDevice, s->stream));
    if (running) KX_CUDA(cudaMemcpyAsync(s->in.running, running, I * 4, cudaMemcpyHostToDevice, s->stream));
    if (waiting) KX_CUDA(cudaMemcpyAsync(s->in.waiting, waiting, I * 4, cudaMemcpyHostToDevice, s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int kx_instances_get_live(kx_sched* s, double* live_kv, int32_t* running, int32_t* waiting,
                          uint8_t* suspended) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    const size_t I = static_cast<size_t>(s->n_inst);
    if (live_kv) KX_CUDA(cudaMemcpyAsync(live_kv, s->in.live_kv, I * 8, cudaMemcpyDeviceToHost, s->stream));
    if (running) KX_CUDA(cudaMemcpyAsync(running, s->in.running, I * 4, cudaMemcpyDeviceToHost, s->stream));
    if (waiting) KX_CUDA(cudaMemcpyAsync(waiting, s->in.waiting, I * 4, cudaMemcpyDeviceToHost, s->stream));
    if (suspended) KX_CUDA(cudaMemcpyAsync(suspended, s->in.suspended, I, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int kx_ledger_try_place(kx_sched* s, int32_t instance_id, double prefill_tokens, double decode_rate,
                        double t_start, double expected_duration, int32_t* fits,
                        double* predicted_peak, int64_t* violating_slot) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    const int i = instance_index(s, instance_id);
    launch_ledger_try_place(s->in, i, s->ring, prefill_tokens, decode_rate, t_start,
                            expected_duration, s->dcfg.slot_len, s->scratch_d, s->scratch_i,
                            s->scratch_s, s->stream);
    double pk = 0;
    int64_t viol = 0;
    int state = 0;
    KX_CUDA(cudaMemcpyAsync(&pk, s->scratch_d, 8, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaMemcpyAsync(&viol, s->scratch_i, 8, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaMemcpyAsync(&state, s->scratch_s, 4, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
    if (state < 0) fail(KX_ERR_CAPACITY, "request span leaves the ledger's slot ring");
    if (fits) *fits = state == 2 ? 1 : 0;
    if (predicted_peak) *predicted_peak = state == 2 ? pk : 0.0;
    if (violating_slot) *violating_slot = state == 2 ? 0 : viol;
  });
}

int kx_ledger_commit(kx_sched* s, int32_t instance_id, uint64_t uid, double prefill_tokens,
                     double decode_rate, double t_start, double expected_duration) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    const int i = instance_index(s, instance_id);
    launch_ledger_commit(s->in, i, s->ring, uid, prefill_tokens, decode_rate, t_start,
                         expected_duration, s->dcfg.slot_len, s->scratch_s, s->stream);
    int st = 0;
    KX_CUDA(cudaMemcpyAsync(&st, s->scratch_s, 4, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
    if (st == KX_ERR_LOGIC) throw std::logic_error("commit after Exceeds is a contract violation");
    if (st == KX_ERR_CAPACITY) fail(KX_ERR_CAPACITY, "ledger slot ring / active table capacity exceeded");
  });
}

int kx_ledger_commit_batch(kx_sched* s, int64_t n, const int32_t* instance_id, const uint64_t* uid,
                           const double* prefill_tokens, const double* decode_rate,
                           const double* t_start, const double* expected_duration,
                           uint8_t* fits_out) {
  return guard([&] {
    require(s, "null handle");
    require(n >= 0, "negative count");
    if (n == 0) return;
    require(instance_id && uid && prefill_tokens && decode_rate && t_start && expected_duration,
            "null argument");
    KX_CUDA(cudaSetDevice(s->device));
    std::vector<int64_t> cnt(static_cast<size_t>(s->n_inst) + 1, 0);
    std::vector<int> idx(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) {
      idx[static_cast<size_t>(j)] = instance_index(s, instance_id[j]);
      cnt[static_cast<size_t>(idx[static_cast<size_t>(j)]) + 1] += 1;
    }
    for (int i = 0; i < s->n_inst; ++i) cnt[i + 1] += cnt[i];
    std::vector<int64_t> order(static_cast<size_t>(n));
    std::vector<int64_t> cur(cnt.begin(), cnt.end() - 1);
    for (int64_t j = 0; j < n; ++j) order[static_cast<size_t>(cur[idx[static_cast<size_t>(j)]]++)] = j;
    const size_t N = static_cast<size_t>(n);
    char* buf = nullptr;
    const size_t bytes = (s->n_inst + 1) * 8 + N * (8 + 8 + 8 * 4 + 1) + 64;
    KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), bytes, s->stream));
    auto* d_off = reinterpret_cast<int64_t*>(buf);
    auto* d_ord = d_off + s->n_inst + 1;
    auto* d_uid = reinterpret_cast<uint64_t*>(d_ord + N);
    auto* d_P = reinterpret_cast<double*>(d_uid + N);
    auto* d_k = d_P + N;
    auto* d_t0 = d_k + N;
    auto* d_T = d_t0 + N;
    auto* d_fit = reinterpret_cast<uint8_t*>(d_T + N);
    KX_CUDA(cudaMemcpyAsync(d_off, cnt.data(), (s->n_inst + 1) * 8, cudaMemcpyHostToDevice, s->stream));
    KX_CUDA(cudaMemcpyAsync(d_ord, order.data(), N * 8, cudaMemcpyHostToDevice, s->stream));
    KX_CUDA(cudaMemcpyAsync(d_uid, uid, N * 8, cudaMemcpyHostToDevice, s->stream));
    KX_CUDA(cudaMemcpyAsync(d_P, prefill_tokens, N * 8, cudaMemcpyHostToDevice, s->stream));
    KX_CUDA(cudaMemcpyAsync(d_k, decode_rate, N * 8, cudaMemcpyHostToDevice, s->stream));
    KX_CUDA(cudaMemcpyAsync(d_t0, t_start, N * 8, cudaMemcpyHostToDevice, s->stream));
    KX_CUDA(cudaMemcpyAsync(d_T, expected_duration, N * 8, cudaMemcpyHostToDevice, s->stream));
    KX_CUDA(cudaMemsetAsync(s->scratch_s, 0, 4, s->stream));
    launch_ledger_commit_batch(s->in, s->n_inst, s->ring, d_off, d_ord, d_uid, d_P, d_k, d_t0, d_T,
                               s->dcfg.slot_len, d_fit, s->scratch_s, s->stream);
    std::vector<uint8_t> fits(N);
    int st = 0;
    KX_CUDA(cudaMemcpyAsync(fits.data(), d_fit, N, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaMemcpyAsync(&st, s->scratch_s, 4, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaFreeAsync(buf, s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
    if (st == KX_ERR_CAPACITY) fail(KX_ERR_CAPACITY, "ledger slot ring / active table capacity exceeded");
    if (fits_out) std::memcpy(fits_out, fits.data(), N);
  });
}

int kx_on_request_finished(kx_sched* s, int32_t instance_id, uint64_t uid, double actual_end) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    const int i = instance_index(s, instance_id);
    if (s->dcfg.policy != KX_DISPATCH_TIME_SLOT) return;
    launch_ledger_finish(s->in, i, s->ring, uid, actual_end, s->dcfg.slot_len, s->stream);
    KX_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int kx_on_overload(kx_sched* s, int32_t instance_id) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    const int i = instance_index(s, instance_id);
    if (s->dcfg.policy != KX_DISPATCH_TIME_SLOT) return;
    launch_on_overload(s->in, i, s->stream);
    KX_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int kx_on_live_usage(kx_sched* s, int32_t instance_id, double live_kv) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    const int i = instance_index(s, instance_id);
    launch_on_live_usage(s->in, i, live_kv, s->dcfg.resume_watermark, s->stream);
    KX_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int kx_gc(kx_sched* s, double now) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    launch_gc_all(s->in, s->n_inst, s->ring, now, s->dcfg.slot_len, s->stream);
    KX_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int kx_ledger_read(kx_sched* s, int32_t instance_id, int64_t* base_slot, double* usage,
                   uint8_t* exists, int32_t* active_requests) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    const int i = instance_index(s, instance_id);
    const int R = s->ring;
    int64_t base = 0;
    std::vector<double> ring_usage(R);
    std::vector<uint8_t> ring_ex(R);
    int32_t na = 0;
    KX_CUDA(cudaMemcpyAsync(&base, s->in.base_slot + i, 8, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaMemcpyAsync(ring_usage.data(), s->in.usage + int64_t(i) * R, R * 8,
                            cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaMemcpyAsync(ring_ex.data(), s->in.exists + int64_t(i) * R, R,
                            cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaMemcpyAsync(&na, s->in.n_active + i, 4, cudaMemcpyDeviceToHost, s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
    if (base_slot) *base_slot = base;
    for (int k = 0; k < R; ++k) {
      const int64_t slot = base + k;
      const uint32_t pos = static_cast<uint32_t>(slot) & (R - 1);
      if (usage) usage[k] = ring_usage[pos];
      if (exists) exists[k] = ring_ex[pos];
    }
    if (active_requests) *active_requests = na;
  });
}

int kx_state_checkpoint(kx_sched* s) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    if (!s->inst_ckpt_blob.base) alloc_blob(s->inst_ckpt_blob, s->inst_mut_blob.size);
    KX_CUDA(cudaMemcpyAsync(s->inst_ckpt_blob.base, s->inst_mut_blob.base, s->inst_mut_blob.size,
                            cudaMemcpyDeviceToDevice, s->stream));
    // waiting-list contents go with their counts
    if (s->wrec && s->wckpt_cap != s->wcap) {
      if (s->wckpt) KX_CUDA(cudaFree(s->wckpt));
      KX_CUDA(cudaMalloc(reinterpret_cast<void**>(&s->wckpt), size_t(s->n_inst) * s->wcap * sizeof(WaitRec)));
      s->wckpt_cap = s->wcap;
    }
    if (s->wrec)
      KX_CUDA(cudaMemcpyAsync(s->wckpt, s->wrec, size_t(s->n_inst) * s->wcap * sizeof(WaitRec),
                              cudaMemcpyDeviceToDevice, s->stream));
    KX_CUDA(cudaStreamSynchronize(s->stream));
    s->have_ckpt = true;
  });
}

int kx_state_restore(kx_sched* s) {
  return guard([&] {
    require(s, "null handle");
    if (!s->have_ckpt) throw std::logic_error("no checkpoint to restore");
    KX_CUDA(cudaSetDevice(s->device));
    KX_CUDA(cudaMemcpyAsync(s->inst_mut_blob.base, s->inst_ckpt_blob.base, s->inst_mut_blob.size,
                            cudaMemcpyDeviceToDevice, s->stream));
    if (s->wrec && s->wckpt_cap == s->wcap)
      KX_CUDA(cudaMemcpyAsync(s->wrec, s->wckpt, size_t(s->n_inst) * s->wcap * sizeof(WaitRec),
                              cudaMemcpyDeviceToDevice, s->stream));
  });
}

// CUDA graph of a repeated step: every call between begin and end (on this
// handle, from this thread) is captured from the handle's stream, including
// the side stream's overlapped dispatch, and kx_graph_launch replays it with
// one launch. The captured calls must be asynchronous (no fetches, no
// profiling); the graph is valid while the queue size and handle state
// shapes stay the same.
int kx_graph_capture_begin(kx_sched* s) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    if (s->prof.enabled) throw std::logic_error("disable profiling before capturing a graph");
    if (s->q_mapped) {  // the graph keeps the queue's addresses
      const bool dv = s->dispatch_valid, ov = s->order_valid;
      unmap_queue(s);
      s->dispatch_valid = dv;
      s->order_valid = ov;
    }
    if (s->graph_exec) {
      cudaGraphExecDestroy(s->graph_exec);
      s->graph_exec = nullptr;
    }
    if (s->graph) {
      cudaGraphDestroy(s->graph);
      s->graph = nullptr;
    }
    KX_CUDA(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
  });
}

int kx_graph_capture_end(kx_sched* s) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    KX_CUDA(cudaStreamEndCapture(s->stream, &s->graph));
    KX_CUDA(cudaGraphInstantiate(&s->graph_exec, s->graph, 0));
    s->graph_n = s->n;
    s->graph_queue_base = s->queue_blob.base;
    s->graph_order_valid = s->order_valid;
    s->graph_dispatch_valid = s->dispatch_valid;
    s->graph_order = s->order;
  });
}

int kx_graph_release(kx_sched* s) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    KX_CUDA(cudaStreamSynchronize(s->stream));
    if (s->graph_exec) {
      cudaGraphExecDestroy(s->graph_exec);
      s->graph_exec = nullptr;
    }
    if (s->graph) {
      cudaGraphDestroy(s->graph);
      s->graph = nullptr;
    }
  });
}

int kx_graph_launch(kx_sched* s) {
  return guard([&] {
    require(s, "null handle");
    if (!s->graph_exec) throw std::logic_error("no captured graph");
    if (s->q_mapped) throw std::logic_error("the queue was uploaded mapped since the capture: capture again");
    // The captured kernels carry the queue size and buffer addresses of the
    // capture: a pop or an enqueue that changed the size needs a new capture.
    if (s->n != s->graph_n || s->queue_blob.base != s->graph_queue_base)
      throw std::logic_error("queue size changed since the graph was captured: capture again");
    KX_CUDA(cudaSetDevice(s->device));
    KX_CUDA(cudaGraphLaunch(s->graph_exec, s->stream));
    s->order = s->graph_order;
    s->order_valid = s->graph_order_valid;
    s->order_n = s->n;
    s->dispatch_valid = s->graph_dispatch_valid;
  });
}

int kx_profile_enable(kx_sched* s, int32_t enable) {
  return guard([&] {
    require(s, "null handle");
    KX_CUDA(cudaSetDevice(s->device));
    s->prof.reset();
    s->prof.enabled = enable != 0;
  });
}

int kx_profile_read(kx_sched* s, kx_phase_stat* out, int32_t cap, int32_t* n_out) {
  return guard([&] {
    require(s && n_out, "null argument");
    KX_CUDA(cudaSetDevice(s->device));
    s->prof.drain();
    const int32_t n = static_cast<int32_t>(s->prof.phases.size());
    *n_out = n;
    for (int32_t i = 0; i < n && i < cap && out; ++i) {
      const auto& p = s->prof.phases[static_cast<size_t>(i)];
      std::memset(out[i].name, 0, sizeof(out[i].name));
      std::strncpy(out[i].name, p.name.c_str(), sizeof(out[i].name) - 1);
      out[i].total_ms = p.ms;
      out[i].launches = p.launches;
      out[i].alg_bytes = p.bytes;
    }
  });
}

int64_t kx_launch_count(void) { return kx::g_kx_launches.load(); }

// Diagnostics: globaltimer stamps of the last batched dispatch kernel (pool 0).
int kx_debug_dispatch_timers(uint64_t* out16) {
  return guard([&] { kx::read_dispatch_debug(reinterpret_cast<unsigned long long*>(out16)); });
}

// Diagnostics: per-stage resolver cycles of pool 0 (KX_DISPATCH_TIMERS=2 builds).
int kx_debug_dispatch_stages(uint64_t* out16) {
  return guard([&] { kx::read_dispatch_stages(reinterpret_cast<unsigned long long*>(out16)); });
}

// Diagnostics: decisions taken by the register-resident resolver and heads
// on the exact path, summed over chain-kernel launches (read, then reset).
int kx_debug_dispatch_counts(uint64_t* out2, int32_t reset) {
  return guard([&] { kx::read_dispatch_counts(reinterpret_cast<unsigned long long*>(out2), reset != 0); });
}

// Diagnostics: phase-3 dispatch start / end per pool (globaltimer, KX_DISPATCH_TIMERS builds).
int kx_debug_dispatch_pool_times(uint64_t* out128) {
  return guard([&] { kx::read_dispatch_pool_times(reinterpret_cast<unsigned long long*>(out128)); });
}

// Diagnostics: globaltimer at the end of the last key generation.
int kx_debug_keys_done(uint64_t* out1) {
  return guard([&] { kx::read_keys_done(reinterpret_cast<unsigned long long*>(out1)); });
}

// Diagnostics: clock stamps of 8 register-resolver steps of pool 0 (KX_DISPATCH_TIMERS=3 builds).
int kx_debug_dispatch_trace(uint64_t* out128) {
  return guard([&] { kx::read_dispatch_trace(reinterpret_cast<unsigned long long*>(out128)); });
}

// Diagnostics: per-pass tile phase sums of the radix passes (KX_SORT_TIMERS builds).
int kx_debug_sort_timers(uint64_t* out64, int32_t reset) {
  return guard([&] { kx::read_sort_debug(reinterpret_cast<unsigned long long*>(out64), reset != 0); });
}

int kx_sorting_accuracy(int64_t n, const int32_t* agent, const double* remaining,
                        const uint8_t* present, int32_t scope_all, uint64_t* pairs, double* correct,
                        double* accuracy) {
  return guard([&] {
    require(n >= 0, "negative size");
    require(n == 0 || (agent && remaining), "null argument");
    for (int64_t i = 0; i < n; ++i) require(agent[i] >= 0, "negative agent index");
    ensure_device(0);
    int dev = 0;
    KX_CUDA(cudaGetDevice(&dev));
    cudaStream_t st = nullptr;
    KX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct SG {
      cudaStream_t s;
      ~SG() { cudaStreamDestroy(s); }
    } sg{st};
    uint64_t p = 0;
    double c = 0.0;
    sorting_accuracy(n, agent, remaining, present, scope_all, &p, &c, sm_count(dev), st);
    if (pairs) *pairs = p;
    if (correct) *correct = c;
    if (accuracy) *accuracy = p ? c / static_cast<double>(p) : std::nan("");
  });
}

int kx_profiler_create(int32_t n_agents, const kx_convergence_config* exec,
                       const kx_convergence_config* remaining, int64_t capacity, int32_t device,
                       kx_profiler** out) {
  return guard([&] {
    require(out && exec && remaining, "null argument");
    require(n_agents > 0, "no agents");
    require(capacity > 0, "capacity must be positive");
    for (const kx_convergence_config* c : {exec, remaining}) {
      require(c->window_cap >= 0, "negative window_cap");
      if (c->window_cap > 0) require(capacity >= c->window_cap + 1, "capacity below window_cap + 1");
    }
    ensure_device(device);
    auto p = std::make_unique<kx_profiler>();
    p->device = device;
    p->n_agents = n_agents;
    p->cap = capacity;
    p->cfg[0] = *exec;
    p->cfg[1] = *remaining;
    KX_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    const size_t nd = size_t(2) * n_agents, C = static_cast<size_t>(capacity);
    Layout L;
    const size_t o_s = L.take<double>(nd * C), o_r = L.take<double>(nd * C), o_sn = L.take<double>(nd * C),
                 o_n = L.take<int64_t>(nd), o_h = L.take<int64_t>(nd), o_snn = L.take<int64_t>(nd),
                 o_t = L.take<uint64_t>(nd), o_cp = L.take<uint64_t>(nd), o_c = L.take<uint8_t>(nd),
                 o_l = L.take<double>(nd), o_ci = L.take<int64_t>(nd), o_cfg = L.take<DistCfg>(nd),
                 o_st = L.take<int>(1);
    KX_CUDA(cudaMalloc(&p->blob, L.off));
    KX_CUDA(cudaMemset(p->blob, 0, L.off));
    char* b = static_cast<char*>(p->blob);
    DistDev& dd = p->dd;
    dd.cap = capacity;
    dd.sorted = reinterpret_cast<double*>(b + o_s);
    dd.ring = reinterpret_cast<double*>(b + o_r);
    dd.snap = reinterpret_cast<double*>(b + o_sn);
    dd.n = reinterpret_cast<int64_t*>(b + o_n);
    dd.ring_head = reinterpret_cast<int64_t*>(b + o_h);
    dd.snap_n = reinterpret_cast<int64_t*>(b + o_snn);
    dd.total = reinterpret_cast<uint64_t*>(b + o_t);
    dd.next_cp = reinterpret_cast<uint64_t*>(b + o_cp);
    dd.conv = reinterpret_cast<uint8_t*>(b + o_c);
    dd.last_dist = reinterpret_cast<double*>(b + o_l);
    dd.conv_item = reinterpret_cast<int64_t*>(b + o_ci);
    p->d_cfg = reinterpret_cast<DistCfg*>(b + o_cfg);
    dd.cfg = p->d_cfg;
    p->status = reinterpret_cast<int*>(b + o_st);
    // EmpiricalDistribution(cfg): next_checkpoint_ = min_samples, last distance -1
    std::vector<DistCfg> cfgs(nd);
    std::vector<uint64_t> ncp(nd);
    std::vector<double> last(nd, -1.0);
    for (size_t d = 0; d < nd; ++d) {
      const kx_convergence_config& c = p->cfg[d / size_t(n_agents)];
      cfgs[d] = DistCfg{c.min_samples, c.relative_threshold, c.window_cap};
      ncp[d] = c.min_samples;
    }
    KX_CUDA(cudaMemcpy(p->d_cfg, cfgs.data(), nd * sizeof(DistCfg), cudaMemcpyHostToDevice));
    KX_CUDA(cudaMemcpy(dd.next_cp, ncp.data(), nd * 8, cudaMemcpyHostToDevice));
    KX_CUDA(cudaMemcpy(dd.last_dist, last.data(), nd * 8, cudaMemcpyHostToDevice));
    KX_CUDA(cudaStreamSynchronize(cudaStreamLegacy));  // the DMA has landed before p->stream uses it
    *out = p.release();
  });
}

int kx_profiler_destroy(kx_profiler* p) {
  return guard([&] {
    if (!p) return;
    cudaSetDevice(p->device);
    if (p->stream) cudaStreamSynchronize(p->stream);
    if (p->blob) cudaFree(p->blob);
    if (p->stream) cudaStreamDestroy(p->stream);
    delete p;
  });
}

int kx_profiler_record_execution(kx_profiler* p, int64_t n, const int32_t* agent, const double* latency) {
  return guard([&] {
    require(p, "null handle");
    require(n >= 0, "negative count");
    if (n == 0) return;
    require(agent && latency, "null argument");
    const int32_t A = p->n_agents;
    std::vector<int64_t> off(size_t(2) * A + 1, 0);
    for (int64_t j = 0; j < n; ++j) {
      require(agent[j] >= 0 && agent[j] < A, "agent index out of range");
      // LatencyProfiler::record_execution (profiler.cpp:20-29)
      if (!(latency[j] >= 0.0)) fail(KX_ERR_INVALID, "negative execution latency");
      ++off[size_t(agent[j]) + 1];
    }
    for (size_t d = 1; d < off.size(); ++d) off[d] += off[d - 1];
    std::vector<int64_t> fill(off.begin(), off.end() - 1), item(static_cast<size_t>(n));
    std::vector<double> values(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) {
      const int64_t k = fill[size_t(agent[j])]++;
      values[size_t(k)] = latency[j];
      item[size_t(k)] = j;
    }
    KX_CUDA(cudaSetDevice(p->device));
    profiler_ingest(p, off, values, item);
  });
}

int kx_profiler_record_remaining(kx_profiler* p, int64_t n_workflows, const int64_t* rec_offsets,
                                 const int32_t* agent, const double* exec_start, const double* exec_end,
                                 uint8_t* newly_converged) {
  return guard([&] {
    require(p, "null handle");
    require(n_workflows >= 0, "negative count");
    if (n_workflows == 0) return;
    require(rec_offsets && rec_offsets[0] == 0, "offsets must start at 0");
    const int64_t nr = rec_offsets[n_workflows];
    require(nr == 0 || (agent && exec_start && exec_end), "null argument");
    const int32_t A = p->n_agents;
    std::vector<double> sample(static_cast<size_t>(nr));
    std::vector<int64_t> off(size_t(2) * A + 1, 0);
    for (int64_t w = 0; w < n_workflows; ++w) {
      const int64_t b = rec_offsets[w], e = rec_offsets[w + 1];
      require(e >= b, "offsets must be non-decreasing");
      if (b == e) continue;  // record_remaining returns on an empty instance
      // finish = max exec_end seeded with the first record (profiler.cpp:33-35)
      double finish = exec_end[b];
      for (int64_t r = b; r < e; ++r) finish = finish < exec_end[r] ? exec_end[r] : finish;
      for (int64_t r = b; r < e; ++r) {
        require(agent[r] >= 0 && agent[r] < A, "agent index out of range");
        sample[size_t(r)] = finish - exec_start[r];
        // EmpiricalDistribution::add rejects negatives (distribution.cpp:92-94);
        // the batch is validated before any sample is applied
        if (!(sample[size_t(r)] >= 0.0)) fail(KX_ERR_INVALID, "latency sample must be non-negative");
        ++off[size_t(A + agent[r]) + 1];
      }
    }
    for (size_t d = 1; d < off.size(); ++d) off[d] += off[d - 1];
    std::vector<int64_t> fill(off.begin(), off.end() - 1), item(static_cast<size_t>(nr));
    std::vector<double> values(static_cast<size_t>(nr));
    for (int64_t w = 0; w < n_workflows; ++w)
      for (int64_t r = rec_offsets[w]; r < rec_offsets[w + 1]; ++r) {
        const int64_t k = fill[size_t(A + agent[r])]++;
        values[size_t(k)] = sample[size_t(r)];
        item[size_t(k)] = w;
      }
    KX_CUDA(cudaSetDevice(p->device));
    const std::vector<int64_t> conv = profiler_ingest(p, off, values, item);
    if (newly_converged) {
      std::memset(newly_converged, 0, size_t(n_workflows));
      for (int32_t a = 0; a < A; ++a) {
        const int64_t w = conv[size_t(A + a)];
        if (w >= 0 && w < n_workflows) newly_converged[w] = 1;
      }
    }
  });
}

int kx_profiler_read(kx_profiler* p, int32_t kind, int32_t agent, int64_t cap, double* samples, int64_t* n,
                     uint64_t* total_added, int32_t* converged, double* last_distance) {
  return guard([&] {
    require(p, "null handle");
    require(kind == 0 || kind == 1, "kind must be 0 (execution) or 1 (remaining)");
    require(agent >= 0 && agent < p->n_agents, "agent index out of range");
    KX_CUDA(cudaSetDevice(p->device));
    const int64_t d = int64_t(kind) * p->n_agents + agent;
    int64_t nn = 0;
    uint64_t tot = 0;
    uint8_t cv = 0;
    double ld = 0.0;
    cudaStream_t st = p->stream;
    KX_CUDA(cudaMemcpyAsync(&nn, p->dd.n + d, 8, cudaMemcpyDeviceToHost, st));
    KX_CUDA(cudaMemcpyAsync(&tot, p->dd.total + d, 8, cudaMemcpyDeviceToHost, st));
    KX_CUDA(cudaMemcpyAsync(&cv, p->dd.conv + d, 1, cudaMemcpyDeviceToHost, st));
    KX_CUDA(cudaMemcpyAsync(&ld, p->dd.last_dist + d, 8, cudaMemcpyDeviceToHost, st));
    KX_CUDA(cudaStreamSynchronize(st));
    if (n) *n = nn;
    if (total_added) *total_added = tot;
    if (converged) *converged = cv;
    if (last_distance) *last_distance = ld;
    const int64_t m = std::min(nn, cap);
    if (samples && m > 0) {
      KX_CUDA(cudaMemcpyAsync(samples, p->dd.sorted + d * p->cap, size_t(m) * 8, cudaMemcpyDeviceToHost, st));
      KX_CUDA(cudaStreamSynchronize(st));
    }
  });
}

int kx_w1_matrix(int32_t n_agents, const int64_t* offsets, const double* samples, double* out) {
  return guard([&] {
    require(n_agents >= 0, "negative agent count");
    require(offsets && out, "null argument");
    // build_matrix's checks (priority.cpp:17-27): no agents, empty set
    if (n_agents == 0) fail(KX_ERR_INVALID, "no converged agent distributions");
    require(offsets[0] == 0, "offsets must start at 0");
    for (int32_t a = 0; a < n_agents; ++a)
      if (offsets[a + 1] <= offsets[a]) fail(KX_ERR_INVALID, "empty distribution for agent " + std::to_string(a));
    const int64_t ns = offsets[n_agents];
    require(ns == 0 || samples, "null samples");
    ensure_device(0);
    int dev = 0;
    KX_CUDA(cudaGetDevice(&dev));
    cudaStream_t st = nullptr;
    KX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct SG {
      cudaStream_t s;
      ~SG() { cudaStreamDestroy(s); }
    } sg{st};
    const int64_t m = int64_t(n_agents) + 1;
    int64_t* d_off = nullptr;
    double *d_s = nullptr, *d_m = nullptr;
    KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_off), size_t(m) * 8, st));
    KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_s), size_t(std::max<int64_t>(ns, 1)) * 8, st));
    KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_m), size_t(m * m) * 8, st));
    KX_CUDA(cudaMemcpyAsync(d_off, offsets, size_t(m) * 8, cudaMemcpyHostToDevice, st));
    if (ns) KX_CUDA(cudaMemcpyAsync(d_s, samples, size_t(ns) * 8, cudaMemcpyHostToDevice, st));
    launch_w1_matrix(n_agents, d_off, d_s, d_m, sm_count(dev), st);
    KX_CUDA(cudaMemcpyAsync(out, d_m, size_t(m * m) * 8, cudaMemcpyDeviceToHost, st));
    KX_CUDA(cudaFreeAsync(d_off, st));
    KX_CUDA(cudaFreeAsync(d_s, st));
    KX_CUDA(cudaFreeAsync(d_m, st));
    KX_CUDA(cudaStreamSynchronize(st));
  });
}

int kx_expected_exec_times(int32_t n_agents, const int64_t* offsets, const double* samples,
                           int64_t min_samples, double fallback, double* out) {
  return guard([&] {
    require(n_agents >= 0, "negative agent count");
    if (n_agents == 0) return;
    require(offsets && out, "null argument");
    require(offsets[0] == 0, "offsets must start at 0");
    for (int32_t a = 0; a < n_agents; ++a) require(offsets[a + 1] >= offsets[a], "offsets must be non-decreasing");
    const int64_t ns = offsets[n_agents];
    require(ns == 0 || samples, "null samples");
    for (int32_t a = 0; a < n_agents; ++a)  // mode_estimate expects a sorted set
      for (int64_t k = offsets[a] + 1; k < offsets[a + 1]; ++k)
        require(samples[k - 1] <= samples[k], "sample sets must be sorted ascending");
    ensure_device(0);
    cudaStream_t st = nullptr;
    KX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct SG {
      cudaStream_t s;
      ~SG() { cudaStreamDestroy(s); }
    } sg{st};
    int64_t* d_off = nullptr;
    double *d_s = nullptr, *d_o = nullptr;
    KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_off), size_t(n_agents + 1) * 8, st));
    KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_s), size_t(std::max<int64_t>(ns, 1)) * 8, st));
    KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_o), size_t(n_agents) * 8, st));
    KX_CUDA(cudaMemcpyAsync(d_off, offsets, size_t(n_agents + 1) * 8, cudaMemcpyHostToDevice, st));
    if (ns) KX_CUDA(cudaMemcpyAsync(d_s, samples, size_t(ns) * 8, cudaMemcpyHostToDevice, st));
    launch_expected_T(n_agents, d_off, d_s, min_samples, fallback, d_o, st);
    KX_CUDA(cudaMemcpyAsync(out, d_o, size_t(n_agents) * 8, cudaMemcpyDeviceToHost, st));
    KX_CUDA(cudaFreeAsync(d_off, st));
    KX_CUDA(cudaFreeAsync(d_s, st));
    KX_CUDA(cudaFreeAsync(d_o, st));
    KX_CUDA(cudaStreamSynchronize(st));
  });
}

int kx_aggregate_metrics(int32_t n_rows, const double* rows, double* out) {
  return guard([&] {
    require(n_rows >= 0 && (rows || n_rows == 0) && out, "null argument");
    for (int k = 0; k < kEngineMetrics; ++k) out[k] = 0.0;
    if (n_rows == 0) return;
    // Sums for counts, plain means (accumulated as x / n in replica order,
    // metrics.cpp:98-118) for the rates, max for the end time.
    const double n = static_cast<double>(n_rows);
    for (int r = 0; r < n_rows; ++r) {
      const double* m = rows + int64_t(r) * kEngineMetrics;
      out[0] += m[0];
      out[1] += m[1];
      for (int k : {2, 3, 4, 5, 6, 7, 8, 11, 13}) out[k] += m[k] / n;
      out[9] += m[9];
      out[10] += m[10];
      out[12] += m[12];
      out[14] = std::max(out[14], m[14]);
      out[15] += m[15];
    }
  });
}

int kx_replicas_run(const kx_engine_config* cfg, const kx_replica_batch* batch, kx_replica_results* out,
                    double* device_ms) {
  return guard([&] { replicas_run_impl(cfg, batch, out, device_ms); });
}

int kx_orchestrator_dp(int64_t n_workflows, const int64_t* wf_offsets, const int32_t* parent,
                       const int64_t* prompt_tokens, const int64_t* target_tokens,
                       double prefill_rate, double decode_rate, uint64_t uid_base,
                       uint64_t* uid_out, double* pure_exec_out, double* remaining_out,
                       int32_t mem) {
  return guard([&] {
    require(n_workflows >= 0, "negative workflow count");
    require(prefill_rate > 0.0 && decode_rate > 0.0, "rates must be positive");
    if (n_workflows == 0) return;
    require(wf_offsets && parent && prompt_tokens && target_tokens && uid_out && pure_exec_out &&
                remaining_out,
            "null argument");
    ensure_device(0);
    int dev = 0;
    KX_CUDA(cudaGetDevice(&dev));
    const int sms = sm_count(dev);
    cudaStream_t st = nullptr;
    KX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    int64_t n_calls = 0;
    const int64_t* off_d = wf_offsets;
    const int32_t* par_d = parent;
    const int64_t* pr_d = prompt_tokens;
    const int64_t* tg_d = target_tokens;
    uint64_t* uid_d = uid_out;
    double* pure_d = pure_exec_out;
    double* rem_d = remaining_out;
    int* err_d = nullptr;
    std::vector<void*> owned;
    auto dalloc = [&](size_t bytes) {
      void* p = nullptr;
      KX_CUDA(cudaMallocAsync(&p, std::max<size_t>(bytes, 8), st));
      owned.push_back(p);
      return p;
    };
    struct FreeGuard {
      std::vector<void*>* v;
      cudaStream_t s;
      ~FreeGuard() {
        for (void* p : *v) cudaFreeAsync(p, s);
        cudaStreamSynchronize(s);
      }
    } fg{&owned, st};
    if (mem == KX_MEM_HOST) {
      n_calls = wf_offsets[n_workflows];
      require(wf_offsets[0] == 0 && n_calls >= 0, "wf_offsets must start at 0");
      for (int64_t w = 0; w < n_workflows; ++w)
        require(wf_offsets[w + 1] >= wf_offsets[w], "wf_offsets must be non-decreasing");
      const size_t C = static_cast<size_t>(n_calls);
      auto* o = static_cast<int64_t*>(dalloc((n_workflows + 1) * 8));
      auto* pa = static_cast<int32_t*>(dalloc(C * 4));
      auto* pr = static_cast<int64_t*>(dalloc(C * 8));
      auto* tg = static_cast<int64_t*>(dalloc(C * 8));
      uid_d = static_cast<uint64_t*>(dalloc(C * 8));
      pure_d = static_cast<double*>(dalloc(C * 8));
      rem_d = static_cast<double*>(dalloc(C * 8));
      KX_CUDA(cudaMemcpyAsync(o, wf_offsets, (n_workflows + 1) * 8, cudaMemcpyHostToDevice, st));
      KX_CUDA(cudaMemcpyAsync(pa, parent, C * 4, cudaMemcpyHostToDevice, st));
      KX_CUDA(cudaMemcpyAsync(pr, prompt_tokens, C * 8, cudaMemcpyHostToDevice, st));
      KX_CUDA(cudaMemcpyAsync(tg, target_tokens, C * 8, cudaMemcpyHostToDevice, st));
      off_d = o;
      par_d = pa;
      pr_d = pr;
      tg_d = tg;
    } else {
      KX_CUDA(cudaMemcpyAsync(&n_calls, wf_offsets + n_workflows, 8, cudaMemcpyDeviceToHost, st));
      KX_CUDA(cudaStreamSynchronize(st));
    }
    err_d = static_cast<int*>(dalloc(4));
    KX_CUDA(cudaMemsetAsync(err_d, 0, 4, st));
    launch_orchestrator_dp(n_workflows, off_d, par_d, pr_d, tg_d, prefill_rate, decode_rate,
                           uid_base, uid_d, pure_d, rem_d, err_d, sms, st);
    int err = 0;
    KX_CUDA(cudaMemcpyAsync(&err, err_d, 4, cudaMemcpyDeviceToHost, st));
    if (mem == KX_MEM_HOST && n_calls > 0) {
      const size_t C = static_cast<size_t>(n_calls);
      KX_CUDA(cudaMemcpyAsync(uid_out, uid_d, C * 8, cudaMemcpyDeviceToHost, st));
      KX_CUDA(cudaMemcpyAsync(pure_exec_out, pure_d, C * 8, cudaMemcpyDeviceToHost, st));
      KX_CUDA(cudaMemcpyAsync(remaining_out, rem_d, C * 8, cudaMemcpyDeviceToHost, st));
    }
    KX_CUDA(cudaStreamSynchronize(st));
    if (err) fail(KX_ERR_INVALID, "parent link is not parents-first (parent >= node id)");
  });
}

int kx_record_remaining(int64_t n_workflows, const int64_t* rec_offsets, const double* exec_start,
                        const double* exec_end, double* finish_out, double* samples_out,
                        int32_t mem) {
  return guard([&] {
    require(n_workflows >= 0, "negative workflow count");
    if (n_workflows == 0) return;
    require(rec_offsets && exec_start && exec_end && finish_out && samples_out, "null argument");
    ensure_device(0);
    int dev = 0;
    KX_CUDA(cudaGetDevice(&dev));
    const int sms = sm_count(dev);
    cudaStream_t st = nullptr;
    KX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    if (mem == KX_MEM_DEVICE) {
      launch_record_remaining(n_workflows, rec_offsets, exec_start, exec_end, finish_out,
                              samples_out, sms, st);
      KX_CUDA(cudaStreamSynchronize(st));
      return;
    }
    const int64_t n_rec = rec_offsets[n_workflows];
    require(rec_offsets[0] == 0 && n_rec >= 0, "rec_offsets must start at 0");
    const size_t R = static_cast<size_t>(n_rec), W = static_cast<size_t>(n_workflows);
    char* buf = nullptr;
    const size_t bytes = (W + 1) * 8 + R * 8 * 3 + W * 8 + 64;
    KX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), bytes, st));
    auto* o = reinterpret_cast<int64_t*>(buf);
    auto* es = reinterpret_cast<double*>(buf + (W + 1) * 8);
    auto* ee = es + R;
    auto* sm = ee + R;
    auto* fin = sm + R;
    KX_CUDA(cudaMemcpyAsync(o, rec_offsets, (W + 1) * 8, cudaMemcpyHostToDevice, st));
    KX_CUDA(cudaMemcpyAsync(es, exec_start, R * 8, cudaMemcpyHostToDevice, st));
    KX_CUDA(cudaMemcpyAsync(ee, exec_end, R * 8, cudaMemcpyHostToDevice, st));
    launch_record_remaining(n_workflows, o, es, ee, fin, sm, sms, st);
    KX_CUDA(cudaMemcpyAsync(samples_out, sm, R * 8, cudaMemcpyDeviceToHost, st));
    KX_CUDA(cudaMemcpyAsync(finish_out, fin, W * 8, cudaMemcpyDeviceToHost, st));
    KX_CUDA(cudaFreeAsync(buf, st));
    KX_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"

// Trace CSV I/O and workflow reconstruction on the device.
//
// Replaces
//   read_trace / parse_trace_line / validate   trace.cpp:14-127
//   write_trace / format_seconds               trace.cpp:29-48
//   WorkflowAnalyzer::ingest_trace             workflow.cpp:319-343
//     WorkflowGraph::ingest / ingest_instance  workflow.cpp:49-111
//     classify_fanout                          workflow.cpp:19-47
// for whole trace files: the bytes are split into lines by a newline scan,
// every line is parsed and validated by one thread (the reference's checks
// in its order; the first bad line by line number is reported with the
// reference's message), strings are interned by a 64-bit hash with a
// byte-compare of every equal-hash pair (a collision fails loudly), and the
// call graph's evidence is reduced with stable radix sorts: edge counts,
// entries, per-(instance, upstream) fan-out classification and the entry
// conflicts. The small graph algorithms over the result (feedback edges,
// downstream paths, topological depth, the report) run on the host
// (paper_2508_06948_b200/workflow.py).
//
// Numbers: the reference parses with std::stod/std::stoll. The device
// parser is exact (correctly rounded, half-even, like glibc's strtod) for
// decimal forms whose significand has at most 19 significant digits and
// whose power of ten is within +-22: one correctly rounded multiply or
// divide when the significand is <= 2^53 (Clinger's fast path), else the
// exact 128-bit quotient/product rounded with a sticky bit. That covers
// every number format_seconds writes below 10^10 s; other forms strtod
// accepts (hex, inf/nan, longer significands, larger exponents) are refused
// with KX_ERR_INVALID rather than parsed approximately.
// format_seconds' "%.9f" is produced exactly: round-half-even of
// x * 10^9 in 128-bit integer arithmetic.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/kairos_b200.h"
#include "kx_common.cuh"
#include "kx_sortlib.cuh"

namespace kx {
void set_last_error(const char* m);  // kx_abi.cu
}

using namespace kx;

namespace {

constexpr char kTraceHeader[] =
    "msg_id,agent,upstream,exec_start,exec_end,prompt_tokens,output_tokens,app_start";  // trace.cpp:10-12
constexpr int kHeaderLen = sizeof(kTraceHeader) - 1;
__device__ __constant__ char c_header[kHeaderLen + 1] =
    "msg_id,agent,upstream,exec_start,exec_end,prompt_tokens,output_tokens,app_start";
constexpr int64_t kChunk = 4096;  // bytes per thread in the newline scan

// Per-line parse outcome (first failing check, the reference's order).
enum : int32_t {
  kOk = 0,
  kSkip = 1,          // empty line or the header
  kFieldCount = 2,    // "expected 8 fields, got N"
  kBadNumber = 3,     // "bad numeric field '<f>': <s>"   (field in err_field)
  kBadCount = 4,      // "bad count field '<f>': <s>"
  kUnsupported = 5,   // a form std::stod accepts that the exact device parser does not
  kInvalid = 6,       // "invalid record: <why>"          (why in err_field)
};
const char* kFieldNames[8] = {"msg_id", "agent", "upstream", "exec_start", "exec_end",
                              "prompt_tokens", "output_tokens", "app_start"};
const char* kWhy[8] = {"empty msg_id", "empty agent", "empty upstream name", "app_start < 0",
                       "exec_start < app_start", "exec_end < exec_start", "prompt_tokens < 1",
                       "output_tokens < 1"};

__device__ __forceinline__ bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

__device__ __constant__ double c_pow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,
                                              1e8,  1e9,  1e10, 1e11, 1e12, 1e13, 1e14, 1e15,
                                              1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};

__device__ __forceinline__ int bitlen128(unsigned __int128 x) {
  const uint64_t hi = static_cast<uint64_t>(x >> 64);
  return hi ? 128 - __clzll(static_cast<long long>(hi)) : 64 - __clzll(static_cast<long long>(static_cast<uint64_t>(x)));
}

// m * 10^e10 correctly rounded (half-even) for a significand above 2^53
// (|e10| <= 22): the exact quotient/product in 128-bit integers, rounded to
// 53 bits with a sticky remainder. false when the product leaves 128 bits.
__device__ bool round_wide(uint64_t m, int e10, double* out) {
  unsigned __int128 p10 = 1;
  for (int i = 0; i < (e10 < 0 ? -e10 : e10); ++i) p10 *= 10u;
  unsigned __int128 q;
  int scale;        // value = q * 2^scale (+ the sticky remainder)
  bool sticky = false;
  if (e10 >= 0) {
    if (bitlen128(m) + bitlen128(p10) > 128) return false;
    q = static_cast<unsigned __int128>(m) * p10;
    scale = 0;
  } else {
    const int sh = 128 - bitlen128(m);
    const unsigned __int128 N = static_cast<unsigned __int128>(m) << sh;
    q = N / p10;
    sticky = N - q * p10 != 0;
    scale = -sh;
  }
  const int bq = bitlen128(q);
  if (bq <= 53) return false;  // not reached for |e10| <= 22
  int drop = bq - 53;
  uint64_t mant = static_cast<uint64_t>(q >> drop);
  const unsigned __int128 rem = q & ((static_cast<unsigned __int128>(1) << drop) - 1);
  const unsigned __int128 half = static_cast<unsigned __int128>(1) << (drop - 1);
  if (rem > half || (rem == half && (sticky || (mant & 1)))) {
    ++mant;
    if (mant == (uint64_t(1) << 53)) {
      mant >>= 1;
      ++drop;
    }
  }
  *out = scalbn(static_cast<double>(mant), drop + scale);  // exact: mant < 2^53, normal range
  return true;
}

// std::stod on [s, e): 0 ok, 1 invalid, 2 valid but outside the exact decimal forms.
__device__ int parse_double_dev(const char* s, const char* e, double* out) {
  const char* p = s;
  while (p < e && is_space(*p)) ++p;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  if (p < e && (*p == 'i' || *p == 'I' || *p == 'n' || *p == 'N')) return 2;  // inf / nan
  if (p + 1 < e && p[0] == '0' && (p[1] == 'x' || p[1] == 'X')) return 2;     // hex float
  uint64_t m = 0;
  int sig = 0, dropped = 0, frac = 0;
  bool any = false;
  for (; p < e && *p >= '0' && *p <= '9'; ++p) {
    any = true;
    if (m == 0 && *p == '0') continue;
    if (sig < 19) {
      m = m * 10 + uint64_t(*p - '0');
      ++sig;
    } else {
      ++dropped;
      if (*p != '0') return 2;
    }
  }
  if (p < e && *p == '.') {
    ++p;
    for (; p < e && *p >= '0' && *p <= '9'; ++p) {
      any = true;
      if (m == 0 && *p == '0') {
        ++frac;
        continue;
      }
      if (sig < 19) {
        m = m * 10 + uint64_t(*p - '0');
        ++sig;
        ++frac;
      } else if (*p != '0') {
        return 2;
      }
    }
  }
  if (!any) return 1;
  int64_t exp10 = 0;
  if (p < e && (*p == 'e' || *p == 'E')) {
    const char* q = p + 1;
    bool eneg = false;
    if (q < e && (*q == '+' || *q == '-')) eneg = *q++ == '-';
    if (q < e && *q >= '0' && *q <= '9') {  // a valid exponent; else strtod stops before 'e'
      int64_t v = 0;
      for (; q < e && *q >= '0' && *q <= '9'; ++q) v = v < 100000 ? v * 10 + (*q - '0') : v;
      exp10 = eneg ? -v : v;
      p = q;
    }
  }
  if (p != e) return 1;  // trailing characters (trace.cpp:66)
  if (m == 0) {
    *out = neg ? -0.0 : 0.0;
    return 0;
  }
  const int64_t e10 = exp10 + dropped - frac;
  if (e10 > 22 || e10 < -22) return 2;
  double v;
  if (m <= (uint64_t(1) << 53)) {  // Clinger: both operands exact, one correctly rounded op
    v = static_cast<double>(m);
    v = e10 >= 0 ? __dmul_rn(v, c_pow10[e10]) : __ddiv_rn(v, c_pow10[-e10]);
  } else if (!round_wide(m, static_cast<int>(e10), &v)) {
    return 2;
  }
  *out = neg ? -v : v;
  return 0;
}

// std::stoll on [s, e): 0 ok, 1 invalid or out of range.
__device__ int parse_count_dev(const char* s, const char* e, int64_t* out) {
  const char* p = s;
  while (p < e && is_space(*p)) ++p;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  if (p >= e || *p < '0' || *p > '9') return 1;
  uint64_t v = 0;
  const uint64_t lim = neg ? (uint64_t(1) << 63) : (uint64_t(1) << 63) - 1;
  for (; p < e && *p >= '0' && *p <= '9'; ++p) {
    const uint64_t d = uint64_t(*p - '0');
    if (v > (lim - d) / 10) return 1;
    v = v * 10 + d;
  }
  if (p != e) return 1;
  *out = neg ? static_cast<int64_t>(0 - v) : static_cast<int64_t>(v);
  return 0;
}

__device__ __forceinline__ uint64_t fnv1a(const char* s, const char* e) {
  uint64_t h = 1469598103934665603ull;
  for (; s < e; ++s) h = (h ^ static_cast<uint8_t>(*s)) * 1099511628211ull;
  return h;
}

struct LineOut {
  int32_t code, field;
};

// Newlines per chunk.
__global__ void k_count_lines(const char* __restrict__ b, int64_t n, int64_t* __restrict__ counts) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t lo = c * kChunk;
  if (lo >= n) return;
  const int64_t hi = lo + kChunk < n ? lo + kChunk : n;
  int64_t k = 0;
  for (int64_t i = lo; i < hi; ++i) k += b[i] == '\n';
  counts[c] = k;
}

// Line start offsets (line 0 starts at 0; every '\n' at i starts a line at i + 1).
__global__ void k_line_starts(const char* __restrict__ b, int64_t n, const int64_t* __restrict__ excl,
                              int64_t* __restrict__ starts) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t lo = c * kChunk;
  if (lo >= n) return;
  const int64_t hi = lo + kChunk < n ? lo + kChunk : n;
  int64_t k = excl[c] + 1;
  if (c == 0) starts[0] = 0;
  for (int64_t i = lo; i < hi; ++i)
    if (b[i] == '\n') starts[k++] = i + 1;
}

struct ParsedCols {
  double *es, *ee, *as;
  int64_t *prompt, *output;
  uint64_t *h_msg, *h_agent, *h_up;
  int64_t *off;          // [3 * lines]: start offsets of msg, agent, upstream
  int32_t *len;          // [3 * lines]
  uint8_t *keep;         // 1 = a record
};

// parse_trace_line + validate (trace.cpp:14-27, 90-109), one thread per line.
__global__ void k_parse_lines(const char* __restrict__ b, int64_t n_lines, const int64_t* __restrict__ starts,
                              int64_t newlines, int64_t n_bytes, ParsedCols c, LineOut* __restrict__ out,
                              unsigned long long* __restrict__ first_bad) {
  const int64_t L = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (L >= n_lines) return;
  const int64_t s = starts[L];
  int64_t e = L < newlines ? starts[L + 1] - 1 : n_bytes;  // exclusive of the '\n' ending line L
  if (e < s) e = s;
  c.keep[L] = 0;
  LineOut r{kOk, 0};
  const int64_t len = e - s;
  bool header = L == 0 && len == kHeaderLen;
  for (int i = 0; header && i < kHeaderLen; ++i) header = b[s + i] == c_header[i];
  if (len == 0 || header) {
    out[L] = LineOut{kSkip, 0};
    return;
  }
  int64_t fs[8], fe[8];
  int nf = 0;
  int64_t cur = s;
  for (int64_t i = s; i < e; ++i)
    if (b[i] == ',') {
      if (nf < 8) {
        fs[nf] = cur;
        fe[nf] = i;
      }
      ++nf;
      cur = i + 1;
    }
  if (nf < 8) {
    fs[nf] = cur;
    fe[nf] = e;
  }
  ++nf;
  double es = 0, ee = 0, as = 0;
  int64_t pt = 0, ot = 0;
  if (nf != 8) {
    r = LineOut{kFieldCount, nf};
  } else {
    int q;
    if ((q = parse_double_dev(b + fs[3], b + fe[3], &es)) != 0) r = LineOut{q == 1 ? kBadNumber : kUnsupported, 3};
    else if ((q = parse_double_dev(b + fs[4], b + fe[4], &ee)) != 0) r = LineOut{q == 1 ? kBadNumber : kUnsupported, 4};
    else if (parse_count_dev(b + fs[5], b + fe[5], &pt)) r = LineOut{kBadCount, 5};
    else if (parse_count_dev(b + fs[6], b + fe[6], &ot)) r = LineOut{kBadCount, 6};
    else if ((q = parse_double_dev(b + fs[7], b + fe[7], &as)) != 0) r = LineOut{q == 1 ? kBadNumber : kUnsupported, 7};
    // validate (trace.cpp:14-27), in order
    else if (fe[0] == fs[0]) r = LineOut{kInvalid, 0};
    else if (fe[1] == fs[1]) r = LineOut{kInvalid, 1};
    else if (as < 0.0) r = LineOut{kInvalid, 3};
    else if (es < as) r = LineOut{kInvalid, 4};
    else if (ee < es) r = LineOut{kInvalid, 5};
    else if (pt < 1) r = LineOut{kInvalid, 6};
    else if (ot < 1) r = LineOut{kInvalid, 7};
  }
  out[L] = r;
  if (r.code != kOk) {
    atomicMin(first_bad, static_cast<unsigned long long>(L));
    return;
  }
  c.keep[L] = 1;
  c.es[L] = es;
  c.ee[L] = ee;
  c.as[L] = as;
  c.prompt[L] = pt;
  c.output[L] = ot;
  for (int f = 0; f < 3; ++f) {
    c.off[3 * L + f] = fs[f];
    c.len[3 * L + f] = static_cast<int32_t>(fe[f] - fs[f]);
  }
  c.h_msg[L] = fnv1a(b + fs[0], b + fe[0]);
  c.h_agent[L] = fnv1a(b + fs[1], b + fe[1]);
  c.h_up[L] = fe[2] > fs[2] ? fnv1a(b + fs[2], b + fe[2]) : 0;
}

// Exclusive scan of 0/1 flags (one block per 1024 elements; block sums
// scanned by the host, added by k_add_offsets).
__global__ void k_flag_scan(const uint8_t* __restrict__ f, int64_t n, int64_t* __restrict__ excl,
                            int64_t* __restrict__ block_sum) {
  __shared__ int64_t s[1024];
  const int64_t i = int64_t(blockIdx.x) * 1024 + threadIdx.x;
  s[threadIdx.x] = i < n ? f[i] : 0;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int64_t v = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
    __syncthreads();
    s[threadIdx.x] += v;
    __syncthreads();
  }
  if (i < n) excl[i] = s[threadIdx.x] - (i < n ? f[i] : 0);
  if (threadIdx.x == 1023) block_sum[blockIdx.x] = s[1023];
}

__global__ void k_add_offsets(int64_t* __restrict__ excl, int64_t n, const int64_t* __restrict__ block_off) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) excl[i] += block_off[i / 1024];
}

// Gathers the kept lines into record order (file order).
__global__ void k_compact(int64_t n_lines, const uint8_t* __restrict__ keep, const int64_t* __restrict__ pos,
                          int64_t* __restrict__ rec_line) {
  const int64_t L = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (L < n_lines && keep[L]) rec_line[pos[L]] = L;
}

// String-interning keys: (hash, record * 4 + field) for every string occurrence.
__global__ void k_string_keys(int64_t n, const int64_t* __restrict__ rec_line, const uint64_t* __restrict__ h_msg,
                              const uint64_t* __restrict__ h_agent, const uint64_t* __restrict__ h_up,
                              const int32_t* __restrict__ len, uint64_t* __restrict__ msg_key,
                              uint64_t* __restrict__ ag_key, uint32_t* __restrict__ ag_val, uint32_t* __restrict__ n_ag) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t L = rec_line[r];
  msg_key[r] = h_msg[L];
  // agents: every record's agent, plus its upstream when present
  const uint32_t k = atomicAdd(n_ag, len[3 * L + 2] > 0 ? 2u : 1u);
  ag_key[k] = h_agent[L];
  ag_val[k] = static_cast<uint32_t>(r * 2);
  if (len[3 * L + 2] > 0) {
    ag_key[k + 1] = h_up[L];
    ag_val[k + 1] = static_cast<uint32_t>(r * 2 + 1);
  }
}

// Run heads of sorted hashes + byte-compare of every member with its head.
__global__ void k_unique_check(const char* __restrict__ b, int64_t n, const uint64_t* __restrict__ key,
                               const uint32_t* __restrict__ val, const int64_t* __restrict__ rec_line,
                               const int64_t* __restrict__ off, const int32_t* __restrict__ len, int field_base,
                               int agent_mode, uint8_t* __restrict__ head, int* __restrict__ collision) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool h = i == 0 || key[i] != key[i - 1];
  head[i] = h ? 1 : 0;
  if (h) return;
  const int64_t j = i - 1;  // equal to its predecessor => equal to the whole run
  auto where = [&](uint32_t v, int64_t* o, int32_t* l) {
    const int64_t r = agent_mode ? v >> 1 : v;
    const int f = agent_mode ? ((v & 1) ? 2 : 1) : field_base;
    const int64_t L = rec_line[r];
    *o = off[3 * L + f];
    *l = len[3 * L + f];
  };
  int64_t oa, ob;
  int32_t la, lb;
  where(val[i], &oa, &la);
  where(val[j], &ob, &lb);
  bool same = la == lb;
  for (int32_t k = 0; same && k < la; ++k) same = b[oa + k] == b[ob + k];
  if (!same) atomicExch(collision, 1);
}

// Compaction of the run heads: unique keys and the value of each run's head.
__global__ void k_compact_heads(int64_t n, const uint8_t* __restrict__ head, const int64_t* __restrict__ pos,
                                const uint64_t* __restrict__ key, const uint32_t* __restrict__ val,
                                uint64_t* __restrict__ ukey, uint32_t* __restrict__ uval) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && head[i]) {
    ukey[pos[i]] = key[i];
    uval[pos[i]] = val[i];
  }
}

// (offset, length) of the string behind an agent-dictionary value (record * 2 + upstream?).
__global__ void k_agent_strings(int64_t n, const uint32_t* __restrict__ val, const int64_t* __restrict__ rec_line,
                                const int64_t* __restrict__ off, const int32_t* __restrict__ len,
                                int64_t* __restrict__ o, int32_t* __restrict__ l) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t v = val[i];
  const int64_t L = rec_line[v >> 1];
  const int f = (v & 1) ? 2 : 1;
  o[i] = off[3 * L + f];
  l[i] = len[3 * L + f];
}

// Dictionary index of every record's msg / agent / upstream: binary search of
// the sorted unique hashes.
__device__ __forceinline__ int64_t find_hash(const uint64_t* u, int64_t n, uint64_t h) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (u[m] < h) lo = m + 1;
    else hi = m;
  }
  return lo;
}

__global__ void k_assign_ids(int64_t n, const int64_t* __restrict__ rec_line, const uint64_t* __restrict__ h_msg,
                             const uint64_t* __restrict__ h_agent, const uint64_t* __restrict__ h_up,
                             const int32_t* __restrict__ len, const uint64_t* __restrict__ umsg, int64_t n_msg,
                             const uint64_t* __restrict__ uag, int64_t n_ag, const int32_t* __restrict__ rank,
                             int64_t* __restrict__ msg, int32_t* __restrict__ agent, int32_t* __restrict__ up) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t L = rec_line[r];
  msg[r] = find_hash(umsg, n_msg, h_msg[L]);
  agent[r] = rank[find_hash(uag, n_ag, h_agent[L])];
  up[r] = len[3 * L + 2] > 0 ? rank[find_hash(uag, n_ag, h_up[L])] : -1;
}

// ---- format_seconds (trace.cpp:29-33): "%.9f", exact ----------------------
// round-half-even(x * 10^9) with x = m * 2^e and 5^9 * m < 2^74: 128-bit
// integer arithmetic; returns the digit count written (no terminator), or
// -1 when x * 10^9 does not fit 127 bits.
__device__ int fmt9(double x, char* out) {
  int n = 0;
  uint64_t bits = static_cast<uint64_t>(__double_as_longlong(x));
  if (bits >> 63) out[n++] = '-';
  bits &= ~(uint64_t(1) << 63);
  const int be = static_cast<int>(bits >> 52);
  uint64_t m = bits & ((uint64_t(1) << 52) - 1);
  int e;
  if (be == 0) {
    e = -1074;
  } else {
    m |= uint64_t(1) << 52;
    e = be - 1075;
  }
  if (be == 2047) return -1;  // inf / nan
  const unsigned __int128 P = static_cast<unsigned __int128>(m) * 1953125u;  // 5^9
  const int sh = e + 9;
  unsigned __int128 N;
  if (sh >= 0) {
    if (sh > 127 - 74) return -1;
    N = P << sh;
  } else {
    const int s = -sh;
    if (s >= 128) {
      N = 0;
    } else {
      const unsigned __int128 q = P >> s;
      const unsigned __int128 rem = P - (q << s);
      const unsigned __int128 half = static_cast<unsigned __int128>(1) << (s - 1);
      N = q + ((rem > half || (rem == half && (q & 1))) ? 1 : 0);
    }
  }
  char d[48];
  int nd = 0;
  do {
    d[nd++] = static_cast<char>('0' + static_cast<int>(N % 10));
    N /= 10;
  } while (N != 0);
  while (nd < 10) d[nd++] = '0';  // at least "0.000000000"
  for (int i = nd - 1; i >= 9; --i) out[n++] = d[i];
  out[n++] = '.';
  for (int i = 8; i >= 0; --i) out[n++] = d[i];
  return n;
}

__device__ int fmt_int(int64_t v, char* out) {
  int n = 0;
  uint64_t u = v < 0 ? 0 - static_cast<uint64_t>(v) : static_cast<uint64_t>(v);
  if (v < 0) out[n++] = '-';
  char d[24];
  int nd = 0;
  do {
    d[nd++] = static_cast<char>('0' + u % 10);
    u /= 10;
  } while (u);
  for (int i = nd - 1; i >= 0; --i) out[n++] = d[i];
  return n;
}

// write_trace_record (trace.cpp:37-43): pass 0 measures, pass 1 writes.
__global__ void k_format(const char* __restrict__ b, int64_t n, const int64_t* __restrict__ rec_line,
                         const int64_t* __restrict__ off, const int32_t* __restrict__ len,
                         const double* __restrict__ es, const double* __restrict__ ee, const double* __restrict__ as,
                         const int64_t* __restrict__ pt, const int64_t* __restrict__ ot, int pass,
                         int64_t* __restrict__ line_len, const int64_t* __restrict__ line_off, char* __restrict__ out,
                         int* __restrict__ bad) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t L = rec_line[r];
  char buf[256];
  int k = 0;
  auto str = [&](int f) {
    const int64_t o = off[3 * L + f];
    const int32_t l = len[3 * L + f];
    if (pass == 1)
      for (int32_t i = 0; i < l; ++i) out[line_off[r] + k + i] = b[o + i];
    k += l;
  };
  auto put = [&](const char* s, int l) {
    if (pass == 1)
      for (int i = 0; i < l; ++i) out[line_off[r] + k + i] = s[i];
    k += l;
  };
  const char comma = ',';
  str(0);
  put(&comma, 1);
  str(1);
  put(&comma, 1);
  str(2);
  put(&comma, 1);
  int l = fmt9(es[L], buf);
  if (l < 0) atomicExch(bad, 1);
  put(buf, l < 0 ? 0 : l);
  put(&comma, 1);
  l = fmt9(ee[L], buf);
  if (l < 0) atomicExch(bad, 1);
  put(buf, l < 0 ? 0 : l);
  put(&comma, 1);
  put(buf, fmt_int(pt[L], buf));
  put(&comma, 1);
  put(buf, fmt_int(ot[L], buf));
  put(&comma, 1);
  l = fmt9(as[L], buf);
  if (l < 0) atomicExch(bad, 1);
  put(buf, l < 0 ? 0 : l);
  const char nl = '\n';
  put(&nl, 1);
  if (pass == 0) line_len[r] = k;
}

// ---- reconstruction ---------------------------------------------------------
__device__ __forceinline__ uint64_t time_bits(double x) {  // ordered bits, -0 == +0 (operator<)
  if (x == 0.0) x = 0.0;
  const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
  return (u >> 63) ? ~u : (u | (uint64_t(1) << 63));
}

template <typename K>
__global__ void k_gather_key(int64_t n, const uint32_t* __restrict__ perm, int which, const double* __restrict__ es,
                             const double* __restrict__ ee, const int32_t* __restrict__ agent,
                             const int32_t* __restrict__ up, const int64_t* __restrict__ msg, K* __restrict__ key) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t r = perm[i];
  uint64_t k = 0;
  switch (which) {
    case 0: k = time_bits(ee[r]); break;
    case 1: k = static_cast<uint32_t>(agent[r]); break;
    case 2: k = time_bits(es[r]); break;
    case 3: k = static_cast<uint64_t>(msg[r]); break;
    default: k = (static_cast<uint64_t>(msg[r]) << 24) | static_cast<uint32_t>(up[r] + 1); break;  // (msg, upstream)
  }
  key[i] = static_cast<K>(k);
}

__global__ void k_permute(int64_t n, const uint32_t* __restrict__ perm, const uint32_t* __restrict__ sorted_pos,
                          uint32_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = perm[sorted_pos[i]];
}

// WorkflowGraph::ingest (workflow.cpp:49-57): node/entry flags and the
// (upstream, agent) keys of the edges.
__global__ void k_edge_keys(int64_t n, const int32_t* __restrict__ agent, const int32_t* __restrict__ up,
                            int32_t n_agents, uint8_t* __restrict__ is_entry, uint32_t* __restrict__ ekey,
                            uint32_t* __restrict__ n_edges_rec) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  if (up[r] < 0) {
    is_entry[agent[r]] = 1;
    return;
  }
  const uint32_t k = atomicAdd(n_edges_rec, 1u);
  ekey[k] = static_cast<uint32_t>(up[r]) * static_cast<uint32_t>(n_agents) + static_cast<uint32_t>(agent[r]);
}

__global__ void k_run_heads_u32(int64_t n, const uint32_t* __restrict__ key, uint32_t* __restrict__ head_pos,
                                uint32_t* __restrict__ n_heads) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0 || key[i] != key[i - 1]) head_pos[atomicAdd(n_heads, 1u)] = static_cast<uint32_t>(i);
}

__global__ void k_run_heads_u64(int64_t n, const uint64_t* __restrict__ key, uint32_t* __restrict__ head_pos,
                                uint32_t* __restrict__ n_heads) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0 || key[i] != key[i - 1]) head_pos[atomicAdd(n_heads, 1u)] = static_cast<uint32_t>(i);
}

// ingest_instance's entry diagnostics (workflow.cpp:59-76): records of one
// instance in (exec_start, agent, exec_end) order; the first upstream-less
// record names the entry, every later one with another agent is reported.
__global__ void k_entry_conflicts(int64_t n_groups, const uint32_t* __restrict__ heads, int64_t n,
                                  const uint64_t* __restrict__ key, const uint32_t* __restrict__ order,
                                  const int32_t* __restrict__ agent, const int32_t* __restrict__ up,
                                  int64_t* __restrict__ d_msg, int32_t* __restrict__ d_pos,
                                  int32_t* __restrict__ d_entry, int32_t* __restrict__ d_other,
                                  uint32_t* __restrict__ n_diag, uint32_t cap) {
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  const int64_t s = heads[g];
  int32_t entry = -1;
  for (int64_t i = s; i < n && (i == s || key[i] == key[s]); ++i) {
    const uint32_t r = order[i];
    if (up[r] >= 0) continue;
    if (entry < 0) {
      entry = agent[r];
    } else if (agent[r] != entry) {
      const uint32_t k = atomicAdd(n_diag, 1u);
      if (k < cap) {
        d_msg[k] = static_cast<int64_t>(key[s]);
        d_pos[k] = static_cast<int32_t>(i - s);
        d_entry[k] = entry;
        d_other[k] = agent[r];
      }
    }
  }
}

// classify_fanout (workflow.cpp:19-47) of one (instance, upstream) group.
constexpr int kFanMax = 64;  // spans per group evaluated in registers/local memory
__global__ void k_fanouts(int64_t n_groups, const uint32_t* __restrict__ heads, int64_t n,
                          const uint64_t* __restrict__ key, const uint32_t* __restrict__ order,
                          const int32_t* __restrict__ agent, const int32_t* __restrict__ up,
                          const double* __restrict__ es, const double* __restrict__ ee,
                          unsigned long long* __restrict__ tallies, int* __restrict__ bad) {
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  const int64_t s = heads[g];
  const uint32_t r0 = order[s];
  if (up[r0] < 0) return;  // upstream-less records: no fan-out evidence
  int64_t e = s + 1;
  while (e < n && key[e] == key[s]) ++e;
  const int cnt = static_cast<int>(e - s);
  // distinct downstream agents
  int distinct = 0;
  for (int64_t i = s; i < e; ++i) {
    bool seen = false;
    for (int64_t j = s; j < i && !seen; ++j) seen = agent[order[j]] == agent[order[i]];
    distinct += seen ? 0 : 1;
  }
  int kind;  // 0 parallel, 1 sequential, 2 single
  if (distinct < 2) {
    kind = 2;
  } else if (cnt > kFanMax) {
    atomicExch(bad, 1);
    return;
  } else {
    // events in span order: (start, +1), (end, -1); libstdc++'s insertion
    // sort (std::sort below 17 elements) with the reference's comparator
    double t[2 * kFanMax];
    int d[2 * kFanMax];
    int m = 0;
    for (int64_t i = s; i < e; ++i) {
      const uint32_t r = order[i];
      t[m] = es[r];
      d[m++] = +1;
      t[m] = ee[r];
      d[m++] = -1;
    }
    auto less = [&](double ta, int da, double tb, int db) {
      const double diff = ta - tb;
      if ((diff < 0 ? -diff : diff) > kTimeEpsilon) return ta < tb;
      return da < db;
    };
    for (int i = 1; i < m; ++i) {
      const double tv = t[i];
      const int dv = d[i];
      int j = i;
      if (less(tv, dv, t[0], d[0])) {
        for (; j > 0; --j) {
          t[j] = t[j - 1];
          d[j] = d[j - 1];
        }
      } else {
        while (less(tv, dv, t[j - 1], d[j - 1])) {
          t[j] = t[j - 1];
          d[j] = d[j - 1];
          --j;
        }
      }
      t[j] = tv;
      d[j] = dv;
    }
    int open = 0;
    kind = 1;
    for (int i = 0; i < m; ++i) {
      open += d[i];
      if (open >= 2) {
        kind = 0;
        break;
      }
    }
  }
  atomicAdd(&tallies[3 * up[r0] + kind], 1ull);
}

}  // namespace

struct kx_trace {
  int dev = 0;
  cudaStream_t st = nullptr;
  int64_t n_bytes = 0, n_lines = 0, newlines = 0, n = 0;
  char* bytes = nullptr;
  // per line
  int64_t* starts = nullptr;
  int64_t* off = nullptr;
  int32_t* len = nullptr;
  double *es = nullptr, *ee = nullptr, *as = nullptr;
  int64_t *prompt = nullptr, *output = nullptr;
  // per record
  int64_t* rec_line = nullptr;
  int64_t* msg = nullptr;
  int32_t *agent = nullptr, *up = nullptr;
  double *r_es = nullptr, *r_ee = nullptr;
  // dictionaries
  std::vector<std::string> agents;  // std::string order
  int64_t n_msgs = 0;
  uint64_t* umsg = nullptr;         // sorted unique msg hashes
  uint32_t* msg_first_dev = nullptr;  // a record of each msg index (device)
  std::vector<void*> allocs;
  // reconstruction
  bool built = false;
  std::vector<int32_t> e_from, e_to;
  std::vector<uint64_t> e_count;
  std::vector<uint8_t> is_entry;
  std::vector<uint64_t> tallies;  // [3 * n_agents]: parallel, sequential, single
  std::vector<int64_t> d_msg;
  std::vector<int32_t> d_entry, d_other;

  template <typename T>
  T* dalloc(size_t count) {
    void* p = nullptr;
    KX_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
  ~kx_trace() {
    for (void* p : allocs) cudaFree(p);
    if (st) cudaStreamDestroy(st);
  }
};

// Byte spans (offset, length in the parsed bytes) of msg indices, and the
// msg_id strings themselves gathered into one packed buffer: a handful of
// transfers however many diagnostics a trace has.
__global__ void k_msg_spans(int64_t k, const int64_t* __restrict__ msgs, const uint32_t* __restrict__ msg_first,
                            const int64_t* __restrict__ rec_line, const int64_t* __restrict__ off,
                            const int32_t* __restrict__ len, int64_t* __restrict__ off_out,
                            int32_t* __restrict__ len_out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= k) return;
  const int64_t L = rec_line[msg_first[msgs[i]]];
  off_out[i] = off[3 * L];
  len_out[i] = len[3 * L];
}

__global__ void k_gather_spans(int64_t k, const char* __restrict__ bytes, const int64_t* __restrict__ off,
                               const int32_t* __restrict__ len, const int64_t* __restrict__ pos,
                               char* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.y + threadIdx.y;
  if (i >= k) return;
  for (int j = threadIdx.x; j < len[i]; j += blockDim.x) out[pos[i] + j] = bytes[off[i] + j];
}

// Host <-> device copies of the trace, ordered on its (non-blocking) stream:
// a plain cudaMemcpy runs on the legacy stream, which does not wait for it.
static void tcopy(const kx_trace* t, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  KX_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, t->st));
  KX_CUDA(cudaStreamSynchronize(t->st));
}

static void msg_spans_dev(const kx_trace* t, int64_t k, const int64_t* msgs_host, int64_t* doff, int32_t* dlen) {
  int64_t* dm = nullptr;
  KX_CUDA(cudaMalloc(&dm, size_t(k) * 8));
  KX_CUDA(cudaMemcpyAsync(dm, msgs_host, size_t(k) * 8, cudaMemcpyHostToDevice, t->st));
  k_msg_spans<<<static_cast<unsigned>((k + 255) / 256), 256, 0, t->st>>>(k, dm, t->msg_first_dev, t->rec_line, t->off,
                                                                       t->len, doff, dlen);
  KX_CHECK_LAUNCH();
  KX_CUDA(cudaStreamSynchronize(t->st));
  KX_CUDA(cudaFree(dm));
}

static std::vector<std::string> fetch_msg_names(const kx_trace* t, const std::vector<int64_t>& msgs) {
  const int64_t k = static_cast<int64_t>(msgs.size());
  std::vector<std::string> out(msgs.size());
  if (k == 0) return out;
  int64_t *doff = nullptr, *dpos = nullptr;
  int32_t* dlen = nullptr;
  KX_CUDA(cudaMalloc(&doff, size_t(k) * 8));
  KX_CUDA(cudaMalloc(&dpos, size_t(k) * 8));
  KX_CUDA(cudaMalloc(&dlen, size_t(k) * 4));
  msg_spans_dev(t, k, msgs.data(), doff, dlen);
  std::vector<int32_t> len(static_cast<size_t>(k));
  tcopy(t, len.data(), dlen, size_t(k) * 4, cudaMemcpyDeviceToHost);
  std::vector<int64_t> pos(static_cast<size_t>(k) + 1, 0);
  for (int64_t i = 0; i < k; ++i) pos[i + 1] = pos[i] + len[i];
  char* dbuf = nullptr;
  KX_CUDA(cudaMalloc(&dbuf, size_t(std::max<int64_t>(pos[k], 1))));
  KX_CUDA(cudaMemcpyAsync(dpos, pos.data(), size_t(k) * 8, cudaMemcpyHostToDevice, t->st));
  const dim3 blk(32, 8);
  k_gather_spans<<<static_cast<unsigned>((k + 7) / 8), blk, 0, t->st>>>(k, t->bytes, doff, dlen, dpos, dbuf);
  KX_CHECK_LAUNCH();
  std::string packed(static_cast<size_t>(pos[k]), '\0');
  if (pos[k]) KX_CUDA(cudaMemcpyAsync(packed.data(), dbuf, size_t(pos[k]), cudaMemcpyDeviceToHost, t->st));
  KX_CUDA(cudaStreamSynchronize(t->st));
  for (int64_t i = 0; i < k; ++i) out[i] = packed.substr(static_cast<size_t>(pos[i]), static_cast<size_t>(len[i]));
  KX_CUDA(cudaFree(doff));
  KX_CUDA(cudaFree(dpos));
  KX_CUDA(cudaFree(dlen));
  KX_CUDA(cudaFree(dbuf));
  return out;
}

namespace {

unsigned grid_of(int64_t n, int t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

// Host exclusive scan of device counts (small arrays).
std::vector<int64_t> host_excl(const int64_t* d, int64_t n, cudaStream_t st, int64_t* total) {
  std::vector<int64_t> h(static_cast<size_t>(n));
  if (n) KX_CUDA(cudaMemcpyAsync(h.data(), d, n * 8, cudaMemcpyDeviceToHost, st));
  KX_CUDA(cudaStreamSynchronize(st));
  int64_t acc = 0;
  for (auto& v : h) {
    const int64_t c = v;
    v = acc;
    acc += c;
  }
  *total = acc;
  return h;
}

std::string line_text(kx_trace* t, int64_t L) {
  int64_t s = 0, e = 0;
  tcopy(t, &s, t->starts + L, 8, cudaMemcpyDeviceToHost);
  if (L < t->newlines) {
    tcopy(t, &e, t->starts + L + 1, 8, cudaMemcpyDeviceToHost);
    e -= 1;
  } else {
    e = t->n_bytes;
  }
  std::string out(static_cast<size_t>(std::max<int64_t>(e - s, 0)), '\0');
  if (!out.empty()) tcopy(t, out.data(), t->bytes + s, out.size(), cudaMemcpyDeviceToHost);
  return out;
}

std::vector<std::string> split(const std::string& line) {
  std::vector<std::string> f(1);
  for (char c : line) {
    if (c == ',') f.emplace_back();
    else f.back().push_back(c);
  }
  return f;
}

void parse(kx_trace* t, const char* host_bytes, int64_t n_bytes) {
  cudaStream_t st = t->st;
  t->n_bytes = n_bytes;
  t->bytes = t->dalloc<char>(static_cast<size_t>(n_bytes) + 1);
  if (n_bytes) KX_CUDA(cudaMemcpyAsync(t->bytes, host_bytes, n_bytes, cudaMemcpyHostToDevice, st));
  // lines: split on '\n' (std::getline); a final '\n' ends the last line
  const int64_t chunks = (n_bytes + kChunk - 1) / kChunk;
  int64_t* counts = t->dalloc<int64_t>(chunks);
  if (chunks) {
    k_count_lines<<<grid_of(chunks), 256, 0, st>>>(t->bytes, n_bytes, counts);
    KX_CHECK_LAUNCH();
  }
  int64_t newlines = 0;
  std::vector<int64_t> excl = host_excl(counts, chunks, st, &newlines);
  const bool trailing_nl = n_bytes > 0 && host_bytes[n_bytes - 1] == '\n';
  t->n_lines = n_bytes == 0 ? 0 : newlines + (trailing_nl ? 0 : 1);
  t->newlines = newlines;
  t->starts = t->dalloc<int64_t>(static_cast<size_t>(newlines) + 1);
  if (chunks) {
    KX_CUDA(cudaMemcpyAsync(counts, excl.data(), chunks * 8, cudaMemcpyHostToDevice, st));
    k_line_starts<<<grid_of(chunks), 256, 0, st>>>(t->bytes, n_bytes, counts, t->starts);
    KX_CHECK_LAUNCH();
  }
  const int64_t NL = t->n_lines;
  ParsedCols c{};
  c.es = t->es = t->dalloc<double>(NL);
  c.ee = t->ee = t->dalloc<double>(NL);
  c.as = t->as = t->dalloc<double>(NL);
  c.prompt = t->prompt = t->dalloc<int64_t>(NL);
  c.output = t->output = t->dalloc<int64_t>(NL);
  c.h_msg = t->dalloc<uint64_t>(NL);
  c.h_agent = t->dalloc<uint64_t>(NL);
  c.h_up = t->dalloc<uint64_t>(NL);
  c.off = t->off = t->dalloc<int64_t>(3 * NL);
  c.len = t->len = t->dalloc<int32_t>(3 * NL);
  c.keep = t->dalloc<uint8_t>(NL);
  LineOut* lo = t->dalloc<LineOut>(NL);
  unsigned long long* first_bad = t->dalloc<unsigned long long>(1);
  KX_CUDA(cudaMemsetAsync(first_bad, 0xff, 8, st));
  if (NL) {
    k_parse_lines<<<grid_of(NL, 128), 128, 0, st>>>(t->bytes, NL, t->starts, newlines, n_bytes, c, lo, first_bad);
    KX_CHECK_LAUNCH();
  }
  unsigned long long bad = 0;
  KX_CUDA(cudaMemcpyAsync(&bad, first_bad, 8, cudaMemcpyDeviceToHost, st));
  KX_CUDA(cudaStreamSynchronize(st));
  if (bad != ~0ull) {  // read_trace's message for the first bad line (trace.cpp:118-123)
    LineOut r{};
    tcopy(t, &r, lo + bad, sizeof(r), cudaMemcpyDeviceToHost);
    const std::string line = line_text(t, static_cast<int64_t>(bad));
    const auto f = split(line);
    std::string m;
    switch (r.code) {
      case kFieldCount: m = "expected 8 fields, got " + std::to_string(f.size()); break;
      case kBadNumber: m = std::string("bad numeric field '") + kFieldNames[r.field] + "': " + f[r.field]; break;
      case kBadCount: m = std::string("bad count field '") + kFieldNames[r.field] + "': " + f[r.field]; break;
      case kUnsupported:
        throw KxError(KX_ERR_INVALID, "trace line " + std::to_string(bad + 1) + ": numeric field '" +
                                          kFieldNames[r.field] + "': " + f[r.field] +
                                          " is outside the device parser's exact decimal forms");
      default: m = std::string("invalid record: ") + kWhy[r.field]; break;
    }
    throw KxError(KX_ERR_INVALID, "trace line " + std::to_string(bad + 1) + ": " + m);
  }
  // records in file order
  const int64_t blocks = (NL + 1023) / 1024;
  int64_t* pos = t->dalloc<int64_t>(NL);
  int64_t* bsum = t->dalloc<int64_t>(blocks);
  if (NL) {
    k_flag_scan<<<static_cast<unsigned>(blocks), 1024, 0, st>>>(c.keep, NL, pos, bsum);
    KX_CHECK_LAUNCH();
  }
  int64_t n = 0;
  std::vector<int64_t> boff = host_excl(bsum, blocks, st, &n);
  if (blocks) {
    KX_CUDA(cudaMemcpyAsync(bsum, boff.data(), blocks * 8, cudaMemcpyHostToDevice, st));
    k_add_offsets<<<grid_of(NL), 256, 0, st>>>(pos, NL, bsum);
    KX_CHECK_LAUNCH();
  }
  if (n >= (int64_t(1) << 31)) throw KxError(KX_ERR_CAPACITY, "trace: more than 2^31 records");
  t->n = n;
  t->rec_line = t->dalloc<int64_t>(n);
  if (NL) {
    k_compact<<<grid_of(NL), 256, 0, st>>>(NL, c.keep, pos, t->rec_line);
    KX_CHECK_LAUNCH();
  }
  // string interning: sorted unique hashes, each run byte-compared with its head
  uint64_t* mkey = t->dalloc<uint64_t>(n);
  uint64_t* akey = t->dalloc<uint64_t>(2 * n);
  uint32_t* aval = t->dalloc<uint32_t>(2 * n);
  uint32_t* n_agk = t->dalloc<uint32_t>(1);
  KX_CUDA(cudaMemsetAsync(n_agk, 0, 4, st));
  if (n) {
    k_string_keys<<<grid_of(n), 256, 0, st>>>(n, t->rec_line, c.h_msg, c.h_agent, c.h_up, c.len, mkey, akey, aval,
                                               n_agk);
    KX_CHECK_LAUNCH();
  }
  uint32_t na = 0;
  KX_CUDA(cudaMemcpyAsync(&na, n_agk, 4, cudaMemcpyDeviceToHost, st));
  KX_CUDA(cudaStreamSynchronize(st));
  int* collision = t->dalloc<int>(1);
  KX_CUDA(cudaMemsetAsync(collision, 0, 4, st));
  // sorted unique hashes (device) and the value of each run head
  auto unique_sorted = [&](uint64_t* key, int64_t cnt, uint32_t* val_in, bool agent_mode, uint64_t** ukey,
                           uint32_t** uval) -> int64_t {
    uint64_t* k2 = t->dalloc<uint64_t>(cnt);
    uint32_t* v = t->dalloc<uint32_t>(cnt);
    uint32_t* v2 = t->dalloc<uint32_t>(cnt);
    if (val_in && cnt) KX_CUDA(cudaMemcpyAsync(v, val_in, cnt * 4, cudaMemcpyDeviceToDevice, st));
    bool alt = false;
    sort_pairs<uint64_t>(key, v, k2, v2, cnt, 0, 64, val_in == nullptr, &alt, st);
    uint64_t* ks = alt ? k2 : key;
    uint32_t* vs = alt ? v2 : v;
    uint8_t* head = t->dalloc<uint8_t>(cnt);
    const int64_t nb = (cnt + 1023) / 1024;
    int64_t* hp = t->dalloc<int64_t>(cnt);
    int64_t* hs = t->dalloc<int64_t>(nb);
    int64_t uniq = 0;
    if (cnt) {
      k_unique_check<<<grid_of(cnt), 256, 0, st>>>(t->bytes, cnt, ks, vs, t->rec_line, c.off, c.len, 0,
                                                    agent_mode ? 1 : 0, head, collision);
      KX_CHECK_LAUNCH();
      k_flag_scan<<<static_cast<unsigned>(nb), 1024, 0, st>>>(head, cnt, hp, hs);
      KX_CHECK_LAUNCH();
    }
    std::vector<int64_t> ho = host_excl(hs, nb, st, &uniq);
    *ukey = t->dalloc<uint64_t>(uniq);
    *uval = t->dalloc<uint32_t>(uniq);
    if (cnt) {
      KX_CUDA(cudaMemcpyAsync(hs, ho.data(), nb * 8, cudaMemcpyHostToDevice, st));
      k_add_offsets<<<grid_of(cnt), 256, 0, st>>>(hp, cnt, hs);
      k_compact_heads<<<grid_of(cnt), 256, 0, st>>>(cnt, head, hp, ks, vs, *ukey, *uval);
      KX_CHECK_LAUNCH();
    }
    return uniq;
  };
  uint64_t *umsg = nullptr, *uag = nullptr;
  uint32_t *fmsg = nullptr, *fag = nullptr;
  const int64_t n_msg = unique_sorted(mkey, n, nullptr, false, &umsg, &fmsg);
  const int64_t n_ag = unique_sorted(akey, na, aval, true, &uag, &fag);
  int col = 0;
  tcopy(t, &col, collision, 4, cudaMemcpyDeviceToHost);
  if (col) throw KxError(KX_ERR_RUNTIME, "trace: 64-bit string hash collision (distinct ids share a hash)");
  // agent names (std::string order, the std::set/std::map order of the
  // graph); msg ids stay in hash order (only their grouping matters, plus
  // the names of diagnosed instances)
  int64_t* ao = t->dalloc<int64_t>(n_ag);
  int32_t* al = t->dalloc<int32_t>(n_ag);
  if (n_ag) {
    k_agent_strings<<<grid_of(n_ag), 256, 0, st>>>(n_ag, fag, t->rec_line, c.off, c.len, ao, al);
    KX_CHECK_LAUNCH();
  }
  std::vector<int64_t> hao(static_cast<size_t>(n_ag));
  std::vector<int32_t> hal(static_cast<size_t>(n_ag));
  if (n_ag) {
    tcopy(t, hao.data(), ao, n_ag * 8, cudaMemcpyDeviceToHost);
    tcopy(t, hal.data(), al, n_ag * 4, cudaMemcpyDeviceToHost);
  }
  std::vector<std::string> names(static_cast<size_t>(n_ag));
  for (int64_t u = 0; u < n_ag; ++u) names[u].assign(host_bytes + hao[u], static_cast<size_t>(hal[u]));
  std::vector<int32_t> order(static_cast<size_t>(n_ag));
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return names[a] < names[b]; });
  std::vector<int32_t> rank(static_cast<size_t>(n_ag));
  t->agents.resize(static_cast<size_t>(n_ag));
  for (size_t i = 0; i < order.size(); ++i) {
    rank[order[i]] = static_cast<int32_t>(i);
    t->agents[i] = names[order[i]];
  }
  t->n_msgs = n_msg;
  t->umsg = umsg;
  t->msg_first_dev = fmsg;
  int32_t* drank = t->dalloc<int32_t>(n_ag);
  if (n_ag) tcopy(t, drank, rank.data(), rank.size() * 4, cudaMemcpyHostToDevice);
  t->msg = t->dalloc<int64_t>(n);
  t->agent = t->dalloc<int32_t>(n);
  t->up = t->dalloc<int32_t>(n);
  if (n) {
    k_assign_ids<<<grid_of(n), 256, 0, st>>>(n, t->rec_line, c.h_msg, c.h_agent, c.h_up, c.len, t->umsg, n_msg,
                                              uag, n_ag, drank, t->msg, t->agent, t->up);
    KX_CHECK_LAUNCH();
  }
  KX_CUDA(cudaStreamSynchronize(st));
}

template <typename T>
__global__ void k_gather_rec(int64_t n, const int64_t* __restrict__ rec_line, const T* __restrict__ src,
                             T* __restrict__ dst) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < n) dst[r] = src[rec_line[r]];
}

void reconstruct(kx_trace* t) {
  if (t->built) return;
  cudaStream_t st = t->st;
  const int64_t n = t->n;
  const int32_t A = static_cast<int32_t>(t->agents.size());
  if (int64_t(A) * A >= (int64_t(1) << 32)) throw KxError(KX_ERR_CAPACITY, "workflow: more than 65535 agents");
  t->r_es = t->dalloc<double>(n);
  t->r_ee = t->dalloc<double>(n);
  if (n) {
    k_gather_rec<double><<<grid_of(n), 256, 0, st>>>(n, t->rec_line, t->es, t->r_es);
    k_gather_rec<double><<<grid_of(n), 256, 0, st>>>(n, t->rec_line, t->ee, t->r_ee);
    KX_CHECK_LAUNCH();
  }
  // instance order: stable sorts by exec_end, agent, exec_start, msg
  // (complete_instance's std::tie order, workflow.cpp:328-332)
  uint32_t* perm = t->dalloc<uint32_t>(n);
  uint32_t* pos = t->dalloc<uint32_t>(n);
  uint32_t* pos2 = t->dalloc<uint32_t>(n);
  uint32_t* tmp = t->dalloc<uint32_t>(n);
  uint64_t* k64 = t->dalloc<uint64_t>(n);
  uint64_t* k64b = t->dalloc<uint64_t>(n);
  std::vector<uint32_t> iota(static_cast<size_t>(n));
  std::iota(iota.begin(), iota.end(), 0u);
  if (n) KX_CUDA(cudaMemcpyAsync(perm, iota.data(), n * 4, cudaMemcpyHostToDevice, st));
  auto stable_by = [&](int which, int bits) {
    if (!n) return;
    k_gather_key<uint64_t><<<grid_of(n), 256, 0, st>>>(n, perm, which, t->r_es, t->r_ee, t->agent, t->up, t->msg,
                                                       k64);
    KX_CHECK_LAUNCH();
    bool alt = false;
    sort_pairs<uint64_t>(k64, pos, k64b, pos2, n, 0, bits, true, &alt, st);
    k_permute<<<grid_of(n), 256, 0, st>>>(n, perm, alt ? pos2 : pos, tmp);
    KX_CHECK_LAUNCH();
    std::swap(perm, tmp);
    if (alt) std::swap(k64, k64b);  // k64 holds the sorted keys
  };
  int mbits = 1;
  while ((int64_t(1) << mbits) < std::max<int64_t>(t->n_msgs, 2)) ++mbits;
  int abits = 1;
  while ((int64_t(1) << abits) < std::max<int32_t>(A + 1, 2)) ++abits;
  stable_by(0, 64);
  stable_by(1, abits);
  stable_by(2, 64);
  stable_by(3, mbits);
  // entry conflicts per instance (k64 = msg of each record in instance order)
  uint32_t* heads = t->dalloc<uint32_t>(n);
  uint32_t* n_heads = t->dalloc<uint32_t>(1);
  KX_CUDA(cudaMemsetAsync(n_heads, 0, 4, st));
  if (n) {
    k_run_heads_u64<<<grid_of(n), 256, 0, st>>>(n, k64, heads, n_heads);
    KX_CHECK_LAUNCH();
  }
  uint32_t groups = 0;
  KX_CUDA(cudaMemcpyAsync(&groups, n_heads, 4, cudaMemcpyDeviceToHost, st));
  KX_CUDA(cudaStreamSynchronize(st));
  const uint32_t dcap = static_cast<uint32_t>(std::min<int64_t>(n, int64_t(1) << 24));
  int64_t* d_msg = t->dalloc<int64_t>(dcap);
  int32_t* d_pos = t->dalloc<int32_t>(dcap);
  int32_t* d_entry = t->dalloc<int32_t>(dcap);
  int32_t* d_other = t->dalloc<int32_t>(dcap);
  uint32_t* n_diag = t->dalloc<uint32_t>(1);
  KX_CUDA(cudaMemsetAsync(n_diag, 0, 4, st));
  if (groups) {
    k_entry_conflicts<<<grid_of(groups), 256, 0, st>>>(groups, heads, n, k64, perm, t->agent, t->up, d_msg, d_pos,
                                                       d_entry, d_other, n_diag, dcap);
    KX_CHECK_LAUNCH();
  }
  // (instance, upstream) groups, instance order kept inside each
  stable_by(4, 24 + mbits);
  KX_CUDA(cudaMemsetAsync(n_heads, 0, 4, st));
  if (n) {
    k_run_heads_u64<<<grid_of(n), 256, 0, st>>>(n, k64, heads, n_heads);
    KX_CHECK_LAUNCH();
  }
  KX_CUDA(cudaMemcpyAsync(&groups, n_heads, 4, cudaMemcpyDeviceToHost, st));
  KX_CUDA(cudaStreamSynchronize(st));
  unsigned long long* tallies = t->dalloc<unsigned long long>(3 * size_t(A));
  int* bad = t->dalloc<int>(1);
  KX_CUDA(cudaMemsetAsync(tallies, 0, 3 * size_t(A) * 8, st));
  KX_CUDA(cudaMemsetAsync(bad, 0, 4, st));
  if (groups) {
    k_fanouts<<<grid_of(groups, 128), 128, 0, st>>>(groups, heads, n, k64, perm, t->agent, t->up, t->r_es, t->r_ee,
                                               tallies, bad);
    KX_CHECK_LAUNCH();
  }
  // edges: (upstream, agent) keys sorted, run heads
  uint8_t* is_entry = t->dalloc<uint8_t>(A);
  uint32_t* ekey = t->dalloc<uint32_t>(n);
  uint32_t* ekey2 = t->dalloc<uint32_t>(n);
  uint32_t* n_er = t->dalloc<uint32_t>(1);
  KX_CUDA(cudaMemsetAsync(is_entry, 0, std::max<int32_t>(A, 1), st));
  KX_CUDA(cudaMemsetAsync(n_er, 0, 4, st));
  if (n) {
    k_edge_keys<<<grid_of(n), 256, 0, st>>>(n, t->agent, t->up, A, is_entry, ekey, n_er);
    KX_CHECK_LAUNCH();
  }
  uint32_t ne = 0;
  KX_CUDA(cudaMemcpyAsync(&ne, n_er, 4, cudaMemcpyDeviceToHost, st));
  KX_CUDA(cudaStreamSynchronize(st));
  bool alt = false;
  sort_pairs<uint32_t>(ekey, pos, ekey2, pos2, ne, 0, 32, true, &alt, st);
  uint32_t* ek = alt ? ekey2 : ekey;
  KX_CUDA(cudaMemsetAsync(n_heads, 0, 4, st));
  if (ne) {
    k_run_heads_u32<<<grid_of(ne), 256, 0, st>>>(ne, ek, heads, n_heads);
    KX_CHECK_LAUNCH();
  }
  uint32_t nh = 0, nd = 0;
  int hb = 0;
  KX_CUDA(cudaMemcpyAsync(&nh, n_heads, 4, cudaMemcpyDeviceToHost, st));
  KX_CUDA(cudaMemcpyAsync(&nd, n_diag, 4, cudaMemcpyDeviceToHost, st));
  KX_CUDA(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, st));
  KX_CUDA(cudaStreamSynchronize(st));
  if (hb) throw KxError(KX_ERR_CAPACITY, "workflow: an upstream calls more than 64 downstreams in one instance");
  if (nd > dcap) throw KxError(KX_ERR_CAPACITY, "workflow: too many entry diagnostics");
  std::vector<uint32_t> hpos(nh), hkey(nh);
  if (nh) {
    tcopy(t, hpos.data(), heads, nh * 4, cudaMemcpyDeviceToHost);
    std::sort(hpos.begin(), hpos.end());
    for (uint32_t i = 0; i < nh; ++i) tcopy(t, &hkey[i], ek + hpos[i], 4, cudaMemcpyDeviceToHost);
  }
  // edges_ is a std::map keyed by (from name, to name): ranks are name order
  t->e_from.clear();
  t->e_to.clear();
  t->e_count.clear();
  for (uint32_t i = 0; i < nh; ++i) {
    const uint32_t end = i + 1 < nh ? hpos[i + 1] : ne;
    t->e_from.push_back(static_cast<int32_t>(hkey[i] / static_cast<uint32_t>(A)));
    t->e_to.push_back(static_cast<int32_t>(hkey[i] % static_cast<uint32_t>(A)));
    t->e_count.push_back(end - hpos[i]);
  }
  t->is_entry.resize(static_cast<size_t>(A));
  t->tallies.resize(3 * static_cast<size_t>(A));
  if (A) {
    tcopy(t, t->is_entry.data(), is_entry, A, cudaMemcpyDeviceToHost);
    tcopy(t, t->tallies.data(), tallies, 3 * size_t(A) * 8, cudaMemcpyDeviceToHost);
  }
  // diagnostics in ingest order: msg_id string order, then record order
  std::vector<int64_t> dm(nd);
  std::vector<int32_t> dp(nd), de(nd), dot(nd);
  if (nd) {
    tcopy(t, dm.data(), d_msg, nd * 8, cudaMemcpyDeviceToHost);
    tcopy(t, dp.data(), d_pos, nd * 4, cudaMemcpyDeviceToHost);
    tcopy(t, de.data(), d_entry, nd * 4, cudaMemcpyDeviceToHost);
    tcopy(t, dot.data(), d_other, nd * 4, cudaMemcpyDeviceToHost);
  }
  std::map<int64_t, std::string> mname;
  std::vector<uint32_t> idx(nd);
  std::iota(idx.begin(), idx.end(), 0u);
  {
    std::vector<int64_t> uniq(dm.begin(), dm.end());
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    const std::vector<std::string> names = fetch_msg_names(t, uniq);
    for (size_t i = 0; i < uniq.size(); ++i) mname[uniq[i]] = names[i];
  }
  std::sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) {
    const std::string& ma = mname[dm[a]];
    const std::string& mb = mname[dm[b]];
    if (ma != mb) return ma < mb;
    return dp[a] < dp[b];
  });
  t->d_msg.clear();
  t->d_entry.clear();
  t->d_other.clear();
  for (uint32_t i : idx) {
    t->d_msg.push_back(dm[i]);
    t->d_entry.push_back(de[i]);
    t->d_other.push_back(dot[i]);
  }
  t->built = true;
}

template <typename F>
int tguard(F&& f) {
  try {
    f();
    kx::set_last_error("");
    return KX_OK;
  } catch (const KxError& e) {
    kx::set_last_error(e.what());
    return e.code;
  } catch (const std::invalid_argument& e) {
    kx::set_last_error(e.what());
    return KX_ERR_INVALID;
  } catch (const std::bad_alloc&) {
    kx::set_last_error("out of host memory");
    return KX_ERR_CAPACITY;
  } catch (const std::exception& e) {
    kx::set_last_error(e.what());
    return KX_ERR_RUNTIME;
  }
}

}  // namespace

extern "C" {

int kx_trace_parse(const char* bytes, int64_t n_bytes, int32_t device, kx_trace** out) {
  return tguard([&] {
    if (!out || (n_bytes > 0 && !bytes) || n_bytes < 0) throw std::invalid_argument("kx_trace_parse: bad arguments");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device)
      throw KxError(KX_ERR_CUDA, "no CUDA device available (the kairos_b200 path has no CPU fallback)");
    KX_CUDA(cudaSetDevice(device));
    auto* t = new kx_trace();
    t->dev = device;
    try {
      KX_CUDA(cudaStreamCreateWithFlags(&t->st, cudaStreamNonBlocking));
      parse(t, bytes, n_bytes);
    } catch (...) {
      delete t;
      throw;
    }
    *out = t;
  });
}

void kx_trace_free(kx_trace* t) { delete t; }

int kx_trace_sizes(const kx_trace* t, int64_t* n_records, int32_t* n_agents, int64_t* n_msgs,
                   int64_t* agent_name_bytes) {
  return tguard([&] {
    if (!t) throw std::invalid_argument("null trace");
    if (n_records) *n_records = t->n;
    if (n_agents) *n_agents = static_cast<int32_t>(t->agents.size());
    if (n_msgs) *n_msgs = t->n_msgs;
    if (agent_name_bytes) {
      int64_t s = 0;
      for (const auto& a : t->agents) s += static_cast<int64_t>(a.size());
      *agent_name_bytes = s;
    }
  });
}

int kx_trace_agents(const kx_trace* t, char* names, int64_t* offsets) {
  return tguard([&] {
    if (!t) throw std::invalid_argument("null trace");
    int64_t o = 0;
    for (size_t i = 0; i < t->agents.size(); ++i) {
      if (offsets) offsets[i] = o;
      if (names) std::memcpy(names + o, t->agents[i].data(), t->agents[i].size());
      o += static_cast<int64_t>(t->agents[i].size());
    }
    if (offsets) offsets[t->agents.size()] = o;
  });
}

int kx_trace_columns(const kx_trace* t, int64_t* msg, int32_t* agent, int32_t* upstream, double* exec_start,
                     double* exec_end, int64_t* prompt_tokens, int64_t* output_tokens, double* app_start) {
  return tguard([&] {
    if (!t) throw std::invalid_argument("null trace");
    const int64_t n = t->n;
    KX_CUDA(cudaSetDevice(t->dev));
    if (!n) return;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst) tcopy(t, dst, src, bytes, cudaMemcpyDeviceToHost);
    };
    cp(msg, t->msg, n * 8);
    cp(agent, t->agent, n * 4);
    cp(upstream, t->up, n * 4);
    // per-line columns gathered into record order
    std::vector<int64_t> rl(n);
    tcopy(t, rl.data(), t->rec_line, n * 8, cudaMemcpyDeviceToHost);
    auto gather = [&](auto* dst, const auto* src) {
      if (!dst) return;
      using T = std::remove_pointer_t<decltype(dst)>;
      std::vector<T> all(static_cast<size_t>(t->n_lines));
      tcopy(t, all.data(), src, t->n_lines * sizeof(T), cudaMemcpyDeviceToHost);
      for (int64_t r = 0; r < n; ++r) dst[r] = all[rl[r]];
    };
    gather(exec_start, t->es);
    gather(exec_end, t->ee);
    gather(prompt_tokens, t->prompt);
    gather(output_tokens, t->output);
    gather(app_start, t->as);
  });
}

int kx_trace_msg_id(const kx_trace* t, int64_t msg, char* buf, int64_t cap, int64_t* len) {
  return tguard([&] {
    if (!t || msg < 0 || msg >= t->n_msgs) throw std::invalid_argument("kx_trace_msg_id: bad msg index");
    KX_CUDA(cudaSetDevice(t->dev));
    int64_t L = 0, off = 0;
    int32_t l = 0;
    uint32_t r = 0;
    tcopy(t, &r, t->msg_first_dev + msg, 4, cudaMemcpyDeviceToHost);
    tcopy(t, &L, t->rec_line + r, 8, cudaMemcpyDeviceToHost);
    tcopy(t, &off, t->off + 3 * L, 8, cudaMemcpyDeviceToHost);
    tcopy(t, &l, t->len + 3 * L, 4, cudaMemcpyDeviceToHost);
    if (len) *len = l;
    if (buf && cap >= l && l) tcopy(t, buf, t->bytes + off, l, cudaMemcpyDeviceToHost);
  });
}

int kx_trace_msg_spans(const kx_trace* t, int64_t k, const int64_t* msgs, int64_t* off_out, int32_t* len_out) {
  return tguard([&] {
    if (!t || k < 0 || (k && (!msgs || !off_out || !len_out))) throw std::invalid_argument("kx_trace_msg_spans: bad argument");
    for (int64_t i = 0; i < k; ++i)
      if (msgs[i] < 0 || msgs[i] >= t->n_msgs) throw std::invalid_argument("kx_trace_msg_spans: bad msg index");
    if (k == 0) return;
    KX_CUDA(cudaSetDevice(t->dev));
    int64_t* doff = nullptr;
    int32_t* dlen = nullptr;
    KX_CUDA(cudaMalloc(&doff, size_t(k) * 8));
    KX_CUDA(cudaMalloc(&dlen, size_t(k) * 4));
    msg_spans_dev(t, k, msgs, doff, dlen);
    tcopy(t, off_out, doff, size_t(k) * 8, cudaMemcpyDeviceToHost);
    tcopy(t, len_out, dlen, size_t(k) * 4, cudaMemcpyDeviceToHost);
    KX_CUDA(cudaFree(doff));
    KX_CUDA(cudaFree(dlen));
  });
}

int kx_trace_format(kx_trace* t, char* out, int64_t cap, int64_t* n_out) {
  return tguard([&] {
    if (!t) throw std::invalid_argument("null trace");
    KX_CUDA(cudaSetDevice(t->dev));
    cudaStream_t st = t->st;
    const int64_t n = t->n;
    int64_t* ll = t->dalloc<int64_t>(n);
    int* bad = t->dalloc<int>(1);
    KX_CUDA(cudaMemsetAsync(bad, 0, 4, st));
    if (n) {
      k_format<<<grid_of(n, 128), 128, 0, st>>>(t->bytes, n, t->rec_line, t->off, t->len, t->es, t->ee, t->as, t->prompt,
                                           t->output, 0, ll, nullptr, nullptr, bad);
      KX_CHECK_LAUNCH();
    }
    int hb = 0;
    KX_CUDA(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, st));
    int64_t body = 0;
    std::vector<int64_t> offs = host_excl(ll, n, st, &body);
    if (hb) throw KxError(KX_ERR_INVALID, "kx_trace_format: a time is not finite or beyond 1.7e29 s");
    const int64_t total = kHeaderLen + 1 + body;  // write_trace_header + records
    if (n_out) *n_out = total;
    if (!out) return;
    if (cap < total) throw std::invalid_argument("kx_trace_format: output buffer too small");
    for (auto& o : offs) o += kHeaderLen + 1;
    int64_t* doff = t->dalloc<int64_t>(n);
    char* dout = t->dalloc<char>(static_cast<size_t>(total));
    if (n) {
      KX_CUDA(cudaMemcpyAsync(doff, offs.data(), n * 8, cudaMemcpyHostToDevice, st));
      k_format<<<grid_of(n, 128), 128, 0, st>>>(t->bytes, n, t->rec_line, t->off, t->len, t->es, t->ee, t->as, t->prompt,
                                           t->output, 1, nullptr, doff, dout, bad);
      KX_CHECK_LAUNCH();
    }
    std::memcpy(out, kTraceHeader, kHeaderLen);
    out[kHeaderLen] = '\n';
    if (body) KX_CUDA(cudaMemcpyAsync(out + kHeaderLen + 1, dout + kHeaderLen + 1, body, cudaMemcpyDeviceToHost, st));
    KX_CUDA(cudaStreamSynchronize(st));
  });
}

int kx_workflow_reconstruct(kx_trace* t, kx_workflow_sizes* sizes) {
  return tguard([&] {
    if (!t) throw std::invalid_argument("null trace");
    KX_CUDA(cudaSetDevice(t->dev));
    reconstruct(t);
    if (sizes) {
      sizes->n_edges = static_cast<int64_t>(t->e_from.size());
      sizes->n_diagnostics = static_cast<int64_t>(t->d_msg.size());
      sizes->instances = t->n_msgs;
    }
  });
}

int kx_workflow_fetch(const kx_trace* t, int32_t* edge_from, int32_t* edge_to, uint64_t* edge_count,
                      uint8_t* is_entry, uint64_t* fan_parallel, uint64_t* fan_sequential, uint64_t* fan_single,
                      int64_t* diag_msg, int32_t* diag_entry, int32_t* diag_other) {
  return tguard([&] {
    if (!t || !t->built) throw std::logic_error("kx_workflow_fetch before kx_workflow_reconstruct");
    for (size_t i = 0; i < t->e_from.size(); ++i) {
      if (edge_from) edge_from[i] = t->e_from[i];
      if (edge_to) edge_to[i] = t->e_to[i];
      if (edge_count) edge_count[i] = t->e_count[i];
    }
    for (size_t a = 0; a < t->agents.size(); ++a) {
      if (is_entry) is_entry[a] = t->is_entry[a];
      if (fan_parallel) fan_parallel[a] = t->tallies[3 * a];
      if (fan_sequential) fan_sequential[a] = t->tallies[3 * a + 1];
      if (fan_single) fan_single[a] = t->tallies[3 * a + 2];
    }
    for (size_t i = 0; i < t->d_msg.size(); ++i) {
      if (diag_msg) diag_msg[i] = t->d_msg[i];
      if (diag_entry) diag_entry[i] = t->d_entry[i];
      if (diag_other) diag_other[i] = t->d_other[i];
    }
  });
}

}  // extern "C"



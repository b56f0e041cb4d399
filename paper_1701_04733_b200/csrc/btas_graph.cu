// On-device instance generator: the reference's random_graph + graph_to_matrix
// (graph_io.py:273-304, 158-165) as three HBM/ALU-bound passes over one numpy
// PCG64 stream, bit-identical to the host generator.
//
// Stream model (numpy PCG64, XSL-RR 128/64): state_{t+1} = M * state_t + inc
// (mod 2^128) and output t is xslrr(state_{t+1}).  Any position is reachable
// with <= 64 affine jumps from a 2^i table (passed as a kernel parameter), so
// every lane starts at its own position and then strides by 32 outputs with
// one 128-bit multiply-add: lane l of a warp owns outputs base + l + 32 i and a
// warp's 32 outputs of one iteration are consecutive — the ballot of a
// predicate over them is a window of the stream in order, which makes ranks
// (edge index, accepted-draw index) a popcount away.
//
//   presence  count present pairs per warp chunk (u >> 11 < ceil(p 2^53))
//   scan      one CTA: chunk counts -> int64 exclusive bases
//   draw      weight stream past the n(n-1) presence doubles: Lemire bounded
//             draws with numpy's exact rejection rule (32-bit buffered words
//             lo-then-hi, or 64-bit words), or uniform doubles; accepted draws
//             are compacted in stream order into a dense array
//   fill      read stage 1's presence ballots (one word per 32 pairs), rank
//             each present pair, write the dense row-major matrix (diagonal
//             0, absent +inf) through the same float64 -> storage conversion
//             and statistics as btas_ingest
#include <algorithm>
#include <cmath>
#include <type_traits>

#include "btas_common.cuh"
#include "btas_stats.cuh"

namespace btas {
int device_sm_count();

namespace {

constexpr int kGenWarps = 8;
constexpr int kGenThreads = kGenWarps * 32;
constexpr int kGenIters = 128;
constexpr int64_t kWarpUnits = 32 * kGenIters;          // stream outputs per warp chunk
constexpr int64_t kCtaUnits = kWarpUnits * kGenWarps;   // per CTA
constexpr int64_t kDrawSlack = 1 << 20;                  // extra draw units per window
constexpr int kScanThreads = 1024;

// 128-bit arithmetic mod 2^128 on (hi, lo) pairs
struct U128 {
  uint64_t hi, lo;
};

BTAS_HD U128 mul_add(U128 m, U128 s, U128 a) {  // m * s + a
#ifdef __CUDA_ARCH__
  const uint64_t lo = m.lo * s.lo;
  uint64_t hi = __umul64hi(m.lo, s.lo) + m.hi * s.lo + m.lo * s.hi;
#else
  const unsigned __int128 p = (unsigned __int128)m.lo * s.lo;
  const uint64_t lo = (uint64_t)p;
  uint64_t hi = (uint64_t)(p >> 64) + m.hi * s.lo + m.lo * s.hi;
#endif
  const uint64_t r = lo + a.lo;
  hi += a.hi + (r < lo ? 1 : 0);
  return {hi, r};
}

BTAS_D uint64_t xslrr(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// affine maps of 2^i PCG64 steps: state -> mul[i] * state + add[i]
struct PcgJumps {
  U128 mul[64];
  U128 add[64];
  U128 s0;
};

PcgJumps make_jumps(const btas_pcg64& g) {
  PcgJumps j;
  U128 cm = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};  // numpy PCG64 multiplier
  U128 cp = {g.inc_hi, g.inc_lo};
  const U128 zero = {0, 0};
  for (int i = 0; i < 64; ++i) {
    j.mul[i] = cm;
    j.add[i] = cp;
    // (cm + 1) * cp, cm * cm
    cp = mul_add(U128{cm.hi + (cm.lo == ~0ull ? 1 : 0), cm.lo + 1}, cp, zero);
    cm = mul_add(cm, cm, zero);
  }
  j.s0 = {g.state_hi, g.state_lo};
  return j;
}

// state whose xslrr is stream output t (0-based)
BTAS_D U128 state_at(const PcgJumps& J, uint64_t t) {
  U128 s = J.s0;
  uint64_t k = t + 1;
  for (int i = 0; k; ++i, k >>= 1)
    if (k & 1) s = mul_add(J.mul[i], s, J.add[i]);
  return s;
}

BTAS_D U128 stride32(const PcgJumps& J, U128 s) { return mul_add(J.mul[5], s, J.add[5]); }

BTAS_D int warp_excl(unsigned ballot) { return __popc(ballot & ((1u << (threadIdx.x & 31)) - 1u)); }

// per-warp and per-CTA counts of a CTA that already reduced its warps
BTAS_D void store_counts(int cnt, int32_t* warp_cnt, int32_t* cta_cnt) {
  __shared__ int s_cnt[kGenWarps];
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_cnt[warp] = cnt;
    warp_cnt[(int64_t)blockIdx.x * kGenWarps + warp] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kGenWarps; ++w) t += s_cnt[w];
    cta_cnt[blockIdx.x] = t;
  }
}

BTAS_D int64_t warp_base(const int32_t* warp_cnt, const int64_t* cta_base) {
  const int warp = threadIdx.x >> 5;
  int64_t b = cta_base[blockIdx.x];
  for (int w = 0; w < warp; ++w) b += warp_cnt[(int64_t)blockIdx.x * kGenWarps + w];
  return b;
}

// ------------------------------------------------------------------ presence
__global__ void __launch_bounds__(kGenThreads) presence_kernel(const __grid_constant__ PcgJumps J, uint64_t pairs,
                                                               uint64_t thr, int32_t* warp_cnt, int32_t* cta_cnt,
                                                               uint32_t* __restrict__ bits) {
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (uint64_t)blockIdx.x * kCtaUnits + (uint64_t)(threadIdx.x >> 5) * kWarpUnits;
  const uint64_t q0 = w0 + lane;
  int cnt = 0;
  if (w0 < pairs) {  // warp-uniform
    U128 s = state_at(J, q0);
    uint32_t mine = 0;  // lane i keeps the ballot word of iteration i (mod 32)
#pragma unroll 4
    for (int it = 0; it < kGenIters; ++it) {
      const uint64_t q = q0 + 32ull * it;
      const unsigned b = __ballot_sync(0xffffffffu, q < pairs && (xslrr(s) >> 11) < thr);
      cnt += __popc(b);
      if ((it & 31) == lane) mine = b;
      if ((it & 31) == 31) bits[w0 / 32 + (it & ~31) + lane] = mine;  // 32 words, coalesced
      s = stride32(J, s);
    }
  }
  store_counts(cnt, warp_cnt, cta_cnt);
}

// ------------------------------------------------------------------ scan
// exclusive int64 bases of int32 counts; base0 = *init (or 0); *total = sum + base0
__global__ void __launch_bounds__(kScanThreads) scan_kernel(const int32_t* __restrict__ cnt, int64_t count,
                                                            int64_t* __restrict__ base, const int64_t* init,
                                                            int64_t* total) {
  __shared__ int64_t s_sum[kScanThreads];
  __shared__ int64_t s_init;
  const int t = threadIdx.x;
  if (t == 0) s_init = init ? *init : 0;
  const int64_t seg = ceil_div(count, kScanThreads);
  const int64_t b0 = t * seg < count ? t * seg : count, b1 = b0 + seg < count ? b0 + seg : count;
  int64_t sum = 0;
  for (int64_t i = b0; i < b1; ++i) sum += cnt[i];
  s_sum[t] = sum;
  __syncthreads();
  // Hillis-Steele inclusive scan over 1024 partial sums
  for (int o = 1; o < kScanThreads; o <<= 1) {
    const int64_t v = t >= o ? s_sum[t - o] : 0;
    __syncthreads();
    s_sum[t] += v;
    __syncthreads();
  }
  int64_t run = s_init + s_sum[t] - sum;
  for (int64_t i = b0; i < b1; ++i) {
    base[i] = run;
    run += cnt[i];
  }
  if (t == kScanThreads - 1) *total = s_init + s_sum[t];
}

// ------------------------------------------------------------------ draws
enum DrawKind { kLemire32 = 0, kRaw32 = 1, kLemire64 = 2, kRaw64 = 3, kUniform = 4 };

struct DrawMode {
  int kind;
  uint64_t excl;    // range + 1 (bounded)
  uint64_t thresh;  // numpy's rejection threshold (UINT_MAX - range) % (range + 1)
  double low, scale;
};

// one 64-bit stream unit -> up to two accepted draws in stream order
struct Draws {
  bool a0, a1;
  uint64_t v0, v1;
};

BTAS_D Draws draw_unit(const DrawMode& m, uint64_t u) {
  Draws d;
  d.a1 = false;
  d.v1 = 0;
  switch (m.kind) {
    case kLemire32: {
      const uint64_t p0 = (u & 0xFFFFFFFFull) * m.excl, p1 = (u >> 32) * m.excl;
      d.a0 = (p0 & 0xFFFFFFFFull) >= m.thresh;
      d.a1 = (p1 & 0xFFFFFFFFull) >= m.thresh;
      d.v0 = p0 >> 32;
      d.v1 = p1 >> 32;
      break;
    }
    case kRaw32:
      d.a0 = d.a1 = true;
      d.v0 = u & 0xFFFFFFFFull;
      d.v1 = u >> 32;
      break;
    case kLemire64:
      d.a0 = u * m.excl >= m.thresh;
      d.v0 = __umul64hi(u, m.excl);
      break;
    case kRaw64:
      d.a0 = true;
      d.v0 = u;
      break;
    default: {  // uniform: low + scale * next_double, no contraction (numpy's C)
      const double x = __dadd_rn(m.low, __dmul_rn(m.scale, (double)(u >> 11) * 0x1.0p-53));
      d.a0 = true;
      d.v0 = (uint64_t)__double_as_longlong(x);
    }
  }
  return d;
}

template <bool kScatter, class V>
__global__ void __launch_bounds__(kGenThreads) draw_kernel(const __grid_constant__ PcgJumps J, DrawMode mode,
                                                           uint64_t first, uint64_t units, int64_t edges,
                                                           int32_t* warp_cnt, int32_t* cta_cnt,
                                                           const int64_t* cta_base, V* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t k0 = (uint64_t)blockIdx.x * kCtaUnits + (uint64_t)(threadIdx.x >> 5) * kWarpUnits + lane;
  int cnt = 0;
  int64_t rank = 0;
  if constexpr (kScatter) rank = warp_base(warp_cnt, cta_base);
  if (k0 - lane < units) {
    U128 s = state_at(J, first + k0);
#pragma unroll 2
    for (int it = 0; it < kGenIters; ++it) {
      const uint64_t k = k0 + 32ull * it;
      const bool valid = k < units;
      Draws d = draw_unit(mode, xslrr(s));
      d.a0 &= valid;
      d.a1 &= valid;
      const unsigned b0 = __ballot_sync(0xffffffffu, d.a0), b1 = __ballot_sync(0xffffffffu, d.a1);
      if constexpr (kScatter) {
        const int64_t r0 = rank + warp_excl(b0) + warp_excl(b1);
        if (d.a0 && r0 < edges) out[r0] = (V)d.v0;
        if (d.a1 && r0 + d.a0 < edges) out[r0 + d.a0] = (V)d.v1;
        rank += __popc(b0) + __popc(b1);
      } else {
        cnt += __popc(b0) + __popc(b1);
      }
      s = stride32(J, s);
    }
  }
  if constexpr (!kScatter) store_counts(cnt, warp_cnt, cta_cnt);
}

// ------------------------------------------------------------------ fill
// integer weights whose every value is representable exactly (int32:
// |w| < 2^28; float storage: |w| < 2^53): the stored value is a plain
// conversion and every statistic btas_ingest would report is zero, so the
// fast variant skips the per-element validation entirely
template <class D>
BTAS_D D store_int_weight(int64_t w) {
  if constexpr (Traits<D>::dtype == BTAS_I32) return (D)w;
  else return (D)(double)w;  // numpy astype(float64), then the storage rounding
}

template <class D, bool FAST>
__global__ void __launch_bounds__(kGenThreads) fill_kernel(int64_t n, int wmode, bool wide, int64_t low,
                                                           const void* __restrict__ draws, D* __restrict__ out,
                                                           int64_t ld, const uint32_t* __restrict__ bits,
                                                           const int32_t* __restrict__ warp_cnt,
                                                           const int64_t* __restrict__ cta_base, int64_t ctas,
                                                           btas_stats* stats) {
  using A = typename std::conditional<Traits<D>::dtype == BTAS_F32, float, double>::type;
  LocalStats<A> st;
  const D inf = Traits<D>::eps(true);
  const int lane = threadIdx.x & 31;
  const int64_t gtid = (int64_t)blockIdx.x * kGenThreads + threadIdx.x;
  if (gtid < n) {  // graph_to_matrix diagonal
    if constexpr (FAST) out[gtid * ld + gtid] = (D)0;
    else out[gtid * ld + gtid] = ingest_one<double, D, A>(0.0, inf, st);
  }
  const uint64_t pairs = (uint64_t)n * (uint64_t)(n - 1);
  const uint64_t w0 = (uint64_t)blockIdx.x * kCtaUnits + (uint64_t)(threadIdx.x >> 5) * kWarpUnits;
  if (blockIdx.x < ctas && w0 < pairs) {
    int64_t rank = warp_base(warp_cnt, cta_base);
    const int64_t row_len = n - 1;
    const uint64_t q0 = w0 + lane;
    int64_t row = (int64_t)(q0 / (uint64_t)row_len);
    int64_t j = (int64_t)(q0 - (uint64_t)row * row_len);
    const uint32_t* wb = bits + w0 / 32;
    uint32_t mine = 0;
    for (int it = 0; it < kGenIters; ++it) {
      if ((it & 31) == 0) mine = wb[it + lane];  // 32 presence words per coalesced load
      const unsigned b = __shfl_sync(0xffffffffu, mine, it & 31);
      const uint64_t q = q0 + 32ull * it;
      if (q < pairs) {
        const bool present = (b >> lane) & 1u;
        D val;
        if constexpr (FAST) {
          val = inf;
          if (present) {
            int64_t w = low;
            if (wmode == BTAS_WEIGHTS_BOUNDED) {
              const int64_t m = rank + warp_excl(b);
              w = (int64_t)((uint64_t)low + (wide ? static_cast<const uint64_t*>(draws)[m]
                                                  : (uint64_t) static_cast<const uint32_t*>(draws)[m]));
            }
            val = store_int_weight<D>(w);
          }
        } else {
          double w = INFINITY;
          if (present) {
            const int64_t m = rank + warp_excl(b);
            if (wmode == BTAS_WEIGHTS_CONST) {
              w = (double)low;
            } else if (wmode == BTAS_WEIGHTS_UNIFORM) {
              w = static_cast<const double*>(draws)[m];
            } else {
              const uint64_t v = wide ? static_cast<const uint64_t*>(draws)[m]
                                      : (uint64_t) static_cast<const uint32_t*>(draws)[m];
              w = (double)(int64_t)((uint64_t)low + v);  // numpy: off + draw, then astype(float64)
            }
          }
          val = ingest_one<double, D, A>(w, inf, st);
        }
        out[row * ld + j + (j >= row ? 1 : 0)] = val;
      }
      rank += __popc(b);
      j += 32;
      while (j >= row_len) {
        j -= row_len;
        ++row;
      }
    }
  }
  if constexpr (!FAST) commit(st, stats);
}

// ------------------------------------------------------------------ edge lists
// graph_to_matrix of an explicit edge list (graph_io.py:158-165 after the
// Graph normalisation of :64-83): +inf, diagonal 0, then min-scatter of every
// edge.  The scatter is an atomicMin on an order-preserving integer image of
// the stored value, so duplicates and self-loops resolve exactly as the
// reference's "keep the minimum" in any order.
BTAS_D uint32_t f32_key(float x) {
  const uint32_t b = __float_as_uint(x);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}
BTAS_D float key_f32(uint32_t k) { return __uint_as_float((k >> 31) ? (k & 0x7FFFFFFFu) : ~k); }

enum { kErrIndex = 0, kErrWeight = 1, kErrRange = 2, kErrWords = 3 };

template <class D>
__global__ void edges_init_kernel(D* __restrict__ out, int64_t n, int64_t ld, int64_t m, int64_t* err) {
  if (blockIdx.x == 0 && threadIdx.x < kErrWords) err[threadIdx.x] = m;  // m: no failing edge
  const int64_t total = n * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, c = i - r * n;
    D* p = out + r * ld + c;
    if constexpr (Traits<D>::dtype == BTAS_F64) {
      *reinterpret_cast<unsigned long long*>(p) = f64_key(r == c ? 0.0 : (double)INFINITY);
    } else if constexpr (Traits<D>::dtype == BTAS_F32) {
      *reinterpret_cast<uint32_t*>(p) = f32_key(r == c ? 0.0f : INFINITY);
    } else {
      *p = r == c ? 0 : kI32Inf;
    }
  }
}

template <class D>
__global__ void edges_scatter_kernel(D* __restrict__ out, int64_t n, int64_t ld, const int64_t* __restrict__ src,
                                     const int64_t* __restrict__ dst, const double* __restrict__ w, int64_t m,
                                     int64_t* err) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = src[e], b = dst[e];
    if (a < 0 || a >= n || b < 0 || b >= n) {
      atomicMin(reinterpret_cast<unsigned long long*>(err + kErrIndex), (unsigned long long)e);
      continue;
    }
    double x = w[e];
    if (!isfinite(x)) {
      atomicMin(reinterpret_cast<unsigned long long*>(err + kErrWeight), (unsigned long long)e);
      continue;
    }
    x = x + 0.0;  // -0.0 -> +0.0 (graph_io.py:78-79)
    D* p = out + a * ld + b;
    if constexpr (Traits<D>::dtype == BTAS_F64) {
      atomicMin(reinterpret_cast<unsigned long long*>(p), f64_key(x));
    } else if constexpr (Traits<D>::dtype == BTAS_F32) {
      const float f = (float)x;  // rounding is monotone: min then round == round then min
      if (isinf(f)) {
        atomicMin(reinterpret_cast<unsigned long long*>(err + kErrRange), (unsigned long long)e);
        continue;
      }
      atomicMin(reinterpret_cast<uint32_t*>(p), f32_key(f));
    } else {
      if (x != floor(x) || fabs(x) >= (double)kI32Limit) {
        atomicMin(reinterpret_cast<unsigned long long*>(err + kErrRange), (unsigned long long)e);
        continue;
      }
      atomicMin(reinterpret_cast<int*>(p), (int)x);
    }
  }
}

template <class D>
__global__ void edges_decode_kernel(D* __restrict__ out, int64_t n, int64_t ld) {
  const int64_t total = n * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, c = i - r * n;
    D* p = out + r * ld + c;
    if constexpr (Traits<D>::dtype == BTAS_F64) {
      *p = key_f64(*reinterpret_cast<unsigned long long*>(p));
    } else {
      *p = key_f32(*reinterpret_cast<uint32_t*>(p));
    }
  }
}

template <class D>
int edges_typed(int64_t n, const int64_t* src, const int64_t* dst, const double* w, int64_t m, D* out, int64_t ld,
                int64_t* err, cudaStream_t st) {
  const unsigned cap = (unsigned)device_sm_count() * 8;
  const unsigned g_nn = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n * n, 256), cap));
  edges_init_kernel<D><<<g_nn, 256, 0, st>>>(out, n, ld, m, err);
  BTAS_CUDA_CHECK_LAUNCH();
  if (m > 0) {
    const unsigned g_m = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), cap));
    edges_scatter_kernel<D><<<g_m, 256, 0, st>>>(out, n, ld, src, dst, w, m, err);
    BTAS_CUDA_CHECK_LAUNCH();
  }
  if constexpr (Traits<D>::dtype != BTAS_I32) {
    edges_decode_kernel<D><<<g_nn, 256, 0, st>>>(out, n, ld);
    BTAS_CUDA_CHECK_LAUNCH();
  }
  return BTAS_OK;
}

// ------------------------------------------------------------------ host
struct GraphWs {
  uint32_t* bits;  // presence ballots of stage 1, one word per 32 pairs
  int32_t *p_warp, *p_cta, *d_warp, *d_cta;
  int64_t *p_base, *d_base;
  int64_t p_ctas, d_ctas;
  size_t bytes;
};

GraphWs graph_ws(int64_t n, void* base) {
  GraphWs w{};
  const uint64_t pairs = (uint64_t)n * (uint64_t)(n - 1);
  w.p_ctas = ceil_div((int64_t)pairs, kCtaUnits);
  w.d_ctas = ceil_div((int64_t)pairs + kDrawSlack, kCtaUnits);
  size_t off = 0;
  char* b = static_cast<char*>(base);
  auto take = [&](size_t bytes) {
    void* p = b ? b + off : nullptr;
    off += (size_t)round_up((int64_t)bytes, 256);
    return p;
  };
  w.bits = (uint32_t*)take(sizeof(uint32_t) * std::max<int64_t>(1, w.p_ctas) * (kCtaUnits / 32));
  w.p_warp = (int32_t*)take(sizeof(int32_t) * std::max<int64_t>(1, w.p_ctas) * kGenWarps);
  w.p_cta = (int32_t*)take(sizeof(int32_t) * std::max<int64_t>(1, w.p_ctas));
  w.p_base = (int64_t*)take(sizeof(int64_t) * std::max<int64_t>(1, w.p_ctas));
  w.d_warp = (int32_t*)take(sizeof(int32_t) * w.d_ctas * kGenWarps);
  w.d_cta = (int32_t*)take(sizeof(int32_t) * w.d_ctas);
  w.d_base = (int64_t*)take(sizeof(int64_t) * w.d_ctas);
  w.bytes = off;
  return w;
}

bool graph_n_ok(int64_t n) { return n >= 1 && n <= (int64_t)1 << 31; }

}  // namespace
}  // namespace btas

using namespace btas;

extern "C" size_t btas_graph_workspace_bytes(int64_t n) {
  if (!graph_n_ok(n)) return 0;
  return graph_ws(n, nullptr).bytes;
}

extern "C" int btas_graph_presence(const btas_pcg64* rng, int64_t n, uint64_t p_threshold, void* workspace,
                                   size_t workspace_bytes, int64_t* dev_edges, btas_stream_t stream) {
  if (!rng || !graph_n_ok(n) || !workspace || !dev_edges || p_threshold > (1ull << 53)) return BTAS_ERR_INVALID;
  const GraphWs w = graph_ws(n, workspace);
  if (workspace_bytes < w.bytes) return BTAS_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t pairs = (uint64_t)n * (uint64_t)(n - 1);
  const PcgJumps J = make_jumps(*rng);
  if (w.p_ctas > 0) {
    presence_kernel<<<(unsigned)w.p_ctas, kGenThreads, 0, st>>>(J, pairs, p_threshold, w.p_warp, w.p_cta, w.bits);
    BTAS_CUDA_CHECK_LAUNCH();
  }
  scan_kernel<<<1, kScanThreads, 0, st>>>(w.p_cta, w.p_ctas, w.p_base, nullptr, dev_edges);
  BTAS_CUDA_CHECK_LAUNCH();
  return BTAS_OK;
}

extern "C" int btas_graph_draw(const btas_pcg64* rng, int64_t n, int weights_mode, uint64_t range, double low,
                               double scale, int64_t edges, uint64_t unit0, uint64_t units, void* draws,
                               void* workspace, size_t workspace_bytes, int64_t* dev_accepted,
                               btas_stream_t stream) {
  if (!rng || !graph_n_ok(n) || !workspace || !dev_accepted || edges < 0) return BTAS_ERR_INVALID;
  if (weights_mode != BTAS_WEIGHTS_BOUNDED && weights_mode != BTAS_WEIGHTS_UNIFORM) return BTAS_ERR_INVALID;
  if (weights_mode == BTAS_WEIGHTS_BOUNDED && range == 0) return BTAS_ERR_INVALID;  // CONST draws nothing
  const GraphWs w = graph_ws(n, workspace);
  if (workspace_bytes < w.bytes) return BTAS_ERR_WORKSPACE;
  const uint64_t pairs = (uint64_t)n * (uint64_t)(n - 1);
  if (units > pairs + (uint64_t)kDrawSlack) return BTAS_ERR_INVALID;
  if (units > 0 && edges > 0 && !draws) return BTAS_ERR_INVALID;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  DrawMode m{};
  m.low = low;
  m.scale = scale;
  bool wide = false;
  if (weights_mode == BTAS_WEIGHTS_UNIFORM) {
    m.kind = kUniform;
    wide = true;
  } else if (range < 0xFFFFFFFFull) {
    m.kind = kLemire32;
    m.excl = range + 1;
    m.thresh = (0xFFFFFFFFull - range) % (range + 1);
  } else if (range == 0xFFFFFFFFull) {
    m.kind = kRaw32;
  } else if (range < ~0ull) {
    m.kind = kLemire64;
    wide = true;
    m.excl = range + 1;
    m.thresh = (~0ull - range) % (range + 1);
  } else {
    m.kind = kRaw64;
    wide = true;
  }
  const PcgJumps J = make_jumps(*rng);
  const int64_t ctas = ceil_div((int64_t)units, kCtaUnits);
  const uint64_t first = pairs + unit0;  // weight stream starts after the presence doubles
  if (ctas > 0) {
    if (wide) {
      draw_kernel<false, uint64_t><<<(unsigned)ctas, kGenThreads, 0, st>>>(J, m, first, units, edges, w.d_warp,
                                                                           w.d_cta, nullptr, nullptr);
    } else {
      draw_kernel<false, uint32_t><<<(unsigned)ctas, kGenThreads, 0, st>>>(J, m, first, units, edges, w.d_warp,
                                                                           w.d_cta, nullptr, nullptr);
    }
    BTAS_CUDA_CHECK_LAUNCH();
  }
  scan_kernel<<<1, kScanThreads, 0, st>>>(w.d_cta, ctas, w.d_base, dev_accepted, dev_accepted);
  BTAS_CUDA_CHECK_LAUNCH();
  if (ctas > 0 && edges > 0) {
    if (wide) {
      draw_kernel<true, uint64_t><<<(unsigned)ctas, kGenThreads, 0, st>>>(
          J, m, first, units, edges, w.d_warp, w.d_cta, w.d_base, static_cast<uint64_t*>(draws));
    } else {
      draw_kernel<true, uint32_t><<<(unsigned)ctas, kGenThreads, 0, st>>>(
          J, m, first, units, edges, w.d_warp, w.d_cta, w.d_base, static_cast<uint32_t*>(draws));
    }
    BTAS_CUDA_CHECK_LAUNCH();
  }
  return BTAS_OK;
}

extern "C" int btas_graph_fill(int dtype, const btas_pcg64* rng, int64_t n, uint64_t p_threshold, int weights_mode,
                               uint64_t range, int64_t low, const void* draws, void* D, int64_t ld,
                               const void* workspace, size_t workspace_bytes, btas_stats* stats_dev,
                               btas_stream_t stream) {
  if (!rng || !graph_n_ok(n) || !D || ld < n || !workspace || !stats_dev || p_threshold > (1ull << 53))
    return BTAS_ERR_INVALID;
  if (weights_mode < BTAS_WEIGHTS_CONST || weights_mode > BTAS_WEIGHTS_UNIFORM) return BTAS_ERR_INVALID;
  // draws is read only for present pairs, i.e. when stage 1 counted edges
  const GraphWs w = graph_ws(n, const_cast<void*>(workspace));
  if (workspace_bytes < w.bytes) return BTAS_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool wide = weights_mode == BTAS_WEIGHTS_BOUNDED && range > 0xFFFFFFFFull;
  const int64_t grid = std::max<int64_t>(w.p_ctas, ceil_div(n, kGenThreads));
  if (grid > 0x7FFFFFFF) return BTAS_ERR_UNSUPPORTED;
  // the fast fill needs integer weights that every storage holds exactly
  const int64_t hi = weights_mode == BTAS_WEIGHTS_BOUNDED ? (int64_t)((uint64_t)low + range) : low;
  const double mag = std::max(std::fabs((double)low), std::fabs((double)hi));
  // (float storage: |w| < 2^52 so the f32 rounding cannot reach the 2^53
  // integer limit; float64: exact below 2^53)
  const double fast_limit = dtype == BTAS_I32 ? (double)kI32Limit : (dtype == BTAS_F32 ? 4503599627370496.0
                                                                                       : 9007199254740992.0);
  const bool fast = weights_mode != BTAS_WEIGHTS_UNIFORM &&
                    !(weights_mode == BTAS_WEIGHTS_BOUNDED && range > (1ull << 53)) && mag < fast_limit;
#define BTAS_FILL(T)                                                                                            \
  (fast ? (fill_kernel<T, true><<<(unsigned)grid, kGenThreads, 0, st>>>(n, weights_mode, wide, low, draws,        \
                                                                         static_cast<T*>(D), ld, w.bits, w.p_warp, \
                                                                         w.p_base, w.p_ctas, stats_dev),           \
           0)                                                                                                    \
        : (fill_kernel<T, false><<<(unsigned)grid, kGenThreads, 0, st>>>(n, weights_mode, wide, low, draws,       \
                                                                          static_cast<T*>(D), ld, w.bits,          \
                                                                          w.p_warp, w.p_base, w.p_ctas, stats_dev), \
           0))
  switch (dtype) {
    case BTAS_F32:
      (void)BTAS_FILL(float);
      break;
    case BTAS_I32:
      (void)BTAS_FILL(int32_t);
      break;
    case BTAS_F64:
      (void)BTAS_FILL(double);
      break;
    default:
      return BTAS_ERR_INVALID;
  }
#undef BTAS_FILL
  BTAS_CUDA_CHECK_LAUNCH();
  return BTAS_OK;
}

extern "C" int btas_edges_to_matrix(int dtype, int64_t n, const int64_t* src, const int64_t* dst, const double* weight,
                                    int64_t m, void* D, int64_t ld, int64_t* dev_errors, btas_stream_t stream) {
  if (n < 1 || m < 0 || !D || ld < n || !dev_errors || (m > 0 && (!src || !dst || !weight))) return BTAS_ERR_INVALID;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (dtype) {
    case BTAS_F32:
      return edges_typed<float>(n, src, dst, weight, m, static_cast<float*>(D), ld, dev_errors, st);
    case BTAS_I32:
      return edges_typed<int32_t>(n, src, dst, weight, m, static_cast<int32_t*>(D), ld, dev_errors, st);
    case BTAS_F64:
      return edges_typed<double>(n, src, dst, weight, m, static_cast<double*>(D), ld, dev_errors, st);
    default:
      return BTAS_ERR_INVALID;
  }
}

// HBM-bound kernels of the hot path: ingest/validation, order-statistics
// scans, fills, the closure base, elementwise ⊕ and the batched matvec.
// All are grid-stride, 16-byte vectorised where alignment allows, and sized
// to a multiple of the SM count.
#include <algorithm>
#include <cfloat>
#include <cuda.h>
#include <type_traits>

#include "btas_common.cuh"
#include "btas_stats.cuh"

namespace btas {
int device_sm_count();

namespace {

inline unsigned grid_for(int64_t work, int threads = 256) {
  const int64_t blocks = ceil_div(work, threads);
  const int64_t cap = (int64_t)device_sm_count() * 8;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, cap));
}

__global__ void stats_init_kernel(btas_stats* s) {
  s->nan_count = s->neg_inf_count = s->non_integral = s->over_limit = s->out_of_range = s->finite_count = 0;
  s->max_abs_key = kKeyNone;
  s->min_key = kKeyNoneMin;
  s->max_key = kKeyNone;
}

template <class S, class D>
__global__ void ingest_kernel(bool min_plus, const S* __restrict__ src, int64_t n, D* __restrict__ dst,
                              btas_stats* stats) {
  // statistics arithmetic: float whenever the data is float32 on either side
  using A = typename std::conditional<sizeof(S) == 4 || Traits<D>::dtype == BTAS_F32, float, double>::type;
  LocalStats<A> st;
  const D inf = Traits<D>::eps(min_plus);
  // 4 independent elements per thread per trip: 4 loads in flight per thread
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i0 + 3 * stride < n; i0 += 4 * stride) {
    S xs[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) xs[u] = src[i0 + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u) dst[i0 + u * stride] = ingest_one<S, D, A>(xs[u], inf, st);
  }
  for (int64_t i = i0; i < n; i += stride) dst[i] = ingest_one<S, D, A>(src[i], inf, st);
  commit(st, stats);
}

// ------------------------------------------------------------------ scan
template <class T>
__global__ void scan_kernel(const T* __restrict__ x, int64_t n, btas_stats* stats) {
  // int32 magnitudes up to 2^28 need double to stay exact; f32 stays float
  LocalStats<typename std::conditional<Traits<T>::dtype == BTAS_F32, float, double>::type> st;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T v = x[i];
    if constexpr (Traits<T>::dtype != BTAS_I32) {
      if (v != v) {
        st.nan++;
        continue;
      }
    }
    if (Traits<T>::finite(v)) st.add_finite(v, Traits<T>::int_limit);
  }
  commit(st, stats);
}

template <class T>
__global__ void to_f64_kernel(const T* __restrict__ x, int64_t n, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = Traits<T>::to_f64(x[i]);
}

template <class T>
__global__ void fill_kernel(T* __restrict__ x, int64_t n, T v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = v;
}

template <class T>
__global__ void identity_kernel(T* __restrict__ d, int64_t ld, int64_t n, T inf) {
  const int64_t total = n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    d[i * ld + j] = (i == j) ? (T)0 : inf;
  }
}

template <class T>
__global__ void closure_base_kernel(const T* __restrict__ s, int64_t lds, T* __restrict__ d, int64_t ldd, int64_t n) {
  const int64_t total = n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    T v = s[i * lds + j];
    if (i == j && v > (T)0) v = (T)0;  // np.minimum(diag, 0.0) (apsp.py:88)
    d[i * ldd + j] = v;
  }
}

// elementwise ⊕, 16-byte vectors for the aligned body
template <class T, bool MIN>
__global__ void ewadd_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ o, int64_t n) {
  constexpr int V = 16 / sizeof(T);
  const bool aligned = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                         reinterpret_cast<uintptr_t>(o)) & 15) == 0;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t body = 0;
  if (aligned) {
    body = (n / V) * V;
    const uint4* av = reinterpret_cast<const uint4*>(a);
    const uint4* bv = reinterpret_cast<const uint4*>(b);
    uint4* ov = reinterpret_cast<uint4*>(o);
    auto op = [](uint4 x, uint4 y) {
      uint4 z;
      const T* xs = reinterpret_cast<const T*>(&x);
      const T* ys = reinterpret_cast<const T*>(&y);
      T* zs = reinterpret_cast<T*>(&z);
#pragma unroll
      for (int v = 0; v < V; ++v) zs[v] = MIN ? (ys[v] < xs[v] ? ys[v] : xs[v]) : (ys[v] > xs[v] ? ys[v] : xs[v]);
      return z;
    };
    // two independent vectors per operand in flight per trip, streamed
    // (evict-first) — each byte is touched once
    const int64_t nv = n / V;
    int64_t i = tid;
    for (; i + stride < nv; i += 2 * stride) {
      const uint4 x0 = __ldcs(av + i), y0 = __ldcs(bv + i), x1 = __ldcs(av + i + stride), y1 = __ldcs(bv + i + stride);
      __stcs(ov + i, op(x0, y0));
      __stcs(ov + i + stride, op(x1, y1));
    }
    for (; i < nv; i += stride) __stcs(ov + i, op(__ldcs(av + i), __ldcs(bv + i)));
  }
  for (int64_t i = body + tid; i < n; i += stride) {
    const T x = a[i], y = b[i];
    o[i] = MIN ? (y < x ? y : x) : (y > x ? y : x);
  }
}

template <class T>
__global__ void diag_neg_kernel(const T* __restrict__ d, int64_t ld, int64_t n, int32_t* flags) {
  bool neg = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    neg |= d[i * ld + i] < (T)0;
  if (__any_sync(0xffffffffu, neg) && (threadIdx.x & 31) == 0) atomicOr(&flags[BTAS_FLAG_DIAG_NEG], 1);
}

// ------------------------------------------------------------------ matvec
// Out[b, i] = ⊕_k A[i, k] ⊗ V[b, k].  R rows per CTA, NB vectors per pass.
// The reference always masks overflow here (matrix.py:408-420): a finite ⊗
// finite candidate that overflows (float) or reaches the integer limit
// becomes ε and sets the flag.  The kernel streams A once with plain add +
// min/max (VIADDMNMX for int32) while tracking max|finite| of the A rows and
// of V; only if that exact screen says some candidate could overflow does
// the CTA redo its rows with the per-candidate mask (same result bytes as
// masking everything, at the cost of the screen: one FMNMX per element).
template <class T>
BTAS_D T abs_finite(T x) {
  if constexpr (Traits<T>::dtype == BTAS_I32) {
    const T a = x < 0 ? -x : x;
    return a < (T)kI32Limit ? a : (T)0;
  } else {
    const T a = fabs(x);
    return a < (T)INFINITY ? a : (T)0;
  }
}

template <class T, bool MIN, bool CHECKED>
BTAS_D void mv_acc(T& acc, T a, T v, int int_mode, double limit, bool& sat) {
  if constexpr (!CHECKED) {
    if constexpr (Traits<T>::dtype == BTAS_I32) {
      acc = MIN ? __viaddmin_s32(a, v, acc) : __viaddmax_s32(a, v, acc);
    } else {
      const T s = a + v;
      acc = MIN ? (s < acc ? s : acc) : (s > acc ? s : acc);
    }
  } else {
    T s = a + v;
    bool over;
    if constexpr (Traits<T>::dtype == BTAS_I32) over = (s >= (T)kI32Limit) || (s <= -(T)kI32Limit);
    else over = int_mode ? (fabs(s) >= (T)limit) : isinf(s);
    if (over && Traits<T>::finite(a) && Traits<T>::finite(v)) {
      sat = true;
      s = Traits<T>::eps(MIN);
    }
    acc = MIN ? (s < acc ? s : acc) : (s > acc ? s : acc);
  }
}

// one pass over the CTA's R rows; returns the thread's max|finite| of A and V
// (tracked only when SCREEN: a caller-proven bound makes the screen moot)
template <class T, bool MIN, int R, int NB, bool CHECKED, bool SCREEN = true>
BTAS_D void mv_pass(const T* __restrict__ A, int64_t lda, int64_t M, int64_t K, const T* __restrict__ Vv,
                    int64_t ldv, int nb, int64_t r0, int64_t kvec_end, int int_mode, double limit,
                    T (&acc)[R][NB], T& amax, T& vmax, bool& sat) {
  constexpr int VEC = 16 / sizeof(T);
  for (int64_t k = (int64_t)threadIdx.x * VEC; k < kvec_end; k += (int64_t)blockDim.x * VEC) {
    T vv[NB][VEC];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      if (b < nb) {
        const uint4 u = *reinterpret_cast<const uint4*>(Vv + (int64_t)b * ldv + k);
        const T* p = reinterpret_cast<const T*>(&u);
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          vv[b][e] = p[e];
          if (!CHECKED && SCREEN) vmax = max(vmax, abs_finite(p[e]));
        }
      }
    }
    uint4 au[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t row = r0 + r < M ? r0 + r : M - 1;
      au[r] = __ldcs(reinterpret_cast<const uint4*>(A + row * lda + k));  // streamed once: evict-first
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const T* ap = reinterpret_cast<const T*>(&au[r]);
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (!CHECKED && SCREEN) amax = max(amax, abs_finite(ap[e]));
      if constexpr (!CHECKED && Traits<T>::dtype == BTAS_F32) {
        // f32: FADD2 over a pair of k, then one FMNMX3 into the accumulator
#pragma unroll
        for (int e = 0; e < VEC; e += 2)
#pragma unroll
          for (int b = 0; b < NB; ++b)
            if (b < nb) {
              const float2 s2 = __fadd2_rn(make_float2(ap[e], ap[e + 1]), make_float2(vv[b][e], vv[b][e + 1]));
              acc[r][b] = MIN ? fminf(fminf(acc[r][b], s2.x), s2.y) : fmaxf(fmaxf(acc[r][b], s2.x), s2.y);
            }
      } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e)
#pragma unroll
          for (int b = 0; b < NB; ++b)
            if (b < nb) mv_acc<T, MIN, CHECKED>(acc[r][b], ap[e], vv[b][e], int_mode, limit, sat);
      }
    }
  }
  for (int64_t k = kvec_end + threadIdx.x; k < K; k += blockDim.x) {
#pragma unroll
    for (int b = 0; b < NB; ++b)
      if (b < nb && !CHECKED && SCREEN) vmax = max(vmax, abs_finite(Vv[(int64_t)b * ldv + k]));
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t row = r0 + r < M ? r0 + r : M - 1;
      const T a = A[row * lda + k];
      if (!CHECKED && SCREEN) amax = max(amax, abs_finite(a));
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (b < nb) mv_acc<T, MIN, CHECKED>(acc[r][b], a, Vv[(int64_t)b * ldv + k], int_mode, limit, sat);
    }
  }
}

template <class T>
BTAS_D T block_max(T v, T* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
  __syncthreads();
  T m = scratch[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = scratch[w] > m ? scratch[w] : m;
  return m;
}

// SCREEN = false: the caller proved max|finite A| + max|finite V| below the
// overflow limit (btas_matvec_bounded), so no candidate can overflow and the
// magnitude tracking and the masked rerun are compiled out.
template <class T, bool MIN, int R, int NB, bool SCREEN = true>
__global__ void __launch_bounds__(256) matvec_kernel(const T* __restrict__ A, int64_t lda, int64_t M, int64_t K,
                                                     const T* __restrict__ Vv, int64_t ldv, int nb,
                                                     T* __restrict__ Out, int64_t ldo, int int_mode, double limit,
                                                     int32_t* flags) {
  constexpr int VEC = 16 / sizeof(T);
  const int64_t r0 = (int64_t)blockIdx.x * R;
  const T eps = Traits<T>::eps(MIN);
  T acc[R][NB];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[r][b] = eps;
  bool sat = false;
  const bool vec_ok = ((lda % VEC) == 0) && ((ldv % VEC) == 0) &&
                      ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(Vv)) & 15) == 0;
  const int64_t kvec_end = vec_ok ? (K / VEC) * VEC : 0;
  T amax = 0, vmax = 0;
  mv_pass<T, MIN, R, NB, false, SCREEN>(A, lda, M, K, Vv, ldv, nb, r0, kvec_end, int_mode, limit, acc, amax, vmax,
                                        sat);
  bool possible = false;
  if constexpr (SCREEN) {
    // exact screen: |a + v| <= amax + vmax for every finite pair of this CTA
    __shared__ T scratch[8];
    amax = block_max(amax, scratch);
    vmax = block_max(vmax, scratch);
    if constexpr (Traits<T>::dtype == BTAS_I32) {
      possible = (int64_t)amax + (int64_t)vmax >= (int64_t)kI32Limit;
    } else {
      const T bound = amax + vmax;  // storage arithmetic, rounding is monotone
      possible = int_mode ? ((double)bound >= limit) : isinf(bound);
    }
  }
  if (possible) {  // uniform across the CTA
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int b = 0; b < NB; ++b) acc[r][b] = eps;
    mv_pass<T, MIN, R, NB, true>(A, lda, M, K, Vv, ldv, nb, r0, kvec_end, int_mode, limit, acc, amax, vmax, sat);
  }
  // block reduction of R*NB values
  __shared__ T red[8][R * NB];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      T v = acc[r][b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const T u = __shfl_xor_sync(0xffffffffu, v, o);
        v = MIN ? (u < v ? u : v) : (u > v ? u : v);
      }
      if (l == 0) red[w][r * NB + b] = v;
    }
  __syncthreads();
  if (threadIdx.x < R * NB) {
    const int r = threadIdx.x / NB, b = threadIdx.x % NB;
    T v = red[0][threadIdx.x];
    for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww) {
      const T u = red[ww][threadIdx.x];
      v = MIN ? (u < v ? u : v) : (u > v ? u : v);
    }
    if constexpr (Traits<T>::dtype == BTAS_I32) {
      if (MIN ? v >= (T)kI32Limit : v <= -(T)kI32Limit) v = eps;
    }
    if (r0 + r < M && b < nb) Out[(int64_t)b * ldo + r0 + r] = v;
  }
  if (__any_sync(0xffffffffu, sat) && l == 0) atomicOr(&flags[BTAS_FLAG_SATURATED], 1);
}

// ---- many vectors (5-8) of 4-byte storage: one pass over A -----------------
// With 8 vectors every A element feeds 8 add-min pairs, so the pass is only
// HBM-bound if A streams with enough bytes in flight AND the vectors are not
// re-read from L2 for every few rows.  CTA = 32 rows (warp w: rows 4w..4w+3),
// two CTAs per SM.  Per 256-column chunk one producer thread issues two 2-D
// tensor-map TMA copies (the 32 x 256 A tile and the 8 x 256 vector tile)
// into a 2-stage shared-memory ring (40 KB per stage) with full/empty
// mbarriers, so the next chunk is in flight while the warps compute,
// without registers or issue slots spent on the loads.  The
// finite-magnitude screen costs two integer ops per element (abs_key).  The
// exact overflow screen is the one of matvec_kernel; a CTA whose screen
// fails recomputes its rows with the masked candidates.
constexpr int kWideRows = 32, kWideChunk = 256, kWideNB = 8, kWideThreads = 256, kWideStages = 2;
// one stage: the CTA's 32 x 128 tile of A, then the 8 x 128 vector tile
static_assert(kWideChunk % 128 == 0 && kWideChunk <= 256, "a warp covers 128 columns per step; TMA box <= 256");
constexpr int kWideStageElems = (kWideRows + kWideNB) * kWideChunk;
constexpr uint32_t kWideStageBytes = kWideStageElems * 4;
constexpr size_t kWideSmem = (size_t)kWideStages * kWideStageBytes + 2 * kWideStages * sizeof(uint64_t);

BTAS_D void tma_2d(void* smem_dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// max |finite| bookkeeping in one or two integer ops per element: the
// tracked key is monotone in |x| for finite x and negative for the stored
// Infinity, so a signed max ignores it.  f32: (|x| bits) + 2^23 (inf bits
// become 0x80000000); i32: |x| << 2 (the int32 Inf encoding wraps negative).
template <class T>
BTAS_D int32_t abs_key(T x) {
  if constexpr (Traits<T>::dtype == BTAS_F32) return (int32_t)((__float_as_uint(x) & 0x7FFFFFFFu) + 0x00800000u);
  else return (int32_t)((uint32_t)abs(x) << 2);
}
template <class T>
BTAS_D T key_abs(int32_t k) {
  if constexpr (Traits<T>::dtype == BTAS_F32) return k <= 0 ? 0.0f : __uint_as_float((uint32_t)k - 0x00800000u);
  else return (T)(k >> 2);
}

template <class T, bool MIN, bool SCREEN = true>
__global__ void __launch_bounds__(kWideThreads, 2) matvec_wide_kernel(const __grid_constant__ CUtensorMap mapA,
                                                                   const __grid_constant__ CUtensorMap mapV,
                                                                   const T* __restrict__ A, int64_t lda, int64_t M,
                                                                   int64_t K, const T* __restrict__ Vv, int64_t ldv,
                                                                   int nb, T* __restrict__ Out, int64_t ldo,
                                                                   int int_mode, double limit, int32_t* flags) {
  static_assert(sizeof(T) == 4, "4-byte storage");
  extern __shared__ __align__(128) unsigned char wide_smem[];
  T* stages = reinterpret_cast<T*>(wide_smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(wide_smem + (size_t)kWideStages * kWideStageBytes);
  uint64_t* empty = full + kWideStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * kWideRows;
  const T eps = Traits<T>::eps(MIN);
  const int64_t nchunks = K / kWideChunk;  // the caller guarantees K % kWideChunk == 0
  if (threadIdx.x == 0) {
    for (int st = 0; st < kWideStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kWideThreads / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // thread 0 is the producer: two tensor-map copies per stage (rows past M
  // and vectors past nb arrive zero-filled; their results are never stored)
  auto issue = [&](int64_t c) {
    const int st = (int)(c % kWideStages);
    T* dst = stages + (size_t)st * kWideStageElems;
    mbar_arrive_expect_tx(&full[st], kWideStageBytes);
    tma_2d(dst, &mapA, (int)(c * kWideChunk), (int)r0, &full[st]);
    tma_2d(dst + kWideRows * kWideChunk, &mapV, (int)(c * kWideChunk), 0, &full[st]);
  };
  if (threadIdx.x == 0)
    for (int64_t c = 0; c < nchunks && c < kWideStages; ++c) issue(c);
  T acc[4][kWideNB];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int b = 0; b < kWideNB; ++b) acc[r][b] = eps;
  int32_t akey = 0, vkey = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int st = (int)(c % kWideStages);
    const uint32_t use = (uint32_t)((c / kWideStages) & 1);
    mbar_wait(&full[st], use);
    const T* src = stages + (size_t)st * kWideStageElems;
#pragma unroll
    for (int j = 0; j < kWideChunk / 128; ++j) {
      const int col = j * 128 + lane * 4;
      T v[kWideNB][4];
#pragma unroll
      for (int b = 0; b < kWideNB; ++b) {
        const uint4 u = *reinterpret_cast<const uint4*>(&src[(kWideRows + b) * kWideChunk + col]);
        v[b][0] = __builtin_bit_cast(T, u.x);
        v[b][1] = __builtin_bit_cast(T, u.y);
        v[b][2] = __builtin_bit_cast(T, u.z);
        v[b][3] = __builtin_bit_cast(T, u.w);
        if (SCREEN && warp == 0 && b < nb) {
#pragma unroll
          for (int e = 0; e < 4; ++e) vkey = max(vkey, abs_key(v[b][e]));
        }
      }
      uint4 au[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) au[r] = *reinterpret_cast<const uint4*>(&src[(warp * 4 + r) * kWideChunk + col]);
      if (j == kWideChunk / 128 - 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);  // this warp's reads of the stage are done
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const T a[4] = {__builtin_bit_cast(T, au[r].x), __builtin_bit_cast(T, au[r].y), __builtin_bit_cast(T, au[r].z),
                        __builtin_bit_cast(T, au[r].w)};
        if constexpr (SCREEN)
          akey = max(akey, max(max(abs_key(a[0]), abs_key(a[1])), max(abs_key(a[2]), abs_key(a[3]))));
#pragma unroll
        for (int b = 0; b < kWideNB; ++b) {
          if constexpr (Traits<T>::dtype == BTAS_F32) {
#pragma unroll
            for (int e = 0; e < 4; e += 2) {
              const float2 s2 = __fadd2_rn(make_float2(a[e], a[e + 1]), make_float2(v[b][e], v[b][e + 1]));
              acc[r][b] = MIN ? fminf(fminf(acc[r][b], s2.x), s2.y) : fmaxf(fmaxf(acc[r][b], s2.x), s2.y);
            }
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              acc[r][b] = MIN ? __viaddmin_s32(a[e], v[b][e], acc[r][b]) : __viaddmax_s32(a[e], v[b][e], acc[r][b]);
          }
        }
      }
    }
    if (threadIdx.x == 0 && c + kWideStages < nchunks) {
      mbar_wait(&empty[st], use);  // every warp has read stage st: refill it
      issue(c + kWideStages);
    }
  }
  bool possible = false;
  if constexpr (SCREEN) {
    T amax = key_abs<T>(akey), vmax = key_abs<T>(vkey);
    // exact screen over the CTA (see matvec_kernel)
    __shared__ T scratch[kWideThreads / 32];
    amax = block_max(amax, scratch);
    vmax = block_max(vmax, scratch);
    if constexpr (Traits<T>::dtype == BTAS_I32) {
      possible = (int64_t)amax + (int64_t)vmax >= (int64_t)kI32Limit;
    } else {
      const T bound = amax + vmax;
      possible = int_mode ? ((double)bound >= limit) : isinf(bound);
    }
  }
  if (!possible) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t row = r0 + warp * 4 + r;
#pragma unroll
      for (int b = 0; b < kWideNB; ++b) {
        T v = acc[r][b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const T u = __shfl_xor_sync(0xffffffffu, v, o);
          v = MIN ? (u < v ? u : v) : (u > v ? u : v);
        }
        if constexpr (Traits<T>::dtype == BTAS_I32) {
          if (MIN ? v >= (T)kI32Limit : v <= -(T)kI32Limit) v = eps;
        }
        if (lane == 0 && row < M && b < nb) Out[(int64_t)b * ldo + row] = v;
      }
    }
    return;
  }
  // rare: masked candidates, 4 rows at a time with the whole CTA over k
  bool sat = false;
  __shared__ T red[kWideThreads / 32][4 * kWideNB];
  for (int g = 0; g < kWideRows / 4; ++g) {
    const int64_t rg = r0 + g * 4;
    if (rg >= M) break;
    T acc4[4][kWideNB];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int b = 0; b < kWideNB; ++b) acc4[r][b] = eps;
    T am = 0, vm = 0;
    mv_pass<T, MIN, 4, kWideNB, true>(A, lda, M, K, Vv, ldv, nb, rg, (K / 4) * 4, int_mode, limit, acc4, am, vm,
                                       sat);
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int b = 0; b < kWideNB; ++b) {
        T v = acc4[r][b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const T u = __shfl_xor_sync(0xffffffffu, v, o);
          v = MIN ? (u < v ? u : v) : (u > v ? u : v);
        }
        if (lane == 0) red[warp][r * kWideNB + b] = v;
      }
    __syncthreads();
    if (threadIdx.x < 4 * kWideNB) {
      const int r = threadIdx.x / kWideNB, b = threadIdx.x % kWideNB;
      T v = red[0][threadIdx.x];
      for (int ww = 1; ww < kWideThreads / 32; ++ww) {
        const T u = red[ww][threadIdx.x];
        v = MIN ? (u < v ? u : v) : (u > v ? u : v);
      }
      if constexpr (Traits<T>::dtype == BTAS_I32) {
        if (MIN ? v >= (T)kI32Limit : v <= -(T)kI32Limit) v = eps;
      }
      if (rg + r < M && b < nb) Out[(int64_t)b * ldo + rg + r] = v;
    }
    __syncthreads();
  }
  if (__any_sync(0xffffffffu, sat) && lane == 0) atomicOr(&flags[BTAS_FLAG_SATURATED], 1);
}

// 2-D tensor maps for matvec_wide_kernel (cuTensorMapEncodeTiled through the
// runtime's driver entry point: no link-time libcuda dependency)
using TensorMapEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline TensorMapEncodeFn tensor_map_encoder() {
  static const TensorMapEncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      (void)cudaGetLastError();
      p = nullptr;
    }
    return reinterpret_cast<TensorMapEncodeFn>(p);
  }();
  return fn;
}
// rows x cols row-major 4-byte matrix with leading dimension ld; box of
// kWideChunk columns x box_rows rows; out-of-range rows read as zero
inline bool wide_tensor_map(CUtensorMap* m, bool f32, const void* base, int64_t rows, int64_t cols, int64_t ld,
                            int box_rows) {
  const TensorMapEncodeFn enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {(cuuint32_t)kWideChunk, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_INT32, 2, const_cast<void*>(base), dims,
             strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// true when a caller bound B >= max|finite A| + max|finite V| proves that no
// finite (x) finite candidate overflows: |a + v| <= B below the integer limit
// (integer mode, int32) or below the largest finite value of the storage
// (a sum of magnitude below it rounds to a finite value)
template <class T>
bool bound_proves_no_overflow(double abs_bound, int int_mode) {
  if (!(abs_bound >= 0.0)) return false;  // unknown (negative or NaN)
  if constexpr (Traits<T>::dtype == BTAS_I32) return abs_bound < (double)kI32Limit;
  if (int_mode) return abs_bound < Traits<T>::int_limit;
  return abs_bound < (double)(Traits<T>::dtype == BTAS_F32 ? FLT_MAX : DBL_MAX);
}

template <class T, bool MIN, bool SCREEN>
int matvec_launch(int int_mode, const T* A, int64_t lda, int64_t M, int64_t K, const T* V, int64_t ldv,
                  int64_t batch, T* Out, int64_t ldo, int32_t* flags, cudaStream_t st) {
  const double limit = Traits<T>::dtype == BTAS_I32 ? (double)kI32Limit : Traits<T>::int_limit;
  // 5-8 vectors of 4-byte storage: one pass (matvec_wide_kernel) when the
  // shapes allow 16-byte chunked streaming; otherwise up to 4 vectors per
  // pass (8 vectors through the register-only kernel ran at 2.1 TB/s)
  const bool wide_ok = sizeof(T) == 4 && K % kWideChunk == 0 && lda % 4 == 0 && ldv % 4 == 0 &&
                       ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(V)) & 15) == 0;
  for (int64_t b0 = 0; b0 < batch;) {
    const int64_t left = batch - b0;
    // 5-8 vectors always; 3-4 vectors too when the bound removed the screen
    // (the screen-free wide kernel beats the narrow one there, 6.6 vs 6.2
    // TB/s at 4 vectors; with the screen it does not, tools/matvec_ab.py)
    const bool use_wide = sizeof(T) == 4 && wide_ok && (left > 4 || (!SCREEN && left > 2));
    const int nb = (int)std::min<int64_t>(use_wide ? kWideNB : 4, left);
    const T* Vb = V + b0 * ldv;
    T* Ob = Out + b0 * ldo;
    b0 += nb;
    if constexpr (sizeof(T) == 4) {
      if (use_wide) {
        CUtensorMap mapA, mapV;
        if (!wide_tensor_map(&mapA, Traits<T>::dtype == BTAS_F32, A, M, K, lda, kWideRows) ||
            !wide_tensor_map(&mapV, Traits<T>::dtype == BTAS_F32, Vb, nb, K, ldv, kWideNB))
          return BTAS_ERR_CUDA;
        static unsigned long long configured = 0;
        if (!configured_on_current_device(configured)) {
          if (cudaFuncSetAttribute(matvec_wide_kernel<T, MIN, SCREEN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kWideSmem) != cudaSuccess) {
            (void)cudaGetLastError();
            return BTAS_ERR_CUDA;
          }
          mark_configured(configured);
        }
        matvec_wide_kernel<T, MIN, SCREEN><<<(unsigned)ceil_div(M, kWideRows), kWideThreads, kWideSmem, st>>>(
            mapA, mapV, A, lda, M, K, Vb, ldv, nb, Ob, ldo, int_mode, limit, flags);
        BTAS_CUDA_CHECK_LAUNCH();
        continue;
      }
    }
    // 1-4 vectors: the screened kernel even when a bound proves the screen
    // moot — ptxas schedules the screen-free instantiation with fewer loads
    // in flight (measured 4.6 vs 6.4 TB/s at 4 vectors, tools/matvec_ab.py);
    // at <= 4 add-min pairs per A element the screen is free anyway
    if (nb == 1) {
      matvec_kernel<T, MIN, 16, 1, true><<<(unsigned)ceil_div(M, 16), 256, 0, st>>>(A, lda, M, K, Vb, ldv, nb, Ob, ldo,
                                                                            int_mode, limit, flags);
    } else if (nb <= 2) {
      matvec_kernel<T, MIN, 8, 2, true><<<(unsigned)ceil_div(M, 8), 256, 0, st>>>(A, lda, M, K, Vb, ldv, nb, Ob, ldo,
                                                                          int_mode, limit, flags);
    } else if (nb <= 4) {
      matvec_kernel<T, MIN, 8, 4, true><<<(unsigned)ceil_div(M, 8), 256, 0, st>>>(A, lda, M, K, Vb, ldv, nb, Ob, ldo,
                                                                          int_mode, limit, flags);
    }
    BTAS_CUDA_CHECK_LAUNCH();
  }
  return BTAS_OK;
}

template <class T, bool MIN>
int matvec_typed(int int_mode, double abs_bound, const T* A, int64_t lda, int64_t M, int64_t K, const T* V,
                 int64_t ldv, int64_t batch, T* Out, int64_t ldo, int32_t* flags, cudaStream_t st) {
  return bound_proves_no_overflow<T>(abs_bound, int_mode)
             ? matvec_launch<T, MIN, false>(int_mode, A, lda, M, K, V, ldv, batch, Out, ldo, flags, st)
             : matvec_launch<T, MIN, true>(int_mode, A, lda, M, K, V, ldv, batch, Out, ldo, flags, st);
}

inline bool valid_dtype(int d) { return d == BTAS_F32 || d == BTAS_I32 || d == BTAS_F64; }
inline bool valid_kind(int k) { return k == BTAS_MIN_PLUS || k == BTAS_MAX_PLUS; }

}  // namespace
}  // namespace btas

using namespace btas;

#define BTAS_DISPATCH(dtype, ...)                          \
  switch (dtype) {                                         \
    case BTAS_F32: {                                       \
      using T = float;                                     \
      __VA_ARGS__;                                         \
      break;                                               \
    }                                                      \
    case BTAS_I32: {                                       \
      using T = int32_t;                                   \
      __VA_ARGS__;                                         \
      break;                                               \
    }                                                      \
    case BTAS_F64: {                                       \
      using T = double;                                    \
      __VA_ARGS__;                                         \
      break;                                               \
    }                                                      \
    default:                                               \
      return BTAS_ERR_INVALID;                             \
  }

extern "C" const char* btas_version(void) { return "btas-b200 0.1.0 (sm_100a)"; }

extern "C" const char* btas_status_string(int status) {
  switch (status) {
    case BTAS_OK:
      return "ok";
    case BTAS_ERR_INVALID:
      return "invalid argument";
    case BTAS_ERR_CUDA: {
      return "CUDA error";
    }
    case BTAS_ERR_WORKSPACE:
      return "workspace too small";
    case BTAS_ERR_UNSUPPORTED:
      return "unsupported combination";
    default:
      return "unknown status";
  }
}

extern "C" double btas_key_to_double(unsigned long long key) {
  if (key == kKeyNone || key == kKeyNoneMin) return NAN;
  return key_f64(key);
}

namespace btas {
namespace {
__global__ void export_words_kernel(const uint32_t* __restrict__ src, volatile uint32_t* dst, int64_t words) {
  for (int64_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
}
}  // namespace
}  // namespace btas

extern "C" int btas_export_words(const void* src, void* dst, int64_t words, btas_stream_t stream) {
  if (!src || !dst || words < 0 || words > 4096) return BTAS_ERR_INVALID;
  if (words == 0) return BTAS_OK;
  btas::export_words_kernel<<<1, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint32_t*>(src), static_cast<volatile uint32_t*>(dst), words);
  BTAS_CUDA_CHECK_LAUNCH();
  return BTAS_OK;
}

extern "C" int btas_stats_init(btas_stats* s, btas_stream_t stream) {
  if (!s) return BTAS_ERR_INVALID;
  stats_init_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(s);
  BTAS_CUDA_CHECK_LAUNCH();
  return BTAS_OK;
}

extern "C" int btas_ingest(int kind, int src_dtype, const void* src, int64_t numel, int dst_dtype, void* dst,
                           btas_stats* stats, btas_stream_t stream) {
  if (!src || !dst || !stats || numel < 0 || !valid_kind(kind) || !valid_dtype(dst_dtype)) return BTAS_ERR_INVALID;
  if (src_dtype != BTAS_F64 && src_dtype != BTAS_F32) return BTAS_ERR_INVALID;
  if (numel == 0) return BTAS_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool mn = kind == BTAS_MIN_PLUS;
  const unsigned grid = grid_for(numel);
  if (src_dtype == BTAS_F64) {
    BTAS_DISPATCH(dst_dtype, ingest_kernel<double, T><<<grid, 256, 0, st>>>(mn, (const double*)src, numel, (T*)dst, stats))
  } else {
    BTAS_DISPATCH(dst_dtype, ingest_kernel<float, T><<<grid, 256, 0, st>>>(mn, (const float*)src, numel, (T*)dst, stats))
  }
  BTAS_CUDA_CHECK_LAUNCH();
  return BTAS_OK;
}

extern "C" int btas_scan(int dtype, const void* x, int64_t numel, btas_stats* stats, btas_stream_t stream) {
  if (!x || !stats || numel < 0) return BTAS_ERR_INVALID;
  if (numel == 0) return BTAS_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  BTAS_DISPATCH(dtype, scan_kernel<T><<<grid_for(numel), 256, 0, st>>>((const T*)x, numel, stats))
  BTAS_CUDA_CHECK_LAUNCH();
  return BTAS_OK;
}

extern "C" int btas_to_f64(int dtype, const void* src, int64_t numel, double* dst, btas_stream_t stream) {
  if (!src || !dst || numel < 0) return BTAS_ERR_INVALID;
  if (numel == 0) return BTAS_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  BTAS_DISPATCH(dtype, to_f64_kernel<T><<<grid_for(numel), 256, 0, st>>>((const T*)src, numel, dst))
  BTAS_CUDA_CHECK_LAUNCH();
  return BTAS_OK;
}

extern "C" int btas_fill(int dtype, int kind, void* x, int64_t numel, double value, btas_stream_t stream) {
  if (!x || numel < 0 || !valid_kind(kind) || isnan(value) || value == -INFINITY) return BTAS_ERR_INVALID;
  if (numel == 0) return BTAS_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool mn = kind == BTAS_MIN_PLUS;
  if (dtype == BTAS_I32 && !isinf(value) && (value != floor(value) || fabs(value) >= (double)kI32Limit))
    return BTAS_ERR_INVALID;
  BTAS_DISPATCH(dtype, {
    const T v = isinf(value) ? Traits<T>::eps(mn) : (T)(value + 0.0);
    fill_kernel<T><<<grid_for(numel), 256, 0, st>>>((T*)x, numel, v);
  })
  BTAS_CUDA_CHECK_LAUNCH();
  return BTAS_OK;
}

extern "C" int btas_identity(int dtype, int kind, void* d, int64_t ld, int64_t n, btas_stream_t stream) {
  if (!d || n < 0 || ld < n || !valid_kind(kind)) return BTAS_ERR_INVALID;
  if (n == 0) return BTAS_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool mn = kind == BTAS_MIN_PLUS;
  BTAS_DISPATCH(dtype, identity_kernel<T><<<grid_for(n * n), 256, 0, st>>>((T*)d, ld, n, Traits<T>::eps(mn)))
  BTAS_CUDA_CHECK_LAUNCH();
  return BTAS_OK;
}

extern "C" int btas_closure_base(int dtype, const void* src, int64_t lds, void* dst, int64_t ldd, int64_t n,
                                 btas_stream_t stream) {
  if (!src || !dst || n < 0 || lds < n || ldd < n) return BTAS_ERR_INVALID;
  if (n == 0) return BTAS_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  BTAS_DISPATCH(dtype, closure_base_kernel<T><<<grid_for(n * n), 256, 0, st>>>((const T*)src, lds, (T*)dst, ldd, n))
  BTAS_CUDA_CHECK_LAUNCH();
  return BTAS_OK;
}

extern "C" int btas_ewadd(int dtype, int kind, const void* a, const void* b, void* out, int64_t numel,
                          btas_stream_t stream) {
  if (!a || !b || !out || numel < 0 || !valid_kind(kind)) return BTAS_ERR_INVALID;
  if (numel == 0) return BTAS_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const unsigned grid = grid_for(ceil_div(numel, 4));
  if (kind == BTAS_MIN_PLUS) {
    BTAS_DISPATCH(dtype, ewadd_kernel<T, true><<<grid, 256, 0, st>>>((const T*)a, (const T*)b, (T*)out, numel))
  } else {
    BTAS_DISPATCH(dtype, ewadd_kernel<T, false><<<grid, 256, 0, st>>>((const T*)a, (const T*)b, (T*)out, numel))
  }
  BTAS_CUDA_CHECK_LAUNCH();
  return BTAS_OK;
}

extern "C" int btas_diag_negative(int dtype, const void* d, int64_t ld, int64_t n, int32_t* flags,
                                  btas_stream_t stream) {
  if (!d || !flags || n < 0 || ld < n) return BTAS_ERR_INVALID;
  if (n == 0) return BTAS_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  BTAS_DISPATCH(dtype, diag_neg_kernel<T><<<grid_for(n), 256, 0, st>>>((const T*)d, ld, n, flags))
  BTAS_CUDA_CHECK_LAUNCH();
  return BTAS_OK;
}

// ------------------------------------------------------------------ verifier (elementwise half)
// find_apsp_violation's first two checks (apsp.py:194-200) in one pass:
// first[0] = smallest i with D[i,i] != 0, first[1] = smallest row-major index
// with !(D[i,j] <= base[i,j]) where base = I (+) A (diagonal min(A_ii, 0)).
// One CTA row per grid step, threads along the row (coalesced), four loads
// in flight per thread; atomics only on violations.
template <class T>
__global__ void __launch_bounds__(256) verify_base_kernel(const T* __restrict__ D, int64_t ldd,
                                                          const T* __restrict__ A, int64_t lda, int64_t n,
                                                          unsigned long long* first) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const T* drow = D + i * ldd;
    const T* arow = A + i * lda;
    auto check = [&](int64_t j, T d, T a) {
      if (j == i) {
        if (d != (T)0) atomicMin(&first[0], (unsigned long long)i);
        a = a < (T)0 ? a : (T)0;
      }
      if (!(d <= a)) atomicMin(&first[1], (unsigned long long)(i * n + j));
    };
    int64_t j = threadIdx.x;
    for (; j + 3 * 256 < n; j += 4 * 256) {
      T d[4], a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        d[u] = drow[j + u * 256];
        a[u] = arow[j + u * 256];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) check(j + u * 256, d[u], a[u]);
    }
    for (; j < n; j += 256) check(j, drow[j], arow[j]);
  }
}

extern "C" int btas_verify_base(int dtype, const void* D, int64_t ldd, const void* A, int64_t lda, int64_t n,
                                unsigned long long* first, btas_stream_t stream) {
  if (!D || !A || !first || n < 1 || ldd < n || lda < n || !valid_dtype(dtype)) return BTAS_ERR_INVALID;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const unsigned grid = (unsigned)std::min<int64_t>(n, (int64_t)device_sm_count() * 8);
  BTAS_DISPATCH(dtype, verify_base_kernel<T><<<grid, 256, 0, st>>>((const T*)D, ldd, (const T*)A, lda, n, first))
  BTAS_CUDA_CHECK_LAUNCH();
  return BTAS_OK;
}

extern "C" int btas_matvec_bounded(int dtype, int kind, int integer_mode, const void* A, int64_t lda, int64_t M,
                                   int64_t K, const void* V, int64_t ldv, int64_t batch, void* Out, int64_t ldo,
                                   double abs_bound, int32_t* flags, btas_stream_t stream) {
  if (!A || !V || !Out || !flags || M < 1 || K < 1 || batch < 1 || lda < K || ldv < K || ldo < M ||
      !valid_kind(kind))
    return BTAS_ERR_INVALID;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool mn = kind == BTAS_MIN_PLUS;
  int rc = BTAS_OK;
  BTAS_DISPATCH(dtype, {
    rc = mn ? matvec_typed<T, true>(integer_mode, abs_bound, (const T*)A, lda, M, K, (const T*)V, ldv, batch,
                                    (T*)Out, ldo, flags, st)
            : matvec_typed<T, false>(integer_mode, abs_bound, (const T*)A, lda, M, K, (const T*)V, ldv, batch,
                                     (T*)Out, ldo, flags, st);
  })
  return rc;
}

extern "C" int btas_matvec(int dtype, int kind, int integer_mode, const void* A, int64_t lda, int64_t M, int64_t K,
                           const void* V, int64_t ldv, int64_t batch, void* Out, int64_t ldo, int32_t* flags,
                           btas_stream_t stream) {
  return btas_matvec_bounded(dtype, kind, integer_mode, A, lda, M, K, V, ldv, batch, Out, ldo, -1.0, flags, stream);
}

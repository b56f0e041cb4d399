// Repeated-squaring APSP for small graphs in ONE cooperative kernel.
//
// apsp_by_squaring (reference apsp.py:136-178) at n <= ~1k is launch- and
// host-sync-bound on the general path: every squaring is a dozen launches
// (screen, packing, gated GEMMs) plus a host read of the fixpoint flag, for a
// GEMM that fills only (n/128)^2 of the 148 SMs.  Here the whole loop — every
// squaring, its fixpoint compare, the negative-cycle probe and the result
// copy — runs inside one persistent kernel with grid-wide barriers between
// the dependent steps: 32 x 32 output tiles spread over every SM, operands
// staged through shared memory, and the flags, the multiplication count and
// the exact overflow screen of the next step kept in device memory.
//
// Semantics are the general path's, candidate for candidate: a step uses the
// plain add-min mix when the exact screen (max |finite| of its operands, summed
// in storage arithmetic, rounding is monotone) proves no finite (x) finite
// candidate can overflow / reach the integer limit, else the reference's
// masked candidate (matrix.py:334-342) with the saturation flag.  The k
// dimension is never split, so results are bit-identical to the general path
// and to the reference.
#include <cooperative_groups.h>

#include <algorithm>

#include "btas_common.cuh"

namespace cg = cooperative_groups;

namespace btas {
int device_sm_count();

namespace {

constexpr int kT = 32;         // output tile edge
constexpr int kKC = 32;        // k chunk staged in shared memory
constexpr int kThreads = 256;  // 16 x 16 threads, 2 x 2 outputs each
constexpr int kMaxSteps = 40;

// device control block (workspace)
struct SmallCtl {
  int32_t changed[kMaxSteps + 1], diag[kMaxSteps + 1], sat[kMaxSteps + 1];
  unsigned long long amax[kMaxSteps + 2];  // ordered keys of max |finite| of each operand
  unsigned long long amax_base;
};

template <class T>
struct SmallArgs {
  const T* base;
  int64_t ldb;
  int64_t n;
  T* w0;
  T* w1;
  T* out;
  int64_t ldo;
  int integer_mode;
  double limit;
  int steps;  // squarings the reference loop allows: ceil(log2(n - 1))
  SmallCtl* ctl;
  int32_t* result;  // [multiplications, negative_cycle, saturated, fixpoint]
  int32_t* flags;
};

template <class T>
BTAS_D bool fin(T x) {
  return Traits<T>::finite(x);
}

template <class T>
BTAS_D double abs_fin(T x) {
  return fin(x) ? fabs((double)x) : 0.0;
}

template <class T>
BTAS_D T add_st(T a, T b) {
  if constexpr (Traits<T>::dtype == BTAS_F32) return __fadd_rn(a, b);
  else if constexpr (Traits<T>::dtype == BTAS_F64) return __dadd_rn(a, b);
  else return a + b;
}

// exact screen: can any finite (x) finite candidate overflow?
template <class T>
BTAS_D bool may_overflow(double amax_a, double amax_b, int integer_mode, double limit) {
  if constexpr (Traits<T>::dtype == BTAS_I32) {
    return amax_a + amax_b >= (double)kI32Limit;  // exact in double
  } else {
    const double s = (double)add_st<T>((T)amax_a, (T)amax_b);
    return integer_mode ? s >= limit : isinf(s);
  }
}

template <class T>
BTAS_D T cand_checked(T a, T b, bool& sat, int integer_mode, double limit) {
  T s = a + b;
  bool over;
  if constexpr (Traits<T>::dtype == BTAS_I32) over = (s >= (T)kI32Limit) || (s <= -(T)kI32Limit);
  else if (integer_mode) over = fabs((double)s) >= limit;
  else over = isinf((double)s);
  if (over && fin(a) && fin(b)) {
    sat = true;
    s = Traits<T>::eps(true);
  }
  return s;
}

template <class T>
BTAS_D T finish(T c) {
  if constexpr (Traits<T>::dtype == BTAS_I32) return c >= (T)kI32Limit ? (T)kI32Inf : c;  // canonical Inf
  else return c;
}

template <class T>
BTAS_D bool bits_ne(T a, T b) {
  if constexpr (sizeof(T) == 8) return __double_as_longlong((double)a) != __double_as_longlong((double)b);
  else if constexpr (Traits<T>::dtype == BTAS_F32) return __float_as_uint(a) != __float_as_uint(b);
  else return a != b;
}

template <class T>
BTAS_D unsigned long long amax_key(double v) {
  return f64_key(v);
}

// One tropical product X (x) Y over all tiles (X: n x n, ld ldx; Y likewise).
// STORE: write the product to Cout; always compares against Cmp (bytewise)
// and tests the diagonal.  Per-thread results are folded into the step's
// control words.
template <class T, bool CHECKED, bool STORE>
BTAS_D void product(const SmallArgs<T>& a, const T* X, int64_t ldx, const T* Y, int64_t ldy, const T* Cmp,
                    int64_t ldcmp, T* Cout, int step, T (*As)[kT + 2], T (*Bs)[kT + 2]) {
  const int64_t n = a.n;
  const int tiles_1d = (int)ceil_div(n, kT);
  const int ntiles = tiles_1d * tiles_1d;
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  const T inf = Traits<T>::eps(true);
  bool changed = false, diag = false, sat = false;
  double amax = 0.0;
  constexpr int kPer = kT * kKC / kThreads;  // staged elements per thread per operand
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = (int64_t)(tile / tiles_1d) * kT, c0 = (int64_t)(tile % tiles_1d) * kT;
    T acc[2][2] = {{inf, inf}, {inf, inf}};
    // register prefetch of the next k chunk: X[r0:r0+32, k0:k0+32] (staged
    // transposed) and Y[k0:k0+32, c0:c0+32]; the loads of chunk k0+32 are in
    // flight while chunk k0 is consumed from shared memory
    T pa[kPer], pb[kPer];
    auto fetch = [&](int64_t k0) {
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int e = threadIdx.x + u * kThreads;
        const int r = e / kKC, k = e % kKC;
        const int64_t gr = r0 + r, gk = k0 + k;
        pa[u] = (gr < n && gk < n) ? X[gr * ldx + gk] : inf;
        const int kk = e / kT, c = e % kT;
        const int64_t gk2 = k0 + kk, gc = c0 + c;
        pb[u] = (gk2 < n && gc < n) ? Y[gk2 * ldy + gc] : inf;
      }
    };
    // f32 fast path: k-pair interleaved staging, so one 16-byte load gives a
    // thread its two rows' (k, k+1) values and FADD2 + FMNMX3 form two
    // candidates per add and per min (as in the GEMM kernel)
    constexpr bool kPairs = Traits<T>::dtype == BTAS_F32 && !CHECKED;
    float2(*A2)[kT + 2] = reinterpret_cast<float2(*)[kT + 2]>(&As[0][0]);  // [k/2][r] = (k even, k odd)
    float2(*B2)[kT + 2] = reinterpret_cast<float2(*)[kT + 2]>(&Bs[0][0]);
    fetch(0);
    for (int64_t k0 = 0; k0 < n; k0 += kKC) {
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int e = threadIdx.x + u * kThreads;
        if constexpr (kPairs) {
          const int k = e % kKC, r = e / kKC, kk = e / kT, c = e % kT;
          reinterpret_cast<float*>(&A2[k >> 1][r])[k & 1] = pa[u];
          reinterpret_cast<float*>(&B2[kk >> 1][c])[kk & 1] = pb[u];
        } else {
          As[e % kKC][e / kKC] = pa[u];
          Bs[e / kT][e % kT] = pb[u];
        }
      }
      __syncthreads();
      if (k0 + kKC < n) fetch(k0 + kKC);
      if constexpr (kPairs) {
#pragma unroll 8
        for (int kp = 0; kp < kKC / 2; ++kp) {
          const float4 xa = *reinterpret_cast<const float4*>(&A2[kp][ty * 2]);  // rows ty*2, ty*2+1
          const float4 yb = *reinterpret_cast<const float4*>(&B2[kp][tx * 2]);  // cols tx*2, tx*2+1
          const float2 x[2] = {make_float2(xa.x, xa.y), make_float2(xa.z, xa.w)};
          const float2 y[2] = {make_float2(yb.x, yb.y), make_float2(yb.z, yb.w)};
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const float2 sum = __fadd2_rn(x[i], y[j]);
              acc[i][j] = fminf(fminf(acc[i][j], sum.x), sum.y);
            }
        }
        __syncthreads();
        continue;
      }
#pragma unroll 8
      for (int k = 0; k < kKC; ++k) {
        T x0, x1, y0, y1;
        if constexpr (sizeof(T) == 4) {
          const uint2 xa = *reinterpret_cast<const uint2*>(&As[k][ty * 2]);
          const uint2 yb = *reinterpret_cast<const uint2*>(&Bs[k][tx * 2]);
          x0 = __builtin_bit_cast(T, xa.x);
          x1 = __builtin_bit_cast(T, xa.y);
          y0 = __builtin_bit_cast(T, yb.x);
          y1 = __builtin_bit_cast(T, yb.y);
        } else {
          x0 = As[k][ty * 2];
          x1 = As[k][ty * 2 + 1];
          y0 = Bs[k][tx * 2];
          y1 = Bs[k][tx * 2 + 1];
        }
        if constexpr (CHECKED) {
          const int im = a.integer_mode;
          const double lim = a.limit;
          T s;
          s = cand_checked(x0, y0, sat, im, lim);
          acc[0][0] = s < acc[0][0] ? s : acc[0][0];
          s = cand_checked(x0, y1, sat, im, lim);
          acc[0][1] = s < acc[0][1] ? s : acc[0][1];
          s = cand_checked(x1, y0, sat, im, lim);
          acc[1][0] = s < acc[1][0] ? s : acc[1][0];
          s = cand_checked(x1, y1, sat, im, lim);
          acc[1][1] = s < acc[1][1] ? s : acc[1][1];
        } else if constexpr (Traits<T>::dtype == BTAS_I32) {
          acc[0][0] = __viaddmin_s32(x0, y0, acc[0][0]);
          acc[0][1] = __viaddmin_s32(x0, y1, acc[0][1]);
          acc[1][0] = __viaddmin_s32(x1, y0, acc[1][0]);
          acc[1][1] = __viaddmin_s32(x1, y1, acc[1][1]);
        } else {
          acc[0][0] = min(acc[0][0], add_st<T>(x0, y0));
          acc[0][1] = min(acc[0][1], add_st<T>(x0, y1));
          acc[1][0] = min(acc[1][0], add_st<T>(x1, y0));
          acc[1][1] = min(acc[1][1], add_st<T>(x1, y1));
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int64_t row = r0 + ty * 2 + i;
      if (row >= n) continue;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t col = c0 + tx * 2 + j;
        if (col >= n) continue;
        const T v = finish(acc[i][j]);
        changed |= bits_ne(v, Cmp[row * ldcmp + col]);
        if (row == col) diag |= v < (T)0;
        amax = fmax(amax, abs_fin(v));
        if constexpr (STORE) Cout[row * n + col] = v;
      }
    }
  }
  const int lane = threadIdx.x & 31;
  if (__any_sync(0xffffffffu, changed) && lane == 0) atomicOr(&a.ctl->changed[step], 1);
  if (__any_sync(0xffffffffu, diag) && lane == 0) atomicOr(&a.ctl->diag[step], 1);
  if (__any_sync(0xffffffffu, sat) && lane == 0) atomicOr(&a.ctl->sat[step], 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if (lane == 0 && STORE) atomicMax(&a.ctl->amax[step + 1], amax_key<T>(amax));
}

template <class T>
BTAS_D int32_t ld_cg(const int32_t* p) {
  return __ldcg(p);
}

template <class T>
__global__ void __launch_bounds__(kThreads, 2) apsp_small_kernel(const __grid_constant__ SmallArgs<T> a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ __align__(16) T As[kKC][kT + 2];
  __shared__ __align__(16) T Bs[kKC][kT + 2];
  const int64_t n = a.n;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
  // control block reset + max |finite| of the base (the first step's operands)
  if (gtid < (int64_t)(sizeof(SmallCtl) / 4)) reinterpret_cast<int32_t*>(a.ctl)[gtid] = 0;
  grid.sync();
  {
    double m = 0.0;
    for (int64_t i = gtid; i < n * n; i += gthreads) m = fmax(m, abs_fin(a.base[(i / n) * a.ldb + i % n]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) {
      atomicMax(&a.ctl->amax[0], amax_key<T>(m));
      atomicMax(&a.ctl->amax_base, amax_key<T>(m));
    }
  }
  grid.sync();

  const T* cur = a.base;
  int64_t ldcur = a.ldb;
  int mults = 0;
  bool fixpoint = false;
  int last = -1;
  for (int s = 0; s < a.steps; ++s) {
    const double am = key_f64(__ldcg(&a.ctl->amax[s]));
    T* nxt = (s & 1) ? a.w1 : a.w0;
    if (may_overflow<T>(am, am, a.integer_mode, a.limit))
      product<T, true, true>(a, cur, ldcur, cur, ldcur, cur, ldcur, nxt, s, As, Bs);
    else
      product<T, false, true>(a, cur, ldcur, cur, ldcur, cur, ldcur, nxt, s, As, Bs);
    grid.sync();
    ++mults;
    last = s;
    if (!ld_cg<T>(&a.ctl->changed[s])) {
      fixpoint = true;  // the product equals its operand byte for byte
      break;
    }
    cur = nxt;
    ldcur = n;
  }
  bool negative;
  bool sat = false;
  for (int s = 0; s <= last; ++s) sat |= ld_cg<T>(&a.ctl->sat[s]) != 0;
  if (fixpoint) {
    negative = ld_cg<T>(&a.ctl->diag[last]) != 0;  // diag of the (unchanged) product
  } else {
    // uncounted probe d (x) (I (+) A): changed or a negative diagonal
    const int p = kMaxSteps;
    const double am = key_f64(__ldcg(&a.ctl->amax[last + 1 > 0 ? last + 1 : 0]));
    const double ab = key_f64(__ldcg(&a.ctl->amax_base));
    if (may_overflow<T>(am, ab, a.integer_mode, a.limit))
      product<T, true, false>(a, cur, ldcur, a.base, a.ldb, cur, ldcur, nullptr, p, As, Bs);
    else
      product<T, false, false>(a, cur, ldcur, a.base, a.ldb, cur, ldcur, nullptr, p, As, Bs);
    grid.sync();
    negative = ld_cg<T>(&a.ctl->changed[p]) != 0 || ld_cg<T>(&a.ctl->diag[p]) != 0;
    sat |= ld_cg<T>(&a.ctl->sat[p]) != 0;
  }
  // result: the last operand (at a fixpoint it equals the product)
  for (int64_t i = gtid; i < n * n; i += gthreads) {
    const int64_t r = i / n, c = i % n;
    a.out[r * a.ldo + c] = cur[r * ldcur + c];
  }
  if (gtid == 0) {
    a.result[0] = mults;
    a.result[1] = negative ? 1 : 0;
    a.result[2] = sat ? 1 : 0;
    a.result[3] = fixpoint ? 1 : 0;
    if (sat) atomicOr(&a.flags[BTAS_FLAG_SATURATED], 1);
  }
}

template <class T>
int apsp_small_typed(int integer_mode, const T* base, int64_t ldb, int64_t n, T* out, int64_t ldo,
                     int32_t* result, int32_t* flags, unsigned char* ws, cudaStream_t st) {
  SmallArgs<T> a{};
  a.base = base;
  a.ldb = ldb;
  a.n = n;
  a.w0 = reinterpret_cast<T*>(ws);
  a.w1 = a.w0 + n * n;
  a.ctl = reinterpret_cast<SmallCtl*>(ws + round_up(2 * n * n * (int64_t)sizeof(T), 256));
  a.out = out;
  a.ldo = ldo;
  a.integer_mode = Traits<T>::dtype == BTAS_I32 ? 1 : integer_mode;
  a.limit = Traits<T>::dtype == BTAS_I32 ? (double)kI32Limit : Traits<T>::int_limit;
  int steps = 0;
  for (int64_t power = 1; power < n - 1; power *= 2) ++steps;
  a.steps = steps;
  a.result = result;
  a.flags = flags;
  // co-resident CTAs per SM, per instantiation and device ordinal (the query
  // costs tens of microseconds; a cooperative grid above the co-resident
  // limit of the launching device fails)
  static int per_sm_dev[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    (void)cudaGetLastError();
    return BTAS_ERR_CUDA;
  }
  int& per_sm = per_sm_dev[dev];
  if (per_sm < 1 &&
      (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, apsp_small_kernel<T>, kThreads, 0) != cudaSuccess ||
       per_sm < 1)) {
    (void)cudaGetLastError();
    per_sm = 0;
    return BTAS_ERR_CUDA;
  }
  const int64_t tiles = ceil_div(n, kT) * ceil_div(n, kT);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)per_sm * device_sm_count()));
  void* params[] = {&a};
  if (cudaLaunchCooperativeKernel((const void*)apsp_small_kernel<T>, dim3(grid), dim3(kThreads), params, 0, st) !=
      cudaSuccess) {
    (void)cudaGetLastError();
    return BTAS_ERR_CUDA;
  }
  return BTAS_OK;
}

}  // namespace
}  // namespace btas

using namespace btas;

extern "C" size_t btas_apsp_small_workspace_bytes(int dtype, int64_t n) {
  if (n < 1 || n > BTAS_APSP_SMALL_MAX_N) return 0;
  const int64_t es = dtype == BTAS_F64 ? 8 : 4;
  return (size_t)round_up(2 * n * n * es, 256) + sizeof(SmallCtl);
}

extern "C" int btas_apsp_squaring_small(int dtype, int integer_mode, const void* base, int64_t ldb, int64_t n,
                                        void* out, int64_t ldo, int32_t* dev_result, int32_t* dev_flags,
                                        void* workspace, size_t workspace_bytes, btas_stream_t stream) {
  if (!base || !out || !dev_result || !dev_flags || !workspace) return BTAS_ERR_INVALID;
  if (n < 2 || n > BTAS_APSP_SMALL_MAX_N || ldb < n || ldo < n) return BTAS_ERR_INVALID;
  if (workspace_bytes < btas_apsp_small_workspace_bytes(dtype, n)) return BTAS_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  switch (dtype) {
    case BTAS_F32:
      return apsp_small_typed<float>(integer_mode, (const float*)base, ldb, n, (float*)out, ldo, dev_result,
                                     dev_flags, ws, st);
    case BTAS_I32:
      return apsp_small_typed<int32_t>(integer_mode, (const int32_t*)base, ldb, n, (int32_t*)out, ldo, dev_result,
                                       dev_flags, ws, st);
    case BTAS_F64:
      return apsp_small_typed<double>(integer_mode, (const double*)base, ldb, n, (double*)out, ldo, dev_result,
                                      dev_flags, ws, st);
    default:
      return BTAS_ERR_INVALID;
  }
}

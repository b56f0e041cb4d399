// Internals of btas_gemm (the matmul drop-in): screen, packing and the
// per-dtype driver.  Included by one translation unit per storage dtype
// (btas_gemm_f32.cu, btas_gemm_i32.cu, btas_gemm_f64.cu) so the kernel
// instantiations compile in parallel.
#pragma once

#include <algorithm>
#include <type_traits>

#include "btas_gemm.cuh"

namespace btas {

// timing hooks (defined in btas_gemm.cu)
extern bool g_timing;
void timing_begin(cudaStream_t st, cudaEvent_t* start);
void timing_end(cudaStream_t st, cudaEvent_t start);
int device_sm_count();

namespace gemm_impl {
namespace {  // internal linkage: one copy per dtype translation unit

constexpr int kKP = 16;    // k pairs per pipeline stage (32/64-bit policies)
constexpr int kKP16 = 32;  // word pairs per pipeline stage of the s16x2 policy

struct Ctrl {
  int32_t path;
  int32_t pad[63];
};

struct WsLayout {
  size_t ctrl, extA, extB, packA, packB, total;
};

template <class T>
struct GemmGeometry {
  static constexpr int BM = sizeof(T) == 8 ? 64 : 128;
  static constexpr int BN = 128;
};

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// column groups of the s16x2 microtile: 4 = 128-wide tiles.  (A 256-wide,
// 8x16 microtile was measured 1 % slower, profiles/r01_experiments.md.)
int s16_gn() { return 4; }

WsLayout ws_layout(int dtype, int64_t M, int64_t N, int64_t K) {
  const size_t es = dtype == BTAS_F64 ? 8 : 4;
  const int64_t BM = dtype == BTAS_F64 ? 64 : 128, BN = 128;
  const int64_t Kp = round_up(K, 2 * kKP);               // 32-bit/64-bit paths
  const int64_t Kw = round_up(ceil_div(K, 2), 2 * kKP16);  // s16 words
  const int64_t Mp = round_up(M, BM), Np = round_up(N, BN);
  const int64_t Mp16 = round_up(M, 128), Np16 = round_up(N, 256);
  const size_t a32 = (size_t)Mp * Kp * es, b32 = (size_t)Np * Kp * es;
  const size_t a16 = (size_t)Mp16 * Kw * 4, b16 = (size_t)Np16 * Kw * 4;
  WsLayout L;
  size_t off = 0;
  L.ctrl = off;
  off += align256(sizeof(Ctrl));
  L.extA = off;
  off += align256((size_t)K * 2 * sizeof(unsigned long long));
  L.extB = off;
  off += align256((size_t)K * 2 * sizeof(unsigned long long));
  L.packA = off;
  off += align256(a32 > a16 ? a32 : a16);
  L.packB = off;
  off += align256(b32 > b16 ? b32 : b16);
  L.total = off;
  return L;
}

// ------------------------------------------------------------------ init
__global__ void init_ws_kernel(Ctrl* ctrl, unsigned long long* extA, unsigned long long* extB, int64_t K) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0) ctrl->path = -1;
  for (int64_t k = t; k < K; k += (int64_t)gridDim.x * blockDim.x) {
    extA[k] = kKeyNone;
    extA[K + k] = kKeyNoneMin;
    extB[k] = kKeyNone;
    extB[K + k] = kKeyNoneMin;
  }
}

// ------------------------------------------------------------------ extremes
// Per-k extremes of the finite entries, accumulated in the storage type
// (B200's FP64 pipe is slow; converting every element to double halved the
// throughput of these passes) and converted once per thread.
template <class T>
BTAS_D T lowest() {
  if constexpr (Traits<T>::dtype == BTAS_I32) return (T)(-kI32Limit);
  else return (T)-INFINITY;
}
template <class T>
BTAS_D T highest() {
  if constexpr (Traits<T>::dtype == BTAS_I32) return (T)kI32Limit;
  else return (T)INFINITY;
}

// A (M x K): per column k, max and min over the finite entries of that column.
template <class T>
__global__ void ext_cols_kernel(const T* __restrict__ A, int64_t lda, int64_t M, int64_t K, int rows_per_cta,
                                unsigned long long* ext) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_cta;
  const int64_t r1 = min(M, r0 + rows_per_cta);
  T mx = lowest<T>(), mn = highest<T>();
  bool any = false;
#pragma unroll 8
  for (int64_t r = r0; r < r1; ++r) {
    const T x = A[r * lda + k];
    if (Traits<T>::finite(x)) {
      mx = x > mx ? x : mx;
      mn = x < mn ? x : mn;
      any = true;
    }
  }
  if (any) {
    atomicMax(&ext[k], f64_key((double)mx));
    atomicMin(&ext[K + k], f64_key((double)mn));
  }
}

// B (K x N): per row k, max and min over the finite entries of that row.
template <class T>
__global__ void ext_rows_kernel(const T* __restrict__ B, int64_t ldb, int64_t K, int64_t N,
                                unsigned long long* ext) {
  const int64_t k = blockIdx.x;
  const T* row = B + k * ldb;
  T mx = lowest<T>(), mn = highest<T>();
  bool any = false;
  auto take = [&](T x) {
    if (Traits<T>::finite(x)) {
      mx = x > mx ? x : mx;
      mn = x < mn ? x : mn;
      any = true;
    }
  };
  const int64_t stride = (int64_t)gridDim.y * blockDim.x;
  int64_t j = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  for (; j + 3 * stride < N; j += 4 * stride) {  // 4 loads in flight per thread
    T xs[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) xs[u] = row[j + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u) take(xs[u]);
  }
  for (; j < N; j += stride) take(row[j]);
  double dmx = any ? (double)mx : -INFINITY, dmn = any ? (double)mn : INFINITY;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dmx = fmax(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
    dmn = fmin(dmn, __shfl_xor_sync(0xffffffffu, dmn, o));
  }
  __shared__ double smx[32], smn[32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    smx[w] = dmx;
    smn[w] = dmn;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    dmx = l < nw ? smx[l] : -INFINITY;
    dmn = l < nw ? smn[l] : INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dmx = fmax(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
      dmn = fmin(dmn, __shfl_xor_sync(0xffffffffu, dmn, o));
    }
    if (l == 0 && dmx >= dmn) {  // at least one finite entry
      atomicMax(&ext[k], f64_key(dmx));
      atomicMin(&ext[K + k], f64_key(dmn));
    }
  }
}

// ------------------------------------------------------------------ screen
template <class T>
BTAS_D double storage_sum(double a, double b) {
  if constexpr (Traits<T>::dtype == BTAS_F32) return (double)__fadd_rn((float)a, (float)b);
  else return a + b;  // f64: the storage op itself; i32: exact in double
}

template <class T>
__global__ void screen_kernel(const unsigned long long* __restrict__ extA, const unsigned long long* __restrict__ extB,
                              int64_t K, int min_plus, int integer_mode, double limit, Ctrl* ctrl,
                              int32_t* flags) {
  bool sat = false, dangerous = false;
  double amax = 0.0, bmax = 0.0;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    const unsigned long long ka = extA[k], kb = extB[k];
    if (ka != kKeyNone) {
      amax = fmax(amax, fmax(fabs(key_f64(ka)), fabs(key_f64(extA[K + k]))));
    }
    if (kb != kKeyNone) {
      bmax = fmax(bmax, fmax(fabs(key_f64(kb)), fabs(key_f64(extB[K + k]))));
    }
    if (ka == kKeyNone || kb == kKeyNone) continue;
    const double hi = storage_sum<T>(key_f64(ka), key_f64(kb));
    const double lo = storage_sum<T>(key_f64(extA[K + k]), key_f64(extB[K + k]));
    bool pos, neg;
    if (integer_mode) {
      pos = hi >= limit;
      neg = lo <= -limit;
    } else {
      pos = isinf(hi);
      neg = isinf(lo);
    }
    sat |= pos || neg;
    dangerous |= min_plus ? neg : pos;
  }
  sat = __syncthreads_or(sat);
  dangerous = __syncthreads_or(dangerous);
  __shared__ double red[2][32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    bmax = fmax(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = amax;
    red[1][threadIdx.x >> 5] = bmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      amax = fmax(amax, red[0][w]);
      bmax = fmax(bmax, red[1][w]);
    }
    int path;
    if (dangerous) {
      path = BTAS_PATH_CHECKED;
    } else if (integer_mode && amax < (double)kS16Limit && bmax < (double)kS16Limit) {
      path = BTAS_PATH_S16X2;
    } else if (Traits<T>::dtype == BTAS_F64 && integer_mode && amax + bmax < (double)kI32Limit) {
      path = BTAS_PATH_I32F64;  // no sum reaches 2^28 (< the 2^53 limit): nothing saturates
    } else {
      path = Traits<T>::dtype == BTAS_F64 ? BTAS_PATH_FAST64 : BTAS_PATH_FAST32;
    }
    ctrl->path = path;
    if (sat) atomicOr(&flags[BTAS_FLAG_SATURATED], 1);
    atomicOr(&flags[BTAS_FLAG_PATH], 1 << path);
  }
}

// ------------------------------------------------------------------ packing
// Packed element: the storage value itself (32/64-bit paths) or an int16x2
// word holding entries k = 2w, 2w+1 (s16 path).
template <class T, bool MIN>
BTAS_D uint32_t to_s16(T x) {
  int v = Traits<T>::finite(x) ? (int)x : (MIN ? kS16Inf : -kS16Inf);
  return (uint32_t)(uint16_t)(int16_t)v;
}

// predecessor keys (MixArgKey): value << 16 | k packs a min-plus candidate
// and its k into one int32, so one VIADDMNMX keeps the first argmin
constexpr int32_t kArgKeyInf = (1 << 30) - (1 << 17);

template <class T, class E, bool S16, bool MIN, int KEYM = 0>
BTAS_D E load_virtual(const T* __restrict__ X, int64_t ld, int64_t rows, int64_t cols, int64_t r, int64_t c,
                      bool c_is_k) {
  // c_is_k: virtual column index c is along k (A operand, row r); otherwise
  // the virtual row index r is along k (B operand, column c).
  if constexpr (KEYM != 0) {  // 1: A operand value << 16; 2: B operand (value << 16) + k
    if (!(r < rows && c < cols)) return (E)kArgKeyInf;
    const T x = X[r * ld + c];
    if (!Traits<T>::finite(x)) return (E)kArgKeyInf;
    const int32_t v = (int32_t)x * 65536;
    return (E)(KEYM == 1 ? v : v + (int32_t)r);
  } else if constexpr (!S16 && std::is_integral<E>::value && !std::is_integral<T>::value) {
    // float64 integer operands packed as int32 (BTAS_PATH_I32F64)
    const T x = (r < rows && c < cols) ? X[r * ld + c] : Traits<T>::eps(MIN);
    return isfinite(x) ? (E)x : (MIN ? (E)kI32Inf : (E)-kI32Inf);
  } else if constexpr (!S16) {
    if (r < rows && c < cols) return (E)X[r * ld + c];
    return (E)Traits<T>::eps(MIN);
  } else {
    uint32_t lo, hi;
    if (c_is_k) {
      const int64_t k0 = 2 * c, k1 = 2 * c + 1;
      lo = (r < rows && k0 < cols) ? to_s16<T, MIN>(X[r * ld + k0]) : to_s16<T, MIN>(Traits<T>::eps(MIN));
      hi = (r < rows && k1 < cols) ? to_s16<T, MIN>(X[r * ld + k1]) : to_s16<T, MIN>(Traits<T>::eps(MIN));
    } else {
      const int64_t k0 = 2 * r, k1 = 2 * r + 1;
      lo = (k0 < rows && c < cols) ? to_s16<T, MIN>(X[k0 * ld + c]) : to_s16<T, MIN>(Traits<T>::eps(MIN));
      hi = (k1 < rows && c < cols) ? to_s16<T, MIN>(X[k1 * ld + c]) : to_s16<T, MIN>(Traits<T>::eps(MIN));
    }
    return (E)(lo | (hi << 16));
  }
}

// A (M x K) -> Ap[mb][kp][BM][2] over virtual k (words for s16): a 32 x 64
// smem transpose so both the row reads and the pair writes are coalesced.
template <class T, class E, bool S16, bool MIN, int BM, int KEYM = 0>
__global__ void pack_a_kernel(const T* __restrict__ A, int64_t lda, int64_t M, int64_t K, int64_t Kv, int64_t Kp2,
                              E* __restrict__ Ap, const Ctrl* ctrl, int gate0, int gate1) {
  if (ctrl != nullptr && ctrl->path != gate0 && ctrl->path != gate1) return;
  __shared__ E tile[32][65];
  const int64_t m0 = (int64_t)blockIdx.y * 32;
  const int64_t k0 = (int64_t)blockIdx.x * 64;  // virtual k
  for (int e = threadIdx.x; e < 32 * 64; e += blockDim.x) {
    const int mr = e >> 6, kc = e & 63;
    const int64_t m = m0 + mr, kv = k0 + kc;
    tile[mr][kc] = load_virtual<T, E, S16, MIN, KEYM>(A, lda, M, K, m, kv, true);  // eps past M / K
  }
  __syncthreads();
  // write pairs: 32 kp x 32 m
  for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
    const int kpl = e >> 5, mr = e & 31;
    const int64_t m = m0 + mr;
    const int64_t kp = (k0 >> 1) + kpl;
    if (kp >= Kp2) continue;
    const int64_t idx = packed_index(m, 2 * kp, Kp2, BM);
    Ap[idx] = tile[mr][2 * kpl];
    Ap[idx + 1] = tile[mr][2 * kpl + 1];
  }
}

// B (K x N) -> Bp[nb][kp][BN][2]: rows 2kp and 2kp+1 interleaved.
template <class T, class E, bool S16, bool MIN, int BN, int KEYM = 0>
__global__ void pack_b_kernel(const T* __restrict__ B, int64_t ldb, int64_t K, int64_t N, int64_t Np, int64_t Kp2,
                              E* __restrict__ Bp, const Ctrl* ctrl, int gate0, int gate1) {
  if (ctrl != nullptr && ctrl->path != gate0 && ctrl->path != gate1) return;
  const int64_t total = Kp2 * Np;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kp = e / Np, n = e - kp * Np;
    const E v0 = load_virtual<T, E, S16, MIN, KEYM>(B, ldb, K, N, 2 * kp, n, false);
    const E v1 = load_virtual<T, E, S16, MIN, KEYM>(B, ldb, K, N, 2 * kp + 1, n, false);
    const int64_t idx = packed_index(n, 2 * kp, Kp2, BN);
    Bp[idx] = v0;
    Bp[idx + 1] = v1;
  }
}

// ------------------------------------------------------------------ driver
template <class T, bool MIN>
int gemm_typed(int integer_mode, const T* A, int64_t lda, const T* B, int64_t ldb, const T* Z, int64_t ldz, T* C,
               int64_t ldc, int64_t M, int64_t N, int64_t K, const T* Cprev, int64_t ldcp, int32_t* flags,
               unsigned char* ws, const WsLayout& L, const GemmExtras& x, cudaStream_t st) {
  void* const* peers = x.peers;
  const int n_peers = x.n_peers;
  using G = GemmGeometry<T>;
  constexpr bool kIsF64 = Traits<T>::dtype == BTAS_F64;
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(ws + L.ctrl);
  unsigned long long* extA = reinterpret_cast<unsigned long long*>(ws + L.extA);
  unsigned long long* extB = reinterpret_cast<unsigned long long*>(ws + L.extB);
  const bool int_mode = Traits<T>::dtype == BTAS_I32 ? true : (integer_mode != 0);
  const double limit = Traits<T>::dtype == BTAS_I32 ? (double)kI32Limit : Traits<T>::int_limit;

  init_ws_kernel<<<(unsigned)std::min<int64_t>(ceil_div(K, 256), 1024), 256, 0, st>>>(ctrl, extA, extB, K);
  {
    const int rows_per_cta = 256;
    dim3 grid((unsigned)ceil_div(K, 256), (unsigned)ceil_div(M, rows_per_cta));
    ext_cols_kernel<T><<<grid, 256, 0, st>>>(A, lda, M, K, rows_per_cta, extA);
  }
  {
    dim3 grid((unsigned)K, (unsigned)std::min<int64_t>(ceil_div(N, 256 * 16), 64));
    ext_rows_kernel<T><<<grid, 256, 0, st>>>(B, ldb, K, N, extB);
  }
  screen_kernel<T><<<1, 1024, 0, st>>>(extA, extB, K, MIN ? 1 : 0, int_mode ? 1 : 0, limit, ctrl, flags);
  BTAS_CUDA_CHECK_LAUNCH();

  const int fast = kIsF64 ? BTAS_PATH_FAST64 : BTAS_PATH_FAST32;
  GemmArgs g{};  // 32/64-bit paths (FAST and CHECKED share the packing)
  {
    const int64_t Kp2 = round_up(K, 2 * kKP) / 2;
    const int64_t Mp = round_up(M, G::BM), Np = round_up(N, G::BN);
    T* Ap = reinterpret_cast<T*>(ws + L.packA);
    T* Bp = reinterpret_cast<T*>(ws + L.packB);
    dim3 ga((unsigned)ceil_div(2 * Kp2, 64), (unsigned)ceil_div(Mp, 32));
    pack_a_kernel<T, T, false, MIN, G::BM><<<ga, 256, 0, st>>>(A, lda, M, K, 2 * Kp2, Kp2, Ap, ctrl, fast,
                                                                BTAS_PATH_CHECKED);
    const int64_t tb = Kp2 * Np;
    pack_b_kernel<T, T, false, MIN, G::BN>
        <<<(unsigned)std::min<int64_t>(ceil_div(tb, 256), 65535), 256, 0, st>>>(B, ldb, K, N, Np, Kp2, Bp, ctrl, fast,
                                                                         BTAS_PATH_CHECKED);
    BTAS_CUDA_CHECK_LAUNCH();
    g.Ap = Ap;
    g.Bp = Bp;
    g.Kp2 = Kp2;
    g.M = M;
    g.N = N;
    g.mblocks = (int)(Mp / G::BM);
    g.nblocks = (int)(Np / G::BN);
    g.Z = Z;
    g.ldz = ldz;
    g.C = C;
    g.ldc = ldc;
    g.Cprev = Cprev;
    g.ldcp = ldcp;
    g.flags = flags;
    g.gate = &ctrl->path;
    g.integer_mode = int_mode ? 1 : 0;
    g.limit = int_mode ? limit : INFINITY;
    g.n_peers = n_peers;
    for (int q = 0; q < n_peers && q < kMaxPeers; ++q) g.peer_C[q] = peers[q];
    g.first_bad = x.first_bad;
    g.verify_mode = x.verify_mode;
  }
  GemmArgs g32{};  // float64 integer operands through the int32 kernel
  if constexpr (kIsF64) {
    if (int_mode) {
      const int64_t Kp2 = round_up(K, 2 * kKP) / 2;
      const int64_t Mp = round_up(M, 128), Np = round_up(N, 128);
      int32_t* Ap = reinterpret_cast<int32_t*>(ws + L.packA);
      int32_t* Bp = reinterpret_cast<int32_t*>(ws + L.packB);
      dim3 ga((unsigned)ceil_div(2 * Kp2, 64), (unsigned)ceil_div(Mp, 32));
      pack_a_kernel<T, int32_t, false, MIN, 128><<<ga, 256, 0, st>>>(A, lda, M, K, 2 * Kp2, Kp2, Ap, ctrl,
                                                                      BTAS_PATH_I32F64, BTAS_PATH_I32F64);
      const int64_t tb = Kp2 * Np;
      pack_b_kernel<T, int32_t, false, MIN, 128><<<(unsigned)std::min<int64_t>(ceil_div(tb, 256), 65535), 256, 0,
                                                    st>>>(B, ldb, K, N, Np, Kp2, Bp, ctrl, BTAS_PATH_I32F64,
                                                          BTAS_PATH_I32F64);
      BTAS_CUDA_CHECK_LAUNCH();
      g32 = g;
      g32.Ap = Ap;
      g32.Bp = Bp;
      g32.Kp2 = Kp2;
      g32.mblocks = (int)(Mp / 128);
      g32.nblocks = (int)(Np / 128);
      g32.gate_value = BTAS_PATH_I32F64;
    }
  }
  GemmArgs g16{};  // int16x2 path (integer operands with |x| < 2^12)
  const int bn16 = 32 * s16_gn();
  if (int_mode) {
    const int64_t Kv = ceil_div(K, 2);              // words
    const int64_t Kp2 = round_up(Kv, 2 * kKP16) / 2;  // word pairs
    const int64_t Mp = round_up(M, 128), Np = round_up(N, bn16);
    uint32_t* Ap = reinterpret_cast<uint32_t*>(ws + L.packA);
    uint32_t* Bp = reinterpret_cast<uint32_t*>(ws + L.packB);
    dim3 ga((unsigned)ceil_div(2 * Kp2, 64), (unsigned)ceil_div(Mp, 32));
    pack_a_kernel<T, uint32_t, true, MIN, 128><<<ga, 256, 0, st>>>(A, lda, M, K, Kv, Kp2, Ap, ctrl,
                                                                    BTAS_PATH_S16X2, BTAS_PATH_S16X2);
    // B: virtual rows are words along k: rows of the virtual matrix = Kv
    const int64_t tb = Kp2 * Np;
    const unsigned gb = (unsigned)std::min<int64_t>(ceil_div(tb, 256), 65535);
    if (bn16 == 256)
      pack_b_kernel<T, uint32_t, true, MIN, 256><<<gb, 256, 0, st>>>(B, ldb, K, N, Np, Kp2, Bp, ctrl,
                                                                      BTAS_PATH_S16X2, BTAS_PATH_S16X2);
    else
      pack_b_kernel<T, uint32_t, true, MIN, 128><<<gb, 256, 0, st>>>(B, ldb, K, N, Np, Kp2, Bp, ctrl,
                                                                      BTAS_PATH_S16X2, BTAS_PATH_S16X2);
    BTAS_CUDA_CHECK_LAUNCH();
    g16 = g;
    g16.Ap = Ap;
    g16.Bp = Bp;
    g16.Kp2 = Kp2;
    g16.mblocks = (int)(Mp / 128);
    g16.nblocks = (int)(Np / bn16);
    g16.gate_value = BTAS_PATH_S16X2;
    g16.integer_mode = 1;
    g16.limit = limit;
  }
  // ---- the GEMM kernels: every path is launched, the gate runs exactly one
  cudaEvent_t t0;
  timing_begin(st, &t0);
  int rc;
  g.gate_value = fast;
  if constexpr (kIsF64) rc = launch_tropical_gemm<MixF64<MIN>, MIN>(g, st);
  else if constexpr (Traits<T>::dtype == BTAS_I32) rc = launch_tropical_gemm<MixI32<MIN>, MIN>(g, st);
  else rc = launch_tropical_gemm<MixF32<MIN>, MIN>(g, st);
  if (rc) return rc;
  g.gate_value = BTAS_PATH_CHECKED;
  rc = launch_tropical_gemm<MixChecked<T, MIN>, MIN>(g, st);
  if (rc) return rc;
  if (int_mode) {
    rc = launch_tropical_gemm<MixS16<MIN, T, 4>, MIN>(g16, st);
    if (rc) return rc;
    if constexpr (kIsF64) {
      rc = launch_tropical_gemm<MixI32F64<MIN>, MIN>(g32, st);
      if (rc) return rc;
    }
  }
  timing_end(st, t0);
  return BTAS_OK;
}


// predecessor product (MixArg): pack A and B (no screen, no gating: the
// operands are min-plus distances / adjacency whose sums the caller bounds)
// and run the argmin kernel; idx receives int32 k indices
template <class T>
int argmin_typed(const T* A, int64_t lda, const T* B, int64_t ldb, const T* Cref, int64_t ldcr, int64_t M, int64_t N,
                 int64_t K, int64_t row0, int32_t* idx, int64_t ldi, bool keys, unsigned char* ws, const WsLayout& L,
                 cudaStream_t st) {
  if (keys) {  // integer operands |x| < 2^12, K <= 2^16: packed (value, k) keys through VIADDMNMX
    using PK = MixArgKey<T>;
    const int64_t Kp2 = round_up(K, 2 * kKP) / 2;
    const int64_t Mp = round_up(M, 128), Np = round_up(N, 128);
    int32_t* Ap = reinterpret_cast<int32_t*>(ws + L.packA);
    int32_t* Bp = reinterpret_cast<int32_t*>(ws + L.packB);
    dim3 ga((unsigned)ceil_div(2 * Kp2, 64), (unsigned)ceil_div(Mp, 32));
    pack_a_kernel<T, int32_t, false, true, 128, 1><<<ga, 256, 0, st>>>(A, lda, M, K, 2 * Kp2, Kp2, Ap, nullptr, 0, 0);
    const int64_t tb = Kp2 * Np;
    pack_b_kernel<T, int32_t, false, true, 128, 2><<<(unsigned)std::min<int64_t>(ceil_div(tb, 256), 65535), 256, 0,
                                                     st>>>(B, ldb, K, N, Np, Kp2, Bp, nullptr, 0, 0);
    BTAS_CUDA_CHECK_LAUNCH();
    GemmArgs g{};
    g.Ap = Ap;
    g.Bp = Bp;
    g.Kp2 = Kp2;
    g.M = M;
    g.N = N;
    g.mblocks = (int)(Mp / 128);
    g.nblocks = (int)(Np / 128);
    g.C = idx;
    g.ldc = ldi;
    g.Cprev = Cref;
    g.ldcp = ldcr;
    g.arg_row0 = row0;
    return launch_gemm_epi<PK, true, kEpiCmp>(g, st);
  }
  using G = GemmGeometry<T>;
  using P = MixArg<T>;
  static_assert(P::GM * 32 == G::BM, "argmin tiles use the 32/64-bit packed geometry");
  const int64_t Kp2 = round_up(K, 2 * kKP) / 2;
  const int64_t Mp = round_up(M, G::BM), Np = round_up(N, G::BN);
  T* Ap = reinterpret_cast<T*>(ws + L.packA);
  T* Bp = reinterpret_cast<T*>(ws + L.packB);
  dim3 ga((unsigned)ceil_div(2 * Kp2, 64), (unsigned)ceil_div(Mp, 32));
  pack_a_kernel<T, T, false, true, G::BM><<<ga, 256, 0, st>>>(A, lda, M, K, 2 * Kp2, Kp2, Ap, nullptr, 0, 0);
  const int64_t tb = Kp2 * Np;
  pack_b_kernel<T, T, false, true, G::BN><<<(unsigned)std::min<int64_t>(ceil_div(tb, 256), 65535), 256, 0, st>>>(
      B, ldb, K, N, Np, Kp2, Bp, nullptr, 0, 0);
  BTAS_CUDA_CHECK_LAUNCH();
  GemmArgs g{};
  g.Ap = Ap;
  g.Bp = Bp;
  g.Kp2 = Kp2;
  g.M = M;
  g.N = N;
  g.mblocks = (int)(Mp / G::BM);
  g.nblocks = (int)(Np / G::BN);
  g.C = idx;
  g.ldc = ldi;
  g.Cprev = Cref;
  g.ldcp = ldcr;
  g.arg_row0 = row0;
  return launch_gemm_epi<P, true, kEpiCmp>(g, st);
}

}  // namespace
}  // namespace gemm_impl

// per-dtype drivers (one per translation unit)
#define BTAS_GEMM_DRIVER_DECL(T, NAME)                                                                       \
  int NAME(bool min_plus, int integer_mode, const T* A, int64_t lda, const T* B, int64_t ldb, const T* Z,      \
           int64_t ldz, T* C, int64_t ldc, int64_t M, int64_t N, int64_t K, const T* Cprev, int64_t ldcp,      \
           int32_t* flags, unsigned char* ws, const GemmExtras& x, cudaStream_t st)
BTAS_GEMM_DRIVER_DECL(float, gemm_f32);
BTAS_GEMM_DRIVER_DECL(int32_t, gemm_i32);
BTAS_GEMM_DRIVER_DECL(double, gemm_f64);
// the max-plus halves live in their own translation units (btas_gemm_*_max.cu)
// so the six kernel families compile in parallel
#define BTAS_GEMM_HALF_DECL(T, NAME)                                                                          \
  int NAME(int integer_mode, const T* A, int64_t lda, const T* B, int64_t ldb, const T* Z, int64_t ldz, T* C,    \
           int64_t ldc, int64_t M, int64_t N, int64_t K, const T* Cprev, int64_t ldcp, int32_t* flags,         \
           unsigned char* ws, const GemmExtras& x, cudaStream_t st)
BTAS_GEMM_HALF_DECL(float, gemm_f32_max);
BTAS_GEMM_HALF_DECL(int32_t, gemm_i32_max);
BTAS_GEMM_HALF_DECL(double, gemm_f64_max);
size_t gemm_ws_total(int dtype, int64_t M, int64_t N, int64_t K);
#define BTAS_ARGMIN_DECL(T, NAME)                                                                                \
  int NAME(const T* A, int64_t lda, const T* B, int64_t ldb, const T* Cref, int64_t ldcr, int64_t M, int64_t N,    \
           int64_t K, int64_t row0, int32_t* idx, int64_t ldi, bool keys, unsigned char* ws, cudaStream_t st)
BTAS_ARGMIN_DECL(float, argmin_f32);
BTAS_ARGMIN_DECL(int32_t, argmin_i32);
BTAS_ARGMIN_DECL(double, argmin_f64);

}  // namespace btas

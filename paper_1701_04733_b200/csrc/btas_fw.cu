// Blocked three-phase Floyd-Warshall, bit-identical to the reference's
// sequential k-round program (apsp.py:93-133).
//
// The reference round k is  d = min(d, add.outer(d[:,k], d[k,:]))  where the
// outer sum is formed from row/column k BEFORE the round updates anything
// (apsp.py:109).  The blocked schedule keeps exactly those operands:
//   phase 1  pivot tile K x K, b sequential rounds in shared memory; records the
//            pivot row/column snapshot of every round (rowsnapP, colsnapP).
//   phase 2  row panels (K x J) and column panels (I x K), b sequential rounds
//            each, driven by the pivot snapshots; every round's panel row /
//            column snapshot is emitted straight into the packed operand
//            layout of phase 3 (Srow, Scol) — 32-bit and int16x2 forms.
//   phase 3  D[I,J] = min(D[I,J], Scol[I,K] (x) Srow[K,J]) for all other tiles:
//            the tropical GEMM kernel with accumulate-in-place, K = b.
// Since min is exact and order-free and every candidate sum uses the same
// operands as the sequential round, D is byte-identical to the reference for
// f32/f64/i32 storage (the candidate sums are the same IEEE/int ops).
//
// Phase 3 runs the int16x2 DPX kernel whenever this round's snapshots all lie
// inside the s16 domain (decided on the device by phases 1/2, no host sync),
// otherwise the 32-bit kernel; the masked variant (reference screen failed)
// uses per-candidate overflow masking throughout.
#include <algorithm>

#include "btas_gemm.cuh"

namespace btas {
namespace {

struct FwCtrl {
  int32_t s16_overflow;  // this round's snapshots leave the s16 domain
  int32_t pad[63];
};

// relaxation candidate of one round
template <class T, bool CHECKED>
BTAS_D T fw_cand(T a, T b, int int_mode, double limit, bool& sat) {
  T s = a + b;
  if constexpr (CHECKED) {
    bool over;
    if constexpr (Traits<T>::dtype == BTAS_I32) over = (s >= (T)kI32Limit) || (s <= -(T)kI32Limit);
    else over = int_mode ? (fabs((double)s) >= limit) : isinf((double)s);
    if (over && Traits<T>::finite(a) && Traits<T>::finite(b)) {
      sat = true;
      return Traits<T>::eps(true);
    }
  }
  if constexpr (Traits<T>::dtype == BTAS_I32) {
    // canonical Inf; clamp inside negative cycles so int32 never wraps
    if (s >= (T)kI32Limit) return (T)kI32Inf;
    if (s < -(T)kI32Limit) return (T)(-kI32Limit);
  }
  return s;
}

template <class T>
BTAS_D T tmin(T a, T b) {
  return b < a ? b : a;
}

template <class T>
BTAS_D bool s16_ok(T v) {
  // representable as an s16 lane value: Infinity, or finite with |v| < 2^12
  return !Traits<T>::finite(v) || fabs((double)v) < (double)kS16Limit;
}

template <class T>
BTAS_D uint32_t s16_lane(T v) {
  const int x = Traits<T>::finite(v) ? (int)v : kS16Inf;  // FW is min-plus
  return (uint32_t)(uint16_t)(int16_t)x;
}

template <class T>
struct FwB {
  static constexpr int b = sizeof(T) == 8 ? 64 : 128;  // pivot block (phase-3 K)
};

struct FwArgs {
  int64_t n, ld, k0;
  int b;
  int nblk;
  int int_mode;
  double limit;
  int BMa, BNb;      // packed block sizes of the 32/64-bit GEMM operands
  int64_t Kp2;       // b / 2
  int64_t Kp2w;      // b / 4 (s16 word pairs)
  int emit_s16;      // also emit the int16x2 operands
  int32_t* flags;
  FwCtrl* ctrl;
};

// ------------------------------------------------------------------ phase 1
// smem: tile[b][b+1], rs[b][b] (row snapshots), cs[b][b] (col snapshots as [a][k'])
template <class T, bool CHECKED>
__global__ void __launch_bounds__(512) fw_phase1_kernel(T* __restrict__ D, T* __restrict__ rowsnapP,
                                                        T* __restrict__ colsnapP, T* __restrict__ Scol,
                                                        T* __restrict__ Srow, uint32_t* __restrict__ Scol16,
                                                        uint32_t* __restrict__ Srow16, FwArgs f) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int b = FwB<T>::b, bp = b + 1;
  T* tile = reinterpret_cast<T*>(smem_raw);
  T* rs = tile + b * bp;
  T* cs = rs + b * b;
  const T inf = Traits<T>::eps(true);
  if (threadIdx.x == 0) f.ctrl->s16_overflow = 0;
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int a = e / b, c = e - a * b;
    const int64_t i = f.k0 + a, j = f.k0 + c;
    tile[a * bp + c] = (i < f.n && j < f.n) ? D[i * f.ld + j] : inf;
  }
  bool sat = false;
  for (int k = 0; k < b; ++k) {
    __syncthreads();
    for (int c = threadIdx.x; c < b; c += blockDim.x) {
      rs[k * b + c] = tile[k * bp + c];
      cs[c * b + k] = tile[c * bp + k];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
      const int a = e / b, c = e - a * b;
      const T s = fw_cand<T, CHECKED>(cs[a * b + k], rs[k * b + c], f.int_mode, f.limit, sat);
      tile[a * bp + c] = tmin(tile[a * bp + c], s);
    }
  }
  __syncthreads();
  bool out16 = false;
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int a = e / b, c = e - a * b;
    const int64_t i = f.k0 + a, j = f.k0 + c;
    if (i < f.n && j < f.n) D[i * f.ld + j] = tile[a * bp + c];
    rowsnapP[e] = rs[e];
    colsnapP[e] = cs[e];
    // pivot rows of Scol (A operand: row i, k = c) and pivot cols of Srow (B: k = a, col j)
    Scol[packed_index(i, c, f.Kp2, f.BMa)] = cs[a * b + c];
    Srow[packed_index(f.k0 + c, a, f.Kp2, f.BNb)] = rs[a * b + c];
    out16 |= !s16_ok(cs[e]) || !s16_ok(rs[e]);
  }
  if (f.emit_s16) {
    // words: lanes (k even, k odd)
    for (int e = threadIdx.x; e < b * (b / 2); e += blockDim.x) {
      const int a = e / (b / 2), w = e - a * (b / 2);
      const int64_t i = f.k0 + a;
      Scol16[packed_index(i, w, f.Kp2w, 128)] = s16_lane(cs[a * b + 2 * w]) | (s16_lane(cs[a * b + 2 * w + 1]) << 16);
      const int64_t j = f.k0 + a;  // here a indexes the column
      Srow16[packed_index(j, w, f.Kp2w, 128)] =
          s16_lane(rs[(2 * w) * b + a]) | (s16_lane(rs[(2 * w + 1) * b + a]) << 16);
    }
  }
  if (__syncthreads_or(out16) && threadIdx.x == 0) atomicOr(&f.ctrl->s16_overflow, 1);
  if (CHECKED && __any_sync(0xffffffffu, sat) && (threadIdx.x & 31) == 0) atomicOr(&f.flags[BTAS_FLAG_SATURATED], 1);
}

// ------------------------------------------------------------------ phase 2
// blockIdx.y == 0: row panel (pivot rows, column block blockIdx.x)
// blockIdx.y == 1: column panel (row block blockIdx.x, pivot columns)
template <class T, bool CHECKED>
__global__ void __launch_bounds__(512) fw_phase2_kernel(T* __restrict__ D, const T* __restrict__ rowsnapP,
                                                        const T* __restrict__ colsnapP, T* __restrict__ Scol,
                                                        T* __restrict__ Srow, uint32_t* __restrict__ Scol16,
                                                        uint32_t* __restrict__ Srow16, FwArgs f) {
  const int blk = blockIdx.x;
  if (blk == (int)(f.k0 / f.b)) return;
  const bool row_panel = blockIdx.y == 0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int b = FwB<T>::b, bp = b + 1;
  T* tile = reinterpret_cast<T*>(smem_raw);
  T* ps = tile + b * bp;  // pivot snapshots (b x b)
  T* buf = ps + b * b;    // [2][b] this round's snapshot (double-buffered)
  const T inf = Traits<T>::eps(true);
  const int64_t r0 = row_panel ? f.k0 : (int64_t)blk * b;
  const int64_t c0 = row_panel ? (int64_t)blk * b : f.k0;
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int a = e / b, c = e - a * b;
    const int64_t i = r0 + a, j = c0 + c;
    tile[a * bp + c] = (i < f.n && j < f.n) ? D[i * f.ld + j] : inf;
    ps[e] = row_panel ? colsnapP[e] : rowsnapP[e];  // colsnapP[a][k'] / rowsnapP[k'][c]
  }
  bool sat = false, out16 = false;
  for (int k = 0; k < b; ++k) {
    T* cur = buf + (k & 1) * b;
    __syncthreads();
    for (int x = threadIdx.x; x < b; x += blockDim.x) cur[x] = row_panel ? tile[k * bp + x] : tile[x * bp + k];
    __syncthreads();
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
      const int a = e / b, c = e - a * b;
      const T s = row_panel ? fw_cand<T, CHECKED>(ps[a * b + k], cur[c], f.int_mode, f.limit, sat)
                            : fw_cand<T, CHECKED>(cur[a], ps[k * b + c], f.int_mode, f.limit, sat);
      tile[a * bp + c] = tmin(tile[a * bp + c], s);
    }
    // emit this round's snapshot (k = pivot index) into the phase-3 operands
    for (int x = threadIdx.x; x < b; x += blockDim.x) {
      const T v = cur[x];
      out16 |= !s16_ok(v);
      if (row_panel) Srow[packed_index(c0 + x, k, f.Kp2, f.BNb)] = v;
      else Scol[packed_index(r0 + x, k, f.Kp2, f.BMa)] = v;
      if (f.emit_s16 && (k & 1)) {
        const uint32_t w = s16_lane(buf[x]) | (s16_lane(v) << 16);
        if (row_panel) Srow16[packed_index(c0 + x, k >> 1, f.Kp2w, 128)] = w;
        else Scol16[packed_index(r0 + x, k >> 1, f.Kp2w, 128)] = w;
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int a = e / b, c = e - a * b;
    const int64_t i = r0 + a, j = c0 + c;
    if (i < f.n && j < f.n) D[i * f.ld + j] = tile[a * bp + c];
  }
  if (__syncthreads_or(out16) && threadIdx.x == 0) atomicOr(&f.ctrl->s16_overflow, 1);
  if (CHECKED && __any_sync(0xffffffffu, sat) && (threadIdx.x & 31) == 0) atomicOr(&f.flags[BTAS_FLAG_SATURATED], 1);
}

__global__ void fill_u32_kernel(uint32_t* p, int64_t n, uint32_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
template <class T>
__global__ void fill_t_kernel(T* p, int64_t n, T v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// ------------------------------------------------------------------ gating
// The 32-bit phase-3 kernel must run when snapshots left the s16 domain; the
// GEMM kernel gates on *gate == gate_value, so expose the flag as the gate.

template <class T>
struct FwGeom {
  static constexpr int b = FwB<T>::b;
  static constexpr int BMa = sizeof(T) == 8 ? 64 : 128;
  static constexpr int BNb = 128;
};

template <class T>
int64_t fw_rows(int64_t n) {
  using G = FwGeom<T>;
  const int64_t nb = ceil_div(n, G::b);
  return std::max<int64_t>(round_up(nb * G::b, G::BMa), round_up(nb * G::b, 128));
}
template <class T>
int64_t fw_cols(int64_t n) {
  using G = FwGeom<T>;
  const int64_t nb = ceil_div(n, G::b);
  return std::max<int64_t>(round_up(nb * G::b, G::BNb), round_up(nb * G::b, 128));
}

struct FwWs {
  size_t ctrl, rsp, csp, scol, srow, scol16, srow16, total;
};

inline size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

template <class T>
FwWs fw_ws(int64_t n) {
  using G = FwGeom<T>;
  const int64_t rows = fw_rows<T>(n), cols = fw_cols<T>(n);
  FwWs w;
  size_t off = 0;
  w.ctrl = off;
  off += a256(sizeof(FwCtrl));
  w.rsp = off;
  off += a256((size_t)G::b * G::b * sizeof(T));
  w.csp = off;
  off += a256((size_t)G::b * G::b * sizeof(T));
  w.scol = off;
  off += a256((size_t)rows * G::b * sizeof(T));
  w.srow = off;
  off += a256((size_t)cols * G::b * sizeof(T));
  w.scol16 = off;
  off += a256((size_t)rows * (G::b / 2) * 4);
  w.srow16 = off;
  off += a256((size_t)cols * (G::b / 2) * 4);
  w.total = off;
  return w;
}

template <class T, bool CHECKED>
int fw_typed(int integer_mode, T* D, int64_t ld, int64_t n, double max_abs, double min_finite, int32_t* flags,
             unsigned char* ws, cudaStream_t st) {
  using G = FwGeom<T>;
  const FwWs W = fw_ws<T>(n);
  const int b = G::b;
  const int nblk = (int)ceil_div(n, b);
  const bool int_mode = Traits<T>::dtype == BTAS_I32 || integer_mode;
  const double limit = Traits<T>::dtype == BTAS_I32 ? (double)kI32Limit : Traits<T>::int_limit;
  (void)max_abs;
  (void)min_finite;

  FwCtrl* ctrl = reinterpret_cast<FwCtrl*>(ws + W.ctrl);
  T* rsp = reinterpret_cast<T*>(ws + W.rsp);
  T* csp = reinterpret_cast<T*>(ws + W.csp);
  T* scol = reinterpret_cast<T*>(ws + W.scol);
  T* srow = reinterpret_cast<T*>(ws + W.srow);
  uint32_t* scol16 = reinterpret_cast<uint32_t*>(ws + W.scol16);
  uint32_t* srow16 = reinterpret_cast<uint32_t*>(ws + W.srow16);

  const int64_t rows = fw_rows<T>(n), cols = fw_cols<T>(n);
  // padding rows/cols of the packed operands hold Infinity
  {
    fill_t_kernel<T><<<1024, 256, 0, st>>>(scol, (int64_t)((W.scol16 - W.scol) / sizeof(T)), Traits<T>::eps(true));
    const uint32_t inf16 = (uint32_t)kS16Inf | ((uint32_t)kS16Inf << 16);
    fill_u32_kernel<<<1024, 256, 0, st>>>(scol16, (int64_t)((W.total - W.scol16) / 4), inf16);
  }
  const bool emit_s16 = int_mode && !CHECKED;

  FwArgs f{};
  f.n = n;
  f.ld = ld;
  f.b = b;
  f.nblk = nblk;
  f.int_mode = int_mode ? 1 : 0;
  f.limit = limit;
  f.BMa = G::BMa;
  f.BNb = G::BNb;
  f.Kp2 = b / 2;
  f.Kp2w = b / 4;
  f.emit_s16 = emit_s16 ? 1 : 0;
  f.flags = flags;
  f.ctrl = ctrl;

  const size_t smem1 = ((size_t)b * (b + 1) + 2 * (size_t)b * b) * sizeof(T);
  const size_t smem2 = ((size_t)b * (b + 1) + (size_t)b * b + 2 * (size_t)b) * sizeof(T);
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(fw_phase1_kernel<T, CHECKED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem1) != cudaSuccess ||
        cudaFuncSetAttribute(fw_phase2_kernel<T, CHECKED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem2) != cudaSuccess) {
      (void)cudaGetLastError();
      return BTAS_ERR_CUDA;
    }
    configured = true;
  }

  GemmArgs g{};
  g.Ap = scol;
  g.Bp = srow;
  g.Kp2 = b / 2;
  g.M = n;
  g.N = n;
  g.mblocks = (int)(rows / G::BMa);
  g.nblocks = (int)(cols / G::BNb);
  g.Z = D;
  g.ldz = ld;
  g.C = D;
  g.ldc = ld;
  g.Cprev = nullptr;
  g.flags = flags;
  g.integer_mode = int_mode ? 1 : 0;
  g.limit = int_mode ? limit : INFINITY;
  g.gate = emit_s16 ? &ctrl->s16_overflow : nullptr;
  g.gate_value = 1;

  GemmArgs g16 = g;
  g16.Ap = scol16;
  g16.Bp = srow16;
  g16.Kp2 = b / 4;
  g16.mblocks = (int)(round_up(rows, 128) / 128);
  g16.nblocks = (int)(round_up(cols, 128) / 128);
  g16.gate = &ctrl->s16_overflow;
  g16.gate_value = 0;
  g16.limit = limit;
  g16.integer_mode = 1;

  for (int kb = 0; kb < nblk; ++kb) {
    f.k0 = (int64_t)kb * b;
    fw_phase1_kernel<T, CHECKED><<<1, 512, smem1, st>>>(D, rsp, csp, scol, srow, scol16, srow16, f);
    if (nblk > 1) {
      fw_phase2_kernel<T, CHECKED><<<dim3(nblk, 2), 512, smem2, st>>>(D, rsp, csp, scol, srow, scol16, srow16, f);
    }
    BTAS_CUDA_CHECK_LAUNCH();
    if (nblk > 1) {
      g.skip_lo = g16.skip_lo = f.k0;
      g.skip_hi = g16.skip_hi = f.k0 + b;
      int rc;
      if constexpr (CHECKED) {
        rc = launch_tropical_gemm<MixChecked<T, true>, true>(g, st);
      } else if constexpr (Traits<T>::dtype == BTAS_F64) {
        rc = launch_tropical_gemm<MixF64<true>, true>(g, st);
      } else if constexpr (Traits<T>::dtype == BTAS_I32) {
        rc = launch_tropical_gemm<MixI32<true>, true>(g, st);
      } else {
        rc = launch_tropical_gemm<MixF32<true>, true>(g, st);
      }
      if (rc) return rc;
      if (emit_s16) {
        rc = launch_tropical_gemm<MixS16<true, T>, true>(g16, st);
        if (rc) return rc;
      }
    }
  }
  return BTAS_OK;
}

}  // namespace
}  // namespace btas

using namespace btas;

extern "C" size_t btas_fw_workspace_bytes(int dtype, int64_t n) {
  if (n < 1) return 0;
  switch (dtype) {
    case BTAS_F32:
      return fw_ws<float>(n).total;
    case BTAS_I32:
      return fw_ws<int32_t>(n).total;
    case BTAS_F64:
      return fw_ws<double>(n).total;
    default:
      return 0;
  }
}

extern "C" int btas_fw(int dtype, int integer_mode, void* D, int64_t ld, int64_t n, int masked, double max_abs,
                       double min_finite, int32_t* dev_flags, void* workspace, size_t workspace_bytes,
                       btas_stream_t stream) {
  if (!D || !dev_flags || !workspace || n < 1 || ld < n) return BTAS_ERR_INVALID;
  if (btas_fw_workspace_bytes(dtype, n) == 0) return BTAS_ERR_INVALID;
  if (workspace_bytes < btas_fw_workspace_bytes(dtype, n)) return BTAS_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  int rc;
#define BTAS_FW_CALL(T)                                                                                  \
  (masked ? fw_typed<T, true>(integer_mode, (T*)D, ld, n, max_abs, min_finite, dev_flags, ws, st)        \
          : fw_typed<T, false>(integer_mode, (T*)D, ld, n, max_abs, min_finite, dev_flags, ws, st))
  switch (dtype) {
    case BTAS_F32:
      rc = BTAS_FW_CALL(float);
      break;
    case BTAS_I32:
      rc = BTAS_FW_CALL(int32_t);
      break;
    default:
      rc = BTAS_FW_CALL(double);
      break;
  }
#undef BTAS_FW_CALL
  if (rc) return rc;
  return btas_diag_negative(dtype, D, ld, n, dev_flags, stream);
}

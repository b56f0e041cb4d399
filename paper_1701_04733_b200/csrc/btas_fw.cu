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
#include <cstdlib>
#include <type_traits>

#include "btas_gemm.cuh"

namespace btas {
namespace {

struct FwCtrl {
  // snapshots of some pivot block of the current lookahead group left the
  // s16 domain (reset by the group's first phase 1, OR-ed by every phase)
  int32_t s16_overflow[3];
  int32_t pad[61];  // 256 bytes
};

// ------------------------------------------------------------------ rounds
// Relaxation modes of one round's candidate d = min(d, a (x) b):
//   kFast     a + b straight into the add-min (VIADDMNMX / FADD+FMNMX):
//             int32 with no negative weight (values stay in [0, Inf]) and
//             every float storage (IEEE Inf absorbs)
//   kClamp    int32 with negative weights: canonical Inf, and a clamp at
//             -2^28 so a negative cycle can never wrap int32
//   kChecked  the reference's masked rounds (apsp.py:111-123)
enum { kFast = 0, kClamp = 1, kChecked = 2 };

template <class T, int MODE>
BTAS_D void relax(T& d, T a, T b, int int_mode, double limit, bool& sat) {
  if constexpr (MODE == kFast) {
    if constexpr (Traits<T>::dtype == BTAS_I32) {
      d = __viaddmin_s32(a, b, d);
    } else {
      const T s = a + b;
      d = s < d ? s : d;
    }
  } else {
    T s = a + b;
    if constexpr (MODE == kChecked) {
      bool over;
      if constexpr (Traits<T>::dtype == BTAS_I32) over = (s >= (T)kI32Limit) || (s <= -(T)kI32Limit);
      else over = int_mode ? (fabs((double)s) >= limit) : isinf((double)s);
      if (over && Traits<T>::finite(a) && Traits<T>::finite(b)) {
        sat = true;
        s = Traits<T>::eps(true);
      }
    }
    if constexpr (Traits<T>::dtype == BTAS_I32) {
      if (s >= (T)kI32Limit) s = (T)kI32Inf;
      if (s < -(T)kI32Limit) s = (T)(-kI32Limit);
    }
    d = s < d ? s : d;
  }
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
  int nblk;
  int int_mode;
  double limit;
  int BMa, BNb;      // packed block sizes of the 32/64-bit GEMM operands
  int64_t Kp2;       // k-pair stride of the packed panels (capacity: two pivot blocks = b)
  int64_t Kp2w;      // word-pair stride of the s16 panels (b / 2)
  int koff;          // k offset of this pivot block inside the panels (0 or b)
  int group_start;   // 1: first pivot block of a lookahead group (resets the s16 flag)
  // row slab held by this process: D points at global row slab_r0 and holds
  // rows [slab_r0, slab_r1) (single GPU: the whole matrix)
  int64_t slab_r0, slab_r1;
  int panel_mode;    // phase 2 grid: 0 = y selects row (0) / column (1) panels, 1 = rows only, 2 = columns only
  int col_blk0;      // first row block of the column panels (blockIdx.x offset)
  int emit_s16;      // also emit the int16x2 operands
  // phase 1 ORs its s16 flag into ctrl->s16_overflow[p1_slot]; slot 1 while
  // it runs concurrently with the thin passes gated on slot 0 (a flip of the
  // gate word in mid-launch would split a gated pair); the panel kernel that
  // follows the join folds slot 1 into slot 0 (fold_slot1)
  int p1_slot;
  int fold_slot1;
  // exact-integer distributed program: phase 1 writes the CLOSED pivot tile
  // T* (row-major, b x b) to its row-snapshot buffer (the broadcast slot)
  // instead of the row history, and column panels of ranks that do not hold
  // the pivot rows read T* from there (tstar) instead of from D
  int tstar_out;
  const void* tstar;
  int32_t* flags;
  FwCtrl* ctrl;
  // fused pivot-panel broadcast (distributed FW): every store into this
  // rank's broadcast region [region_lo, region_hi) is repeated at the same
  // offset in up to 7 peers' regions (the other ranks' workspaces, mapped
  // over NVLink / CUDA IPC), so the panel reaches them as it is produced
  unsigned char* region_lo;
  unsigned char* region_hi;
  unsigned char* peer_region[7];
  int n_peers;
};

// store v at p, and at the same region offset in every peer's workspace
template <class V>
BTAS_D void rstore(const FwArgs& f, V* p, V v) {
  *p = v;
  if (f.n_peers > 0) {
    const unsigned char* a = reinterpret_cast<const unsigned char*>(p);
    if (a >= f.region_lo && a < f.region_hi) {
      const size_t off = (size_t)(a - f.region_lo);
      for (int q = 0; q < f.n_peers; ++q) *reinterpret_cast<V*>(f.peer_region[q] + off) = v;
    }
  }
}
BTAS_D void rflag_or(const FwArgs& f, int32_t* p) {
  atomicOr(p, 1);
  if (f.n_peers > 0) {
    const unsigned char* a = reinterpret_cast<const unsigned char*>(p);
    if (a >= f.region_lo && a < f.region_hi) {
      const size_t off = (size_t)(a - f.region_lo);
      for (int q = 0; q < f.n_peers; ++q) atomicOr_system(reinterpret_cast<int32_t*>(f.peer_region[q] + off), 1);
    }
  }
}

// The tile lives in registers: thread (ty, tx) owns rows ty*RI .. +RI and
// cols tx*RJ .. +RJ (phase 1: 32 x 32 threads, phase 2: 16 x 32).  Round k:
// the owners of row k / column k publish the PRE-round values into the
// history arrays (which double as the round's operand buffers — written
// once, so one barrier per round), then every thread relaxes its block.
template <class T, int RI, int RJ>
BTAS_D void load_block(const T* __restrict__ D, const FwArgs& f, int64_t r0, int64_t c0, int ty, int tx,
                       T (&v)[RI][RJ]) {
  const T inf = Traits<T>::eps(true);
#pragma unroll
  for (int i = 0; i < RI; ++i) {
    const int64_t row = r0 + ty * RI + i;
#pragma unroll
    for (int j = 0; j < RJ; ++j) {
      const int64_t col = c0 + tx * RJ + j;
      v[i][j] = (row < f.slab_r1 && col < f.n) ? D[(row - f.slab_r0) * f.ld + col] : inf;
    }
  }
}

template <class T, int RI, int RJ>
BTAS_D void store_block(T* __restrict__ D, const FwArgs& f, int64_t r0, int64_t c0, int ty, int tx,
                        const T (&v)[RI][RJ]) {
#pragma unroll
  for (int i = 0; i < RI; ++i) {
    const int64_t row = r0 + ty * RI + i;
#pragma unroll
    for (int j = 0; j < RJ; ++j) {
      const int64_t col = c0 + tx * RJ + j;
      if (row < f.slab_r1 && col < f.n) D[(row - f.slab_r0) * f.ld + col] = v[i][j];
    }
  }
}

// packed phase-3 operands from a history array h[k][x] (k = pivot round,
// x = row (A operand, Scol) or col (B operand, Srow) inside the block at rc0)
template <class T, int HS = FwB<T>::b>
BTAS_D bool emit_history(const T* __restrict__ h, int64_t rc0, int BLK, const FwArgs& f, T* __restrict__ P,
                         uint32_t* __restrict__ P16) {
  constexpr int b = FwB<T>::b;  // HS: row stride of h (padded histories avoid bank conflicts)
  // rc0 is a multiple of b and b divides the packing blocks, so the b
  // rows/columns stay inside one packed block: packed_index(rc0 + x, koff +
  // 2 kp, Kp2, BLK) = base + (kp * BLK + x) * 2 with the divisions done once
  const int64_t blk = rc0 / BLK, roff = rc0 - blk * BLK;
  T* Pb = P + ((blk * f.Kp2 + f.koff / 2) * BLK + roff) * 2;
  bool out16 = false;
  for (int e = threadIdx.x; e < (b / 2) * b; e += blockDim.x) {
    const int kp = e / b, x = e - kp * b;
    const T v0 = h[(2 * kp) * HS + x], v1 = h[(2 * kp + 1) * HS + x];
    const int64_t idx = ((int64_t)kp * BLK + x) * 2;
    rstore(f, Pb + idx, v0);
    rstore(f, Pb + idx + 1, v1);
    out16 |= !s16_ok(v0) || !s16_ok(v1);
  }
  if (f.emit_s16) {
    const int64_t blk16 = rc0 / 128, roff16 = rc0 - blk16 * 128;
    uint32_t* P16b = P16 + ((blk16 * f.Kp2w + f.koff / 4) * 128 + roff16) * 2;
    for (int e = threadIdx.x; e < (b / 4) * b; e += blockDim.x) {
      const int wp = e / b, x = e - wp * b;
      const int k = 4 * wp;
      const uint32_t w0 = s16_lane(h[k * HS + x]) | (s16_lane(h[(k + 1) * HS + x]) << 16);
      const uint32_t w1 = s16_lane(h[(k + 2) * HS + x]) | (s16_lane(h[(k + 3) * HS + x]) << 16);
      const int64_t idx = ((int64_t)wp * 128 + x) * 2;
      rstore(f, P16b + idx, w0);
      rstore(f, P16b + idx + 1, w1);
    }
  }
  return out16;
}

// ------------------------------------------------------------------ phase 1
// smem: rs[k][c] (pivot-row history), cT[k][a] (pivot-column history)
// One CTA of 16 x 32 threads (RI x RJ = 8 x 4 values each, b = 128; 4 x 2
// for b = 64): the b sequential rounds are barrier-latency-bound, so the
// pivot tile is spread over 16 warps (32 warps of 4 x 4: 1-2 us slower per
// pivot block, profiles/r02_ab_phase1_threads.txt).
#ifndef BTAS_FW1_THREADS
#define BTAS_FW1_THREADS 512
#endif
constexpr int kFw1Threads = BTAS_FW1_THREADS;
#ifndef BTAS_FW_OVERLAP_P1_MIN_BLOCKS
#define BTAS_FW_OVERLAP_P1_MIN_BLOCKS 128
#endif
constexpr int kOverlapP1MinBlocks = BTAS_FW_OVERLAP_P1_MIN_BLOCKS;  // n >= 16384 at b = 128

// env BTAS_FW_OVERLAP_P1_MIN_BLOCKS overrides the threshold (tests force the
// overlapped schedule on small graphs; read per call, it is one getenv)
inline int overlap_p1_min_blocks() {
  const char* e = getenv("BTAS_FW_OVERLAP_P1_MIN_BLOCKS");
  const int v = e ? atoi(e) : 0;
  return v > 0 ? v : kOverlapP1MinBlocks;
}

template <class T>
struct Fw1 {
  static constexpr int b = FwB<T>::b, TY = kFw1Threads / 32, RI = b / TY, RJ = b / 32;
  static constexpr int U = RI > RJ ? RI : RJ;  // rounds per unrolled step (both owners static)
};

template <class T, int MODE>
__global__ void __launch_bounds__(kFw1Threads) fw_phase1_kernel(T* __restrict__ D, T* __restrict__ rowsnapP,
                                                                T* __restrict__ colsnapT, T* __restrict__ Scol,
                                                                T* __restrict__ Srow, uint32_t* __restrict__ Scol16,
                                                                uint32_t* __restrict__ Srow16, FwArgs f) {
  constexpr int b = Fw1<T>::b, RI = Fw1<T>::RI, RJ = Fw1<T>::RJ, U = Fw1<T>::U;
  static_assert(U % RI == 0 && U % RJ == 0, "round unroll covers both owners");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* rs = reinterpret_cast<T*>(smem_raw);
  T* cT = rs + b * b;
  const int ty = threadIdx.x >> 5, tx = threadIdx.x & 31;
  if (threadIdx.x == 0 && f.group_start) {
    rstore(f, &f.ctrl->s16_overflow[0], 0);
    rstore(f, &f.ctrl->s16_overflow[1], 0);
  }
  T v[RI][RJ];
  load_block(D, f, f.k0, f.k0, ty, tx, v);
  bool sat = false;
  for (int kb = 0; kb < b; kb += U) {
#pragma unroll
    for (int kk = 0; kk < U; ++kk) {
      const int k = kb + kk;
      if (ty == k / RI) {
#pragma unroll
        for (int j = 0; j < RJ; ++j) rs[k * b + tx * RJ + j] = v[kk % RI][j];
      }
      if (tx == k / RJ) {
#pragma unroll
        for (int i = 0; i < RI; ++i) cT[k * b + ty * RI + i] = v[i][kk % RJ];
      }
      __syncthreads();
      T rowv[RJ], colv[RI];
#pragma unroll
      for (int j = 0; j < RJ; ++j) rowv[j] = rs[k * b + tx * RJ + j];
#pragma unroll
      for (int i = 0; i < RI; ++i) colv[i] = cT[k * b + ty * RI + i];
#pragma unroll
      for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < RJ; ++j) relax<T, MODE>(v[i][j], colv[i], rowv[j], f.int_mode, f.limit, sat);
    }
  }
  store_block(D, f, f.k0, f.k0, ty, tx, v);
  if (f.tstar_out) {  // the closed tile, row-major (padding rows/cols hold Infinity)
#pragma unroll
    for (int i = 0; i < RI; ++i)
#pragma unroll
      for (int j = 0; j < RJ; ++j) rstore(f, rowsnapP + (ty * RI + i) * b + tx * RJ + j, v[i][j]);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    if (!f.tstar_out) rstore(f, rowsnapP + e, rs[e]);
    rstore(f, colsnapT + e, cT[e]);
  }
  // pivot rows of Scol (A operand) and pivot columns of Srow (B operand)
  bool out16 = emit_history(cT, f.k0 - f.slab_r0, f.BMa, f, Scol, Scol16);  // Scol rows are slab-local
  out16 |= emit_history(rs, f.k0, f.BNb, f, Srow, Srow16);
  if (__syncthreads_or(out16) && threadIdx.x == 0) {
    rflag_or(f, &f.ctrl->s16_overflow[f.p1_slot]);
  }
  if (MODE == kChecked && __any_sync(0xffffffffu, sat) && (threadIdx.x & 31) == 0)
    atomicOr(&f.flags[BTAS_FLAG_SATURATED], 1);
}

// ------------------------------------------------------------------ phase 2
// blockIdx.y == 0: row panel (pivot rows x column block blockIdx.x): own
//                  operand = its row k each round, fixed = pivot-column snapshot
// blockIdx.y == 1: column panel (row block blockIdx.x x pivot columns)
// The fixed operand of every round (the pivot tile's column / row snapshot,
// 64 KB, identical for all CTAs) is read through L1 one round ahead instead
// of being staged in shared memory: a CTA needs only its own history array,
// so two CTAs share an SM and phase 2's latency-bound rounds overlap.
template <class T, int N>
BTAS_D void load_fixed(const T* __restrict__ src, int k, int x0, T (&out)[N]) {
  constexpr int b = FwB<T>::b;
  const T* p = src + (int64_t)k * b + x0;
  if constexpr (N * sizeof(T) % 16 == 0) {
#pragma unroll
    for (int q = 0; q < N * (int)sizeof(T) / 16; ++q) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(p) + q);
      const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
      for (int i = 0; i < 16 / (int)sizeof(T); ++i) out[q * (16 / sizeof(T)) + i] = e[i];
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = __ldg(p + i);
  }
}

// phase-2 thread grid: 16 x 32 threads, RI x RJ values each
constexpr int kFw2Threads = 512;
template <class T>
struct Fw2 {
  static constexpr int RI = FwB<T>::b / 16, RJ = FwB<T>::b / 32;
};

// the b rounds of one panel tile.  Row panel: each round's own operand is
// the tile's row k (history, per column), the fixed one the pivot column
// snapshot (per row).  Column panel: own = the tile's column k (per row),
// fixed = the pivot row snapshot (per column).
template <class T, int MODE, bool ROW>
BTAS_D void phase2_rounds(T (&v)[Fw2<T>::RI][Fw2<T>::RJ], T* hist, const T* __restrict__ fixedg, int ty, int tx,
                          const FwArgs& f, bool& sat) {
  constexpr int b = FwB<T>::b, RI = Fw2<T>::RI, RJ = Fw2<T>::RJ;
  constexpr int NF = ROW ? RI : RJ;  // fixed operand per thread
  constexpr int NO = ROW ? RJ : RI;  // own operand per thread
  constexpr int STEP = ROW ? RI : RJ;  // rounds owned by one thread row / column
  const int fx0 = ROW ? ty * RI : tx * RJ;
  const int ox0 = ROW ? tx * RJ : ty * RI;
  T fx[NF];
  load_fixed(fixedg, 0, fx0, fx);
  for (int kb = 0; kb < b; kb += STEP) {
    const int owner = kb / STEP;
#pragma unroll
    for (int kk = 0; kk < STEP; ++kk) {
      const int k = kb + kk;
      if (ROW) {
        if (ty == owner) {
#pragma unroll
          for (int j = 0; j < RJ; ++j) hist[k * b + tx * RJ + j] = v[kk][j];
        }
      } else {
        if (tx == owner) {
#pragma unroll
          for (int i = 0; i < RI; ++i) hist[k * b + ty * RI + i] = v[i][kk];
        }
      }
      T fxn[NF];
      if (k + 1 < b) load_fixed(fixedg, k + 1, fx0, fxn);  // next round's fixed operand, in flight
      __syncthreads();
      T own[NO];
#pragma unroll
      for (int j = 0; j < NO; ++j) own[j] = hist[k * b + ox0 + j];
#pragma unroll
      for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < RJ; ++j) {
          if (ROW) relax<T, MODE>(v[i][j], fx[i], own[j], f.int_mode, f.limit, sat);
          else relax<T, MODE>(v[i][j], own[i], fx[j], f.int_mode, f.limit, sat);
        }
      if (k + 1 < b) {
#pragma unroll
        for (int i = 0; i < NF; ++i) fx[i] = fxn[i];
      }
    }
  }
}

template <class T, int MODE>
__global__ void __launch_bounds__(kFw2Threads, MODE == kChecked ? 1 : 2)
    fw_phase2_kernel(T* __restrict__ D, const T* __restrict__ rowsnapP, const T* __restrict__ colsnapT,
                     T* __restrict__ Scol, T* __restrict__ Srow, uint32_t* __restrict__ Scol16,
                     uint32_t* __restrict__ Srow16, FwArgs f) {
  constexpr int b = FwB<T>::b, RI = Fw2<T>::RI, RJ = Fw2<T>::RJ;
  const bool row_panel = f.panel_mode == 0 ? blockIdx.y == 0 : f.panel_mode == 1;
  const int blk = row_panel ? (int)blockIdx.x : f.col_blk0 + (int)blockIdx.x;
  if (blk == (int)(f.k0 / b)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* hist = reinterpret_cast<T*>(smem_raw);  // row panel: rs[k][c]; col panel: cT[k][a]
  const int ty = threadIdx.x >> 5, tx = threadIdx.x & 31;
  const int64_t r0 = row_panel ? f.k0 : (int64_t)blk * b;
  const int64_t c0 = row_panel ? (int64_t)blk * b : f.k0;
  T v[RI][RJ];
  load_block(D, f, r0, c0, ty, tx, v);
  bool sat = false;
  if (row_panel) phase2_rounds<T, MODE, true>(v, hist, colsnapT, ty, tx, f, sat);
  else phase2_rounds<T, MODE, false>(v, hist, rowsnapP, ty, tx, f, sat);
  store_block(D, f, r0, c0, ty, tx, v);
  __syncthreads();
  const bool out16 = row_panel ? emit_history(hist, c0, f.BNb, f, Srow, Srow16)
                               : emit_history(hist, r0 - f.slab_r0, f.BMa, f, Scol, Scol16);
  if (__syncthreads_or(out16) && threadIdx.x == 0) {
    rflag_or(f, &f.ctrl->s16_overflow[0]);
  }
  if (MODE == kChecked && __any_sync(0xffffffffu, sat) && (threadIdx.x & 31) == 0)
    atomicOr(&f.flags[BTAS_FLAG_SATURATED], 1);
}

// ------------------------------------------------------------------ phase 2, exact integers
// For exact integer data without negative weights (every candidate an exact
// integer, no negative cycle) the distances do not depend on how the
// candidates are grouped, so the panels take the standard blocked-FW update
// with the closed pivot tile T* that phase 1 left in D:
//   row panel  P' = T* (x) P        column panel  C' = C (x) T*
// (T* has a zero diagonal, so the old value is among the candidates) — one
// min-plus product per 128 x 128 tile instead of b barrier-separated rounds,
// and the FINAL panels are emitted as the phase-3 operands.  Any candidate is
// the length of a real path and every candidate the sequential program uses
// is still formed, so D is the same bytes.
template <class T>
struct FwP {
  static constexpr int b = FwB<T>::b, RI = b / 16, RJ = b / 32;  // 512 threads, RI x RJ outputs each
};
constexpr int kFwPThreads = 512;

template <class T>
__global__ void __launch_bounds__(kFwPThreads, 1) fw_panel_kernel(T* __restrict__ D, T* __restrict__ Scol,
                                                                  T* __restrict__ Srow, uint32_t* __restrict__ Scol16,
                                                                  uint32_t* __restrict__ Srow16, FwArgs f) {
  constexpr int b = FwP<T>::b, RI = FwP<T>::RI, RJ = FwP<T>::RJ;
  const bool row_panel = blockIdx.y == 0;
  const int blk = (int)blockIdx.x;
  if (blk == (int)(f.k0 / b)) return;
  // Ls (the transposed left operand) has an odd row stride, so the
  // transposed stores of a warp hit 32 distinct banks; its reads are warp
  // broadcasts (scalar).  Rs and the history keep 16-byte aligned rows.
  constexpr int LS = b + 1, S = b + 16 / (int)sizeof(T);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Ls = reinterpret_cast<T*>(smem_raw);  // left operand, transposed: Ls[m][i]
  T* Rs = Ls + b * S;                      // right operand: Rs[m][x] (Ls occupies b * LS <= b * S)
  const T inf = Traits<T>::eps(true);
  const int64_t r0 = row_panel ? f.k0 : (int64_t)blk * b;  // the tile's rows / columns in D
  const int64_t c0 = row_panel ? (int64_t)blk * b : f.k0;
  // loads: all of a thread's elements are fetched before any shared-memory
  // store (a load-store loop serialised one memory latency per element)
  constexpr int kPer = b * b / kFwPThreads;  // elements per thread per operand
  T xv[kPer], tv[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = (int)threadIdx.x + u * kFwPThreads;
    const int i = e / b, j = e % b;
    xv[u] = (r0 + i < f.n && c0 + j < f.n) ? D[(r0 + i - f.slab_r0) * f.ld + c0 + j] : inf;
    tv[u] = (f.k0 + i < f.n && f.k0 + j < f.n) ? D[(f.k0 + i - f.slab_r0) * f.ld + f.k0 + j] : inf;
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = (int)threadIdx.x + u * kFwPThreads;
    const int i = e / b, j = e % b;
    if (row_panel) {  // P' = T* (x) P: left T*[k][m], right P[m][x]
      Ls[j * LS + i] = tv[u];
      Rs[i * S + j] = xv[u];
    } else {  // C' = C (x) T*: left C[x][m], right T*[m][k]
      Ls[j * LS + i] = xv[u];
      Rs[i * S + j] = tv[u];
    }
  }
  __syncthreads();
  const int ty = threadIdx.x >> 5, tx = threadIdx.x & 31;
  T acc[RI][RJ];
#pragma unroll
  for (int i = 0; i < RI; ++i)
#pragma unroll
    for (int j = 0; j < RJ; ++j) acc[i][j] = inf;
  bool sat = false;
#pragma unroll 4
  for (int m = 0; m < b; ++m) {
    T l[RI], r[RJ];
#pragma unroll
    for (int i = 0; i < RI; ++i) l[i] = Ls[m * LS + ty * RI + i];  // broadcast within the warp
#pragma unroll
    for (int j = 0; j < RJ; ++j) r[j] = Rs[m * S + tx * RJ + j];
#pragma unroll
    for (int i = 0; i < RI; ++i)
#pragma unroll
      for (int j = 0; j < RJ; ++j) relax<T, kFast>(acc[i][j], l[i], r[j], f.int_mode, f.limit, sat);
  }
  __syncthreads();  // Ls becomes the emission history h[k][x]
  T* h = Ls;
#pragma unroll
  for (int i = 0; i < RI; ++i)
#pragma unroll
    for (int j = 0; j < RJ; ++j) {
      const int oi = ty * RI + i, oj = tx * RJ + j;  // output row / column inside the tile
      const int64_t row = r0 + oi, col = c0 + oj;
      if (row < f.n && col < f.n) D[(row - f.slab_r0) * f.ld + col] = acc[i][j];
      // h[k][x] (row stride S): k along the pivot block, x along the panel
      if (row_panel) h[oi * S + oj] = acc[i][j];
      else h[oj * S + oi] = acc[i][j];
    }
  __syncthreads();
  const bool out16 = row_panel ? emit_history<T, S>(h, c0, f.BNb, f, Srow, Srow16)
                               : emit_history<T, S>(h, r0 - f.slab_r0, f.BMa, f, Scol, Scol16);
  if (__syncthreads_or(out16) && threadIdx.x == 0) rflag_or(f, &f.ctrl->s16_overflow[0]);
}

// Half-tile panels for 4-byte storage (b = 128): CTA (blk, half) computes
// 64 output rows of one panel tile with 256 threads and 100 KB of shared
// memory, so two CTAs share an SM and one CTA's operand loads and emission
// overlap the other's add-min loop (the full-tile kernel above runs one
// 135 KB CTA per SM: load, compute, emit in sequence).  Per k: the left
// operand's 8 rows of a warp are two broadcast LDS.128, the right operand's
// 4 columns of a lane are strided (x = lane + 32 j), so those reads, the D
// stores and both history layouts are bank-conflict free.
constexpr int kFwHThreads = 256;
template <class T>
struct FwH {
  static constexpr int b = 128, HR = 64;         // pivot block, output rows per CTA
  static constexpr int LS = HR + 4, RS = b + 4;  // 16-byte aligned row strides
  static constexpr size_t smem = (size_t)(b * LS + b * RS) * sizeof(T);
};

// packed phase-3 operands from a partial history h[k - k_lo][x - x_lo]
// (k in [k_lo, k_lo + KN), x in [x_lo, x_lo + XN)), as emit_history
template <class T, int HS, int KN, int XN>
BTAS_D bool emit_part(const T* __restrict__ h, int k_lo, int x_lo, int64_t rc0, int BLK, const FwArgs& f,
                      T* __restrict__ P, uint32_t* __restrict__ P16) {
  const int64_t blk = rc0 / BLK, roff = rc0 - blk * BLK;
  T* Pb = P + ((blk * f.Kp2 + f.koff / 2) * BLK + roff) * 2;
  bool out16 = false;
  for (int e = threadIdx.x; e < (KN / 2) * XN; e += blockDim.x) {
    const int kp = e / XN, xl = e - kp * XN;
    const T v0 = h[(2 * kp) * HS + xl], v1 = h[(2 * kp + 1) * HS + xl];
    const int64_t idx = ((int64_t)(k_lo / 2 + kp) * BLK + x_lo + xl) * 2;
    rstore(f, Pb + idx, v0);
    rstore(f, Pb + idx + 1, v1);
    out16 |= !s16_ok(v0) || !s16_ok(v1);
  }
  if (f.emit_s16) {
    const int64_t blk16 = rc0 / 128, roff16 = rc0 - blk16 * 128;
    uint32_t* P16b = P16 + ((blk16 * f.Kp2w + f.koff / 4) * 128 + roff16) * 2;
    for (int e = threadIdx.x; e < (KN / 4) * XN; e += blockDim.x) {
      const int wp = e / XN, xl = e - wp * XN;
      const int k = 4 * wp;
      const uint32_t w0 = s16_lane(h[k * HS + xl]) | (s16_lane(h[(k + 1) * HS + xl]) << 16);
      const uint32_t w1 = s16_lane(h[(k + 2) * HS + xl]) | (s16_lane(h[(k + 3) * HS + xl]) << 16);
      const int64_t idx = ((int64_t)(k_lo / 4 + wp) * 128 + x_lo + xl) * 2;
      rstore(f, P16b + idx, w0);
      rstore(f, P16b + idx + 1, w1);
    }
  }
  return out16;
}

template <class T>
__global__ void __launch_bounds__(kFwHThreads, 2) fw_panel_half_kernel(T* __restrict__ D, T* __restrict__ Scol,
                                                                       T* __restrict__ Srow,
                                                                       uint32_t* __restrict__ Scol16,
                                                                       uint32_t* __restrict__ Srow16, FwArgs f) {
  static_assert(sizeof(T) == 4, "b = 128 storage");
  constexpr int b = FwH<T>::b, HR = FwH<T>::HR, LS = FwH<T>::LS, RS = FwH<T>::RS;
  const bool row_panel = f.panel_mode == 0 ? blockIdx.y == 0 : f.panel_mode == 1;
  const int blk = (row_panel ? 0 : f.col_blk0) + (int)(blockIdx.x >> 1), half = (int)(blockIdx.x & 1);
  if (f.fold_slot1 && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 &&
      *reinterpret_cast<volatile int32_t*>(&f.ctrl->s16_overflow[1]) != 0)
    rflag_or(f, &f.ctrl->s16_overflow[0]);
  if (blk == (int)(f.k0 / b)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Ls = reinterpret_cast<T*>(smem_raw);  // Ls[m][i] = left[i][m]
  T* Rs = Ls + b * LS;                     // Rs[m][x] = right[m][x]
  const T inf = Traits<T>::eps(true);
  const int w = (int)threadIdx.x >> 5, lane = (int)threadIdx.x & 31;
  // the tile in D; row panel P' = T* (x) P, column panel C' = C (x) T*.
  // left[i][m] = D[lr0 + i][k0 + m] (T* rows / C rows of this half),
  // right[m][x] = D[k0 + m][rc0 + x] (P / T*)
  const int64_t r0 = row_panel ? f.k0 : (int64_t)blk * b;
  const int64_t c0 = row_panel ? (int64_t)blk * b : f.k0;
  const int64_t lr0 = (row_panel ? f.k0 : r0) + half * HR;
  const int64_t rc0 = row_panel ? c0 : f.k0;
  auto at = [&](int64_t row, int64_t col) -> T {
    return (row < f.slab_r1 && col < f.n) ? D[(row - f.slab_r0) * f.ld + col] : inf;
  };
  // the right operand of a column panel is T*: from D, or from the
  // broadcast copy when this rank does not hold the pivot rows
  const T* tstar = (!row_panel && f.tstar) ? static_cast<const T*>(f.tstar) : nullptr;
  {  // left operand: a warp reads 4 rows x 8 columns (four full 32-byte
     // sectors) and stores them transposed into 32 distinct banks
    constexpr int kQ = HR * b / 32 / (kFwHThreads / 32);  // patches per warp
    T v[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int p = w + 8 * q;
      const int i = 4 * (p & 15) + (lane & 3), m = 8 * (p >> 4) + (lane >> 2);
      v[q] = at(lr0 + i, f.k0 + m);
    }
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int p = w + 8 * q;
      const int i = 4 * (p & 15) + (lane & 3), m = 8 * (p >> 4) + (lane >> 2);
      Ls[m * LS + i] = v[q];
    }
  }
  {  // right operand: row-major, 4 consecutive columns per thread
    constexpr int kQ = b * b / 4 / kFwHThreads;
    const bool vec = (f.ld % 4) == 0 && (reinterpret_cast<uintptr_t>(D) % 16) == 0 && rc0 + b <= f.n;
    uint4 v[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int e = (int)threadIdx.x + kFwHThreads * q;
      const int m = e >> 5, x = 4 * (e & 31);
      const int64_t row = f.k0 + m;
      if (tstar != nullptr) {
        v[q] = *reinterpret_cast<const uint4*>(tstar + m * b + x);
      } else if (vec && row < f.slab_r1) {
        v[q] = *reinterpret_cast<const uint4*>(D + (row - f.slab_r0) * f.ld + rc0 + x);
      } else {
        v[q].x = __builtin_bit_cast(uint32_t, at(row, rc0 + x));
        v[q].y = __builtin_bit_cast(uint32_t, at(row, rc0 + x + 1));
        v[q].z = __builtin_bit_cast(uint32_t, at(row, rc0 + x + 2));
        v[q].w = __builtin_bit_cast(uint32_t, at(row, rc0 + x + 3));
      }
    }
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int e = (int)threadIdx.x + kFwHThreads * q;
      const int m = e >> 5, x = 4 * (e & 31);
      *reinterpret_cast<uint4*>(Rs + m * RS + x) = v[q];
    }
  }
  __syncthreads();
  T acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = inf;
  bool sat = false;
#pragma unroll 4
  for (int m = 0; m < b; ++m) {
    T l[8], r[4];
    lds4(Ls + m * LS + w * 8, l);  // broadcast within the warp
    lds4(Ls + m * LS + w * 8 + 4, l + 4);
#pragma unroll
    for (int j = 0; j < 4; ++j) r[j] = Rs[m * RS + lane + 32 * j];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) relax<T, kFast>(acc[i][j], l[i], r[j], f.int_mode, f.limit, sat);
  }
  __syncthreads();  // the operand buffers become the emission history
  T* h = Ls;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int orow = half * HR + w * 8 + i;  // output row inside the tile
    const int64_t row = r0 + orow;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int x = lane + 32 * j;
      if (row < f.slab_r1 && c0 + x < f.n) D[(row - f.slab_r0) * f.ld + c0 + x] = acc[i][j];
      if (row_panel) h[(w * 8 + i) * RS + x] = acc[i][j];  // h[k - 64 half][x]
    }
  }
  if (!row_panel) {  // h[k][x - 64 half] = C'[x][k]: 8 consecutive x per (thread, k)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      T* hp = h + (lane + 32 * j) * LS + w * 8;
      *reinterpret_cast<uint4*>(hp) = make_uint4(
          __builtin_bit_cast(uint32_t, acc[0][j]), __builtin_bit_cast(uint32_t, acc[1][j]),
          __builtin_bit_cast(uint32_t, acc[2][j]), __builtin_bit_cast(uint32_t, acc[3][j]));
      *reinterpret_cast<uint4*>(hp + 4) = make_uint4(
          __builtin_bit_cast(uint32_t, acc[4][j]), __builtin_bit_cast(uint32_t, acc[5][j]),
          __builtin_bit_cast(uint32_t, acc[6][j]), __builtin_bit_cast(uint32_t, acc[7][j]));
    }
  }
  __syncthreads();
  const bool out16 = row_panel ? emit_part<T, RS, HR, b>(h, half * HR, 0, c0, f.BNb, f, Srow, Srow16)
                               : emit_part<T, LS, b, HR>(h, 0, half * HR, r0 - f.slab_r0, f.BMa, f, Scol, Scol16);
  if (__syncthreads_or(out16) && threadIdx.x == 0) rflag_or(f, &f.ctrl->s16_overflow[0]);
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
  // lookahead group size: 4-byte storage has b == every GEMM tile edge
  static constexpr int look = sizeof(T) == 4 ? 8 : 1;
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
  off += a256((size_t)rows * G::look * G::b * sizeof(T));  // kLook pivot blocks of k
  w.srow = off;
  off += a256((size_t)cols * G::look * G::b * sizeof(T));
  w.scol16 = off;
  off += a256((size_t)rows * G::look * G::b / 2 * 4);
  w.srow16 = off;
  off += a256((size_t)cols * G::look * G::b / 2 * 4);
  w.total = off;
  return w;
}

template <class T, int MODE>
int fw_typed(int integer_mode, T* D, int64_t ld, int64_t n, double max_abs, double min_finite, int32_t* flags,
             unsigned char* ws, cudaStream_t st) {
  using G = FwGeom<T>;
  using T4 = std::conditional_t<sizeof(T) == 4, T, float>;  // the half-tile panel kernel's storage
  const FwWs W = fw_ws<T>(n);
  const int b = G::b;
  const int nblk = (int)ceil_div(n, b);
  const bool int_mode = Traits<T>::dtype == BTAS_I32 || integer_mode;
  const double limit = Traits<T>::dtype == BTAS_I32 ? (double)kI32Limit : Traits<T>::int_limit;
  constexpr bool CHECKED = MODE == kChecked;
  constexpr int kLook = G::look;

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
  // the s16x2 phase-3 kernel streams 32 word pairs per stage: b = 128 (4-byte
  // storage) only
  const bool emit_s16 = int_mode && !CHECKED && sizeof(T) == 4;

  FwArgs f{};
  f.n = n;
  f.ld = ld;
  f.slab_r0 = 0;
  f.slab_r1 = n;
  f.nblk = nblk;
  f.int_mode = int_mode ? 1 : 0;
  f.limit = limit;
  f.BMa = G::BMa;
  f.BNb = G::BNb;
  f.Kp2 = (int64_t)kLook * b / 2;  // panels hold kLook pivot blocks of k
  f.Kp2w = (int64_t)kLook * b / 4;
  f.emit_s16 = emit_s16 ? 1 : 0;
  f.flags = flags;
  f.ctrl = ctrl;

  const size_t smem1 = 2 * (size_t)b * b * sizeof(T);
  const size_t smem2 = (size_t)b * b * sizeof(T);  // phase 2: the history array only
  const size_t smemP = 2 * (size_t)b * (b + 16 / sizeof(T)) * sizeof(T);  // exact-integer panels: both operands
  static unsigned long long configured = 0;
  if (!configured_on_current_device(configured)) {
    if (cudaFuncSetAttribute(fw_phase1_kernel<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem1) != cudaSuccess ||
        cudaFuncSetAttribute(fw_phase2_kernel<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem2) != cudaSuccess ||
        cudaFuncSetAttribute(fw_panel_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemP) !=
            cudaSuccess ||
        (sizeof(T) == 4 && cudaFuncSetAttribute(fw_panel_half_kernel<T4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)FwH<T4>::smem) != cudaSuccess)) {
      (void)cudaGetLastError();
      return BTAS_ERR_CUDA;
    }
    mark_configured(configured);
  }
  // exact integers without negative weights: the panel products
  // (fw_panel_kernel) replace the b sequential phase-2 rounds
  const bool exact_panels =
      MODE == kFast && !CHECKED &&
      (Traits<T>::dtype == BTAS_I32 ||
       (integer_mode && (Traits<T>::dtype == BTAS_F64 || 2.0 * (double)(n + 1) * max_abs < 16777216.0)));

  // base GEMM descriptors over the full D; per launch only the k range
  // (which half of the panels), the row/col window and the skip ranges change
  GemmArgs g{};
  g.Ap = scol;
  g.Bp = srow;
  g.Kp2 = b / 2;
  g.Kp2s = (int64_t)kLook * b / 2;
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
  g.gate_value = 1;
  g.no_diag = 1;  // windows below offset C; FW tests the diagonal once at the end
  GemmArgs g16 = g;
  g16.Ap = scol16;
  g16.Bp = srow16;
  g16.Kp2 = b / 4;
  g16.Kp2s = (int64_t)kLook * b / 4;
  g16.mblocks = (int)(round_up(rows, 128) / 128);
  g16.nblocks = (int)(round_up(cols, 128) / 128);
  g16.gate_value = 0;
  g16.limit = limit;
  g16.integer_mode = 1;

  // one phase-3 style update over K = halves * b (pivot-block slots
  // [0, halves) of the panels): 32-bit kernel gated on "s16 overflow",
  // s16x2 kernel gated on "no overflow"
  auto phase3_on = [&](GemmArgs a, GemmArgs a16, int halves, cudaStream_t s) -> int {
    a.Kp2 = (int64_t)halves * b / 2;
    a16.Kp2 = (int64_t)halves * b / 4;
    a.gate = emit_s16 ? &ctrl->s16_overflow[0] : nullptr;
    a16.gate = &ctrl->s16_overflow[0];
    int rc;
    if constexpr (CHECKED) {
      rc = launch_gemm_epi<MixChecked<T, true>, true, kEpiAcc>(a, s);
    } else if constexpr (Traits<T>::dtype == BTAS_F64) {
      rc = launch_gemm_epi<MixF64<true>, true, kEpiAcc>(a, s);
    } else if constexpr (Traits<T>::dtype == BTAS_I32) {
      rc = launch_gemm_epi<MixI32<true>, true, kEpiAcc>(a, s);
    } else {
      rc = launch_gemm_epi<MixF32<true>, true, kEpiAcc>(a, s);
    }
    if (rc) return rc;
    if (emit_s16) rc = launch_gemm_epi<MixS16<true, T>, true, kEpiAcc>(a16, s);
    return rc;
  };
  auto phase3 = [&](GemmArgs a, GemmArgs a16, int halves) -> int { return phase3_on(a, a16, halves, st); };
  // The row- and column-panel thin passes of a pivot block touch disjoint
  // tiles and each fills only n/128 CTAs: the column pass runs on a side
  // stream, forked from and joined back into the caller's stream (per host
  // thread and device, created once), so both share the SMs.
  cudaStream_t side = nullptr, side2 = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr, join_ev2 = nullptr;
  {
    // created together or not at all (a partial set is destroyed and the
    // device is marked so creation is not retried on every call); they live
    // for the thread's lifetime
    thread_local cudaStream_t t_side[64] = {}, t_side2[64] = {};
    thread_local cudaEvent_t t_fork[64] = {}, t_join[64] = {}, t_join2[64] = {};
    thread_local bool t_failed[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64) {
      if (!t_side[dev] && !t_failed[dev]) {
        cudaStream_t s = nullptr, s2 = nullptr;
        cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&e0, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&e1, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&e2, cudaEventDisableTiming) == cudaSuccess) {
          t_side[dev] = s;
          t_side2[dev] = s2;
          t_fork[dev] = e0;
          t_join[dev] = e1;
          t_join2[dev] = e2;
        } else {
          (void)cudaGetLastError();
          if (e1) cudaEventDestroy(e1);
          if (e0) cudaEventDestroy(e0);
          if (s2) cudaStreamDestroy(s2);
          if (s) cudaStreamDestroy(s);
          t_failed[dev] = true;
        }
      }
      side = t_side[dev];
      side2 = t_side2[dev];
      fork_ev = t_fork[dev];
      join_ev = t_join[dev];
      join_ev2 = t_join2[dev];
    } else {
      (void)cudaGetLastError();
    }
  }
  // Joins the side stream back into the caller's stream on every exit from
  // a forked region, including early error returns, so the caller's stream
  // is always ordered after the side stream's work.
  struct Join {
    cudaStream_t st = nullptr, side = nullptr;
    cudaEvent_t ev = nullptr;
    bool open = false;
    int close() {
      if (!open) return BTAS_OK;
      open = false;
      if (cudaEventRecord(ev, side) != cudaSuccess || cudaStreamWaitEvent(st, ev, 0) != cudaSuccess) {
        (void)cudaGetLastError();
        return BTAS_ERR_CUDA;
      }
      return BTAS_OK;
    }
    ~Join() { (void)close(); }
  };
  auto phase1 = [&](int kb, int slot, int p1_slot) -> int {
    f.k0 = (int64_t)kb * b;
    f.koff = slot * b;
    f.group_start = slot == 0;
    f.p1_slot = p1_slot;
    fw_phase1_kernel<T, MODE><<<1, kFw1Threads, smem1, st>>>(D, rsp, csp, scol, srow, scol16, srow16, f);
    BTAS_CUDA_CHECK_LAUNCH();
    return BTAS_OK;
  };
  auto phase2 = [&](int fold_slot1) -> int {
    f.fold_slot1 = fold_slot1;
    if (nblk > 1) {
      if (exact_panels && sizeof(T) == 4)
        fw_panel_half_kernel<T4><<<dim3(2 * nblk, 2), kFwHThreads, FwH<T4>::smem, st>>>(
            reinterpret_cast<T4*>(D), reinterpret_cast<T4*>(scol), reinterpret_cast<T4*>(srow), scol16, srow16, f);
      else if (exact_panels)
        fw_panel_kernel<T><<<dim3(nblk, 2), kFwPThreads, smemP, st>>>(D, scol, srow, scol16, srow16, f);
      else
        fw_phase2_kernel<T, MODE><<<dim3(nblk, 2), kFw2Threads, smem2, st>>>(D, rsp, csp, scol, srow, scol16,
                                                                            srow16, f);
    }
    f.fold_slot1 = 0;
    BTAS_CUDA_CHECK_LAUNCH();
    return BTAS_OK;
  };
  auto phases12 = [&](int kb, int slot) -> int {
    int r = phase1(kb, slot, 0);
    return r ? r : phase2(0);
  };
  // Large graphs: the pivot tile's pending update runs first and phase 1
  // (one CTA, b dependent rounds) overlaps the rest of the thin passes,
  // which run on the two side streams with their persistent grids capped
  // one SM short (the thin passes span several waves there, phase 1 was
  // serial after them).  Exact-integer panels on 4-byte storage only (the
  // panel kernel folds phase 1's s16 flag word back in).
  const bool overlap_p1 = exact_panels && sizeof(T) == 4 && side != nullptr && side2 != nullptr &&
                          nblk >= overlap_p1_min_blocks();

  // Lookahead groups of kLook pivot blocks (4-byte storage, where b equals
  // the GEMM tile edge).  Inside a group, block kb0+j's row and column
  // panels first receive the pending updates of blocks kb0..kb0+j-1 (thin
  // passes, K = j*b) — exactly what its phases 1/2 read — and every other
  // tile receives all kLook updates at the end in ONE pass with K = kLook*b.
  // Each candidate is formed from the same per-round snapshots as in the
  // sequential program and min is order-free (re-applying a block's
  // candidates to a tile that already has them changes nothing), so D is
  // unchanged; the bulk pass does kLook times the add-min work per epilogue.
  int rc;
  for (int kb0 = 0; kb0 < nblk; kb0 += kLook) {
    const int m = std::min(kLook, nblk - kb0);
    for (int j = 0; j < m; ++j) {
      const int kb = kb0 + j;
      const int64_t kk = (int64_t)kb * b, mk = std::min<int64_t>(b, n - kk);
      if (j > 0 && overlap_p1) {
        if (cudaEventRecord(fork_ev, st) != cudaSuccess || cudaStreamWaitEvent(side, fork_ev, 0) != cudaSuccess ||
            cudaStreamWaitEvent(side2, fork_ev, 0) != cudaSuccess) {
          (void)cudaGetLastError();
          return BTAS_ERR_CUDA;
        }
        Join join1, join2;
        join1.st = join2.st = st;
        join1.side = side;
        join1.ev = join_ev;
        join2.side = side2;
        join2.ev = join_ev2;
        join1.open = join2.open = true;
        const int sms = device_sm_count();
        {  // pending updates -> row block kb except the pivot tile (side stream 1)
          GemmArgs a = g, a16 = g16;
          a.M = a16.M = mk;
          a.mblocks = a16.mblocks = 1;
          a.Ap = static_cast<const T*>(g.Ap) + (size_t)kb * g.Kp2s * G::BMa * 2;
          a16.Ap = static_cast<const uint32_t*>(g16.Ap) + (size_t)kb * g16.Kp2s * 128 * 2;
          a.C = a16.C = D + kk * ld;
          a.Z = a16.Z = D + kk * ld;
          a.skip_col_lo = a16.skip_col_lo = kk;
          a.skip_col_hi = a16.skip_col_hi = kk + b;
          a.max_ctas = a16.max_ctas = sms / 2;
          if ((rc = phase3_on(a, a16, j, side))) return rc;
        }
        {  // pending updates -> column block kb outside the pivot rows (side stream 2)
          GemmArgs a = g, a16 = g16;
          a.N = a16.N = mk;
          a.nblocks = a16.nblocks = 1;
          a.Bp = static_cast<const T*>(g.Bp) + (size_t)kb * g.Kp2s * G::BNb * 2;
          a16.Bp = static_cast<const uint32_t*>(g16.Bp) + (size_t)kb * g16.Kp2s * 128 * 2;
          a.C = a16.C = D + kk;
          a.Z = a16.Z = D + kk;
          a.skip_row_lo = a16.skip_row_lo = kk;
          a.skip_row_hi = a16.skip_row_hi = kk + b;
          a.max_ctas = a16.max_ctas = sms - 1 - sms / 2;
          if ((rc = phase3_on(a, a16, j, side2))) return rc;
        }
        {  // pending updates -> the pivot tile, then phase 1, on the caller's stream
          GemmArgs a = g, a16 = g16;
          a.M = a16.M = a.N = a16.N = mk;
          a.mblocks = a16.mblocks = a.nblocks = a16.nblocks = 1;
          a.Ap = static_cast<const T*>(g.Ap) + (size_t)kb * g.Kp2s * G::BMa * 2;
          a16.Ap = static_cast<const uint32_t*>(g16.Ap) + (size_t)kb * g16.Kp2s * 128 * 2;
          a.Bp = static_cast<const T*>(g.Bp) + (size_t)kb * g.Kp2s * G::BNb * 2;
          a16.Bp = static_cast<const uint32_t*>(g16.Bp) + (size_t)kb * g16.Kp2s * 128 * 2;
          a.C = a16.C = D + kk * ld + kk;
          a.Z = a16.Z = D + kk * ld + kk;
          if ((rc = phase3(a, a16, j))) return rc;
        }
        if ((rc = phase1(kb, j, 1))) return rc;
        if ((rc = join1.close()) || (rc = join2.close())) return rc;
        if ((rc = phase2(1))) return rc;
        continue;
      }
      if (j > 0) {
        const bool fork = side != nullptr;
        Join join;
        if (fork) {
          if (cudaEventRecord(fork_ev, st) != cudaSuccess || cudaStreamWaitEvent(side, fork_ev, 0) != cudaSuccess) {
            (void)cudaGetLastError();
            return BTAS_ERR_CUDA;
          }
          join.st = st;
          join.side = side;
          join.ev = join_ev;
          join.open = true;
        }
        {  // pending updates -> row block kb
          GemmArgs a = g, a16 = g16;
          a.M = a16.M = mk;
          a.mblocks = a16.mblocks = 1;
          a.Ap = static_cast<const T*>(g.Ap) + (size_t)kb * g.Kp2s * G::BMa * 2;
          a16.Ap = static_cast<const uint32_t*>(g16.Ap) + (size_t)kb * g16.Kp2s * 128 * 2;
          a.C = a16.C = D + kk * ld;
          a.Z = a16.Z = D + kk * ld;
          if ((rc = phase3(a, a16, j))) return rc;
        }
        {  // pending updates -> column block kb outside the pivot rows (disjoint from the row pass)
          GemmArgs a = g, a16 = g16;
          a.N = a16.N = mk;
          a.nblocks = a16.nblocks = 1;
          a.Bp = static_cast<const T*>(g.Bp) + (size_t)kb * g.Kp2s * G::BNb * 2;
          a16.Bp = static_cast<const uint32_t*>(g16.Bp) + (size_t)kb * g16.Kp2s * 128 * 2;
          a.C = a16.C = D + kk;
          a.Z = a16.Z = D + kk;
          a.skip_row_lo = a16.skip_row_lo = kk;
          a.skip_row_hi = a16.skip_row_hi = kk + b;
          if ((rc = phase3_on(a, a16, j, fork ? side : st))) return rc;
        }
        if ((rc = join.close())) return rc;
      }
      if ((rc = phases12(kb, j))) return rc;
    }
    if (nblk == 1) break;
    // all kLook updates on every tile outside the last block's row/col panels
    const int64_t kl = (int64_t)(kb0 + m - 1) * b;
    GemmArgs a = g, a16 = g16;
    a.skip_row_lo = a16.skip_row_lo = a.skip_col_lo = a16.skip_col_lo = kl;
    a.skip_row_hi = a16.skip_row_hi = a.skip_col_hi = a16.skip_col_hi = kl + b;
    if ((rc = phase3(a, a16, m))) return rc;
  }
  return BTAS_OK;
}

// ------------------------------------------------------------------ distributed
// Row-slab Floyd-Warshall for P processes (one per GPU) with the single-GPU
// lookahead.  Pivot blocks are taken in GROUPS of up to G::look consecutive
// blocks that lie inside one rank's slab (the owner).  Per group:
//   OWNER (owner only): for each block j of the group, the pending updates
//     of the group's earlier blocks go into the block's row panel and into
//     its column panel over the owner's rows (thin passes, K = j*b), then
//     phase 1, the row panel (phase 2, emits Srow slot j) and the column
//     panel over the owner's rows (emits Scol slot j);
//   exchange: the owner's "broadcast region" — the s16 flag, the pivot-row
//     snapshots of every block of the group and the packed Srow slots in both
//     forms — reaches every rank: stored into the peers' regions by the
//     owner's kernels as they produce it (fused, btas_fw_dist_group_peers)
//     or one NCCL broadcast per group; the host orders REST after it;
//   REST (every rank): a non-owner runs, for each block j, the thin pass of
//     the earlier blocks into its column panel rows and the column panel
//     itself (emits its Scol slot j); then every rank applies all the
//     group's blocks to its rows in ONE GEMM pass with K = m*b.
// The candidates are those of the single-GPU program (same per-round
// snapshots; re-applying a block's candidates is a no-op under min), so D is
// byte-identical for any P, and the bulk pass does m times the add-min work
// per epilogue with one exchange per group instead of per block.
struct FwDistWs {
  size_t ctrl, rsp, srow, srow16, bcast_end, csp, scol, scol16, total;
};

template <class T>
FwDistWs fw_dist_ws(int64_t n, int64_t slab_rows) {
  using G = FwGeom<T>;
  const int64_t rows = std::max<int64_t>(round_up(std::max<int64_t>(slab_rows, 1), 128), G::b);
  const int64_t cols = fw_cols<T>(n);
  FwDistWs w;
  size_t off = 0;
  w.ctrl = off;
  off += a256(sizeof(FwCtrl));
  w.rsp = off;  // pivot-row snapshots of every block of the group
  off += a256((size_t)G::look * G::b * G::b * sizeof(T));
  w.srow = off;
  off += a256((size_t)cols * G::look * G::b * sizeof(T));
  w.srow16 = off;
  off += a256((size_t)cols * G::look * (G::b / 2) * 4);
  w.bcast_end = off;
  w.csp = off;  // pivot-column snapshot (owner-local)
  off += a256((size_t)G::b * G::b * sizeof(T));
  w.scol = off;
  off += a256((size_t)rows * G::look * G::b * sizeof(T));
  w.scol16 = off;
  off += a256((size_t)rows * G::look * (G::b / 2) * 4);
  w.total = off;
  return w;
}

template <class T, int MODE>
int fw_dist_group_typed(int integer_mode, int stage, T* D, int64_t ld, int64_t n, int64_t slab_r0,
                        int64_t slab_rows, int64_t kb0, int m, int32_t* flags, unsigned char* ws, void* const* peers,
                        int n_peers, cudaStream_t st) {
  using G = FwGeom<T>;
  using T4 = std::conditional_t<sizeof(T) == 4, T, float>;  // the half-tile panel kernel's storage
  constexpr int b = G::b, kLook = G::look;
  constexpr bool CHECKED = MODE == kChecked;
  const FwDistWs W = fw_dist_ws<T>(n, slab_rows);
  const int nblk = (int)ceil_div(n, b);
  const bool int_mode = Traits<T>::dtype == BTAS_I32 || integer_mode;
  const double limit = Traits<T>::dtype == BTAS_I32 ? (double)kI32Limit : Traits<T>::int_limit;
  // the s16x2 phase-3 kernel streams 32 word pairs per stage: b = 128 (4-byte
  // storage) only
  const bool emit_s16 = int_mode && !CHECKED && sizeof(T) == 4;
  FwCtrl* ctrl = reinterpret_cast<FwCtrl*>(ws + W.ctrl);
  T* rsp = reinterpret_cast<T*>(ws + W.rsp);
  T* csp = reinterpret_cast<T*>(ws + W.csp);
  T* srow = reinterpret_cast<T*>(ws + W.srow);
  uint32_t* srow16 = reinterpret_cast<uint32_t*>(ws + W.srow16);
  T* scol = reinterpret_cast<T*>(ws + W.scol);
  uint32_t* scol16 = reinterpret_cast<uint32_t*>(ws + W.scol16);
  const int64_t rows_pad = (int64_t)((W.scol16 - W.scol) / sizeof(T)) / ((int64_t)kLook * b);
  const int64_t cols = fw_cols<T>(n);
  const int64_t k_lo = kb0 * b, k_hi = std::min<int64_t>(n, (kb0 + m) * b);
  const bool owner = slab_rows > 0 && k_lo >= slab_r0 && k_lo < slab_r0 + slab_rows;
  if (stage != BTAS_FW_STAGE_INIT && stage != BTAS_FW_STAGE_DIAG) {
    if (m < 1 || m > kLook || kb0 < 0 || k_lo >= n) return BTAS_ERR_INVALID;
    if (owner && k_hi > slab_r0 + slab_rows) return BTAS_ERR_INVALID;  // a group never spans two slabs
    if (stage == BTAS_FW_STAGE_OWNER && !owner) return BTAS_ERR_INVALID;
  }

  FwArgs f{};
  f.n = n;
  f.ld = ld;
  f.slab_r0 = slab_r0;
  f.slab_r1 = slab_r0 + slab_rows;
  f.nblk = nblk;
  f.int_mode = int_mode ? 1 : 0;
  f.limit = limit;
  f.BMa = G::BMa;
  f.BNb = G::BNb;
  f.Kp2 = (int64_t)kLook * b / 2;  // panels hold kLook pivot blocks of k
  f.Kp2w = (int64_t)kLook * b / 4;
  f.emit_s16 = emit_s16 ? 1 : 0;
  f.flags = flags;
  f.ctrl = ctrl;
  f.region_lo = ws + W.ctrl;
  f.region_hi = ws + W.bcast_end;
  f.n_peers = n_peers;
  for (int q = 0; q < n_peers; ++q) f.peer_region[q] = static_cast<unsigned char*>(peers[q]);
  const size_t smem = 2 * (size_t)b * b * sizeof(T);
  const size_t smem2 = (size_t)b * b * sizeof(T);
  static unsigned long long configured = 0;
  if (!configured_on_current_device(configured)) {
    if (cudaFuncSetAttribute(fw_phase1_kernel<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(fw_phase2_kernel<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2) !=
            cudaSuccess ||
        (sizeof(T) == 4 && cudaFuncSetAttribute(fw_panel_half_kernel<T4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)FwH<T4>::smem) != cudaSuccess)) {
      (void)cudaGetLastError();
      return BTAS_ERR_CUDA;
    }
    mark_configured(configured);
  }
  // int32 storage without negative weights: the exact-integer panel products
  // (fw_panel_half_kernel) as in btas_fw; phase 1 broadcasts the closed pivot
  // tile T* in the row-snapshot slot, from which the other ranks' column
  // panels read it
  const bool exact = MODE == kFast && !CHECKED && Traits<T>::dtype == BTAS_I32;
  f.tstar_out = exact ? 1 : 0;

  // GEMM descriptors over this rank's slab (rows slab-local); per launch only
  // the k range (slots), the row/column window and the skips change
  GemmArgs g{};
  g.Ap = scol;
  g.Bp = srow;
  g.Kp2 = b / 2;
  g.Kp2s = (int64_t)kLook * b / 2;
  g.M = slab_rows;
  g.N = n;
  g.mblocks = (int)(rows_pad / G::BMa);
  g.nblocks = (int)(cols / G::BNb);
  g.Z = D;
  g.ldz = ld;
  g.C = D;
  g.ldc = ld;
  g.flags = flags;
  g.integer_mode = int_mode ? 1 : 0;
  g.limit = int_mode ? limit : INFINITY;
  g.gate = emit_s16 ? &ctrl->s16_overflow[0] : nullptr;
  g.gate_value = 1;
  g.no_diag = 1;
  g.skip_row_lo = g.skip_row_hi = g.skip_col_lo = g.skip_col_hi = 0;
  GemmArgs g16 = g;
  g16.Ap = scol16;
  g16.Bp = srow16;
  g16.Kp2 = b / 4;
  g16.Kp2s = (int64_t)kLook * b / 4;
  g16.mblocks = (int)(round_up(rows_pad, 128) / 128);
  g16.nblocks = (int)(round_up(cols, 128) / 128);
  g16.gate = &ctrl->s16_overflow[0];
  g16.gate_value = 0;
  g16.limit = limit;
  g16.integer_mode = 1;
  // one update over K = slots * b (group slots [0, slots)): 32-bit kernel
  // gated on "s16 overflow", s16x2 kernel gated on "no overflow"
  auto update = [&](GemmArgs a, GemmArgs a16, int slots) -> int {
    a.Kp2 = (int64_t)slots * b / 2;
    a16.Kp2 = (int64_t)slots * b / 4;
    int rc;
    if constexpr (CHECKED) rc = launch_gemm_epi<MixChecked<T, true>, true, kEpiAcc>(a, st);
    else if constexpr (Traits<T>::dtype == BTAS_F64) rc = launch_gemm_epi<MixF64<true>, true, kEpiAcc>(a, st);
    else if constexpr (Traits<T>::dtype == BTAS_I32) rc = launch_gemm_epi<MixI32<true>, true, kEpiAcc>(a, st);
    else rc = launch_gemm_epi<MixF32<true>, true, kEpiAcc>(a, st);
    if (rc) return rc;
    if (emit_s16) rc = launch_gemm_epi<MixS16<true, T>, true, kEpiAcc>(a16, st);
    return rc;
  };
  // pending updates (slots 0..j-1) -> column block kb over this rank's rows
  // (the owner skips the block's own rows: the row pass covers them)
  auto thin_cols = [&](int64_t kb, int j) -> int {
    const int64_t kk = kb * b;
    GemmArgs a = g, a16 = g16;
    a.N = a16.N = std::min<int64_t>(b, n - kk);
    a.nblocks = a16.nblocks = 1;
    a.Bp = srow + (size_t)kb * g.Kp2s * G::BNb * 2;
    a16.Bp = srow16 + (size_t)kb * g16.Kp2s * 128 * 2;
    a.C = a16.C = D + kk;
    a.Z = a16.Z = D + kk;
    if (owner) {
      a.skip_row_lo = a16.skip_row_lo = kk - slab_r0;
      a.skip_row_hi = a16.skip_row_hi = kk - slab_r0 + b;
    }
    return update(a, a16, j);
  };
  // phase 2 column panel over this rank's row blocks for block kb (slot j)
  auto cols_panel = [&](int64_t kb, int j) -> int {
    if (nblk == 1) return BTAS_OK;
    FwArgs fc = f;
    fc.k0 = kb * b;
    fc.koff = j * b;
    fc.group_start = 0;
    fc.panel_mode = 2;
    fc.col_blk0 = (int)(slab_r0 / b);
    fc.n_peers = 0;  // column panels are rank-local
    const int nsb = (int)ceil_div(slab_rows, b);
    if (exact) {
      fc.tstar = owner ? nullptr : rsp + (size_t)j * b * b;  // the owner's column panel reads T* from D
      fw_panel_half_kernel<T4><<<dim3(2 * nsb, 1), kFwHThreads, FwH<T4>::smem, st>>>(
          reinterpret_cast<T4*>(D), reinterpret_cast<T4*>(scol), reinterpret_cast<T4*>(srow), scol16, srow16, fc);
    } else {
      fw_phase2_kernel<T, MODE><<<dim3(nsb, 1), kFw2Threads, smem2, st>>>(D, rsp + (size_t)j * b * b, csp, scol,
                                                                         srow, scol16, srow16, fc);
    }
    BTAS_CUDA_CHECK_LAUNCH();
    return BTAS_OK;
  };
  int rc;
  switch (stage) {
    case BTAS_FW_STAGE_INIT: {
      // packed panels: padding rows/cols hold Infinity
      fill_t_kernel<T><<<1024, 256, 0, st>>>(srow, (int64_t)((W.srow16 - W.srow) / sizeof(T)), Traits<T>::eps(true));
      fill_t_kernel<T><<<1024, 256, 0, st>>>(scol, (int64_t)((W.scol16 - W.scol) / sizeof(T)), Traits<T>::eps(true));
      const uint32_t inf16 = (uint32_t)kS16Inf | ((uint32_t)kS16Inf << 16);
      fill_u32_kernel<<<1024, 256, 0, st>>>(srow16, (int64_t)((W.bcast_end - W.srow16) / 4), inf16);
      fill_u32_kernel<<<1024, 256, 0, st>>>(scol16, (int64_t)((W.total - W.scol16) / 4), inf16);
      break;
    }
    case BTAS_FW_STAGE_OWNER: {
      for (int j = 0; j < m; ++j) {
        const int64_t kb = kb0 + j, kk = kb * b;
        if (j > 0) {
          {  // pending updates -> row panel kb (pivot rows x every column)
            GemmArgs a = g, a16 = g16;
            a.M = a16.M = std::min<int64_t>(b, n - kk);
            a.mblocks = a16.mblocks = 1;
            a.Ap = scol + (size_t)((kk - slab_r0) / G::BMa) * g.Kp2s * G::BMa * 2;
            a16.Ap = scol16 + (size_t)((kk - slab_r0) / 128) * g16.Kp2s * 128 * 2;
            a.C = a16.C = D + (kk - slab_r0) * ld;
            a.Z = a16.Z = D + (kk - slab_r0) * ld;
            if ((rc = update(a, a16, j))) return rc;
          }
          if ((rc = thin_cols(kb, j))) return rc;
        }
        FwArgs fp = f;
        fp.k0 = kk;
        fp.koff = j * b;
        fp.group_start = j == 0;
        T* rsp_j = rsp + (size_t)j * b * b;
        fw_phase1_kernel<T, MODE><<<1, kFw1Threads, smem, st>>>(D, rsp_j, csp, scol, srow, scol16, srow16, fp);
        if (nblk > 1) {
          fp.panel_mode = 1;
          if (exact)
            fw_panel_half_kernel<T4><<<dim3(2 * nblk, 1), kFwHThreads, FwH<T4>::smem, st>>>(
                reinterpret_cast<T4*>(D), reinterpret_cast<T4*>(scol), reinterpret_cast<T4*>(srow), scol16, srow16,
                fp);
          else
            fw_phase2_kernel<T, MODE><<<dim3(nblk, 1), kFw2Threads, smem2, st>>>(D, rsp_j, csp, scol, srow, scol16,
                                                                                srow16, fp);
        }
        BTAS_CUDA_CHECK_LAUNCH();
        if ((rc = cols_panel(kb, j))) return rc;
      }
      break;
    }
    case BTAS_FW_STAGE_REST: {
      if (slab_rows == 0) break;
      if (!owner) {
        for (int j = 0; j < m; ++j) {
          if (j > 0 && (rc = thin_cols(kb0 + j, j))) return rc;
          if ((rc = cols_panel(kb0 + j, j))) return rc;
        }
      }
      if (nblk == 1) break;
      // every group block on every tile of this rank outside the last
      // block's row/column panels, K = m*b in one pass
      const int64_t kl = (kb0 + m - 1) * b;
      GemmArgs a = g, a16 = g16;
      a.skip_col_lo = a16.skip_col_lo = kl;
      a.skip_col_hi = a16.skip_col_hi = kl + b;
      if (owner) {
        a.skip_row_lo = a16.skip_row_lo = kl - slab_r0;
        a.skip_row_hi = a16.skip_row_hi = kl - slab_r0 + b;
      }
      if ((rc = update(a, a16, m))) return rc;
      break;
    }
    case BTAS_FW_STAGE_DIAG:
      if (slab_rows > 0) return btas_diag_negative(Traits<T>::dtype, D + slab_r0, ld, slab_rows, flags, st);
      break;
    default:
      return BTAS_ERR_INVALID;
  }
  BTAS_CUDA_CHECK_LAUNCH();
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
  // int32 with a negative weight needs the clamped rounds; floats never do
#define BTAS_FW_CALL(T)                                                                                      \
  (masked ? fw_typed<T, kChecked>(integer_mode, (T*)D, ld, n, max_abs, min_finite, dev_flags, ws, st)        \
   : (dtype == BTAS_I32 && min_finite < 0.0)                                                                 \
       ? fw_typed<T, kClamp>(integer_mode, (T*)D, ld, n, max_abs, min_finite, dev_flags, ws, st)             \
       : fw_typed<T, kFast>(integer_mode, (T*)D, ld, n, max_abs, min_finite, dev_flags, ws, st))
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

extern "C" size_t btas_fw_dist_workspace_bytes(int dtype, int64_t n, int64_t slab_rows, size_t* bcast_offset,
                                               size_t* bcast_bytes) {
  if (n < 1 || slab_rows < 0) return 0;
  size_t total = 0, off = 0, end = 0;
  switch (dtype) {
    case BTAS_F32: {
      const FwDistWs w = fw_dist_ws<float>(n, slab_rows);
      total = w.total, off = w.ctrl, end = w.bcast_end;
      break;
    }
    case BTAS_I32: {
      const FwDistWs w = fw_dist_ws<int32_t>(n, slab_rows);
      total = w.total, off = w.ctrl, end = w.bcast_end;
      break;
    }
    case BTAS_F64: {
      const FwDistWs w = fw_dist_ws<double>(n, slab_rows);
      total = w.total, off = w.ctrl, end = w.bcast_end;
      break;
    }
    default:
      return 0;
  }
  if (bcast_offset) *bcast_offset = off;
  if (bcast_bytes) *bcast_bytes = end - off;
  return total;
}

extern "C" int btas_fw_dist_group_size(int dtype) {
  switch (dtype) {
    case BTAS_F32:
      return FwGeom<float>::look;
    case BTAS_I32:
      return FwGeom<int32_t>::look;
    case BTAS_F64:
      return FwGeom<double>::look;
    default:
      return 0;
  }
}

static int fw_dist_group_entry(int dtype, int integer_mode, int stage, void* D_slab, int64_t ld, int64_t n,
                               int64_t slab_r0, int64_t slab_rows, int64_t kb0, int group_blocks, int masked,
                               double min_finite, int32_t* dev_flags, void* workspace, size_t workspace_bytes,
                               void* const* peers, int n_peers, btas_stream_t stream) {
  if (!dev_flags || !workspace || n < 1 || ld < n || slab_r0 < 0 || slab_rows < 0 || slab_r0 + slab_rows > n)
    return BTAS_ERR_INVALID;
  if (n_peers < 0 || n_peers > 7 || (n_peers > 0 && !peers)) return BTAS_ERR_INVALID;
  for (int q = 0; q < n_peers; ++q)
    if (!peers[q]) return BTAS_ERR_INVALID;
  if (slab_rows > 0 && !D_slab) return BTAS_ERR_INVALID;
  const int64_t b = dtype == BTAS_F64 ? 64 : 128;
  if ((slab_rows > 0 && slab_r0 % 128 != 0) || kb0 < 0 || kb0 * b >= n) return BTAS_ERR_INVALID;
  if (workspace_bytes < btas_fw_dist_workspace_bytes(dtype, n, slab_rows, nullptr, nullptr)) return BTAS_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
#define BTAS_FWD_CALL(T)                                                                                           \
  (masked ? fw_dist_group_typed<T, kChecked>(integer_mode, stage, (T*)D_slab, ld, n, slab_r0, slab_rows, kb0,      \
                                             group_blocks, dev_flags, ws, peers, n_peers, st)                      \
   : (dtype == BTAS_I32 && min_finite < 0.0)                                                                       \
       ? fw_dist_group_typed<T, kClamp>(integer_mode, stage, (T*)D_slab, ld, n, slab_r0, slab_rows, kb0,           \
                                        group_blocks, dev_flags, ws, peers, n_peers, st)                           \
       : fw_dist_group_typed<T, kFast>(integer_mode, stage, (T*)D_slab, ld, n, slab_r0, slab_rows, kb0,            \
                                       group_blocks, dev_flags, ws, peers, n_peers, st))
  switch (dtype) {
    case BTAS_F32:
      return BTAS_FWD_CALL(float);
    case BTAS_I32:
      return BTAS_FWD_CALL(int32_t);
    case BTAS_F64:
      return BTAS_FWD_CALL(double);
    default:
      return BTAS_ERR_INVALID;
  }
#undef BTAS_FWD_CALL
}

extern "C" int btas_fw_dist_group(int dtype, int integer_mode, int stage, void* D_slab, int64_t ld, int64_t n,
                                  int64_t slab_r0, int64_t slab_rows, int64_t kb0, int group_blocks, int masked,
                                  double min_finite, int32_t* dev_flags, void* workspace, size_t workspace_bytes,
                                  btas_stream_t stream) {
  return fw_dist_group_entry(dtype, integer_mode, stage, D_slab, ld, n, slab_r0, slab_rows, kb0, group_blocks, masked,
                             min_finite, dev_flags, workspace, workspace_bytes, nullptr, 0, stream);
}

extern "C" int btas_fw_dist_group_peers(int dtype, int integer_mode, int stage, void* D_slab, int64_t ld, int64_t n,
                                        int64_t slab_r0, int64_t slab_rows, int64_t kb0, int group_blocks,
                                        int masked, double min_finite, int32_t* dev_flags, void* workspace,
                                        size_t workspace_bytes, void* const* peer_regions, int n_peers,
                                        btas_stream_t stream) {
  return fw_dist_group_entry(dtype, integer_mode, stage, D_slab, ld, n, slab_r0, slab_rows, kb0, group_blocks, masked,
                             min_finite, dev_flags, workspace, workspace_bytes, peer_regions, n_peers, stream);
}

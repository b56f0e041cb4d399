// Tropical (min-plus / max-plus) GEMM core for sm_100a, shared by btas_gemm
// (matmul, reference matrix.py:315-400) and the Floyd-Warshall phase-3 update
// (btas_fw.cu).
//
// Design:
//  * Operands are first packed into a k-pair-interleaved, tile-contiguous
//    layout  P[blk][kp][r][2]  (blk = 32*G rows/cols, kp = k/2).  One pipeline
//    stage of a tile is then ONE contiguous chunk, moved global->shared by a
//    single bulk TMA copy (cp.async.bulk, SASS UBLKCP) completing on an
//    mbarrier.  A producer warp keeps STAGES copies in flight; 8 consumer warps
//    compute.  The kernel is persistent (one CTA per SM, static round-robin
//    over output tiles in grouped raster order for L2 reuse).
//  * Each consumer thread owns a (2*GM) x (2*GN) register microtile; rows
//    ty*2 + 32*g + r, cols tx*2 + 32*h + c, so every shared-memory read is a
//    conflict-free LDS.128 returning two rows (or cols) x one k pair.
//  * Inner step per (i, j, k-pair) — the "mix" policies below:
//      f32  : FADD2 {a_ik, a_ik+1} + {b_kj, b_k+1j}, then FMNMX3(acc, s.x, s.y)
//      i32  : VIADDMNMX twice (DPX __viaddmin_s32 / __viaddmax_s32)
//      s16x2: one 32-bit word holds the k and k+1 entries as int16 lanes;
//             VIADDMNMX.S16x2 twice per word pair = 4 candidate pairs
//      f64  : DADD + min
//    min/max are exact and order-independent, every candidate is rounded
//    once, so results are bit-identical to the reference's float64 ufuncs on
//    the same inputs (matrix.py:9-13 determinism contract).
//  * Epilogue fuses: integer-limit saturation clamp, the accumulate_into ⊕,
//    the fixpoint compare against Cprev (apsp.py:161) and the diag<0 test.
#pragma once

#include <type_traits>

#include "btas_common.cuh"

namespace btas {

constexpr int kConsumerWarps = 8;
constexpr int kGemmThreads = (kConsumerWarps + 4) * 32;  // producer warpgroup + 2 consumer warpgroups
constexpr int kProducerRegs = 40;
constexpr int kConsumerRegs = 232;  // 4*40*32 + 8*232*32 = 64512 <= 65536

// ---------------------------------------------------------------------------
// epilogue / kernel arguments
// ---------------------------------------------------------------------------
struct GemmArgs {
  const void* Ap;        // packed A  [mblocks][Kp2][BM][2]
  const void* Bp;        // packed B  [nblocks][Kp2][BN][2]
  int64_t Kp2;           // k pairs in the packed layout (multiple of KP)
  int64_t M, N;
  int mblocks, nblocks;
  const void* Z;         // nullable accumulate operand (storage dtype)
  int64_t ldz;
  void* C;
  int64_t ldc;
  const void* Cprev;     // nullable fixpoint reference
  int64_t ldcp;
  int32_t* flags;        // BTAS_NUM_FLAGS device ints
  const int32_t* gate;   // nullable: run only when *gate == gate_value
  int gate_value;
  // skip tiles whose rows lie inside [skip_row_lo, skip_row_hi) or whose
  // cols lie inside [skip_col_lo, skip_col_hi) (empty ranges: no skipping)
  int64_t skip_row_lo, skip_row_hi, skip_col_lo, skip_col_hi;
  int64_t Kp2s;          // k-pair stride between blocks of the packed buffers (0: = Kp2)
  int no_diag;           // 1: skip the diag<0 test (C is a window, not the whole matrix)
  int max_ctas;          // > 0: cap the persistent grid (leave SMs to a concurrent latency-bound chain)
  // fused all-gather: every output element is also stored, at the same
  // offset, into up to kMaxPeers other buffers — the other ranks' copies
  // mapped into this process (NVLink peer memory), so the exchange of
  // row-sharded results overlaps the add-min work tile by tile
  void* peer_C[7];
  int n_peers;
  int integer_mode;
  double limit;          // saturation limit (integer limit, or +inf for float mode)
  // verifier products (btas_gemm_verify): compare with Cprev instead of
  // storing C; smallest violating row-major index -> *first_bad
  unsigned long long* first_bad;
  int verify_mode;       // BTAS_VERIFY_LE / BTAS_VERIFY_EQ
  int64_t arg_row0;      // predecessor product: global row of output row 0 (i == j test)
};

// per-call options of the btas_gemm drivers beyond the plain product
struct GemmExtras {
  void* const* peers = nullptr;  // fused all-gather targets (btas_gemm_peers)
  int n_peers = 0;
  unsigned long long* first_bad = nullptr;  // verifier product (btas_gemm_verify)
  int verify_mode = 0;
};

// ---------------------------------------------------------------------------
// inner-step policies
// ---------------------------------------------------------------------------
template <bool MIN>
struct MixF32 {
  using E = float;
  using Acc = float;
  using Out = float;
  static constexpr int GM = 4, GN = 4, KP = 16, STAGES = 4;
  static constexpr int path = BTAS_PATH_FAST32;
  static constexpr bool kChecked = false;
  static constexpr bool kArg = false;
  BTAS_D static Acc init() { return MIN ? INFINITY : -INFINITY; }
  BTAS_D static void step(Acc& c, E a0, E a1, E b0, E b1, bool&, const GemmArgs&) {
    float2 s = __fadd2_rn(make_float2(a0, a1), make_float2(b0, b1));
    c = MIN ? fminf(fminf(c, s.x), s.y) : fmaxf(fmaxf(c, s.x), s.y);
  }
  BTAS_D static Out finish(Acc c, const GemmArgs& a) {
    // integer mode: sums at/after the float32 exactness limit saturate to Inf
    // (the benign side; the other side is routed to the checked path)
    if (a.integer_mode && (MIN ? (double)c >= a.limit : (double)c <= -a.limit)) c = MIN ? INFINITY : -INFINITY;
    return c;
  }
};

template <bool MIN>
struct MixI32 {
  using E = int32_t;
  using Acc = int32_t;
  using Out = int32_t;
  static constexpr int GM = 4, GN = 4, KP = 16, STAGES = 4;
  static constexpr int path = BTAS_PATH_FAST32;
  static constexpr bool kChecked = false;
  static constexpr bool kArg = false;
  BTAS_D static Acc init() { return MIN ? kI32Inf : -kI32Inf; }
  BTAS_D static void step(Acc& c, E a0, E a1, E b0, E b1, bool&, const GemmArgs&) {
    if (MIN) {
      c = __viaddmin_s32(a0, b0, c);
      c = __viaddmin_s32(a1, b1, c);
    } else {
      c = __viaddmax_s32(a0, b0, c);
      c = __viaddmax_s32(a1, b1, c);
    }
  }
  BTAS_D static Out finish(Acc c, const GemmArgs&) {
    // canonical Inf, and benign-side saturation at the int32 domain limit.
    // The other side cannot be reached on this path (the screen routes it to
    // CHECKED) except inside a negative cycle of Floyd-Warshall, where the
    // clamp keeps int32 from wrapping so diag < 0 stays detectable.
    if (MIN) return c >= kI32Limit ? kI32Inf : (c < -kI32Limit ? -kI32Limit : c);
    return c <= -kI32Limit ? -kI32Inf : (c > kI32Limit ? kI32Limit : c);
  }
};

// float64 storage, integer operands whose every finite sum stays inside the
// int32 domain (|a| + |b| < 2^28, decided by the exact screen): the packed
// operands are int32 (Inf -> +/-(2^30-1)) and the add-min is VIADDMNMX, 5x the
// DADD+min rate.  Sums are exact integers in both representations, so the
// float64 result is the same bytes.
template <bool MIN>
struct MixI32F64 {
  using E = int32_t;
  using Acc = int32_t;
  using Out = double;
  static constexpr int GM = 4, GN = 4, KP = 16, STAGES = 4;
  static constexpr int path = BTAS_PATH_I32F64;
  static constexpr bool kChecked = false;
  static constexpr bool kArg = false;
  BTAS_D static Acc init() { return MIN ? kI32Inf : -kI32Inf; }
  BTAS_D static void step(Acc& c, E a0, E a1, E b0, E b1, bool&, const GemmArgs&) {
    if (MIN) {
      c = __viaddmin_s32(a0, b0, c);
      c = __viaddmin_s32(a1, b1, c);
    } else {
      c = __viaddmax_s32(a0, b0, c);
      c = __viaddmax_s32(a1, b1, c);
    }
  }
  BTAS_D static Out finish(Acc c, const GemmArgs&) {
    if (MIN) return c >= kI32Limit ? INFINITY : (double)c;
    return c <= -kI32Limit ? -INFINITY : (double)c;
  }
};

template <bool MIN>
struct MixF64 {
  using E = double;
  using Acc = double;
  using Out = double;
  static constexpr int GM = 2, GN = 4, KP = 16, STAGES = 3;
  static constexpr int path = BTAS_PATH_FAST64;
  static constexpr bool kChecked = false;
  static constexpr bool kArg = false;
  BTAS_D static Acc init() { return MIN ? INFINITY : -INFINITY; }
  BTAS_D static void step(Acc& c, E a0, E a1, E b0, E b1, bool&, const GemmArgs&) {
    // ternary compares (DSETP.GEU + 2 FSEL), not fmin/fmax: those lower to
    // DSETP.MIN with NaN handling at half the rate (tools/f64_microbench.cu:
    // 21.7 vs 11.5 pairs/clk/SM).  No NaN and no -0.0 reach the kernel.
    const double s0 = __dadd_rn(a0, b0), s1 = __dadd_rn(a1, b1);
    if (MIN) {
      c = s0 < c ? s0 : c;
      c = s1 < c ? s1 : c;
    } else {
      c = s0 > c ? s0 : c;
      c = s1 > c ? s1 : c;
    }
  }
  BTAS_D static Out finish(Acc c, const GemmArgs& a) {
    if (a.integer_mode && (MIN ? c >= a.limit : c <= -a.limit)) c = MIN ? INFINITY : -INFINITY;
    return c;
  }
};

// int16x2 lanes: E is a word holding (k even, k odd) entries; acc lanes hold
// the running ⊕ of even-k and odd-k candidates, merged in finish().
template <bool MIN, class OutT, int GNv = 4>
struct MixS16 {
  using E = uint32_t;
  using Acc = uint32_t;
  using Out = OutT;
  // GNv = 8: 128 x 256 tiles, 8 x 16 microtile (12 LDS.128 per 256 DPX ops
  // instead of 8 per 128).  32 word pairs (128 k) per stage, 3 stages.
  static constexpr int GM = 4, GN = GNv, KP = 32, STAGES = 3;
  static constexpr int path = BTAS_PATH_S16X2;
  static constexpr bool kChecked = false;
  static constexpr bool kArg = false;
  BTAS_D static Acc init() {
    const uint32_t inf = MIN ? (uint32_t)kS16Inf : (uint32_t)(uint16_t)(-kS16Inf);
    return inf | (inf << 16);
  }
  BTAS_D static void step(Acc& c, E a0, E a1, E b0, E b1, bool&, const GemmArgs&) {
    if (MIN) {
      c = __viaddmin_s16x2(a0, b0, c);
      c = __viaddmin_s16x2(a1, b1, c);
    } else {
      c = __viaddmax_s16x2(a0, b0, c);
      c = __viaddmax_s16x2(a1, b1, c);
    }
  }
  BTAS_D static Out finish(Acc c, const GemmArgs&) {
    int lo = (int)(int16_t)(c & 0xFFFFu);
    int hi = (int)(int16_t)(c >> 16);
    int r = MIN ? min(lo, hi) : max(lo, hi);
    if (MIN ? r >= kS16InfThreshold : r <= -kS16InfThreshold) return Traits<OutT>::eps(MIN);
    return (OutT)r;
  }
};

// Per-candidate overflow masking: the reference's masked tile
// (matrix.py:334-342): a finite (x) finite sum that overflows (float) or
// reaches the integer limit (integer mode) becomes ε and raises the flag.
template <class T, bool MIN>
struct MixChecked {
  using E = T;
  using Acc = T;
  using Out = T;
  static constexpr int GM = sizeof(T) == 8 ? 2 : 4, GN = 4, KP = 16, STAGES = sizeof(T) == 8 ? 3 : 4;
  static constexpr int path = BTAS_PATH_CHECKED;
  static constexpr bool kChecked = true;
  static constexpr bool kArg = false;
  BTAS_D static Acc init() { return Traits<T>::eps(MIN); }
  BTAS_D static T cand(T a, T b, bool& sat, const GemmArgs& g) {
    T s = a + b;
    bool over;
    if (sizeof(T) == 4 && Traits<T>::dtype == BTAS_I32) {
      over = (s >= (T)kI32Limit) || (s <= -(T)kI32Limit);
    } else if (g.integer_mode) {
      over = fabs((double)s) >= g.limit;
    } else {
      over = isinf((double)s);
    }
    if (over && Traits<T>::finite(a) && Traits<T>::finite(b)) {
      sat = true;
      s = Traits<T>::eps(MIN);
    }
    return s;
  }
  BTAS_D static void step(Acc& c, E a0, E a1, E b0, E b1, bool& sat, const GemmArgs& g) {
    T s0 = cand(a0, b0, sat, g), s1 = cand(a1, b1, sat, g);
    if (MIN) {
      c = s0 < c ? s0 : c;
      c = s1 < c ? s1 : c;
    } else {
      c = s0 > c ? s0 : c;
      c = s1 > c ? s1 : c;
    }
  }
  BTAS_D static Out finish(Acc c, const GemmArgs&) {
    if (Traits<T>::dtype == BTAS_I32) {
      if (MIN) return c >= (T)kI32Limit ? (T)kI32Inf : c;
      return c <= -(T)kI32Limit ? (T)(-kI32Inf) : c;
    }
    return c;
  }
};

// Predecessor product (path reconstruction): the
// min-plus product A (x) B together with, per output, the FIRST k attaining
// the minimum (strict < in increasing k; the k dimension is never split, so
// the index is deterministic).  Used as D (x) (A with an infinite diagonal):
// the argmin is the last hop of a shortest path.  The epilogue writes int32
// indices (-1 where the minimum does not reproduce Cprev, the distances).
template <class T>
struct MixArg {
  using E = T;
  using Acc = T;
  using Out = T;
  static constexpr int GM = sizeof(T) == 8 ? 2 : 4, GN = 4, KP = 16, STAGES = sizeof(T) == 8 ? 3 : 4;
  static constexpr int path = BTAS_PATH_CHECKED;  // never gated
  static constexpr bool kChecked = false;
  static constexpr bool kArg = true;
  BTAS_D static Acc init() { return Traits<T>::eps(true); }
  BTAS_D static void step_arg(Acc& c, int32_t& idx, E a0, E a1, E b0, E b1, int32_t k0) {
    // int32 storage: Inf = 2^30-1, sums of two stay below 2^31 and every sum
    // involving Inf stays >= 2^29 > every finite value
    const T s0 = a0 + b0, s1 = a1 + b1;
    if (s0 < c) {
      c = s0;
      idx = k0;
    }
    if (s1 < c) {
      c = s1;
      idx = k0 + 1;
    }
  }
  BTAS_D static void step(Acc&, E, E, E, E, bool&, const GemmArgs&) {}
  BTAS_D static Out finish(Acc c, const GemmArgs&) {
    if constexpr (Traits<T>::dtype == BTAS_I32) return c >= (T)kI32Limit ? (T)kI32Inf : c;
    return c;
  }
};

// The predecessor product for small integer data (|x| < 2^12, K <= 2^16):
// operands packed as keys  a' = a << 16,  b' = (b << 16) + k  (Inf -> a
// large key), so  a' + b' = ((a + b) << 16) + k  and one VIADDMNMX per
// candidate keeps the minimum sum AND, among equal sums, the smallest k — the
// same first argmin as MixArg at the plain int32 GEMM rate.  Decoded in the
// epilogue (value = key >> 16, k = key & 0xFFFF).
template <class T>
struct MixArgKey {
  using E = int32_t;
  using Acc = int32_t;
  using Out = T;  // Cprev (the distances) is read in the storage type
  static constexpr int GM = 4, GN = 4, KP = 16, STAGES = 4;
  static constexpr int path = BTAS_PATH_FAST32;  // never gated
  static constexpr bool kChecked = false;
  static constexpr bool kArg = true;
  static constexpr bool kArgKey = true;
  BTAS_D static Acc init() { return (1 << 30) - 1; }
  BTAS_D static void step(Acc& c, E a0, E a1, E b0, E b1, bool&, const GemmArgs&) {
    c = __viaddmin_s32(a0, b0, c);
    c = __viaddmin_s32(a1, b1, c);
  }
  BTAS_D static void step_arg(Acc&, int32_t&, E, E, E, E, int32_t) {}
  BTAS_D static Out finish(Acc c, const GemmArgs&) { return (Out)c; }  // unused: the key epilogue decodes
};

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
template <class E>
BTAS_D void lds4(const E* p, E out[4]) {
  if constexpr (sizeof(E) == 4) {
    uint4 v = *reinterpret_cast<const uint4*>(p);
    out[0] = __builtin_bit_cast(E, v.x);
    out[1] = __builtin_bit_cast(E, v.y);
    out[2] = __builtin_bit_cast(E, v.z);
    out[3] = __builtin_bit_cast(E, v.w);
  } else {
    double2 v0 = reinterpret_cast<const double2*>(p)[0];
    double2 v1 = reinterpret_cast<const double2*>(p)[1];
    out[0] = v0.x;
    out[1] = v0.y;
    out[2] = v1.x;
    out[3] = v1.y;
  }
}

template <class T>
BTAS_D bool bits_differ(T a, T b) {
  if constexpr (sizeof(T) == 4) return __builtin_bit_cast(uint32_t, a) != __builtin_bit_cast(uint32_t, b);
  else return __builtin_bit_cast(unsigned long long, a) != __builtin_bit_cast(unsigned long long, b);
}

// two adjacent elements as one 8-byte (4-byte T) or 16-byte (8-byte T) access
template <class T>
BTAS_D bool aligned2(const T* p, int64_t ld) {
  return (ld % 2) == 0 && (reinterpret_cast<uintptr_t>(p) % (2 * sizeof(T))) == 0;
}
template <class T>
BTAS_D void ld2(const T* p, T out[2]) {
  if constexpr (sizeof(T) == 4) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    out[0] = __builtin_bit_cast(T, u.x);
    out[1] = __builtin_bit_cast(T, u.y);
  } else {
    const ulonglong2 u = *reinterpret_cast<const ulonglong2*>(p);
    out[0] = __builtin_bit_cast(T, u.x);
    out[1] = __builtin_bit_cast(T, u.y);
  }
}
template <class T>
BTAS_D void st2(T* p, const T v[2]) {
  if constexpr (sizeof(T) == 4) {
    *reinterpret_cast<uint2*>(p) = make_uint2(__builtin_bit_cast(uint32_t, v[0]), __builtin_bit_cast(uint32_t, v[1]));
  } else {
    ulonglong2 u;
    u.x = __builtin_bit_cast(unsigned long long, v[0]);
    u.y = __builtin_bit_cast(unsigned long long, v[1]);
    *reinterpret_cast<ulonglong2*>(p) = u;
  }
}

template <class T, bool MIN>
BTAS_D T combine(T a, T b) {
  if (MIN) return b < a ? b : a;
  return b > a ? b : a;
}

BTAS_D void tile_coords(int tile, int mblocks, int nblocks, int& mb, int& nb) {
  constexpr int kGroup = 8;
  const int per_group = kGroup * nblocks;
  const int gid = tile / per_group;
  const int first = gid * kGroup;
  const int gsz = min(mblocks - first, kGroup);
  const int in = tile - gid * per_group;
  mb = first + in % gsz;
  nb = in / gsz;
}

template <class P>
struct GemmShape {
  static constexpr int BM = 32 * P::GM;
  static constexpr int BN = 32 * P::GN;
  static constexpr int A_ELEMS = P::KP * BM * 2;
  static constexpr int B_ELEMS = P::KP * BN * 2;
  static constexpr size_t smem_bytes =
      (size_t)P::STAGES * (A_ELEMS + B_ELEMS) * sizeof(typename P::E) + 2 * P::STAGES * sizeof(uint64_t);
};

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
// EPI (compile-time epilogue operands): bit 0 = accumulate_into Z present,
// bit 1 = fixpoint reference Cprev present.  Separate instantiations keep the
// plain product's epilogue minimal (measured: a generic epilogue costs the
// n = 16384 GEMM ~1 %, profiles/r01_experiments.md).
// bit 2 = peer stores (fused all-gather); bit 3 = verify (compare with
// Cprev under g.verify_mode, record the first violating index, no store).
enum { kEpiPlain = 0, kEpiAcc = 1, kEpiCmp = 2, kEpiBoth = 3, kEpiPeers = 4, kEpiVerify = 8 };

#ifndef BTAS_KP_UNROLL_PLAIN
#define BTAS_KP_UNROLL_PLAIN 2
#endif
#ifndef BTAS_KP_UNROLL_EPI
#define BTAS_KP_UNROLL_EPI 4
#endif

#ifndef BTAS_L2_HINTS
#define BTAS_L2_HINTS 1
#endif

// verifier epilogue: one output entry against the reference value
template <class Out>
BTAS_D void verify_entry(const GemmArgs& g, Out v, Out ref, int64_t row, int64_t col, bool& bad_any) {
  const bool bad = g.verify_mode == BTAS_VERIFY_LE ? !(ref <= v) : (v != ref);
  if (bad) {
    bad_any = true;
    atomicMin(g.first_bad, (unsigned long long)(row * g.N + col));
  }
}
constexpr int kMaxPeers = 7;

template <class P, class = void>
struct arg_key : std::false_type {};
template <class P>
struct arg_key<P, std::void_t<decltype(P::kArgKey)>> : std::bool_constant<P::kArgKey> {};

template <class P, bool MIN, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1) tropical_gemm_kernel(const __grid_constant__ GemmArgs g) {
  if (g.gate != nullptr && *g.gate != g.gate_value) return;
  using E = typename P::E;
  using Acc = typename P::Acc;
  using Out = typename P::Out;
  using S = GemmShape<P>;
  constexpr int GM = P::GM, GN = P::GN, KP = P::KP, ST = P::STAGES;
  constexpr int BM = S::BM, BN = S::BN;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  E* sA = reinterpret_cast<E*>(smem_raw);
  E* sB = sA + ST * S::A_ELEMS;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + ST * S::B_ELEMS);
  uint64_t* empty = full + ST;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int ntiles = g.mblocks * g.nblocks;
  const int nkb = (int)(g.Kp2 / KP);

  auto skipped = [&](int mb, int nb) {
    const int64_t r0 = (int64_t)mb * BM, c0 = (int64_t)nb * BN;
    return (r0 >= g.skip_row_lo && r0 + BM <= g.skip_row_hi) || (c0 >= g.skip_col_lo && c0 + BN <= g.skip_col_hi);
  };

  // ------------------------------ producer --------------------------------
  // Warp-specialised: warpgroup 0 gives its registers back (setmaxnreg) and
  // one elected thread streams the k-stages with bulk TMA copies into the
  // STAGES-deep mbarrier ring; warpgroups 1-2 (8 warps) compute with up to
  // kConsumerRegs registers per thread.
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProducerRegs));
    if (warp == 0 && lane == 0) {
#if BTAS_L2_HINTS
      const uint64_t polA = l2_policy_evict_last(), polB = l2_policy_evict_first();
#endif
      uint32_t it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int mb, nb;
        tile_coords(tile, g.mblocks, g.nblocks, mb, nb);
        if (skipped(mb, nb)) continue;
        const int64_t kps = g.Kp2s ? g.Kp2s : g.Kp2;
        const E* gA = static_cast<const E*>(g.Ap) + (size_t)mb * kps * BM * 2;
        const E* gB = static_cast<const E*>(g.Bp) + (size_t)nb * kps * BN * 2;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % ST;
          if (it >= (uint32_t)ST) mbar_wait(&empty[s], ((it / ST) - 1) & 1);
          mbar_arrive_expect_tx(&full[s], (uint32_t)((S::A_ELEMS + S::B_ELEMS) * sizeof(E)));
#if BTAS_L2_HINTS
          // A panels are shared by every tile of the 8-row group across the
          // consecutive waves; B panels of a wave are streamed
          bulk_g2s_hint(sA + s * S::A_ELEMS, gA + (size_t)kb * S::A_ELEMS, S::A_ELEMS * sizeof(E), &full[s], polA);
          bulk_g2s_hint(sB + s * S::B_ELEMS, gB + (size_t)kb * S::B_ELEMS, S::B_ELEMS * sizeof(E), &full[s], polB);
#else
          bulk_g2s(sA + s * S::A_ELEMS, gA + (size_t)kb * S::A_ELEMS, S::A_ELEMS * sizeof(E), &full[s]);
          bulk_g2s(sB + s * S::B_ELEMS, gB + (size_t)kb * S::B_ELEMS, S::B_ELEMS * sizeof(E), &full[s]);
#endif
        }
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kConsumerRegs));

  // ------------------------------ consumers -------------------------------
  const int cw = warp - 4;                     // consumer warp 0..7
  const int ty = (cw >> 1) * 4 + (lane >> 3);  // 0..15
  const int tx = (cw & 1) * 8 + (lane & 7);    // 0..15
  bool changed = false, diag_neg = false, sat = false;
  uint32_t it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int mb, nb;
    tile_coords(tile, g.mblocks, g.nblocks, mb, nb);
    if (skipped(mb, nb)) continue;

    // epilogue operands: for interior tiles the Z / Cprev values are loaded
    // at the start of the LAST k-stage (peeled below), so their latency hides
    // behind that stage's add-min work while the main loop runs without 64
    // more live registers (K1, "epilogue operand")
    Out* C = static_cast<Out*>(g.C);
    const Out* Z = (EPI & kEpiAcc) ? static_cast<const Out*>(g.Z) : nullptr;
    const Out* Cp = (EPI & kEpiCmp) ? static_cast<const Out*>(g.Cprev) : nullptr;
    const bool vec2 = aligned2(C, g.ldc) && (Z == nullptr || aligned2(Z, g.ldz)) &&
                      (Cp == nullptr || aligned2(Cp, g.ldcp));
    const Out* X = Z != nullptr ? Z : Cp;  // the pre-loaded operand
    const int64_t ldx = Z != nullptr ? g.ldz : g.ldcp;
    const bool interior = vec2 && (int64_t)(mb + 1) * BM <= g.M && (int64_t)(nb + 1) * BN <= g.N &&
                          !(Z != nullptr && Cp != nullptr);
    const int64_t rb = (int64_t)mb * BM + ty * 2, cb = (int64_t)nb * BN + tx * 2;
    Out xi[GM][2][GN][2];

    Acc acc[GM][2][GN][2];
    int32_t aidx[P::kArg ? GM : 1][2][P::kArg ? GN : 1][2];  // argmin k (predecessor product only)
#pragma unroll
    for (int i = 0; i < GM; ++i)
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int j = 0; j < GN; ++j)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            acc[i][r][j][c] = P::init();
            if constexpr (P::kArg) aidx[i][r][j][c] = -1;
          }

    // k-pair unroll of the inner loop (the register schedule ptxas picks
    // differs per epilogue): 4 for the 32-bit integer mixes with an epilogue
    // operand (accumulate K = 1024 0.912 -> 0.925, K = 8192 0.935 -> 0.947 of
    // the ceiling; compare n = 65536 0.930 -> 0.954) and for MixI32 plain;
    // 2 for the s16x2 plain product (4 measured 0.3 % slower) and for the
    // float / 64-bit policies (they spill at 4).  profiles/r02_ab_unroll.txt
    constexpr bool kNarrowInt = sizeof(Out) == 4 && std::is_integral_v<E> && !P::kChecked && !P::kArg;
    constexpr int kKpUnroll = !kNarrowInt                                         ? 2
                              : EPI != kEpiPlain                                   ? BTAS_KP_UNROLL_EPI
                              : std::is_same_v<E, int32_t> ? 4  // MixI32: 0.987 -> 0.994
                                                           : BTAS_KP_UNROLL_PLAIN;
    auto k_stage = [&](int kb) {
      const int s = it % ST;
      mbar_wait(&full[s], (it / ST) & 1);
      const E* tA = sA + s * S::A_ELEMS + ty * 4;
      const E* tB = sB + s * S::B_ELEMS + tx * 4;
#pragma unroll kKpUnroll
      for (int kp = 0; kp < KP; ++kp) {
        E a[GM][4], b[GN][4];
#pragma unroll
        for (int i = 0; i < GM; ++i) lds4(tA + kp * BM * 2 + i * 64, a[i]);
#pragma unroll
        for (int j = 0; j < GN; ++j) lds4(tB + kp * BN * 2 + j * 64, b[j]);
#pragma unroll
        for (int i = 0; i < GM; ++i)
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int j = 0; j < GN; ++j)
#pragma unroll
              for (int c = 0; c < 2; ++c) {
                if constexpr (P::kArg && !arg_key<P>::value)
                  P::step_arg(acc[i][r][j][c], aidx[i][r][j][c], a[i][2 * r], a[i][2 * r + 1], b[j][2 * c],
                              b[j][2 * c + 1], (int32_t)(2 * ((int64_t)kb * KP + kp)));
                else
                  P::step(acc[i][r][j][c], a[i][2 * r], a[i][2 * r + 1], b[j][2 * c], b[j][2 * c + 1], sat, g);
              }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      ++it;
    };
    for (int kb = 0; kb < nkb - 1; ++kb) k_stage(kb);
    if (interior && X != nullptr) {
#pragma unroll
      for (int i = 0; i < GM; ++i)
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int j = 0; j < GN; ++j) ld2(X + (rb + i * 32 + r) * ldx + cb + j * 32, xi[i][r][j]);
    }
    k_stage(nkb - 1);

    // ------------------------------ epilogue ------------------------------
    // Interior tiles (every tile but the last row/column of tiles): operands
    // already in registers, no bounds tests, 8/16-byte stores, diagonal test
    // only on diagonal tiles.  Edge tiles: two passes (all loads, then all
    // stores — C may alias Z in Floyd-Warshall, so interleaving them would
    // serialise each load's latency).
    if constexpr (P::kArg) {
      // predecessor product: C holds int32 indices; Cprev the distances
      int32_t* Ci = static_cast<int32_t*>(g.C);
#pragma unroll
      for (int i = 0; i < GM; ++i)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int64_t row = (int64_t)mb * BM + i * 32 + ty * 2 + r;
          if (row >= g.M) continue;
#pragma unroll
          for (int j = 0; j < GN; ++j)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int64_t col = (int64_t)nb * BN + j * 32 + tx * 2 + c;
              if (col >= g.N) continue;
              const Out d = Cp[row * g.ldcp + col];
              if constexpr (arg_key<P>::value) {
                const int32_t key = acc[i][r][j][c];
                const bool tight = key < (1 << 29) && Traits<Out>::finite(d) && (Out)(key >> 16) == d &&
                                   row + g.arg_row0 != col;
                Ci[row * g.ldc + col] = tight ? (key & 0xFFFF) : -1;
              } else {
                const Out v = P::finish(acc[i][r][j][c], g);
                const bool tight = Traits<Out>::finite(v) && !bits_differ(v, d) && row + g.arg_row0 != col;
                Ci[row * g.ldc + col] = tight ? aidx[i][r][j][c] : -1;
              }
            }
        }
      continue;
    }
    if (interior) {
      const bool diag_tile = !g.no_diag && (int64_t)mb * BM < (int64_t)(nb + 1) * BN &&
                             (int64_t)nb * BN < (int64_t)(mb + 1) * BM;
#pragma unroll
      for (int i = 0; i < GM; ++i)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int64_t row = rb + i * 32 + r;
#pragma unroll
          for (int j = 0; j < GN; ++j) {
            const int64_t col0 = cb + j * 32;
            Out v[2];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              v[c] = P::finish(acc[i][r][j][c], g);
              if (Z != nullptr) v[c] = combine<Out, MIN>(v[c], xi[i][r][j][c]);
            }
            if constexpr ((EPI & kEpiVerify) != 0) {
              verify_entry(g, v[0], xi[i][r][j][0], row, col0, changed);
              verify_entry(g, v[1], xi[i][r][j][1], row, col0 + 1, changed);
            } else {
              if (Cp != nullptr) changed |= bits_differ(v[0], xi[i][r][j][0]) | bits_differ(v[1], xi[i][r][j][1]);
              if (diag_tile) diag_neg |= (row == col0 && v[0] < (Out)0) | (row == col0 + 1 && v[1] < (Out)0);
              st2(C + row * g.ldc + col0, v);
              if constexpr ((EPI & kEpiPeers) != 0) {
#pragma unroll 1
                for (int q = 0; q < g.n_peers; ++q) st2(static_cast<Out*>(g.peer_C[q]) + row * g.ldc + col0, v);
              }
            }
          }
        }
      continue;
    }
    Out xv[GM][2][GN][2];
    if (X != nullptr) {
#pragma unroll
      for (int i = 0; i < GM; ++i)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int64_t row = (int64_t)mb * BM + i * 32 + ty * 2 + r;
#pragma unroll
          for (int j = 0; j < GN; ++j) {
            const int64_t col0 = (int64_t)nb * BN + j * 32 + tx * 2;
            if (row < g.M && vec2 && col0 + 1 < g.N) {
              ld2(X + row * ldx + col0, xv[i][r][j]);
            } else {
#pragma unroll
              for (int c = 0; c < 2; ++c)
                xv[i][r][j][c] = (row < g.M && col0 + c < g.N) ? X[row * ldx + col0 + c] : (Out)0;
            }
          }
        }
    }
#pragma unroll
    for (int i = 0; i < GM; ++i)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int64_t row = (int64_t)mb * BM + i * 32 + ty * 2 + r;
        if (row >= g.M) continue;
#pragma unroll
        for (int j = 0; j < GN; ++j) {
          const int64_t col0 = (int64_t)nb * BN + j * 32 + tx * 2;
          Out v[2];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            v[c] = P::finish(acc[i][r][j][c], g);
            if (Z != nullptr) v[c] = combine<Out, MIN>(v[c], xv[i][r][j][c]);
          }
          if constexpr ((EPI & kEpiVerify) != 0) {
            if (col0 < g.N) verify_entry(g, v[0], xv[i][r][j][0], row, col0, changed);
            if (col0 + 1 < g.N) verify_entry(g, v[1], xv[i][r][j][1], row, col0 + 1, changed);
            continue;
          }
          if (Cp != nullptr && Z == nullptr) {
            if (col0 < g.N) changed |= bits_differ(v[0], xv[i][r][j][0]);
            if (col0 + 1 < g.N) changed |= bits_differ(v[1], xv[i][r][j][1]);
          } else if (Cp != nullptr) {  // both operands given (rare): second operand read inline
            if (col0 < g.N) changed |= bits_differ(v[0], Cp[row * g.ldcp + col0]);
            if (col0 + 1 < g.N) changed |= bits_differ(v[1], Cp[row * g.ldcp + col0 + 1]);
          }
          if (!g.no_diag) {
            if (row == col0) diag_neg |= (v[0] < (Out)0);
            if (row == col0 + 1 && col0 + 1 < g.N) diag_neg |= (v[1] < (Out)0);
          }
          if (vec2 && col0 + 1 < g.N) {
            st2(C + row * g.ldc + col0, v);
          } else {
            if (col0 < g.N) C[row * g.ldc + col0] = v[0];
            if (col0 + 1 < g.N) C[row * g.ldc + col0 + 1] = v[1];
          }
          if constexpr ((EPI & kEpiPeers) != 0) {
#pragma unroll 1
            for (int q = 0; q < g.n_peers; ++q) {
              Out* Pq = static_cast<Out*>(g.peer_C[q]);
              if (col0 < g.N) Pq[row * g.ldc + col0] = v[0];
              if (col0 + 1 < g.N) Pq[row * g.ldc + col0 + 1] = v[1];
            }
          }
        }
      }
  }
  if constexpr ((EPI & kEpiPeers) != 0) __threadfence_system();  // peer stores visible before completion
  if (__any_sync(0xffffffffu, changed) && lane == 0) atomicOr(&g.flags[BTAS_FLAG_CHANGED], 1);
  if (__any_sync(0xffffffffu, diag_neg) && lane == 0) atomicOr(&g.flags[BTAS_FLAG_DIAG_NEG], 1);
  if (P::kChecked) {
    if (__any_sync(0xffffffffu, sat) && lane == 0) atomicOr(&g.flags[BTAS_FLAG_SATURATED], 1);
  }
}

// host-side launcher for one policy
int device_sm_count();

template <class P, bool MIN, int EPI>
int launch_gemm_epi(const GemmArgs& g, cudaStream_t stream) {
  using S = GemmShape<P>;
  static unsigned long long configured = 0;
  if (!configured_on_current_device(configured)) {
    if (cudaFuncSetAttribute(tropical_gemm_kernel<P, MIN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)S::smem_bytes) != cudaSuccess) {
      (void)cudaGetLastError();
      return BTAS_ERR_CUDA;
    }
    mark_configured(configured);
  }
  if (g.Kp2 < P::KP || g.Kp2 % P::KP != 0) return BTAS_ERR_INVALID;  // whole pipeline stages only
  const int ntiles = g.mblocks * g.nblocks;
  int cap = device_sm_count();
  if (g.max_ctas > 0 && g.max_ctas < cap) cap = g.max_ctas;
  const int grid = ntiles < cap ? ntiles : cap;
  if (grid <= 0) return BTAS_OK;
  tropical_gemm_kernel<P, MIN, EPI><<<grid, kGemmThreads, S::smem_bytes, stream>>>(g);
  BTAS_CUDA_CHECK_LAUNCH();
  return BTAS_OK;
}

template <class P, bool MIN>
int launch_tropical_gemm(const GemmArgs& g, cudaStream_t stream) {
  if (g.first_bad != nullptr) {  // verifier product: min-plus, compare only
    if constexpr (MIN) {
      if (g.Cprev == nullptr || g.Z != nullptr || g.n_peers > 0) return BTAS_ERR_INVALID;
      return launch_gemm_epi<P, MIN, kEpiCmp | kEpiVerify>(g, stream);
    } else {
      return BTAS_ERR_UNSUPPORTED;
    }
  }
  const int epi = (g.Z != nullptr ? kEpiAcc : 0) | (g.Cprev != nullptr ? kEpiCmp : 0);
  if (g.n_peers > 0) {
    // peer-store variants: the squaring step (compare against Cprev) and the plain product
    if (g.n_peers > kMaxPeers) return BTAS_ERR_UNSUPPORTED;
    if (epi == kEpiCmp) return launch_gemm_epi<P, MIN, kEpiCmp | kEpiPeers>(g, stream);
    if (epi == kEpiPlain) return launch_gemm_epi<P, MIN, kEpiPlain | kEpiPeers>(g, stream);
    return BTAS_ERR_UNSUPPORTED;
  }
  switch (epi) {
    case kEpiPlain:
      return launch_gemm_epi<P, MIN, kEpiPlain>(g, stream);
    case kEpiAcc:
      return launch_gemm_epi<P, MIN, kEpiAcc>(g, stream);
    case kEpiCmp:
      return launch_gemm_epi<P, MIN, kEpiCmp>(g, stream);
    default:
      return launch_gemm_epi<P, MIN, kEpiBoth>(g, stream);
  }
}

// packed-layout index: P[blk][kp][r][2]
BTAS_HD int64_t packed_index(int64_t rc, int64_t k, int64_t Kp2, int BLK) {
  const int64_t blk = rc / BLK, r = rc - blk * BLK;
  return ((blk * Kp2 + (k >> 1)) * BLK + r) * 2 + (k & 1);
}

}  // namespace btas

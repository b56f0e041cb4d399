// Shared definitions of the B200 tropical kernels: storage traits (oriented
// Infinity per dtype), ordered keys for order statistics, and the sm_100a
// async-copy / mbarrier primitives used by the GEMM pipeline.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <string.h>

#include "../../include/btas_cuda.h"

#define BTAS_HD __host__ __device__ __forceinline__
#define BTAS_D __device__ __forceinline__

#define BTAS_CUDA_CHECK_LAUNCH()                       \
  do {                                                 \
    if (cudaPeekAtLastError() != cudaSuccess) {        \
      (void)cudaGetLastError();                        \
      return BTAS_ERR_CUDA;                            \
    }                                                  \
  } while (0)

namespace btas {

constexpr int kI32Inf = BTAS_I32_INF;          // 2^30 - 1: Inf + Inf does not wrap
constexpr int kI32Limit = BTAS_I32_LIMIT;      // finite |x| < 2^28
constexpr int kI32InfThreshold = 1 << 29;      // any sum involving Inf stays >= this
// s16x2 lanes: finite |x| < 2^12, Inf = 2^14 - 1, Inf + Inf = 32766 (no wrap)
constexpr int kS16Limit = 1 << 12;
constexpr int kS16Inf = (1 << 14) - 1;
constexpr int kS16InfThreshold = 1 << 13;

// ---------------------------------------------------------------------------
// storage traits
// ---------------------------------------------------------------------------
template <class T> struct Traits;

template <> struct Traits<float> {
  static constexpr int dtype = BTAS_F32;
  // integer-mode saturation limit: the reference's INT_EXACT_LIMIT (2^53,
  // semiring.py:71) for every float storage, so ONE f32 product / matvec /
  // ew_add is the reference's float64 result rounded once to f32 and
  // saturates exactly where the reference does.  Integer-valued f32 data is
  // exact only below 2^24: in chains (matrix_power, APSP) whose sums pass
  // 2^24 the per-step rounding compounds and the result is no longer the
  // reference's chain rounded once (INTEGRATION.md "float32 storage";
  // float64 or int32 storage keep integer chains exact).
  static constexpr double int_limit = 9007199254740992.0;
  BTAS_HD static float eps(bool min_plus) { return min_plus ? INFINITY : -INFINITY; }
  BTAS_HD static bool finite(float x) { return isfinite(x); }
  BTAS_HD static double to_f64(float x) { return (double)x; }
};

template <> struct Traits<double> {
  static constexpr int dtype = BTAS_F64;
  static constexpr double int_limit = 9007199254740992.0;  // 2^53
  BTAS_HD static double eps(bool min_plus) { return min_plus ? INFINITY : -INFINITY; }
  BTAS_HD static bool finite(double x) { return isfinite(x); }
  BTAS_HD static double to_f64(double x) { return x; }
};

template <> struct Traits<int32_t> {
  static constexpr int dtype = BTAS_I32;
  static constexpr double int_limit = (double)kI32Limit;
  BTAS_HD static int32_t eps(bool min_plus) { return min_plus ? kI32Inf : -kI32Inf; }
  BTAS_HD static bool finite(int32_t x) { return x < kI32Limit && x > -kI32Limit; }
  BTAS_HD static double to_f64(int32_t x) {
    return x >= kI32Limit ? INFINITY : (x <= -kI32Limit ? -INFINITY : (double)x);
  }
};

// ---------------------------------------------------------------------------
// ordered 64-bit keys: key(a) < key(b)  <=>  a < b  for non-NaN doubles
// ---------------------------------------------------------------------------
BTAS_HD unsigned long long f64_key(double x) {
#ifdef __CUDA_ARCH__
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
#else
  unsigned long long b;
  memcpy(&b, &x, 8);
#endif
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
BTAS_HD double key_f64(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  double x;
  memcpy(&x, &b, 8);
  return x;
#endif
}
// sentinels: no finite entry seen
constexpr unsigned long long kKeyNone = 0ull;           // for max keys
constexpr unsigned long long kKeyNoneMin = ~0ull;       // for min keys

// ---------------------------------------------------------------------------
// sm_90+/sm_100a async copy (bulk TMA) and mbarrier primitives
// ---------------------------------------------------------------------------
BTAS_D uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
BTAS_D void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
BTAS_D void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
BTAS_D void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
BTAS_D void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
BTAS_D void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "BTAS_WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra BTAS_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared through the TMA unit (UBLKCP), completion
// signalled on an mbarrier as transaction bytes.
// the same copy with an L2 eviction-priority hint (createpolicy descriptor)
BTAS_D void bulk_g2s_hint(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
BTAS_D uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
BTAS_D uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

BTAS_D void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// one bit per device: per-function attributes (dynamic shared memory limits)
// are set once per device the process launches on
inline bool configured_on_current_device(unsigned long long& mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return dev < 64 && ((mask >> dev) & 1ull);
}
inline void mark_configured(unsigned long long& mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess && dev < 64) mask |= 1ull << dev;
}

BTAS_HD int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
BTAS_HD int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

}  // namespace btas

// Per-element validation statistics shared by the ingest kernels
// (btas_elementwise.cu) and the on-device instance generator (btas_graph.cu):
// one definition of how a float64 value becomes oriented storage and what it
// contributes to btas_stats, so both ingest routes agree bit for bit.
#pragma once

#include "btas_common.cuh"

namespace btas {
namespace {

// ------------------------------------------------------------------ stats
// Per-thread statistics in the narrowest exact arithmetic A (float for f32
// data: B200 FP64 is a slow pipe), 32-bit per-thread counters, folded into
// the 64-bit device struct once per warp.
template <class A>
struct LocalStats {
  uint32_t nan = 0, neg_inf = 0, non_integral = 0, over = 0, out_of_range = 0, finite = 0;
  A max_abs = (A)-1;  // < 0: none
  A mn = (A)INFINITY, mx = (A)-INFINITY;

  BTAS_D void add_finite(A v, A int_limit) {
    finite++;
    if (v != floor(v)) non_integral++;
    const A a = fabs(v);
    if (a >= int_limit) over++;
    max_abs = a > max_abs ? a : max_abs;
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
  }
};

BTAS_D unsigned long long warp_sum(uint32_t v32) {
  unsigned long long v = v32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
BTAS_D double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
BTAS_D double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// warp-aggregated commit: one set of atomics per warp
template <class A>
BTAS_D void commit(const LocalStats<A>& s, btas_stats* out) {
  const unsigned long long nan = warp_sum(s.nan), neg_inf = warp_sum(s.neg_inf),
                           non_integral = warp_sum(s.non_integral), over = warp_sum(s.over),
                           out_of_range = warp_sum(s.out_of_range), finite = warp_sum(s.finite);
  const double max_abs = warp_max((double)s.max_abs), mn = warp_min((double)s.mn), mx = warp_max((double)s.mx);
  if ((threadIdx.x & 31) != 0) return;
  if (nan) atomicAdd(&out->nan_count, nan);
  if (neg_inf) atomicAdd(&out->neg_inf_count, neg_inf);
  if (non_integral) atomicAdd(&out->non_integral, non_integral);
  if (over) atomicAdd(&out->over_limit, over);
  if (out_of_range) atomicAdd(&out->out_of_range, out_of_range);
  if (finite) {
    atomicAdd(&out->finite_count, finite);
    atomicMax(&out->max_abs_key, f64_key(max_abs));
    atomicMin(&out->min_key, f64_key(mn));
    atomicMax(&out->max_key, f64_key(mx));
  }
}

// ------------------------------------------------------------------ ingest
template <class S, class D, class A>
BTAS_D D ingest_one(S x, D inf, LocalStats<A>& st) {
  D out;
  if (x != x) {
    st.nan++;
    out = inf;
  } else if (x == (S)-INFINITY) {
    st.neg_inf++;
    out = inf;
  } else if (x == (S)INFINITY) {
    out = inf;  // symbolic Infinity -> oriented (matrix.py:92-94)
  } else {
    const S v = x + (S)0;  // -0.0 -> +0.0 (matrix.py:92)
    if constexpr (Traits<D>::dtype == BTAS_I32) {
      if (v != floor(v) || fabs(v) >= (S)kI32Limit) {
        st.out_of_range++;
        out = 0;
      } else {
        out = (int32_t)v;
      }
      st.add_finite((A)v, (A)Traits<D>::int_limit);
    } else {
      out = (D)v;
      if (isinf(out)) {
        st.out_of_range++;  // finite double beyond the float range
      } else {
        st.add_finite((A)out, (A)Traits<D>::int_limit);
      }
    }
  }
  return out;
}

}  // namespace
}  // namespace btas

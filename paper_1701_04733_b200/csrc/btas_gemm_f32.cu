// btas_gemm driver (min-plus half) instantiated for float storage (see btas_gemm_impl.cuh).
#include "btas_gemm_impl.cuh"

namespace btas {

BTAS_GEMM_DRIVER_DECL(float, gemm_f32) {
  if (!min_plus) return gemm_f32_max(integer_mode, A, lda, B, ldb, Z, ldz, C, ldc, M, N, K, Cprev, ldcp, flags, ws,
                                     x, st);
  const gemm_impl::WsLayout L = gemm_impl::ws_layout(Traits<float>::dtype, M, N, K);
  return gemm_impl::gemm_typed<float, true>(integer_mode, A, lda, B, ldb, Z, ldz, C, ldc, M, N, K, Cprev, ldcp, flags, ws,
                                         L, x, st);
}

size_t gemm_ws_total(int dtype, int64_t M, int64_t N, int64_t K) {
  return gemm_impl::ws_layout(dtype, M, N, K).total;
}

BTAS_ARGMIN_DECL(float, argmin_f32) {
  const gemm_impl::WsLayout L = gemm_impl::ws_layout(Traits<float>::dtype, M, N, K);
  return gemm_impl::argmin_typed<float>(A, lda, B, ldb, Cref, ldcr, M, N, K, row0, idx, ldi, keys, ws, L, st);
}

}  // namespace btas

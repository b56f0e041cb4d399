// btas_gemm driver (min-plus half) instantiated for int32_t storage (see btas_gemm_impl.cuh).
#include "btas_gemm_impl.cuh"

namespace btas {

BTAS_GEMM_DRIVER_DECL(int32_t, gemm_i32) {
  if (!min_plus) return gemm_i32_max(integer_mode, A, lda, B, ldb, Z, ldz, C, ldc, M, N, K, Cprev, ldcp, flags, ws,
                                     x, st);
  const gemm_impl::WsLayout L = gemm_impl::ws_layout(Traits<int32_t>::dtype, M, N, K);
  return gemm_impl::gemm_typed<int32_t, true>(integer_mode, A, lda, B, ldb, Z, ldz, C, ldc, M, N, K, Cprev, ldcp, flags, ws,
                                         L, x, st);
}

BTAS_ARGMIN_DECL(int32_t, argmin_i32) {
  const gemm_impl::WsLayout L = gemm_impl::ws_layout(Traits<int32_t>::dtype, M, N, K);
  return gemm_impl::argmin_typed<int32_t>(A, lda, B, ldb, Cref, ldcr, M, N, K, row0, idx, ldi, keys, ws, L, st);
}

}  // namespace btas

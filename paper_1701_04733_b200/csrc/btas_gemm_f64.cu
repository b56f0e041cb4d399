// btas_gemm driver (min-plus half) instantiated for double storage (see btas_gemm_impl.cuh).
#include "btas_gemm_impl.cuh"

namespace btas {

BTAS_GEMM_DRIVER_DECL(double, gemm_f64) {
  if (!min_plus) return gemm_f64_max(integer_mode, A, lda, B, ldb, Z, ldz, C, ldc, M, N, K, Cprev, ldcp, flags, ws,
                                     x, st);
  const gemm_impl::WsLayout L = gemm_impl::ws_layout(Traits<double>::dtype, M, N, K);
  return gemm_impl::gemm_typed<double, true>(integer_mode, A, lda, B, ldb, Z, ldz, C, ldc, M, N, K, Cprev, ldcp, flags, ws,
                                         L, x, st);
}

BTAS_ARGMIN_DECL(double, argmin_f64) {
  const gemm_impl::WsLayout L = gemm_impl::ws_layout(Traits<double>::dtype, M, N, K);
  return gemm_impl::argmin_typed<double>(A, lda, B, ldb, Cref, ldcr, M, N, K, row0, idx, ldi, keys, ws, L, st);
}

}  // namespace btas

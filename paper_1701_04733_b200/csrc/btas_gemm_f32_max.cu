// btas_gemm max-plus half for float storage (see btas_gemm_impl.cuh).
#include "btas_gemm_impl.cuh"

namespace btas {

BTAS_GEMM_HALF_DECL(float, gemm_f32_max) {
  const gemm_impl::WsLayout L = gemm_impl::ws_layout(Traits<float>::dtype, M, N, K);
  return gemm_impl::gemm_typed<float, false>(integer_mode, A, lda, B, ldb, Z, ldz, C, ldc, M, N, K, Cprev, ldcp, flags,
                                          ws, L, x, st);
}

}  // namespace btas

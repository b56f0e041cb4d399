// btas_gemm: the drop-in body of reference `matmul` (matrix.py:349-400),
// including its saturation screen (matrix.py:297-312) and masked tile
// (matrix.py:334-342).  Device pipeline, all stream-ordered, no host sync:
//
//   init → ext(A), ext(B)      per-k extremes of the finite entries
//        → screen              exact overflow test + kernel-path choice
//        → pack32 | pack16     operands into the packed tile layout (gated)
//        → gemm FAST | S16X2 | CHECKED                              (gated)
//
// The screen is exact, not a bound: for every k it forms
// max_i A[i,k] (x) max_j B[k,j] and min_i A[i,k] (x) min_j B[k,j] in the
// storage arithmetic (rounding is monotone), so "some finite (x) finite
// candidate overflows" is decided precisely and the saturation flag matches
// the reference's per-candidate mask bit for bit.  Overflow on the side that
// cannot win the ⊕ (min-plus: too large) is absorbed by the epilogue clamp;
// overflow that could win (min-plus: too negative) routes to the CHECKED path.
#include <utility>
#include <vector>

#include "btas_gemm_impl.cuh"

namespace btas {

// SM count of the CURRENT device, cached per device ordinal (one process may
// drive several GPUs; a MIG slice or a mixed box has different counts).
int device_sm_count() {
  constexpr int kMaxDev = 64;
  static int sms[kMaxDev] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    (void)cudaGetLastError();
    dev = 0;
  }
  int* slot = dev >= 0 && dev < kMaxDev ? &sms[dev] : nullptr;
  if (slot && *slot > 0) return *slot;
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
    (void)cudaGetLastError();
    v = 148;
  }
  if (slot) *slot = v;
  return v;
}

// Optional CUDA-event bracketing of the GEMM kernel launches (bench.py's
// roofline timing of the dominant kernel on the launching stream).
bool g_timing = false;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_timing_events;

void timing_begin(cudaStream_t st, cudaEvent_t* start) {
  *start = nullptr;
  if (!g_timing) return;
  if (cudaEventCreate(start) == cudaSuccess) cudaEventRecord(*start, st);
}
void timing_end(cudaStream_t st, cudaEvent_t start) {
  if (!g_timing || start == nullptr) return;
  cudaEvent_t stop;
  if (cudaEventCreate(&stop) == cudaSuccess) {
    cudaEventRecord(stop, st);
    g_timing_events.emplace_back(start, stop);
  }
}

}  // namespace btas

using namespace btas;

extern "C" int btas_gemm_timing(int enable) {
  for (auto& e : g_timing_events) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  g_timing_events.clear();
  g_timing = enable != 0;
  return BTAS_OK;
}

extern "C" int btas_gemm_timing_read(double* total_ms, int* count) {
  if (!total_ms || !count) return BTAS_ERR_INVALID;
  double sum = 0.0;
  for (auto& e : g_timing_events) {
    if (cudaEventSynchronize(e.second) != cudaSuccess) return BTAS_ERR_CUDA;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.first, e.second);
    sum += ms;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  *count = (int)g_timing_events.size();
  *total_ms = sum;
  g_timing_events.clear();
  return BTAS_OK;
}

extern "C" size_t btas_gemm_workspace_bytes(int dtype, int64_t M, int64_t N, int64_t K) {
  if (M < 1 || N < 1 || K < 1) return 0;
  return gemm_ws_total(dtype, M, N, K);
}

static int gemm_entry(int dtype, int kind, int integer_mode, const void* A, int64_t lda, const void* B, int64_t ldb,
                      const void* Z, int64_t ldz, void* C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                      const void* Cprev, int64_t ldcp, int32_t* dev_flags, void* workspace, size_t workspace_bytes,
                      const GemmExtras& x, btas_stream_t stream) {
  const int n_peers = x.n_peers;
  if (n_peers < 0 || n_peers > kMaxPeers || (n_peers > 0 && !x.peers)) return BTAS_ERR_INVALID;
  for (int q = 0; q < n_peers; ++q)
    if (!x.peers[q]) return BTAS_ERR_INVALID;
  if (!A || !B || !C || !dev_flags || !workspace) return BTAS_ERR_INVALID;
  if (M < 1 || N < 1 || K < 1 || lda < K || ldb < N || ldc < N) return BTAS_ERR_INVALID;
  if (Z && ldz < N) return BTAS_ERR_INVALID;
  if (Cprev && ldcp < N) return BTAS_ERR_INVALID;
  if (kind != BTAS_MIN_PLUS && kind != BTAS_MAX_PLUS) return BTAS_ERR_INVALID;
  if (dtype != BTAS_F32 && dtype != BTAS_I32 && dtype != BTAS_F64) return BTAS_ERR_INVALID;
  if ((int64_t)ceil_div(M, 32) > 65535) return BTAS_ERR_UNSUPPORTED;
  if (workspace_bytes < gemm_ws_total(dtype, M, N, K)) return BTAS_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  const bool mn = kind == BTAS_MIN_PLUS;
  switch (dtype) {
    case BTAS_F32:
      return gemm_f32(mn, integer_mode, (const float*)A, lda, (const float*)B, ldb, (const float*)Z, ldz, (float*)C,
                      ldc, M, N, K, (const float*)Cprev, ldcp, dev_flags, ws, x, st);
    case BTAS_I32:
      return gemm_i32(mn, integer_mode, (const int32_t*)A, lda, (const int32_t*)B, ldb, (const int32_t*)Z, ldz,
                      (int32_t*)C, ldc, M, N, K, (const int32_t*)Cprev, ldcp, dev_flags, ws, x, st);
    default:
      return gemm_f64(mn, integer_mode, (const double*)A, lda, (const double*)B, ldb, (const double*)Z, ldz,
                      (double*)C, ldc, M, N, K, (const double*)Cprev, ldcp, dev_flags, ws, x, st);
  }
}

extern "C" int btas_gemm(int dtype, int kind, int integer_mode, const void* A, int64_t lda, const void* B,
                         int64_t ldb, const void* Z, int64_t ldz, void* C, int64_t ldc, int64_t M, int64_t N,
                         int64_t K, const void* Cprev, int64_t ldcp, int32_t* dev_flags, void* workspace,
                         size_t workspace_bytes, btas_stream_t stream) {
  return gemm_entry(dtype, kind, integer_mode, A, lda, B, ldb, Z, ldz, C, ldc, M, N, K, Cprev, ldcp, dev_flags,
                    workspace, workspace_bytes, GemmExtras{}, stream);
}

extern "C" int btas_gemm_verify(int dtype, int kind, int integer_mode, const void* A, int64_t lda, const void* B,
                                int64_t ldb, const void* Cref, int64_t ldcr, int64_t M, int64_t N, int64_t K, int mode,
                                unsigned long long* first_bad, int32_t* dev_flags, void* workspace,
                                size_t workspace_bytes, btas_stream_t stream) {
  if (!Cref || !first_bad || kind != BTAS_MIN_PLUS || (mode != BTAS_VERIFY_LE && mode != BTAS_VERIFY_EQ))
    return BTAS_ERR_INVALID;
  GemmExtras x;
  x.first_bad = first_bad;
  x.verify_mode = mode;
  // C is never written by the verifier kernels; Cref stands in for the
  // pointer argument checks
  return gemm_entry(dtype, kind, integer_mode, A, lda, B, ldb, nullptr, 0, const_cast<void*>(Cref), ldcr, M, N, K,
                    Cref, ldcr, dev_flags, workspace, workspace_bytes, x, stream);
}

extern "C" int btas_gemm_peers(int dtype, int kind, int integer_mode, const void* A, int64_t lda, const void* B,
                               int64_t ldb, void* C, int64_t ldc, int64_t M, int64_t N, int64_t K, const void* Cprev,
                               int64_t ldcp, void* const* peer_C, int n_peers, int32_t* dev_flags, void* workspace,
                               size_t workspace_bytes, btas_stream_t stream) {
  GemmExtras x;
  x.peers = peer_C;
  x.n_peers = n_peers;
  return gemm_entry(dtype, kind, integer_mode, A, lda, B, ldb, nullptr, 0, C, ldc, M, N, K, Cprev, ldcp, dev_flags,
                    workspace, workspace_bytes, x, stream);
}

extern "C" int btas_gemm_argmin(int dtype, int integer_mode, double operand_bound, const void* A, int64_t lda,
                                const void* B, int64_t ldb, const void* Cref, int64_t ldcr, int64_t M, int64_t N,
                                int64_t K, int64_t row0, int32_t* idx, int64_t ldi, void* workspace,
                                size_t workspace_bytes, btas_stream_t stream) {
  if (!A || !B || !Cref || !idx || !workspace || M < 1 || N < 1 || K < 1 || lda < K || ldb < N || ldcr < N ||
      ldi < N || row0 < 0)
    return BTAS_ERR_INVALID;
  if (K > 0x7FFFFFFFLL) return BTAS_ERR_UNSUPPORTED;
  if ((int64_t)ceil_div(M, 32) > 65535) return BTAS_ERR_UNSUPPORTED;
  if (workspace_bytes < gemm_ws_total(dtype, M, N, K)) return BTAS_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  // (value, k) keys when every finite operand is an integer below 2^12 in
  // magnitude (then every finite sum key stays below 2^29) and k fits 16 bits
  const bool keys = (dtype == BTAS_I32 || integer_mode) && operand_bound >= 0.0 &&
                    operand_bound < (double)kS16Limit && K <= 65536;
  switch (dtype) {
    case BTAS_F32:
      return argmin_f32((const float*)A, lda, (const float*)B, ldb, (const float*)Cref, ldcr, M, N, K, row0, idx, ldi,
                        keys, ws, st);
    case BTAS_I32:
      return argmin_i32((const int32_t*)A, lda, (const int32_t*)B, ldb, (const int32_t*)Cref, ldcr, M, N, K, row0,
                        idx, ldi, keys, ws, st);
    case BTAS_F64:
      return argmin_f64((const double*)A, lda, (const double*)B, ldb, (const double*)Cref, ldcr, M, N, K, row0, idx,
                        ldi, keys, ws, st);
    default:
      return BTAS_ERR_INVALID;
  }
}

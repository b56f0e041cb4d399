// btas_probe_ceiling: the live roofline denominator for the tropical GEMM.
// Runs the GEMM inner loop without global traffic — an 8x8 register
// microtile, A operands in registers, B operands streamed from shared memory
// with LDS.128 — for the instruction mix of each kernel path, one 512-thread
// CTA per SM, and reports candidate pairs per SM clock plus the SM clock the
// run saw (from clock64 vs. event time).  tools/pipe_microbench.cu is the
// standalone, wider version of the same measurement.
#include <algorithm>
#include <vector>

#include "btas_common.cuh"

namespace btas {
int device_sm_count();
namespace {

constexpr int kProbeIters = 8192;

// f64 (mix 3): the MixF64 step — DADD over a k pair, two ternary compares —
// on a 4 x 4 double microtile with register operands (the FP64 compare is the
// limiter, not shared memory)
__global__ void __launch_bounds__(256) probe_f64_kernel(const double* __restrict__ gin, double* gout,
                                                        long long* cycles) {
  double a[4][2], b[4][2], acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    a[i][0] = gin[(threadIdx.x + i) & 255];
    a[i][1] = gin[(threadIdx.x + 3 * i + 1) & 255];
    b[i][0] = gin[(threadIdx.x * 7 + i) & 255];
    b[i][1] = gin[(threadIdx.x * 5 + i + 9) & 255];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 1e300;
  const long long t0 = clock64();
  for (int it = 0; it < kProbeIters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double s0 = __dadd_rn(a[i][0], b[j][0]), s1 = __dadd_rn(a[i][1], b[j][1]);
        double& c = acc[i][j];
        c = s0 < c ? s0 : c;
        c = s1 < c ? s1 : c;
      }
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i][0] += 1.0;
  }
  const long long t1 = clock64();
  double r = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) r += acc[i][j];
  gout[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int run_probe_f64(double* ppc, double* mhz, double* tps) {
  const int nsm = device_sm_count();
  double *din = nullptr, *dout = nullptr;
  long long* dcyc = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = BTAS_ERR_CUDA;
  std::vector<double> h(256);
  std::vector<long long> hc(nsm);
  for (int i = 0; i < 256; ++i) h[i] = 1.0 + (i * 37 % 101) * 0.37;
  if (cudaMalloc(&din, 256 * 8) || cudaMalloc(&dout, (size_t)nsm * 256 * 8) || cudaMalloc(&dcyc, nsm * 8)) goto done;
  if (cudaMemcpy(din, h.data(), 256 * 8, cudaMemcpyHostToDevice)) goto done;
  probe_f64_kernel<<<nsm, 256>>>(din, dout, dcyc);
  if (cudaDeviceSynchronize()) goto done;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe_f64_kernel<<<nsm, 256>>>(din, dout, dcyc);
  cudaEventRecord(e1);
  if (cudaEventSynchronize(e1)) goto done;
  {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (cudaMemcpy(hc.data(), dcyc, nsm * 8, cudaMemcpyDeviceToHost)) goto done;
    const long long mx = *std::max_element(hc.begin(), hc.end());
    const double pairs = 32.0 * kProbeIters * 256.0 * nsm;
    *ppc = pairs / nsm / (double)mx;
    *mhz = (double)mx / (ms * 1e-3) / 1e6;
    *tps = pairs / (ms * 1e-3) / 1e12;
    rc = BTAS_OK;
  }
done:
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFree(din);
  cudaFree(dout);
  cudaFree(dcyc);
  (void)cudaGetLastError();
  return rc;
}

// 16 warps per SM: enough latency hiding that the issue / pipe limit of the
// mix, not the dependency chains, sets the figure (8 warps read 3 % low for
// FADD2+FMNMX3: the GEMM kernel itself exceeded that ceiling)
constexpr int kProbeThreads = 512;

template <int MIX>
__global__ void __launch_bounds__(kProbeThreads, 1) probe_kernel(const uint32_t* __restrict__ gin, uint32_t* gout,
                                                    long long* cycles) {
  __shared__ __align__(16) uint32_t sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = gin[i];
  __syncthreads();
  const long long t0 = clock64();
  uint32_t a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = gin[(threadIdx.x + i * 7) & 1023];
  uint32_t acc[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) acc[i] = MIX == 2 ? 0x3fff3fffu : (MIX == 1 ? 0x3fffffffu : 0x7f800000u);
  const int lane_off = (threadIdx.x & 7) * 4;
  for (int it = 0; it < kProbeIters; ++it) {
    const uint4* bp = reinterpret_cast<const uint4*>(sm + (((it * 16) + lane_off) & 1023));
    const uint4 b0 = bp[0], b1 = bp[1], b2 = bp[2], b3 = bp[3];
    const uint32_t b[16] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w,
                            b2.x, b2.y, b2.z, b2.w, b3.x, b3.y, b3.z, b3.w};
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint32_t& c = acc[i * 8 + j];
        if (MIX == 0) {
          const float2 s = __fadd2_rn(make_float2(__uint_as_float(a[2 * i]), __uint_as_float(a[2 * i + 1])),
                                      make_float2(__uint_as_float(b[2 * j]), __uint_as_float(b[2 * j + 1])));
          c = __float_as_uint(fminf(fminf(__uint_as_float(c), s.x), s.y));
        } else if (MIX == 1) {
          c = (uint32_t)__viaddmin_s32((int)a[2 * i], (int)b[2 * j], (int)c);
          c = (uint32_t)__viaddmin_s32((int)a[2 * i + 1], (int)b[2 * j + 1], (int)c);
        } else {
          c = __viaddmin_s16x2(a[2 * i], b[2 * j], c);
          c = __viaddmin_s16x2(a[2 * i + 1], b[2 * j + 1], c);
        }
      }
  }
  const long long t1 = clock64();
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) r ^= acc[i];
  gout[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MIX>
int run_probe(double* ppc, double* mhz, double* tps) {
  const int nsm = device_sm_count();
  uint32_t *din = nullptr, *dout = nullptr;
  long long* dcyc = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = BTAS_ERR_CUDA;
  std::vector<uint32_t> h(2048);
  std::vector<long long> hc(nsm);
  for (int i = 0; i < 2048; ++i) h[i] = MIX == 0 ? 0x3f800000u + (uint32_t)(i * 2654435761u % 100000u) : (uint32_t)(i % 97);
  if (cudaMalloc(&din, 2048 * 4) || cudaMalloc(&dout, (size_t)nsm * kProbeThreads * 4) || cudaMalloc(&dcyc, nsm * 8))
    goto done;
  if (cudaMemcpy(din, h.data(), 2048 * 4, cudaMemcpyHostToDevice)) goto done;
  probe_kernel<MIX><<<nsm, kProbeThreads>>>(din, dout, dcyc);  // warm-up
  if (cudaDeviceSynchronize()) goto done;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe_kernel<MIX><<<nsm, kProbeThreads>>>(din, dout, dcyc);
  cudaEventRecord(e1);
  if (cudaEventSynchronize(e1)) goto done;
  {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (cudaMemcpy(hc.data(), dcyc, nsm * 8, cudaMemcpyDeviceToHost)) goto done;
    const long long mx = *std::max_element(hc.begin(), hc.end());
    const double pairs = 128.0 * (MIX == 2 ? 2.0 : 1.0) * kProbeIters * (double)kProbeThreads * nsm;
    *ppc = pairs / nsm / (double)mx;
    *mhz = (double)mx / (ms * 1e-3) / 1e6;
    *tps = pairs / (ms * 1e-3) / 1e12;
    rc = BTAS_OK;
  }
done:
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFree(din);
  cudaFree(dout);
  cudaFree(dcyc);
  (void)cudaGetLastError();
  return rc;
}

}  // namespace
}  // namespace btas

extern "C" int btas_probe_ceiling(int mix, double* pairs_per_clk_sm, double* sm_mhz, double* tpairs_per_s) {
  if (!pairs_per_clk_sm || !sm_mhz || !tpairs_per_s) return BTAS_ERR_INVALID;
  switch (mix) {
    case 0:
      return btas::run_probe<0>(pairs_per_clk_sm, sm_mhz, tpairs_per_s);
    case 1:
      return btas::run_probe<1>(pairs_per_clk_sm, sm_mhz, tpairs_per_s);
    case 2:
      return btas::run_probe<2>(pairs_per_clk_sm, sm_mhz, tpairs_per_s);
    case 3:
      return btas::run_probe_f64(pairs_per_clk_sm, sm_mhz, tpairs_per_s);
    default:
      return BTAS_ERR_INVALID;
  }
}

// f64 add-min instruction-mix microbenchmark (register resident, no memory
// traffic in the loop): how many (DADD + min) pairs per SM clock each
// formulation reaches on sm_100a.  nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o /tmp/f64mb tools/f64_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 2048, NA = 8, NB = 4;  // 8 x 4 accumulators, 2 k per step

template <int MODE>
__global__ void __launch_bounds__(256) kern(const double* __restrict__ gin, double* gout, long long* cyc) {
  double a[NA][2], b[NB][2];
#pragma unroll
  for (int i = 0; i < NA; ++i) { a[i][0] = gin[(threadIdx.x + i) & 255]; a[i][1] = gin[(threadIdx.x + 3 * i + 1) & 255]; }
#pragma unroll
  for (int j = 0; j < NB; ++j) { b[j][0] = gin[(threadIdx.x * 7 + j) & 255]; b[j][1] = gin[(threadIdx.x * 5 + j + 9) & 255]; }
  double acc[NA][NB];
#pragma unroll
  for (int i = 0; i < NA; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[i][j] = 1e300;
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NA; ++i)
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        double& c = acc[i][j];
        if (MODE == 0) {  // fmin chain (current MixF64)
          const double s0 = __dadd_rn(a[i][0], b[j][0]), s1 = __dadd_rn(a[i][1], b[j][1]);
          c = fmin(fmin(c, s0), s1);
        } else if (MODE == 1) {  // tree: min of the pair first
          const double s0 = __dadd_rn(a[i][0], b[j][0]), s1 = __dadd_rn(a[i][1], b[j][1]);
          c = fmin(c, fmin(s0, s1));
        } else if (MODE == 2) {  // adds only
          c = __dadd_rn(__dadd_rn(c, a[i][0]), b[j][1]);
        } else if (MODE == 3) {  // mins only
          c = fmin(fmin(c, a[i][0]), b[j][1]);
        } else if (MODE == 4) {  // int64 key compare (non-negative doubles)
          const double s0 = __dadd_rn(a[i][0], b[j][0]), s1 = __dadd_rn(a[i][1], b[j][1]);
          long long k = __double_as_longlong(c), k0 = __double_as_longlong(s0), k1 = __double_as_longlong(s1);
          k = k0 < k ? k0 : k;
          k = k1 < k ? k1 : k;
          c = __longlong_as_double(k);
        } else if (MODE == 6) {  // ternary chain
          const double s0 = __dadd_rn(a[i][0], b[j][0]), s1 = __dadd_rn(a[i][1], b[j][1]);
          c = s0 < c ? s0 : c;
          c = s1 < c ? s1 : c;
        } else if (MODE == 7) {  // predicate-only cost: DSETP + one 32-bit select (not a real min)
          const double s0 = __dadd_rn(a[i][0], b[j][0]), s1 = __dadd_rn(a[i][1], b[j][1]);
          const bool p0 = s0 < c, p1 = s1 < c;
          c = __hiloint2double(p0 ? __double2hiint(s0) : __double2hiint(c), p1 ? __double2loint(s1) : __double2loint(c));
        } else if (MODE == 8 || MODE == 9) {  // hybrid: part of the accumulators compare
          // on the FP64 pipe (DSETP), the rest as signed int64 keys on the ALU
          // pipe (exact for non-negative doubles and +-inf): 8 = half, 9 = 3/4 on the ALU
          const double s0 = __dadd_rn(a[i][0], b[j][0]), s1 = __dadd_rn(a[i][1], b[j][1]);
          const bool alu = MODE == 8 ? (j & 1) != 0 : (j & 3) != 0;
          if (alu) {
            long long k = __double_as_longlong(c), k0 = __double_as_longlong(s0), k1 = __double_as_longlong(s1);
            k = k0 < k ? k0 : k;
            k = k1 < k ? k1 : k;
            c = __longlong_as_double(k);
          } else {
            c = s0 < c ? s0 : c;
            c = s1 < c ? s1 : c;
          }
        } else if (MODE == 5) {  // ternary compare (DSETP + 2 SEL)
          const double s0 = __dadd_rn(a[i][0], b[j][0]), s1 = __dadd_rn(a[i][1], b[j][1]);
          const double m = s1 < s0 ? s1 : s0;
          c = m < c ? m : c;
        }
      }
#pragma unroll
    for (int i = 0; i < NA; ++i) { a[i][0] += 1.0; }
  }
  const long long t1 = clock64();
  double r = 0;
#pragma unroll
  for (int i = 0; i < NA; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) r += acc[i][j];
  gout[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int bps) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *din, *dout;
  long long* dc;
  cudaMalloc(&din, 256 * 8);
  cudaMalloc(&dout, (size_t)nsm * bps * 256 * 8);
  cudaMalloc(&dc, nsm * bps * 8);
  double h[256];
  for (int i = 0; i < 256; ++i) h[i] = 1.0 + (i * 37 % 101);
  cudaMemcpy(din, h, sizeof h, cudaMemcpyHostToDevice);
  kern<MODE><<<nsm * bps, 256>>>(din, dout, dc);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<MODE><<<nsm * bps, 256>>>(din, dout, dc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long hc[4096], mx = 0;
  cudaMemcpy(hc, dc, nsm * bps * 8, cudaMemcpyDeviceToHost);
  for (int i = 0; i < nsm * bps; ++i) mx = hc[i] > mx ? hc[i] : mx;
  const double pairs = 2.0 * NA * NB * ITERS * 256.0 * nsm * bps;
  printf("{\"mix\": \"%s\", \"blocks_per_sm\": %d, \"pairs_per_clk_sm\": %.2f, \"mhz\": %.0f}\n", name, bps,
         pairs / nsm / (double)mx, mx / (ms * 1e-3) / 1e6);
  cudaFree(din);
  cudaFree(dout);
  cudaFree(dc);
}

int main() {
  for (int bps = 1; bps <= 2; ++bps) {
    run<0>("f64 DADD + fmin chain", bps);
    run<1>("f64 DADD + fmin tree", bps);
    run<2>("f64 DADD only (2 per pair)", bps);
    run<3>("f64 fmin only (2 per pair)", bps);
    run<4>("f64 DADD + int64 key min", bps);
    run<5>("f64 DADD + ternary tree", bps);
    run<6>("f64 DADD + ternary chain", bps);
    run<7>("f64 DADD + DSETP + 1 SEL (cost probe)", bps);
    run<8>("f64 DADD + hybrid 1/2 DSETP, 1/2 int64 key", bps);
    run<9>("f64 DADD + hybrid 1/4 DSETP, 3/4 int64 key", bps);
  }
  return 0;
}

/*
 * tropical_oracle.c — plain-C restatement of the reference hot path.
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the checker for GPU
 * parity at sizes the NumPy restatement is too slow for.  Never linked into
 * or called by the product library.
 *
 * Operates on ORIENTED float64 arrays (reference storage form,
 * /root/reference/pkg/src/btas/matrix.py:3-7).  `storage` restates the
 * arithmetic of the element type under test:
 *   0 f64: candidate a+b in double, integer-mode limit 2^53 (matrix.py:297-312)
 *   1 f32: candidate rounded once to float (exact for float operands up to
 *          innocuous double rounding), limit 2^53 in integer mode
 *   2 i32: exact integers, limit 2^28 always
 * Masking rule of _product_tile (matrix.py:334-342): a finite (x) finite
 * candidate that overflows (float) or reaches the limit (integer) becomes
 * the oriented Infinity and sets *saturated.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static double round_storage(double s, int storage) {
  if (storage == 1) return (double)(float)s;
  return s;
}

static double limit_for(int storage, int integer_mode) {
  if (storage == 2) return 268435456.0; /* 2^28 */
  return integer_mode ? 9007199254740992.0 : INFINITY;
}

/* C[M x N] = (+)_k A[M x K] (x) B[K x N]; returns 0 */
int oracle_gemm(int min_plus, int storage, int integer_mode, const double* A, const double* B, double* C, int64_t M,
                int64_t N, int64_t K, int* saturated) {
  const double eps = min_plus ? INFINITY : -INFINITY;
  const double limit = limit_for(storage, integer_mode);
  const int int_lim = !isinf(limit);
  double* Bt = (double*)malloc((size_t)N * (size_t)K * sizeof(double));
  if (!Bt) return 1;
  for (int64_t k = 0; k < K; ++k)
    for (int64_t j = 0; j < N; ++j) Bt[j * K + k] = B[k * N + j];
  int sat = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : sat)
  for (int64_t i = 0; i < M; ++i) {
    const double* a = A + i * K;
    for (int64_t j = 0; j < N; ++j) {
      const double* b = Bt + j * K;
      double acc = eps;
      for (int64_t k = 0; k < K; ++k) {
        double s = round_storage(a[k] + b[k], storage);
        const int over = int_lim ? (fabs(s) >= limit) : isinf(s);
        if (over && isfinite(a[k]) && isfinite(b[k])) {
          s = eps;
          sat = 1;
        }
        if (min_plus) {
          if (s < acc) acc = s;
        } else {
          if (s > acc) acc = s;
        }
      }
      C[i * N + j] = acc;
    }
  }
  free(Bt);
  if (saturated) *saturated = sat;
  return 0;
}

/* Sequential k-rounds of apsp.py:93-133 on D (n x n, oriented min-plus,
 * already the closure base).  masked selects the overflow-masking rounds. */
int oracle_fw(int storage, int integer_mode, double* D, int64_t n, int masked, int* negative_cycle, int* saturated) {
  double limit = limit_for(storage, integer_mode);
  if (storage == 1 && !integer_mode) limit = INFINITY;
  const int int_lim = !isinf(limit);
  double* col = (double*)malloc((size_t)n * sizeof(double));
  double* row = (double*)malloc((size_t)n * sizeof(double));
  if (!col || !row) return 1;
  int sat = 0;
  for (int64_t k = 0; k < n; ++k) {
    for (int64_t i = 0; i < n; ++i) {
      col[i] = D[i * n + k];
      row[i] = D[k * n + i];
    }
#pragma omp parallel for schedule(static) reduction(| : sat)
    for (int64_t i = 0; i < n; ++i) {
      double* d = D + i * n;
      const double ci = col[i];
      for (int64_t j = 0; j < n; ++j) {
        double s = round_storage(ci + row[j], storage);
        if (masked) {
          const int over = int_lim ? (fabs(s) >= limit) : isinf(s);
          if (over && isfinite(ci) && isfinite(row[j])) {
            s = INFINITY;
            sat = 1;
          }
        }
        if (s < d[j]) d[j] = s;
      }
    }
  }
  int neg = 0;
  for (int64_t i = 0; i < n; ++i) neg |= D[i * n + i] < 0.0;
  free(col);
  free(row);
  if (negative_cycle) *negative_cycle = neg;
  if (saturated) *saturated = sat;
  return 0;
}

/* Sampled-row closure oracle (SURVEY §8(c) "At-scale verification"): rows of
 * (I (+) A)* by row-wise Bellman-Ford, R <- R (x) base until R stops
 * changing — the restatement of apsp.py:136-178's result row by row, valid
 * without a negative cycle.  Works on float32 values that the caller has
 * proven exact (every finite candidate |sum| < 2^24, checked by the caller
 * from max|base| and max|R|), so no rounding and no overflow mask arise and
 * the float32 add is the reference's float64 add.  base: n x n oriented
 * min-plus (+inf absent), row-major; R: s x n, in: base rows, out: closure
 * rows.  Returns the number of products (the last one detected the
 * fixpoint) or -1.
 *
 * Blocking (speed only; min is exact, so any order gives the same bits):
 * 16 sampled rows x 32 columns of accumulators live in registers, a 64-row
 * k panel of 512 columns of base stays in L2 while the 16 column strips
 * sweep it; threads own 512-column blocks.  AVX-512 / AVX2 / scalar
 * variants are picked at run time (the GPU box's host CPU is not this
 * container's). */
#include <immintrin.h>

#define CR_ROWS 16
#define CR_JB 512
#define CR_KB 64

__attribute__((target("avx512f"))) static void cr_block_avx512(const float* base, int64_t n, const float* Rt,
                                                               float* acc, int64_t j0, int64_t j1, int64_t k0,
                                                               int64_t k1) {
  for (int64_t jj = j0; jj < j1; jj += 32) {
    float* a = acc + (jj - j0) * CR_ROWS; /* [16 rows][32 cols] per 32-column strip */
    __m512 lo[CR_ROWS], hi[CR_ROWS];
    for (int r = 0; r < CR_ROWS; ++r) {
      lo[r] = _mm512_loadu_ps(a + r * 32);
      hi[r] = _mm512_loadu_ps(a + r * 32 + 16);
    }
    for (int64_t k = k0; k < k1; ++k) {
      const __m512 b0 = _mm512_loadu_ps(base + k * n + jj);
      const __m512 b1 = _mm512_loadu_ps(base + k * n + jj + 16);
      const float* rk = Rt + k * CR_ROWS;
      for (int r = 0; r < CR_ROWS; ++r) {
        const __m512 x = _mm512_set1_ps(rk[r]);
        lo[r] = _mm512_min_ps(lo[r], _mm512_add_ps(x, b0));
        hi[r] = _mm512_min_ps(hi[r], _mm512_add_ps(x, b1));
      }
    }
    for (int r = 0; r < CR_ROWS; ++r) {
      _mm512_storeu_ps(a + r * 32, lo[r]);
      _mm512_storeu_ps(a + r * 32 + 16, hi[r]);
    }
  }
}

__attribute__((target("avx2"))) static void cr_block_avx2(const float* base, int64_t n, const float* Rt, float* acc,
                                                          int64_t j0, int64_t j1, int64_t k0, int64_t k1) {
  for (int64_t jj = j0; jj < j1; jj += 32) {
    float* a = acc + (jj - j0) * CR_ROWS;
    for (int half = 0; half < 4; ++half) { /* 4 rows x 32 columns = 16 ymm accumulators per pass */
      __m256 c[4][4];
      for (int r = 0; r < 4; ++r)
        for (int q = 0; q < 4; ++q) c[r][q] = _mm256_loadu_ps(a + (half * 4 + r) * 32 + q * 8);
      for (int64_t k = k0; k < k1; ++k) {
        const float* brow = base + k * n + jj;
        const __m256 b0 = _mm256_loadu_ps(brow), b1 = _mm256_loadu_ps(brow + 8);
        const __m256 b2 = _mm256_loadu_ps(brow + 16), b3 = _mm256_loadu_ps(brow + 24);
        const float* rk = Rt + k * CR_ROWS + half * 4;
        for (int r = 0; r < 4; ++r) {
          const __m256 x = _mm256_set1_ps(rk[r]);
          c[r][0] = _mm256_min_ps(c[r][0], _mm256_add_ps(x, b0));
          c[r][1] = _mm256_min_ps(c[r][1], _mm256_add_ps(x, b1));
          c[r][2] = _mm256_min_ps(c[r][2], _mm256_add_ps(x, b2));
          c[r][3] = _mm256_min_ps(c[r][3], _mm256_add_ps(x, b3));
        }
      }
      for (int r = 0; r < 4; ++r)
        for (int q = 0; q < 4; ++q) _mm256_storeu_ps(a + (half * 4 + r) * 32 + q * 8, c[r][q]);
    }
  }
}

static void cr_block_scalar(const float* base, int64_t n, const float* Rt, float* acc, int64_t j0, int64_t j1,
                            int64_t k0, int64_t k1) {
  for (int64_t jj = j0; jj < j1; jj += 32) {
    float* a = acc + (jj - j0) * CR_ROWS;
    for (int64_t k = k0; k < k1; ++k)
      for (int r = 0; r < CR_ROWS; ++r) {
        const float x = Rt[k * CR_ROWS + r];
        for (int q = 0; q < 32; ++q) {
          const float c = x + base[k * n + jj + q];
          if (c < a[r * 32 + q]) a[r * 32 + q] = c;
        }
      }
  }
}

int oracle_closure_rows_f32(const float* base, int64_t n, float* R, int64_t s, int max_iter) {
  if (s < 1 || s > CR_ROWS || n < 1) return -1;
  const int64_t np = (n + 31) / 32 * 32; /* padded column count */
  float* Rt = (float*)malloc((size_t)n * CR_ROWS * sizeof(float)); /* R transposed: [k][row] */
  float* nxt = (float*)malloc((size_t)CR_ROWS * (size_t)np * sizeof(float));
  float* bpad = NULL;
  const float* B = base;
  int64_t ld = n;
  if (np != n) { /* pad base columns to a multiple of 32 with +inf */
    bpad = (float*)malloc((size_t)n * (size_t)np * sizeof(float));
    if (bpad)
      for (int64_t k = 0; k < n; ++k) {
        memcpy(bpad + k * np, base + k * n, (size_t)n * sizeof(float));
        for (int64_t j = n; j < np; ++j) bpad[k * np + j] = INFINITY;
      }
    B = bpad;
    ld = np;
  }
  if (!Rt || !nxt || (np != n && !bpad)) {
    free(Rt);
    free(nxt);
    free(bpad);
    return -1;
  }
  void (*blk)(const float*, int64_t, const float*, float*, int64_t, int64_t, int64_t, int64_t) = cr_block_scalar;
  __builtin_cpu_init();
  if (__builtin_cpu_supports("avx512f"))
    blk = cr_block_avx512;
  else if (__builtin_cpu_supports("avx2"))
    blk = cr_block_avx2;
  int result = -1;
  for (int it = 1; it <= max_iter; ++it) {
    for (int64_t k = 0; k < n; ++k)
      for (int r = 0; r < CR_ROWS; ++r) Rt[k * CR_ROWS + r] = r < s ? R[r * n + k] : INFINITY;
    int changed = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : changed)
    for (int64_t j0 = 0; j0 < np; j0 += CR_JB) {
      const int64_t j1 = j0 + CR_JB < np ? j0 + CR_JB : np;
      float* acc = nxt + j0 * CR_ROWS; /* this block's [col strip][row][32] accumulators */
      for (int64_t i = 0; i < (j1 - j0) * CR_ROWS; ++i) acc[i] = INFINITY;
      for (int64_t k0 = 0; k0 < n; k0 += CR_KB) blk(B, ld, Rt, acc, j0, j1, k0, k0 + CR_KB < n ? k0 + CR_KB : n);
      for (int64_t jj = j0; jj < j1; jj += 32)
        for (int r = 0; r < s; ++r)
          for (int q = 0; q < 32 && jj + q < n; ++q) changed |= acc[(jj - j0) * CR_ROWS + r * 32 + q] != R[r * n + jj + q];
    }
    /* R <- product (the compares above read R before any write) */
    for (int64_t jj = 0; jj < np; jj += 32)
      for (int r = 0; r < s; ++r)
        for (int q = 0; q < 32 && jj + q < n; ++q) R[r * n + jj + q] = nxt[jj * CR_ROWS + r * 32 + q];
    if (!changed) {
      result = it;
      break;
    }
  }
  free(Rt);
  free(nxt);
  free(bpad);
  return result;
}

/* max |finite| and min finite of a float32 array (the exactness screen of
 * oracle_closure_rows_f32; 0 when nothing is finite). */
void oracle_f32_finite_range(const float* x, int64_t count, float* max_abs, float* min_finite) {
  float mx = 0.0f, mn = 0.0f;
#pragma omp parallel for schedule(static) reduction(max : mx) reduction(min : mn)
  for (int64_t i = 0; i < count; ++i) {
    const float v = x[i];
    if (isfinite(v)) {
      const float a = fabsf(v);
      mx = a > mx ? a : mx;
      mn = v < mn ? v : mn;
    }
  }
  *max_abs = mx;
  *min_finite = mn;
}

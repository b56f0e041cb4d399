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

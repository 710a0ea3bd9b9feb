/*
 * ORACLE — test infrastructure only.  Never linked into the product path.
 *
 * Plain-C restatement of the reference's low-precision triangular
 * matrix-equation solver, stril(T L - L T) = -E for strictly lower L:
 *
 *   solve_block          /root/reference/pkg/src/ddschur/trisolve.py:243-262
 *   _block_solve         trisolve.py:223-240   (recursive halving, n1 = n // 2)
 *   _sylvester_tri       trisolve.py:164-196   (column-wise shifted back-substitution)
 *   _stril_inplace_add   trisolve.py:217-220
 *   _scalar_solve_inplace trisolve.py:121-145  (column j bottom-up substitution)
 *   _check_separation    trisolve.py:104-113   (exact duplicate diagonal)
 *   _check_finite        trisolve.py:116-118
 *   matmul_lp order      matmul.py:84-110 + _numba_kernels.py:49-69
 *                        (32-wide k panels, left-to-right inside a panel,
 *                         panel partials merged left to right)
 *
 * Compiled twice: SCALAR = double complex (the reference's binary64 lp,
 * dd mode) and SCALAR = float complex (FP64 mode, lp = complex64).
 * Matrices are row-major with leading dimension ld (element (i, j) at
 * i*ld + j); the reference is column-major, which only changes strides.
 *
 * Return codes follow include/sr.h: 0 ok, 1 bad argument, 2 separation,
 * 3 non-finite.
 */
#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define PANEL 32

#define DEFINE_SOLVER(SUF, SCALAR, REAL, CABS, ISFIN)                                   \
  static void mm_panel_##SUF(int m, int k, int p, const SCALAR* a, int lda,              \
                             const SCALAR* b, int ldb, SCALAR* c, int ldc) {             \
    /* c = a(m x k) * b(k x p) in the reference panel order (matmul.py:84-110,           \
       _numba_kernels.py:49-69); per-entry order fixed, rows run in parallel */          \
    _Pragma("omp parallel for schedule(static) if ((long long)m * k * p > 262144)")      \
    for (int i = 0; i < m; ++i) {                                                        \
      REAL* buf = (REAL*)malloc(sizeof(REAL) * 4 * (size_t)(p > 0 ? p : 1));             \
      REAL *acc_r = buf, *acc_i = buf + p, *pr = buf + 2 * p, *pi = buf + 3 * p;         \
      for (int j = 0; j < p; ++j) acc_r[j] = acc_i[j] = 0;                               \
      for (int p0 = 0; p0 < k; p0 += PANEL) {                                            \
        int p1 = p0 + PANEL < k ? p0 + PANEL : k;                                        \
        for (int j = 0; j < p; ++j) pr[j] = pi[j] = 0;                                   \
        for (int kk = p0; kk < p1; ++kk) {                                               \
          SCALAR x = a[(size_t)i * lda + kk];                                            \
          REAL xr = creal(x), xi = cimag(x);                                             \
          const SCALAR* brow = b + (size_t)kk * ldb;                                     \
          for (int j = 0; j < p; ++j) {                                                  \
            REAL yr = creal(brow[j]), yi = cimag(brow[j]);                               \
            REAL tr = xr * yr - xi * yi;                                                 \
            REAL ti = xr * yi + xi * yr;                                                 \
            pr[j] = pr[j] + tr;                                                          \
            pi[j] = pi[j] + ti;                                                          \
          }                                                                              \
        }                                                                                \
        for (int j = 0; j < p; ++j) {                                                    \
          acc_r[j] = acc_r[j] + pr[j];                                                   \
          acc_i[j] = acc_i[j] + pi[j];                                                   \
        }                                                                                \
      }                                                                                  \
      for (int j = 0; j < p; ++j) c[(size_t)i * ldc + j] = acc_r[j] + acc_i[j] * I;      \
      free(buf);                                                                         \
    }                                                                                    \
  }                                                                                      \
                                                                                         \
  static SCALAR dot_##SUF(int len, const SCALAR* x, int incx, const SCALAR* y,           \
                          int incy) {                                                    \
    SCALAR s = 0;                                                                        \
    for (int q = 0; q < len; ++q) s += x[(size_t)q * incx] * y[(size_t)q * incy];        \
    return s;                                                                            \
  }                                                                                      \
                                                                                         \
  /* trisolve.py:121-145 */                                                              \
  static long long scalar_solve_##SUF(int n, const SCALAR* t, int ldt, SCALAR* e,        \
                                      int lde, SCALAR* l, int ldl, REAL clip) {          \
    long long clipped = 0;                                                               \
    for (int j = 0; j < n - 1; ++j)                                                      \
      for (int i = n - 1; i > j; --i) {                                                  \
        SCALAR acc = e[(size_t)i * lde + j];                                             \
        if (i + 1 < n)                                                                   \
          acc = acc + dot_##SUF(n - i - 1, t + (size_t)i * ldt + i + 1, 1,               \
                                l + (size_t)(i + 1) * ldl + j, ldl);                     \
        if (j > 0)                                                                       \
          acc = acc - dot_##SUF(j, l + (size_t)i * ldl, 1, t + j, ldt);                  \
        e[(size_t)i * lde + j] = acc;                                                    \
        SCALAR val = -acc / (t[(size_t)i * ldt + i] - t[(size_t)j * ldt + j]);           \
        if (clip > 0 && CABS(val) > clip) {                                              \
          val = 0;                                                                       \
          clipped++;                                                                     \
        }                                                                                \
        l[(size_t)i * ldl + j] = val;                                                    \
      }                                                                                  \
    return clipped;                                                                      \
  }                                                                                      \
                                                                                         \
  /* trisolve.py:164-196: T22 X - X T11 = C, x written into x (ldx) */                   \
  static int sylvester_##SUF(int m, int p, const SCALAR* t22, const SCALAR* t11,         \
                             int ldt, const SCALAR* c, int ldc, SCALAR* x, int ldx,      \
                             REAL clip, long long* clipped) {                            \
    SCALAR* rhs = (SCALAR*)malloc(sizeof(SCALAR) * (size_t)(m > 0 ? m : 1));             \
    for (int j = 0; j < p; ++j) {                                                        \
      for (int i = 0; i < m; ++i) rhs[i] = c[(size_t)i * ldc + j];                        \
      if (j > 0) {                                                                       \
        _Pragma("omp parallel for schedule(static) if ((long long)m * j > 65536)")       \
        for (int i = 0; i < m; ++i)                                                      \
          rhs[i] += dot_##SUF(j, x + (size_t)i * ldx, 1, t11 + j, ldt);                  \
      }                                                                                  \
      SCALAR mu = t11[(size_t)j * ldt + j];                                              \
      for (int i = m - 1; i >= 0; --i) {                                                 \
        SCALAR acc = rhs[i];                                                             \
        if (i + 1 < m)                                                                   \
          acc = acc - dot_##SUF(m - i - 1, t22 + (size_t)i * ldt + i + 1, 1,             \
                                x + (size_t)(i + 1) * ldx + j, ldx);                     \
        SCALAR piv = t22[(size_t)i * ldt + i] - mu;                                      \
        if (piv == 0) {                                                                  \
          free(rhs);                                                                     \
          return 2;                                                                      \
        }                                                                                \
        SCALAR val = acc / piv;                                                          \
        if (clip > 0 && CABS(val) > clip) {                                              \
          val = 0;                                                                       \
          (*clipped)++;                                                                  \
        }                                                                                \
        x[(size_t)i * ldx + j] = val;                                                    \
      }                                                                                  \
    }                                                                                    \
    free(rhs);                                                                           \
    return 0;                                                                            \
  }                                                                                      \
                                                                                         \
  /* trisolve.py:223-240 */                                                              \
  static int block_solve_##SUF(int n, const SCALAR* t, int ldt, SCALAR* e, int lde,      \
                               SCALAR* l, int ldl, int n_min, REAL clip,                 \
                               long long* clipped) {                                     \
    if (n <= n_min) {                                                                    \
      *clipped += scalar_solve_##SUF(n, t, ldt, e, lde, l, ldl, clip);                   \
      return 0;                                                                          \
    }                                                                                    \
    int n1 = n / 2, n2 = n - n1;                                                         \
    const SCALAR* t11 = t;                                                               \
    const SCALAR* t12 = t + n1;                                                          \
    const SCALAR* t22 = t + (size_t)n1 * ldt + n1;                                       \
    SCALAR* c = (SCALAR*)malloc(sizeof(SCALAR) * (size_t)n2 * n1);                       \
    for (int i = 0; i < n2; ++i)                                                         \
      for (int j = 0; j < n1; ++j) c[(size_t)i * n1 + j] = -e[(size_t)(n1 + i) * lde + j]; \
    SCALAR* x = l + (size_t)n1 * ldl; /* L21 block, n2 x n1 */                           \
    int rc = sylvester_##SUF(n2, n1, t22, t11, ldt, c, n1, x, ldl, clip, clipped);       \
    free(c);                                                                             \
    if (rc) return rc;                                                                   \
    /* E11 += stril(T12 X); E22 -= stril(X T12) (trisolve.py:236-237) */                 \
    SCALAR* prod = (SCALAR*)malloc(sizeof(SCALAR) * (size_t)(n1 > n2 ? n1 : n2) *        \
                                   (n1 > n2 ? n1 : n2));                                 \
    mm_panel_##SUF(n1, n2, n1, t12, ldt, x, ldl, prod, n1);                              \
    for (int j = 0; j < n1; ++j)                                                         \
      for (int i = j + 1; i < n1; ++i) e[(size_t)i * lde + j] += prod[(size_t)i * n1 + j]; \
    mm_panel_##SUF(n2, n1, n2, x, ldl, t12, ldt, prod, n2);                              \
    SCALAR* e22 = e + (size_t)n1 * lde + n1;                                             \
    for (int j = 0; j < n2; ++j)                                                         \
      for (int i = j + 1; i < n2; ++i)                                                   \
        e22[(size_t)i * lde + j] += -1.0 * prod[(size_t)i * n2 + j];                     \
    free(prod);                                                                          \
    rc = block_solve_##SUF(n1, t11, ldt, e, lde, l, ldl, n_min, clip, clipped);          \
    if (rc) return rc;                                                                   \
    return block_solve_##SUF(n2, t22, ldt, e22, lde, l + (size_t)n1 * ldl + n1, ldl,     \
                             n_min, clip, clipped);                                      \
  }                                                                                      \
                                                                                         \
  static int cmp_##SUF(const void* pa, const void* pb) {                                 \
    const REAL* a = (const REAL*)pa;                                                     \
    const REAL* b = (const REAL*)pb;                                                     \
    if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;                                       \
    if (a[1] != b[1]) return a[1] < b[1] ? -1 : 1;                                       \
    return 0;                                                                            \
  }                                                                                      \
                                                                                         \
  /* solve_block, trisolve.py:243-262.  clip <= 0 disables clipping. */                  \
  int oracle_solve_block_##SUF(int n, const SCALAR* t, const SCALAR* e, SCALAR* l,       \
                               int n_min, REAL clip, long long* clipped_out) {           \
    if (n < 0 || n_min < 2) return 1;                                                    \
    for (int i = 0; i < n; ++i)                                                          \
      for (int j = 0; j < n; ++j) {                                                      \
        if (j < i && t[(size_t)i * n + j] != 0) return 1;                                \
        if (j >= i && e[(size_t)i * n + j] != 0) return 1;                               \
      }                                                                                  \
    /* exact-duplicate diagonal check (trisolve.py:104-113), O(n log n) */               \
    REAL* d = (REAL*)malloc(sizeof(REAL) * 2 * (size_t)(n > 0 ? n : 1));                 \
    for (int i = 0; i < n; ++i) {                                                        \
      d[2 * i] = creal(t[(size_t)i * n + i]);                                            \
      d[2 * i + 1] = cimag(t[(size_t)i * n + i]);                                        \
    }                                                                                    \
    qsort(d, n, 2 * sizeof(REAL), cmp_##SUF);                                            \
    for (int i = 0; i + 1 < n; ++i)                                                      \
      if (d[2 * i] == d[2 * i + 2] && d[2 * i + 1] == d[2 * i + 3]) {                    \
        free(d);                                                                         \
        return 2;                                                                        \
      }                                                                                  \
    free(d);                                                                             \
    SCALAR* ew = (SCALAR*)malloc(sizeof(SCALAR) * (size_t)(n > 0 ? n * n : 1));          \
    memcpy(ew, e, sizeof(SCALAR) * (size_t)n * n);                                       \
    memset(l, 0, sizeof(SCALAR) * (size_t)n * n);                                        \
    long long clipped = 0;                                                               \
    int rc = block_solve_##SUF(n, t, n, ew, n, l, n, n_min, clip, &clipped);             \
    free(ew);                                                                            \
    *clipped_out = clipped;                                                              \
    if (rc) return rc;                                                                   \
    for (size_t q = 0; q < (size_t)n * n; ++q)                                           \
      if (!ISFIN(creal(l[q])) || !ISFIN(cimag(l[q]))) return 3;                          \
    return 0;                                                                            \
  }                                                                                      \
                                                                                         \
  /* solve_scalar, trisolve.py:148-161 */                                                \
  int oracle_solve_scalar_##SUF(int n, const SCALAR* t, const SCALAR* e, SCALAR* l,      \
                                REAL clip, long long* clipped_out) {                     \
    return oracle_solve_block_##SUF(n, t, e, l, n > 2 ? n : 2, clip, clipped_out);       \
  }

DEFINE_SOLVER(c128, double complex, double, cabs, isfinite)
DEFINE_SOLVER(c64, float complex, float, cabsf, isfinite)

/*
 * ORACLE — test infrastructure only.  Never linked into the product path.
 *
 * Plain-C restatement of the reference's double-double complex GEMM:
 *   dd EFTs     /root/reference/pkg/src/ddschur/dd.py:53-180 (two_sum,
 *               quick_two_sum, Dekker split/two_prod without FMA, add, mul, cmul)
 *   gemm_hp     /root/reference/pkg/src/ddschur/_numba_kernels.py:18-46
 *               (per output: 32-wide k panels, dd.cmul then dd.add inside a
 *                panel left to right, panel partials folded left to right)
 * Compiled with -ffp-contract=off so no FMA is formed: the result is bit
 * identical to the reference kernel on the same inputs.
 * Planes are row-major: element (i, j) at i*ld + j.
 */
#include <stddef.h>

static const double SPLITTER = 134217729.0; /* 2^27 + 1, dd.py:26 */

static inline void two_sum(double a, double b, double* s, double* e) {
  double ss = a + b, bb = ss - a;
  *e = (a - (ss - bb)) + (b - bb);
  *s = ss;
}
static inline void quick_two_sum(double a, double b, double* s, double* e) {
  double ss = a + b;
  *e = b - (ss - a);
  *s = ss;
}
static inline void split(double a, double* hi, double* lo) {
  double t = SPLITTER * a;
  double h = t - (t - a);
  *hi = h;
  *lo = a - h;
}
static inline void two_prod(double a, double b, double* p, double* e) {
  double pp = a * b, ah, al, bh, bl;
  split(a, &ah, &al);
  split(b, &bh, &bl);
  *e = ((ah * bh - pp) + ah * bl + al * bh) + al * bl;
  *p = pp;
}
static inline void dd_add(double ah, double al, double bh, double bl, double* rh, double* rl) {
  double s1, s2, t1, t2;
  two_sum(ah, bh, &s1, &s2);
  two_sum(al, bl, &t1, &t2);
  s2 += t1;
  quick_two_sum(s1, s2, &s1, &s2);
  s2 += t2;
  quick_two_sum(s1, s2, rh, rl);
}
static inline void dd_sub(double ah, double al, double bh, double bl, double* rh, double* rl) {
  dd_add(ah, al, -bh, -bl, rh, rl);
}
static inline void dd_mul(double ah, double al, double bh, double bl, double* rh, double* rl) {
  double p, e;
  two_prod(ah, bh, &p, &e);
  double cross = ah * bl + al * bh;
  e += cross + al * bl;
  quick_two_sum(p, e, rh, rl);
}
static inline void dd_cmul(double arh, double arl, double aih, double ail, double brh, double brl,
                           double bih, double bil, double* rh, double* rl, double* ih, double* il) {
  double ph, pl, qh, ql, sh, sl, th, tl;
  dd_mul(arh, arl, brh, brl, &ph, &pl);
  dd_mul(aih, ail, bih, bil, &qh, &ql);
  dd_sub(ph, pl, qh, ql, rh, rl);
  dd_mul(arh, arl, bih, bil, &sh, &sl);
  dd_mul(aih, ail, brh, brl, &th, &tl);
  dd_add(sh, sl, th, tl, ih, il);
}

/* C(m x n) = A(m x k) B(k x n), all double-double complex planes. */
void oracle_gemm_dd(int m, int n, int k, int panel,
                    const double* arh, const double* arl, const double* aih, const double* ail,
                    const double* brh, const double* brl, const double* bih, const double* bil,
                    double* orh, double* orl, double* oih, double* oil) {
#pragma omp parallel for schedule(static)
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) {
      double acc_rh = 0, acc_rl = 0, acc_ih = 0, acc_il = 0;
      for (int p0 = 0; p0 < k; p0 += panel) {
        int p1 = p0 + panel < k ? p0 + panel : k;
        double prh = 0, prl = 0, pih = 0, pil = 0;
        for (int kk = p0; kk < p1; ++kk) {
          size_t ia = (size_t)i * k + kk, ib = (size_t)kk * n + j;
          double crh, crl, cih, cil;
          dd_cmul(arh[ia], arl[ia], aih[ia], ail[ia], brh[ib], brl[ib], bih[ib], bil[ib],
                  &crh, &crl, &cih, &cil);
          dd_add(prh, prl, crh, crl, &prh, &prl);
          dd_add(pih, pil, cih, cil, &pih, &pil);
        }
        dd_add(acc_rh, acc_rl, prh, prl, &acc_rh, &acc_rl);
        dd_add(acc_ih, acc_il, pih, pil, &acc_ih, &acc_il);
      }
      size_t io = (size_t)i * n + j;
      orh[io] = acc_rh;
      orl[io] = acc_rl;
      oih[io] = acc_ih;
      oil[io] = acc_il;
    }
}

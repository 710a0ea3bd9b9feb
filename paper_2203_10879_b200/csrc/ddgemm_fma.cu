// Double-double complex GEMM with FMA error-free transformations on the FP64
// pipe — the comparison point north_star item 2 asks for ("FMA-based
// TwoProd/TwoSum GEMM kernels or an Ozaki-split ... picked by measured
// throughput"), against the Ozaki-II int8 products (ozaki.cu / oz_gemm.cu)
// that dd mode uses.  Replaces the same call site as those: the reference's
// gemm_hp (/root/reference/pkg/src/ddschur/_numba_kernels.py:18-46, EFTs of
// dd.py:53-180 — Dekker's split, no FMA), here with the FMA forms:
//
//   two_prod(a, b) = (p, fma(a, b, -p))                    2 ops (Dekker: 17)
//   dd x dd        = p + (e + a.h b.l + a.l b.h)            4 ops
//   acc += term    two_sum on the hi parts, lo parts summed 8 ops
//
// 48 FP64 instructions per complex dd multiply-accumulate (the reference's
// Dekker cmul + two dd adds: ~184).  C = op(A) B, planar row-major dd planes
// (re_hi, re_lo, im_hi, im_lo), op = N or C (conjugate transpose).  Tiles:
// 32 x 32 outputs per 256-thread block, 2 x 2 complex outputs per thread,
// k-tiles of 16 staged in shared memory; the hi/lo accumulators are
// renormalised (quick_two_sum) at the end of every k-tile.
#include "sr_common.cuh"

namespace {

constexpr int BM = 32, BN = 32, BK = 16;

struct dd2 {
  double h, l;
};

// acc += s * (a * b) for dd a, b and s = +-1 (unnormalised accumulator:
// two_sum on the hi parts, every low-order term folded into acc.l)
__device__ __forceinline__ void fma_acc(dd2& acc, double ah, double al, double bh, double bl, double s) {
  const double p = s * (ah * bh);
  double e = fma(s * ah, bh, -p);
  e = fma(s * ah, bl, e);
  e = fma(s * al, bh, e);
  const double t = acc.h + p;
  const double bb = t - acc.h;
  const double err = (acc.h - (t - bb)) + (p - bb);
  acc.h = t;
  acc.l += err + e;
}

__device__ __forceinline__ void renorm(dd2& a) {
  const double s = a.h + a.l;
  a.l = a.l - (s - a.h);
  a.h = s;
}

struct Plane4 {
  const double *rh, *rl, *ih, *il;
};

template <int OPA>
__global__ void __launch_bounds__(256) ddgemm_fma_kernel(int m, int n, int k, Plane4 A, long long lda, Plane4 B,
                                                         long long ldb, double* crh, double* crl, double* cih,
                                                         double* cil, long long ldc) {
  __shared__ double sa[4][BK][BM + 1];  // [plane][k][i]
  __shared__ double sb[4][BK][BN + 1];  // [plane][k][j]
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int i0 = blockIdx.y * BM, j0 = blockIdx.x * BN;
  dd2 accr[2][2], acci[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) accr[a][b] = acci[a][b] = {0.0, 0.0};
  for (int k0 = 0; k0 < k; k0 += BK) {
    // stage op(A)[i0 .. i0+32][k0 .. k0+16] and B[k0 .. k0+16][j0 .. j0+32]
    for (int idx = threadIdx.x; idx < BM * BK; idx += 256) {
      int i, kk;
      size_t off;
      if (OPA == 0) {
        i = idx / BK, kk = idx % BK;
        off = (size_t)(i0 + i) * lda + (k0 + kk);
      } else {  // A^H: element (i, kk) = conj(A[kk][i]), coalesced along i
        kk = idx / BM, i = idx % BM;
        off = (size_t)(k0 + kk) * lda + (i0 + i);
      }
      const bool in = (i0 + i) < m && (k0 + kk) < k;
      const double sg = OPA ? -1.0 : 1.0;
      sa[0][kk][i] = in ? A.rh[off] : 0.0;
      sa[1][kk][i] = in ? A.rl[off] : 0.0;
      sa[2][kk][i] = in ? sg * A.ih[off] : 0.0;
      sa[3][kk][i] = in ? sg * A.il[off] : 0.0;
    }
    for (int idx = threadIdx.x; idx < BK * BN; idx += 256) {
      const int kk = idx / BN, j = idx % BN;
      const bool in = (k0 + kk) < k && (j0 + j) < n;
      const size_t off = (size_t)(k0 + kk) * ldb + (j0 + j);
      sb[0][kk][j] = in ? B.rh[off] : 0.0;
      sb[1][kk][j] = in ? B.rl[off] : 0.0;
      sb[2][kk][j] = in ? B.ih[off] : 0.0;
      sb[3][kk][j] = in ? B.il[off] : 0.0;
    }
    __syncthreads();
#pragma unroll 2
    for (int kk = 0; kk < BK; ++kk) {
      double a[2][4], b[2][4];
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int pl = 0; pl < 4; ++pl) {
          a[r][pl] = sa[pl][kk][ty + 16 * r];
          b[r][pl] = sb[pl][kk][tx + 16 * r];
        }
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          // (ar + i ai)(br + i bi): re = ar br - ai bi, im = ar bi + ai br
          fma_acc(accr[r][c], a[r][0], a[r][1], b[c][0], b[c][1], 1.0);
          fma_acc(accr[r][c], a[r][2], a[r][3], b[c][2], b[c][3], -1.0);
          fma_acc(acci[r][c], a[r][0], a[r][1], b[c][2], b[c][3], 1.0);
          fma_acc(acci[r][c], a[r][2], a[r][3], b[c][0], b[c][1], 1.0);
        }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        renorm(accr[r][c]);
        renorm(acci[r][c]);
      }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int i = i0 + ty + 16 * r, j = j0 + tx + 16 * c;
      if (i < m && j < n) {
        const size_t o = (size_t)i * ldc + j;
        crh[o] = accr[r][c].h;
        crl[o] = accr[r][c].l;
        cih[o] = acci[r][c].h;
        cil[o] = acci[r][c].l;
      }
    }
}

}  // namespace

extern "C" int sr_zgemm_dd_fma(int op_a, int m, int n, int k, const double* a_rh, const double* a_rl,
                               const double* a_ih, const double* a_il, long long lda, const double* b_rh,
                               const double* b_rl, const double* b_ih, const double* b_il, long long ldb,
                               double* c_rh, double* c_rl, double* c_ih, double* c_il, long long ldc, void* stream) {
  if (m < 0 || n < 0 || k < 0 || (op_a != SR_OP_N && op_a != SR_OP_C)) return SR_EINVAL;
  if ((long long)m * n == 0) return SR_OK;
  const Plane4 A{a_rh, a_rl, a_ih, a_il}, B{b_rh, b_rl, b_ih, b_il};
  const dim3 grid(sr_ceil_div(n, BN), sr_ceil_div(m, BM));
  if (op_a == SR_OP_N)
    ddgemm_fma_kernel<0><<<grid, 256, 0, (cudaStream_t)stream>>>(m, n, k, A, lda, B, ldb, c_rh, c_rl, c_ih, c_il,
                                                                 ldc);
  else
    ddgemm_fma_kernel<1><<<grid, 256, 0, (cudaStream_t)stream>>>(m, n, k, A, lda, B, ldb, c_rh, c_rl, c_ih, c_il,
                                                                 ldc);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

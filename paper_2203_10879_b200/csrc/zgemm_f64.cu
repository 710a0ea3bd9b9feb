// FP64 complex GEMM on the sm_100a FP64 tensor pipe (DMMA, mma.sync m16n8k8 f64).
//
//   C = alpha * op(A) * B  (+ diag_shift on the diagonal),   op(A) = A or A^H
//
// Planar complex storage (separate re / im planes, row-major, leading
// dimension in elements).  B may be real (b_im == NULL): the Q^H A product
// of config 3 then costs two real products instead of four.
//
// Replaces the reference's hp product in FP64 mode:
//   matmul_hp      /root/reference/pkg/src/ddschur/matmul.py:52-81
//   gemm_hp        /root/reference/pkg/src/ddschur/_numba_kernels.py:18-46
// Summation order is the DMMA k8 chain over 16-wide k tiles, fixed for a
// given launch configuration (deterministic, like the reference's fixed
// panel order; not bit-identical to it).
//
// Tiling: CTA 128 x 64 complex outputs, 8 warps (4 x 2), warp tile 32 x 32,
// k tile 16, 3-stage cp.async pipeline (LDGSTS, 16-byte granules with
// zero-fill at the edges).  Shared-memory rows are padded so every 64-bit
// fragment read is conflict-free.
#include "sr_common.cuh"

namespace {

constexpr int BM = 128, BN = 64, BK = 16, STAGES = 3;
constexpr int NTHREADS = 256;
constexpr int SA_N = BK + 4;   // A tile [m][k] (op N): padded row stride
constexpr int SA_C = BM + 4;   // A tile [k][m] (op C): padded row stride
constexpr int SB = BN + 4;     // B tile [k][n]
constexpr int A_PLANE = (BM * SA_N > BK * SA_C) ? BM * SA_N : BK * SA_C;  // doubles
constexpr int B_PLANE = BK * SB;
constexpr int STAGE_DOUBLES = 2 * A_PLANE + 2 * B_PLANE;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_DOUBLES * sizeof(double);
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");

__device__ __forceinline__ void dmma(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// Load one pair of doubles (16 bytes) with zero fill beyond `limit` columns.
__device__ __forceinline__ void load_pair(double* s, const double* g, int col, int limit, bool row_ok) {
  int bytes = 0;
  if (row_ok) bytes = (col + 1 < limit) ? 16 : (col < limit ? 8 : 0);
  cp_async_16(s, g, bytes);
}

template <int OPA, bool BREAL>
__device__ __forceinline__ void load_stage(double* st, const double* __restrict__ ar,
                                           const double* __restrict__ ai, long long lda,
                                           const double* __restrict__ br, const double* __restrict__ bi,
                                           long long ldb, int m0, int n0, int k0, int M, int N, int K) {
  const int tid = threadIdx.x;
  double* sar = st;
  double* sai = st + A_PLANE;
  double* sbr = st + 2 * A_PLANE;
  double* sbi = sbr + B_PLANE;
  if (OPA == 0) {
    // A tile rows m0..m0+127, cols k0..k0+15: 128 rows x 8 pairs = 1024 pairs / plane
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int idx = tid + r * NTHREADS;
      int row = idx >> 3, pc = (idx & 7) * 2;
      int gm = m0 + row, gk = k0 + pc;
      bool ok = gm < M;
      size_t off = (size_t)(ok ? gm : 0) * lda + (gk < K ? gk : 0);
      load_pair(sar + row * SA_N + pc, ar + off, gk, K, ok);
      load_pair(sai + row * SA_N + pc, ai + off, gk, K, ok);
    }
  } else {
    // A^H tile: read A rows k0..k0+15, cols m0..m0+127 (contiguous): 16 x 64 pairs
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int idx = tid + r * NTHREADS;
      int row = idx >> 6, pc = (idx & 63) * 2;
      int gk = k0 + row, gm = m0 + pc;
      bool ok = gk < K;
      size_t off = (size_t)(ok ? gk : 0) * lda + (gm < M ? gm : 0);
      load_pair(sar + row * SA_C + pc, ar + off, gm, M, ok);
      load_pair(sai + row * SA_C + pc, ai + off, gm, M, ok);
    }
  }
  // B tile rows k0..k0+15, cols n0..n0+63: 16 x 32 pairs = 512 pairs / plane
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    int idx = tid + r * NTHREADS;
    int row = idx >> 5, pc = (idx & 31) * 2;
    int gk = k0 + row, gn = n0 + pc;
    bool ok = gk < K;
    size_t off = (size_t)(ok ? gk : 0) * ldb + (gn < N ? gn : 0);
    load_pair(sbr + row * SB + pc, br + off, gn, N, ok);
    if (!BREAL) load_pair(sbi + row * SB + pc, bi + off, gn, N, ok);
  }
}

template <int OPA, bool BREAL>
__global__ void __launch_bounds__(NTHREADS, 1)
    zgemm_f64_kernel(int M, int N, int K, double alpha, double diag_shift, const double* __restrict__ ar,
                     const double* __restrict__ ai, long long lda, const double* __restrict__ br,
                     const double* __restrict__ bi, long long ldb, double* __restrict__ cr,
                     double* __restrict__ ci, long long ldc) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 3, wn = warp >> 2;  // 4 x 2 warps
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int ktiles = (K + BK - 1) / BK;

  double accr[2][4][4], acci[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) accr[i][j][v] = acci[i][j][v] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles)
      load_stage<OPA, BREAL>(smem + s * STAGE_DOUBLES, ar, ai, lda, br, bi, ldb, m0, n0, s * BK, M, N, K);
    cp_async_commit();
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {  // prefetch tile kt + STAGES - 1 into the slot freed at iteration kt - 1
      int nk = kt + STAGES - 1;
      if (nk < ktiles)
        load_stage<OPA, BREAL>(smem + (nk % STAGES) * STAGE_DOUBLES, ar, ai, lda, br, bi, ldb, m0, n0,
                               nk * BK, M, N, K);
      cp_async_commit();
    }
    const double* st = smem + (kt % STAGES) * STAGE_DOUBLES;
    const double* sar = st;
    const double* sai = st + A_PLANE;
    const double* sbr = st + 2 * A_PLANE;
    const double* sbi = sbr + B_PLANE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 8) {
      double fa_r[2][4], fa_i[2][4], fa_n[2][4], fb_r[4][2], fb_i[4][2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        int mr = wm * 32 + i * 16 + g;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          int m = mr + (v & 1) * 8, k = kk + t + (v >> 1) * 4;
          double xr, xi;
          if (OPA == 0) {
            xr = sar[m * SA_N + k];
            xi = sai[m * SA_N + k];
          } else {
            xr = sar[k * SA_C + m];
            xi = sai[k * SA_C + m];
          }
          fa_r[i][v] = xr;
          fa_i[i][v] = xi;
          fa_n[i][v] = -xi;
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int n = wn * 32 + j * 8 + g;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          int k = kk + t + v * 4;
          fb_r[j][v] = sbr[k * SB + n];
          if (!BREAL) fb_i[j][v] = sbi[k * SB + n];
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma(accr[i][j], fa_r[i], fb_r[j]);
          if (OPA == 0) {
            // (ar + i ai)(br + i bi)
            dmma(acci[i][j], fa_i[i], fb_r[j]);
            if (!BREAL) {
              dmma(accr[i][j], fa_n[i], fb_i[j]);
              dmma(acci[i][j], fa_r[i], fb_i[j]);
            }
          } else {
            // conj(a): (ar - i ai)(br + i bi)
            dmma(acci[i][j], fa_n[i], fb_r[j]);
            if (!BREAL) {
              dmma(accr[i][j], fa_i[i], fb_i[j]);
              dmma(acci[i][j], fa_r[i], fb_i[j]);
            }
          }
        }
    }
  }
  cp_async_wait<0>();

  // epilogue: c[v] = C[g + 8 (v>>1)][2t + (v&1)]
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int m = m0 + wm * 32 + i * 16 + g + h * 8;
        int n = n0 + wn * 32 + j * 8 + 2 * t;
        if (m >= M) continue;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (n + e >= N) continue;
          double vr = alpha * accr[i][j][h * 2 + e];
          double vi = alpha * acci[i][j][h * 2 + e];
          if (m == n + e) vr += diag_shift;
          size_t off = (size_t)m * ldc + n + e;
          cr[off] = vr;
          ci[off] = vi;
        }
      }
}

template <int OPA, bool BREAL>
int launch(int m, int n, int k, double alpha, double shift, const double* ar, const double* ai, long long lda,
           const double* br, const double* bi, long long ldb, double* cr, double* ci, long long ldc,
           cudaStream_t st) {
  auto kern = zgemm_f64_kernel<OPA, BREAL>;
  static bool configured[SR_MAX_DEVICES] = {};  // function attributes are per device
  int slot = 0;
  if (sr_device_slot(&slot) != SR_OK) return SR_EINVAL;
  if (!configured[slot]) {
    SR_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
    configured[slot] = true;
  }
  dim3 grid(sr_ceil_div(n, BN), sr_ceil_div(m, BM));
  kern<<<grid, NTHREADS, SMEM_BYTES, st>>>(m, n, k, alpha, shift, ar, ai, lda, br, bi, ldb, cr, ci, ldc);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

}  // namespace

extern "C" int sr_zgemm_f64(int op_a, int m, int n, int k, double alpha, double diag_shift, const double* a_re,
                            const double* a_im, long long lda, const double* b_re, const double* b_im,
                            long long ldb, double* c_re, double* c_im, long long ldc, void* stream) {
  if (m < 0 || n < 0 || k < 0 || !a_re || !a_im || !b_re || !c_re || !c_im) return SR_EINVAL;
  if ((lda | ldb | ldc) & 1) return SR_EINVAL;  // 16-byte row alignment for cp.async
  if (((uintptr_t)a_re | (uintptr_t)a_im | (uintptr_t)b_re | (uintptr_t)(b_im ? b_im : b_re)) & 15)
    return SR_EINVAL;
  if (m == 0 || n == 0) return SR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  bool breal = (b_im == nullptr);
  if (op_a == SR_OP_N)
    return breal ? launch<0, true>(m, n, k, alpha, diag_shift, a_re, a_im, lda, b_re, b_im, ldb, c_re, c_im, ldc, st)
                 : launch<0, false>(m, n, k, alpha, diag_shift, a_re, a_im, lda, b_re, b_im, ldb, c_re, c_im, ldc, st);
  if (op_a == SR_OP_C)
    return breal ? launch<1, true>(m, n, k, alpha, diag_shift, a_re, a_im, lda, b_re, b_im, ldb, c_re, c_im, ldc, st)
                 : launch<1, false>(m, n, k, alpha, diag_shift, a_re, a_im, lda, b_re, b_im, ldb, c_re, c_im, ldc, st);
  return SR_EINVAL;
}

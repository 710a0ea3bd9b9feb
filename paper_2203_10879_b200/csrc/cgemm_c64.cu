// lp complex64 GEMM on the FP32 pipe: C = A * B (complex64, interleaved).
//
// Replaces the reference's lp product in FP64 mode (lp = complex64):
//   matmul_lp  /root/reference/pkg/src/ddschur/matmul.py:84-110
//   gemm_lp    /root/reference/pkg/src/ddschur/_numba_kernels.py:49-69
// used for Y W, W^2, W^3 (and W^2 Y, W^2 Y W) in merged_update
// (orthogonal.py:188-199).
//
// CTA tile 64 x 64, 256 threads, 4 x 4 complex outputs per thread, k tile 16,
// register-staged double buffering; A is stored k-major in shared memory so
// each thread reads its 4 A values as two 16-byte vectors.
#include "sr_common.cuh"

namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;
constexpr int PADA = 4, PADB = 4;

__global__ void __launch_bounds__(NT) cgemm_c64_kernel(int M, int N, int K, const float2* __restrict__ A,
                                                       long long lda, const float2* __restrict__ B, long long ldb,
                                                       float2* __restrict__ C, long long ldc) {
  __shared__ __align__(16) float2 As[2][BK][BM + PADA];
  __shared__ __align__(16) float2 Bs[2][BK][BN + PADB];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  float2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);

  float2 ra[4], rb[4];
  auto gload = [&](int k0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int idx = tid + r * NT;       // A: 64 rows x 16 k
      int row = idx / BK, kk = idx % BK;
      int gm = m0 + row, gk = k0 + kk;
      ra[r] = (gm < M && gk < K) ? A[(size_t)gm * lda + gk] : make_float2(0.f, 0.f);
      int brow = idx / BN, bc = idx % BN;  // B: 16 k x 64 cols
      int gk2 = k0 + brow, gn = n0 + bc;
      rb[r] = (gk2 < K && gn < N) ? B[(size_t)gk2 * ldb + gn] : make_float2(0.f, 0.f);
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int idx = tid + r * NT;
      As[buf][idx % BK][idx / BK] = ra[r];
      Bs[buf][idx / BN][idx % BN] = rb[r];
    }
  };

  const int ktiles = (K + BK - 1) / BK;
  if (ktiles > 0) {
    gload(0);
    sstore(0);
  }
  __syncthreads();
  for (int kt = 0; kt < ktiles; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < ktiles) gload((kt + 1) * BK);
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float4 a01 = *reinterpret_cast<const float4*>(&As[buf][k][4 * ty]);
      float4 a23 = *reinterpret_cast<const float4*>(&As[buf][k][4 * ty + 2]);
      float4 b01 = *reinterpret_cast<const float4*>(&Bs[buf][k][4 * tx]);
      float4 b23 = *reinterpret_cast<const float4*>(&Bs[buf][k][4 * tx + 2]);
      float2 a[4] = {make_float2(a01.x, a01.y), make_float2(a01.z, a01.w), make_float2(a23.x, a23.y),
                     make_float2(a23.z, a23.w)};
      float2 b[4] = {make_float2(b01.x, b01.y), make_float2(b01.z, b01.w), make_float2(b23.x, b23.y),
                     make_float2(b23.z, b23.w)};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j].x = fmaf(a[i].x, b[j].x, acc[i][j].x);
          acc[i][j].x = fmaf(-a[i].y, b[j].y, acc[i][j].x);
          acc[i][j].y = fmaf(a[i].x, b[j].y, acc[i][j].y);
          acc[i][j].y = fmaf(a[i].y, b[j].x, acc[i][j].y);
        }
    }
    if (kt + 1 < ktiles) {
      sstore(buf ^ 1);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + 4 * ty + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + 4 * tx + j;
      if (n < N) C[(size_t)m * ldc + n] = acc[i][j];
    }
  }
}

}  // namespace

extern "C" int sr_cgemm_c64(int op_a, int m, int n, int k, const void* a, long long lda, const void* b,
                            long long ldb, void* c, long long ldc, void* stream) {
  if (op_a != SR_OP_N || m < 0 || n < 0 || k < 0 || !a || !b || !c) return SR_EINVAL;
  if (m == 0 || n == 0) return SR_OK;
  dim3 grid(sr_ceil_div(n, BN), sr_ceil_div(m, BM));
  cgemm_c64_kernel<<<grid, NT, 0, (cudaStream_t)stream>>>(m, n, k, (const float2*)a, lda, (const float2*)b, ldb,
                                                          (float2*)c, ldc);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

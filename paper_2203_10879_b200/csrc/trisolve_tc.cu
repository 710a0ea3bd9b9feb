// Far updates of the complex64 lp solver on the 5th-generation tensor cores.
//
// trisolve.cu's wavefront applies ~93 % of the solver's n^3/3 complex
// multiply-adds as FAR updates: once the four levels of batch b are solved,
//   COL  Rf[strip, M] -= T[strip, K0..K0+3] L[K0..K0+3, M]    (strip = 4 tiles of column M)
//   ROW  Rf[I, strip] += L[I, J0..J0+3] T[J0..J0+3, strip]    (strip = 4 tiles of row I)
// (index sets in trisolve.cu).  Here each strip is one tcgen05 GEMM tile:
//   * complex as real: with A' = a complex row read as interleaved (re, im)
//     floats and B'^T rows 2c, 2c+1 = conj(b_c), i conj(b_c) (interleaved), the
//     real product A' B' is the interleaved complex product, so every operand is
//     a plain K-major fp32 matrix and the accumulator columns come out as
//     (re, im) pairs;
//   * 3xTF32: every operand is split x = hi + lo (hi = x with the low 13
//     mantissa bits cleared, exactly representable in TF32; lo = x - hi), and
//     D += A_hi B_hi + A_hi B_lo + A_lo B_hi in FP32 TMEM accumulators, which is
//     complex64-grade accuracy (the lp arithmetic of FP64 mode);
//   * COL: M = 128 strip rows, N = 64 (32 complex columns of tile M), K = 256
//     (4 source tiles x 32 complex);  ROW runs the transposed product
//     C^T = T^T L^T so that its 128 strip columns are the MMA's M dimension.
// Operand forms (built on the far stream, never on the critical path):
//   tform / ttform  hi, lo planes of T and T^T (once per solve)
//   lb              rows 2c, 2c+1 = conj(L[:, c]), i conj(L[:, c])   (COL B operand)
//   lc              rows 2i, 2i+1 = conj(L[i, :]), i conj(L[i, :])   (ROW B operand)
// (the L forms of batch b are written right before its far updates).  TMA
// loads both planes of a 64-byte K block per operand (64-byte swizzle, zero
// fill outside the matrix, which also supplies the non-existent source tiles),
// a 2-stage mbarrier ring feeds the single-thread MMA issuer (4 CTAs per SM), and four
// epilogue warps read the 128 x 64 accumulator with tcgen05.ld and update Rf.
#include "trisolve_tc.cuh"
#include "tc_common.cuh"

namespace {

constexpr int NB = 32;
constexpr int BW = 4;
constexpr int KB_F = 16;                           // fp32 per 64-byte K block
constexpr int NKB = BW * NB * 2 / KB_F;            // 16 K blocks per strip
constexpr int TC_STAGES = 2;  // 50 KB of shared memory: 4 CTAs per SM hide each other's latency
constexpr int A_PLANE = 128 * 64;                  // bytes: 128 rows x 64 B
constexpr int B_PLANE = 64 * 64;                   // bytes: 64 rows x 64 B
constexpr int TC_STAGE = 2 * A_PLANE + 2 * B_PLANE;
constexpr int TC_THREADS = 192;
constexpr uint32_t TC_TMEM_COLS = 64;

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// hi / lo planes of T (row-major) and T^T, as interleaved fp32
__global__ void __launch_bounds__(256) tforms_kernel(int n, const float2* __restrict__ T, long long ld,
                                                     float* __restrict__ tf, float* __restrict__ ttf, int P) {
  __shared__ float2 s[NB][NB + 1];
  const int r0 = blockIdx.y * NB, c0 = blockIdx.x * NB;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const size_t plane = (size_t)n * P;
  for (int r = ty; r < NB; r += 8) {
    const int gr = r0 + r, gc = c0 + tx;
    float2 v = make_float2(0.f, 0.f);
    if (gr < n && gc < n) {
      v = T[(size_t)gr * ld + gc];
      const float2 h = make_float2(tf32_hi(v.x), tf32_hi(v.y));
      *reinterpret_cast<float2*>(tf + (size_t)gr * P + 2 * gc) = h;
      *reinterpret_cast<float2*>(tf + plane + (size_t)gr * P + 2 * gc) = make_float2(v.x - h.x, v.y - h.y);
    }
    s[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < NB; r += 8) {  // T^T[c0 + r][r0 + tx] = T[r0 + tx][c0 + r]
    const int gr = c0 + r, gc = r0 + tx;
    if (gr < n && gc < n) {
      const float2 v = s[tx][r];
      const float2 h = make_float2(tf32_hi(v.x), tf32_hi(v.y));
      *reinterpret_cast<float2*>(ttf + (size_t)gr * P + 2 * gc) = h;
      *reinterpret_cast<float2*>(ttf + plane + (size_t)gr * P + 2 * gc) = make_float2(v.x - h.x, v.y - h.y);
    }
  }
}

__device__ __forceinline__ void put_split(float* base, size_t plane, size_t off, float x, float y) {
  const float2 h = make_float2(tf32_hi(x), tf32_hi(y));
  *reinterpret_cast<float2*>(base + off) = h;
  *reinterpret_cast<float2*>(base + plane + off) = make_float2(x - h.x, y - h.y);
}

// L forms of the tiles on levels 4b .. 4b+3 (blockIdx.y = level - 4b, blockIdx.x = M)
__global__ void __launch_bounds__(256) lforms_kernel(int n, int N, int b, const float2* __restrict__ L, long long ld,
                                                     float* __restrict__ lb, float* __restrict__ lc, int P) {
  __shared__ float2 s[NB][NB + 1];
  const int level = BW * b + blockIdx.y;
  const int M = blockIdx.x;
  if (level > N - 1 || M > level) return;
  const int I = M + N - 1 - level;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < NB; r += 8) {
    const int gr = I * NB + r, gc = M * NB + tx;
    s[r][tx] = (gr < n && gc < n) ? L[(size_t)gr * ld + gc] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  const size_t plane = (size_t)2 * n * P;
  for (int c = ty; c < NB; c += 8) {  // LB rows 2C, 2C+1 (C = column of L), cols 2K (K = row of L)
    const int C = M * NB + c, K = I * NB + tx;
    if (C < n && K < n) {
      const float2 v = s[tx][c];
      put_split(lb, plane, (size_t)(2 * C) * P + 2 * K, v.x, -v.y);
      put_split(lb, plane, (size_t)(2 * C + 1) * P + 2 * K, v.y, v.x);
    }
  }
  for (int i = ty; i < NB; i += 8) {  // LC rows 2R, 2R+1 (R = row of L), cols 2K (K = column of L)
    const int R = I * NB + i, K = M * NB + tx;
    if (R < n && K < n) {
      const float2 v = s[i][tx];
      put_split(lc, plane, (size_t)(2 * R) * P + 2 * K, v.x, -v.y);
      put_split(lc, plane, (size_t)(2 * R + 1) * P + 2 * K, v.y, v.x);
    }
  }
}

__device__ __forceinline__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

struct FarTcArgs {
  int n, N, b, h, first;
  long long ld;
};

template <bool ROW>
__global__ void __launch_bounds__(TC_THREADS, 1)
    far_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                  const __grid_constant__ FarTcArgs p, float2* __restrict__ Rf) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + TC_STAGES * TC_STAGE);  // full[S], empty[S], done
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * TC_STAGES + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (TC_STAGES + s); };
  const uint32_t done_bar = bar0 + 8u * (2 * TC_STAGES);

  const int N = p.N, b = p.b;
  const int line = p.first + blockIdx.y;
  const int t0 = BW * blockIdx.x;
  int a_row0, b_row0, k0;  // A rows (strip), B rows (2 x the tile's rows / cols), first K' column
  if (!ROW) {
    const int M = line;
    a_row0 = (M + t0) * NB;
    b_row0 = 2 * M * NB;
    k0 = (M + N - BW * b - BW) * NB * 2;
  } else {
    const int I = line;
    a_row0 = (I - N + BW * b + 2 * BW + 1 + t0) * NB;
    b_row0 = 2 * I * NB;
    k0 = (I - N + 1 + BW * b) * NB * 2;
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&map_b) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(TC_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      for (int kb = 0; kb < NKB; ++kb) {
        const int s = kb % TC_STAGES;
        if (kb >= TC_STAGES) mbar_wait(empty_bar(s), ((kb / TC_STAGES) - 1) & 1);
        uint8_t* st = smem + s * TC_STAGE;
        mbar_expect_tx(full_bar(s), TC_STAGE);
        tma_load_3d(smem_u32(st), &map_a, full_bar(s), k0 + kb * KB_F, a_row0, 0);
        tma_load_3d(smem_u32(st + 2 * A_PLANE), &map_b, full_bar(s), k0 + kb * KB_F, b_row0, 0);
      }
    }
  } else if (warp == 1) {  // MMA issuer
    const uint32_t id = idesc_tf32(128, 64);
    for (int kb = 0; kb < NKB; ++kb) {
      const int s = kb % TC_STAGES;
      mbar_wait(full_bar(s), (kb / TC_STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (lane == 0) {
        const uint32_t sa = smem_u32(smem + s * TC_STAGE);
        const uint32_t sb = sa + 2 * A_PLANE;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {  // two K = 8 tf32 steps per 64-byte block
          const uint64_t ahi = umma_desc_sw64(sa + ks * 32), alo = umma_desc_sw64(sa + A_PLANE + ks * 32);
          const uint64_t bhi = umma_desc_sw64(sb + ks * 32), blo = umma_desc_sw64(sb + B_PLANE + ks * 32);
          umma_tf32(tmem_base, ahi, bhi, id, (kb | ks) != 0);
          umma_tf32(tmem_base, ahi, blo, id, 1u);
          umma_tf32(tmem_base, alo, bhi, id, 1u);
        }
        umma_commit(empty_bar(s));
        if (kb == NKB - 1) umma_commit(done_bar);
      }
      __syncwarp();
    }
  } else {  // epilogue: warps 2..5, TMEM lane quadrant warp & 3
    const int ew = warp & 3;
    mbar_wait(done_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    uint32_t v[64];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t (&vq)[16] = *reinterpret_cast<uint32_t(*)[16]>(&v[16 * q]);
      tmem_ld16(tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(16 * q), vq);
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    const int n = p.n;
    const long long ld = p.ld;
    const int tgt = t0 + ew;  // target tile index along the line
    const int idx = a_row0 + ew * 32 + lane;  // COL: global row;  ROW: global column
    if (tgt < p.h && (!ROW || idx < n)) {
      if (!ROW) {
        // stage the warp's 32 x 32 block in (now idle) pipeline smem, then
        // update Rf row by row with coalesced 256-byte accesses
        float2* buf = reinterpret_cast<float2*>(smem) + ew * 32 * 33;
#pragma unroll
        for (int c = 0; c < NB; ++c) buf[lane * 33 + c] = make_float2(__uint_as_float(v[2 * c]), __uint_as_float(v[2 * c + 1]));
        __syncwarp();
        const int c0 = line * NB, row0 = a_row0 + ew * 32;
        for (int r = 0; r < 32 && row0 + r < n; ++r) {
          if (c0 + lane < n) {
            float2* dst = Rf + (size_t)(row0 + r) * ld + c0 + lane;
            const float2 a = buf[r * 33 + lane];
            float2 q = *dst;
            q.x -= a.x;
            q.y -= a.y;
            *dst = q;
          }
        }
      } else {
        const int r0 = line * NB;
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          if (r0 + i < n) {
            float2* dst = Rf + (size_t)(r0 + i) * ld + idx;
            float2 r = *dst;
            r.x += __uint_as_float(v[2 * i]);
            r.y += __uint_as_float(v[2 * i + 1]);
            *dst = r;
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base),
                              "r"(TC_TMEM_COLS));
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline int pitch_f(int n) { return 2 * (n + (n & 1)); }  // fp32 per row: 2 even(n), a multiple of 4

// 3-d map over [2 planes][rows][P] fp32 (logical width 2n), box (16, box_rows, 2), 64-byte swizzle
int make_form_map(CUtensorMap* map, const float* base, int n, int rows, int P, int box_rows) {
  auto enc = get_encode();
  if (!enc) return SR_ECUDA;
  cuuint64_t dims[3] = {(cuuint64_t)(2 * n), (cuuint64_t)rows, 2};
  cuuint64_t strides[2] = {(cuuint64_t)P * 4, (cuuint64_t)P * 4 * (cuuint64_t)rows};
  cuuint32_t box[3] = {(cuuint32_t)KB_F, (cuuint32_t)box_rows, 2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? SR_OK : SR_ECUDA;
}

}  // namespace

size_t far_tc_forms_bytes(int n) {
  if (n <= 0) return 0;
  const size_t P = (size_t)pitch_f(n);
  const size_t t = align_up(2 * (size_t)n * P * 4, 1024);
  const size_t l = align_up(2 * (size_t)(2 * n) * P * 4, 1024);
  return 2 * t + 2 * l + 1024;
}

int far_tc_prepare(FarTcPlan* plan, int n, const float2* T, long long ld, void* base, cudaStream_t st) {
  const int P = pitch_f(n);
  const size_t t = align_up(2 * (size_t)n * P * 4, 1024);
  const size_t l = align_up(2 * (size_t)(2 * n) * P * 4, 1024);
  char* p0 = (char*)(((uintptr_t)base + 1023) & ~(uintptr_t)1023);
  plan->n = n;
  plan->P = P;
  plan->tform = (float*)p0;
  plan->ttform = (float*)(p0 + t);
  plan->lb = (float*)(p0 + 2 * t);
  plan->lc = (float*)(p0 + 2 * t + l);
  if (make_form_map(&plan->a_col, plan->tform, n, n, P, 128) != SR_OK ||
      make_form_map(&plan->a_row, plan->ttform, n, n, P, 128) != SR_OK ||
      make_form_map(&plan->b_col, plan->lb, n, 2 * n, P, 64) != SR_OK ||
      make_form_map(&plan->b_row, plan->lc, n, 2 * n, P, 64) != SR_OK)
    return sr_set_cuda_error(cudaErrorInvalidValue, "cuTensorMapEncodeTiled(solver forms)");
  const dim3 g(sr_ceil_div(n, NB), sr_ceil_div(n, NB));
  tforms_kernel<<<g, 256, 0, st>>>(n, T, ld, plan->tform, plan->ttform, P);
  SR_LAUNCH_CHECK();
  static bool configured = false;
  if (!configured) {
    const int smem = 1024 + TC_STAGES * TC_STAGE + 256;
    SR_CUDA_CHECK(cudaFuncSetAttribute(far_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    SR_CUDA_CHECK(cudaFuncSetAttribute(far_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  return SR_OK;
}

int far_tc_batch(const FarTcPlan& plan, int N, int b, int h, const float2* L, long long ld, float2* Rf,
                 cudaStream_t st) {
  const int n = plan.n;
  lforms_kernel<<<dim3(BW * b + BW, BW), 256, 0, st>>>(n, N, b, L, ld, plan.lb, plan.lc, plan.P);
  SR_LAUNCH_CHECK();
  const int strips = (h + BW - 1) / BW;
  const int smem = 1024 + TC_STAGES * TC_STAGE + 256;
  FarTcArgs a{n, N, b, h, 0, ld};
  far_tc_kernel<false><<<dim3(strips, min(BW * b + BW, N)), TC_THREADS, smem, st>>>(plan.a_col, plan.b_col, a, Rf);
  SR_LAUNCH_CHECK();
  a.first = N - BW - BW * b;
  far_tc_kernel<true><<<dim3(strips, N - a.first), TC_THREADS, smem, st>>>(plan.a_row, plan.b_row, a, Rf);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

// Far updates of the complex64 lp solver on the 5th-generation tensor cores.
//
// trisolve.cu's wavefront applies ~93 % of the solver's n^3/3 complex
// multiply-adds as FAR updates: once the four levels of batch b are solved,
//   COL  Rf[strip, M] -= T[strip, K0..K0+3] L[K0..K0+3, M]    (strip = 4 tiles of column M)
//   ROW  Rf[I, strip] += L[I, J0..J0+3] T[J0..J0+3, strip]    (strip = 4 tiles of row I)
// (index sets in trisolve.cu).  Here each strip is one tcgen05 GEMM tile:
//   * complex as real: with A' = a complex row read as interleaved (re, im)
//     values and B'^T rows 2c, 2c+1 = conj(b_c), i conj(b_c) (interleaved), the
//     real product A' B' is the interleaved complex product, so every operand is
//     a plain K-major matrix and the accumulator columns come out as (re, im);
//   * scaled two-piece FP16: every A row and every B column is scaled by a power
//     of two 2^-e to below 1 in magnitude (T: per row / per column of T, fixed
//     for the solve; L: per column / row over the four source tiles of the
//     batch), split x = hi + lo with hi = fp16(x), lo = fp16(x - hi), and
//     D += A_hi B_hi + A_hi B_lo + A_lo B_hi (kind::f16, FP32 accumulation in
//     TMEM) — ~22 significant bits per operand relative to its row / column
//     maximum, i.e. complex64-grade products; the epilogue multiplies by
//     2^(e_row + e_col) before updating Rf;
//   * COL: M = 128 strip rows, N = 64 (32 complex columns of tile M), K = 256
//     (4 source tiles x 32 complex);  ROW runs the transposed product
//     C^T = T^T L^T so that its 128 strip columns are the MMA's M dimension.
// Operand forms (built on the far stream, never on the critical path):
//   tform / ttform  hi, lo planes of scaled T and T^T (once per solve; the
//                   row / column maxima of T in tmax_r / tmax_c)
//   lb              rows 2c, 2c+1 = conj(L[:, c]), i conj(L[:, c])   (COL B operand)
//   lc              rows 2i, 2i+1 = conj(L[i, :]), i conj(L[i, :])   (ROW B operand)
//                   (per batch, right before its far updates; scaled by the
//                   column / row maxima of the batch's source tiles, lmax_c / lmax_r)
// TMA loads both planes of a 64-byte K block per operand (64-byte swizzle, zero
// fill outside the matrix, which also supplies the non-existent source tiles),
// persistent CTAs (one per SM) loop over the strips: a 4-stage mbarrier ring
// feeds the single-thread MMA issuer, and four epilogue warps drain one of two
// 64-column TMEM accumulators while the MMAs of the next strip run.
#include <cuda_fp16.h>

#include "trisolve_tc.cuh"
#include "tc_common.cuh"

namespace {

SR_TL_DECLARE(g_tl_tc)  // kinds: 2 far COL, 3 far ROW, 4 lforms, 5 lmax (slot = batch)


constexpr int NB = 32;
constexpr int BW = 4;
constexpr int KB_H = 32;                           // fp16 per 64-byte K block
constexpr int NKB = BW * NB * 2 / KB_H;            // 8 K blocks per strip
// persistent CTAs, one per SM; 4 stages keep 130 KB of shared memory so a
// critical-path SOLVE CTA (84 KB) still fits beside it on the same SM
#ifndef SR_FAR_STAGES
#define SR_FAR_STAGES 3
#endif
constexpr int TC_STAGES = SR_FAR_STAGES;
constexpr int A_PLANE = 128 * 64;                  // bytes: 128 rows x 64 B
constexpr int B_PLANE = 64 * 64;                   // bytes: 64 rows x 64 B
constexpr int TC_STAGE = 2 * A_PLANE + 2 * B_PLANE;
#ifndef SR_FAR_EPI_WARPS
#define SR_FAR_EPI_WARPS 8  // two per TMEM lane quadrant, each owning half of the unit's 32 line entries
#endif
constexpr int EPI_W = SR_FAR_EPI_WARPS;
constexpr int EPI_HALF = EPI_W / 4;   // warps per quadrant (1 or 2)
constexpr int EPI_SPAN = NB / EPI_HALF;  // line entries (COL: columns, ROW: rows) per epilogue warp
constexpr int TC_THREADS = 64 + 32 * EPI_W;
constexpr uint32_t TC_TMEM_COLS = 128;             // two 64-column accumulators
constexpr int EPI_BYTES = 2 * 4 * 32 * 33 * 8;      // epilogue staging, double-buffered (2 x 4 warps x 32 x 33 float2)
constexpr int TC_SMEM = 1024 + TC_STAGES * TC_STAGE + EPI_BYTES + 256;

// exponent e with max < 2^e (0 for an all-zero line): the line is scaled by 2^-e
__device__ __forceinline__ int line_exp(float mx) { return mx > 0.f ? ilogbf(mx) + 1 : 0; }

// x * 2^k: one multiply by an exact power of two for |k| <= 126 (every line
// scale of non-extreme data), ldexpf beyond (no overflow of the factor)
__device__ __forceinline__ float scale_pow2(float x, int k) {
  return (k >= -126 && k <= 126) ? x * __int_as_float((k + 127) << 23) : ldexpf(x, k);
}

__device__ __forceinline__ void put_h2(__half* base, size_t plane, size_t off, float x, float y) {
  const __half2 h = __floats2half2_rn(x, y);
  const float2 hf = __half22float2(h);
  *reinterpret_cast<__half2*>(base + off) = h;
  *reinterpret_cast<__half2*>(base + plane + off) = __floats2half2_rn(x - hf.x, y - hf.y);
}

__device__ __forceinline__ void atomic_max_pos(float* a, float v) {  // v >= 0: float order == int order
  atomicMax(reinterpret_cast<int*>(a), __float_as_int(v));
}

__device__ __forceinline__ float max4(const float* a, size_t n, int i) {
  return fmaxf(fmaxf(a[i], a[n + i]), fmaxf(a[2 * n + i], a[3 * n + i]));
}

// The far updates read T only in tiles (I, K) with K - I >= 4 FAR_LA + 1 >= 5
// (COL: K - I = N - 4b - 4 + k - t with t < N - 4b - 8; ROW alike): the tiles
// nearer the diagonal — the diagonal itself, whose eigenvalues dwarf the
// strict upper part — are kept out of the line maxima that scale the FP16
// forms (and written as zeros there), so every far operand keeps its full
// ~22 bits relative to the entries the far updates actually read.
constexpr int FAR_TILE_GAP = 4;  // excluded: tile distance K - I < FAR_TILE_GAP (far reads >= 5)

// row / column maxima of |re|, |im| of T over the tiles the far updates read
// (arrays zeroed by the caller)
__global__ void __launch_bounds__(256) tmax_kernel(int n, const float2* __restrict__ T, long long ld,
                                                   float* __restrict__ rmax, float* __restrict__ cmax) {
  const int r0 = blockIdx.y * NB, c0 = blockIdx.x * NB;
  if ((int)blockIdx.x - (int)blockIdx.y < FAR_TILE_GAP) return;  // lower part (zero), diagonal band
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  float cm = 0.f;
  for (int r = ty; r < NB; r += 8) {
    const int gr = r0 + r, gc = c0 + tx;
    float m = 0.f;
    if (gr < n && gc < n) {
      const float2 v = T[(size_t)gr * ld + gc];
      m = fmaxf(fabsf(v.x), fabsf(v.y));
    }
    cm = fmaxf(cm, m);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (tx == 0 && gr < n && m > 0.f) atomic_max_pos(rmax + gr, m);
  }
  if (c0 + tx < n && cm > 0.f) atomic_max_pos(cmax + c0 + tx, cm);
}

// hi / lo planes of the scaled T (rows scaled by tmax_r) and T^T (rows = columns of T, scaled by tmax_c)
__global__ void __launch_bounds__(256) tforms_kernel(int n, const float2* __restrict__ T, long long ld,
                                                     const float* __restrict__ rmax, const float* __restrict__ cmax,
                                                     __half* __restrict__ tf, __half* __restrict__ ttf, int P) {
  __shared__ float2 s[NB][NB + 1];
  const int r0 = blockIdx.y * NB, c0 = blockIdx.x * NB;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const size_t plane = (size_t)n * P;
  const bool read = (int)blockIdx.x - (int)blockIdx.y >= FAR_TILE_GAP;  // a tile the far updates read
  for (int r = ty; r < NB; r += 8) {
    const int gr = r0 + r, gc = c0 + tx;
    float2 v = make_float2(0.f, 0.f);
    if (gr < n && gc < n) {
      if (read) v = T[(size_t)gr * ld + gc];
      const int e = line_exp(rmax[gr]);
      put_h2(tf, plane, (size_t)gr * P + 2 * gc, scale_pow2(v.x, -e), scale_pow2(v.y, -e));
    }
    s[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < NB; r += 8) {  // T^T[c0 + r][r0 + tx] = T[r0 + tx][c0 + r]
    const int gr = c0 + r, gc = r0 + tx;
    if (gr < n && gc < n) {
      const float2 v = s[tx][r];
      const int e = line_exp(cmax[gr]);
      put_h2(ttf, plane, (size_t)gr * P + 2 * gc, scale_pow2(v.x, -e), scale_pow2(v.y, -e));
    }
  }
}

// Column / row maxima of the L tiles on levels 4b .. 4b+3 into lmax_c[level - 4b][.],
// lmax_r[level - 4b][.] (zeroed by the caller; blockIdx.y = level - 4b, blockIdx.x = M)
__global__ void __launch_bounds__(256) lmax_kernel(int n, int N, int b, const float2* __restrict__ L, long long ld,
                                                   float* __restrict__ lmax_c, float* __restrict__ lmax_r) {
  __shared__ float s[NB][NB + 1];
  const int level = BW * b + blockIdx.y;
  const int M = blockIdx.x;
  if (threadIdx.x == 0) SR_TL_MARK(g_tl_tc, 5, b, 0);
  if (level > N - 1 || M > level) return;
  const int I = M + N - 1 - level;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < NB; r += 8) {
    const int gr = I * NB + r, gc = M * NB + tx;
    float m = 0.f;
    if (gr < n && gc < n) {
      const float2 v = L[(size_t)gr * ld + gc];
      m = fmaxf(fabsf(v.x), fabsf(v.y));
    }
    s[r][tx] = m;
  }
  __syncthreads();
  if (ty == 0) {  // column maxima
    float m = 0.f;
    for (int r = 0; r < NB; ++r) m = fmaxf(m, s[r][tx]);
    if (M * NB + tx < n) lmax_c[(size_t)blockIdx.y * n + M * NB + tx] = m;
  } else if (ty == 1) {  // row maxima
    float m = 0.f;
    for (int c = 0; c < NB; ++c) m = fmaxf(m, s[tx][c]);
    if (I * NB + tx < n) lmax_r[(size_t)blockIdx.y * n + I * NB + tx] = m;
  }
  if (threadIdx.x == 0) SR_TL_MARK(g_tl_tc, 5, b, 1);
}

// L forms of the tiles on levels 4b .. 4b+3 (blockIdx.y = level - 4b, blockIdx.x = M)
__global__ void __launch_bounds__(256) lforms_kernel(int n, int N, int b, const float2* __restrict__ L, long long ld,
                                                     const float* __restrict__ lmax_c,
                                                     const float* __restrict__ lmax_r, __half* __restrict__ lb,
                                                     __half* __restrict__ lc, int P) {
  __shared__ float2 s[NB][NB + 1];
  __shared__ int ec[NB], er[NB];
  const int level = BW * b + blockIdx.y;
  const int M = blockIdx.x;
  if (threadIdx.x == 0) SR_TL_MARK(g_tl_tc, 4, b, 0);
  if (level > N - 1 || M > level) return;
  const int I = M + N - 1 - level;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < NB; r += 8) {
    const int gr = I * NB + r, gc = M * NB + tx;
    s[r][tx] = (gr < n && gc < n) ? L[(size_t)gr * ld + gc] : make_float2(0.f, 0.f);
  }
  if (ty == 0) ec[tx] = M * NB + tx < n ? line_exp(max4(lmax_c, n, M * NB + tx)) : 0;
  if (ty == 1) er[tx] = I * NB + tx < n ? line_exp(max4(lmax_r, n, I * NB + tx)) : 0;
  __syncthreads();
  const size_t plane = (size_t)2 * n * P;
  for (int c = ty; c < NB; c += 8) {  // LB rows 2C, 2C+1 (C = column of L), cols 2K (K = row of L)
    const int C = M * NB + c, K = I * NB + tx;
    if (C < n && K < n) {
      const float2 v = s[tx][c];
      const float x = scale_pow2(v.x, -ec[c]), y = scale_pow2(v.y, -ec[c]);
      put_h2(lb, plane, (size_t)(2 * C) * P + 2 * K, x, -y);
      put_h2(lb, plane, (size_t)(2 * C + 1) * P + 2 * K, y, x);
    }
  }
  for (int i = ty; i < NB; i += 8) {  // LC rows 2R, 2R+1 (R = row of L), cols 2K (K = column of L)
    const int R = I * NB + i, K = M * NB + tx;
    if (R < n && K < n) {
      const float2 v = s[i][tx];
      const float x = scale_pow2(v.x, -er[i]), y = scale_pow2(v.y, -er[i]);
      put_h2(lc, plane, (size_t)(2 * R) * P + 2 * K, x, -y);
      put_h2(lc, plane, (size_t)(2 * R + 1) * P + 2 * K, y, x);
    }
  }
  if (threadIdx.x == 0) SR_TL_MARK(g_tl_tc, 4, b, 1);
}

__device__ __forceinline__ constexpr uint32_t idesc_f16(int m, int n) {
  // D = F32, A = B = F16, K-major operands
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

struct FarTcArgs {
  int n, N, b, h, first, lines, strips;
  int first_level;  // first far target level
  long long ld;
  const float* a_max;  // A-line maxima: T rows (COL) or T columns (ROW)
  const float* b_max;  // [4][n] source-tile maxima: L columns (COL) or L rows (ROW)
};

template <bool ROW>
// At most 216 registers per thread: the two epilogue-heavy warp pairs then
// leave 2304 registers free in every SM sub-partition, so a 4-warp SOLVE
// CTA (72 registers) can be resident beside a far CTA (254 registers would
// fill two sub-partitions completely and serialise the critical path behind
// every far launch).
#ifndef SR_FAR_TC_MAXNREG
#define SR_FAR_TC_MAXNREG (EPI_W == 8 ? 168 : 216)  // room for a 4-warp SOLVE CTA beside a far CTA
#endif
__global__ void __maxnreg__(SR_FAR_TC_MAXNREG)
    far_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                  const __grid_constant__ FarTcArgs p, float2* __restrict__ Rf) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ float eb_s[EPI_W][32];  // 2^(e_b) of the tile's B lines (per epilogue warp)
  __shared__ int eb_x[EPI_W][32];    // e_b itself (the out-of-range path)
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float2* stage_buf = reinterpret_cast<float2*>(smem + TC_STAGES * TC_STAGE);  // COL epilogue staging, 4 x 32 x 33
  uint64_t* bars = (uint64_t*)(smem + TC_STAGES * TC_STAGE + EPI_BYTES);
  // full[S], empty[S], tfull[2], tempty[2]; then the TMEM base slot
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * TC_STAGES + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (TC_STAGES + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * TC_STAGES + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * TC_STAGES + 2 + a); };

  const int N = p.N, b = p.b;
  const int units = p.lines * p.strips;
  if (threadIdx.x == 0) SR_TL_MARK(g_tl_tc, ROW ? 3 : 2, b, 0);
  // unit -> (line, first target t0) and the A / B / K origins of its strip
  auto unit = [&](int u, int& line, int& t0, int& a_row0, int& b_row0, int& k0) {
    line = p.first + u / p.strips;
    t0 = BW * (u % p.strips);
    if (!ROW) {
      a_row0 = (line + t0) * NB;
      b_row0 = 2 * line * NB;
      k0 = (line + N - BW * b - BW) * NB * 2;
    } else {
      a_row0 = (line - N + 1 + p.first_level + t0) * NB;
      b_row0 = 2 * line * NB;
      k0 = (line - N + 1 + BW * b) * NB * 2;
    }
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 32 * EPI_W);
    }
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
    if (lane == 0) {  // TMA producer: runs ahead across units through the stage ring
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int line, t0, a_row0, b_row0, k0;
        unit(u, line, t0, a_row0, b_row0, k0);
        for (int kb = 0; kb < NKB; ++kb, ++it) {
          const int s = it % TC_STAGES;
          if (it >= TC_STAGES) mbar_wait(empty_bar(s), ((it / TC_STAGES) - 1) & 1);
          uint8_t* st = smem + s * TC_STAGE;
          mbar_expect_tx(full_bar(s), TC_STAGE);
          tma_load_3d(smem_u32(st), &map_a, full_bar(s), k0 + kb * KB_H, a_row0, 0);
          tma_load_3d(smem_u32(st + 2 * A_PLANE), &map_b, full_bar(s), k0 + kb * KB_H, b_row0, 0);
        }
      }
    }
  } else if (warp == 1) {  // MMA issuer: two TMEM accumulators, epilogue of unit i overlaps MMAs of unit i+1
    const uint32_t id = idesc_f16(128, 64);
    int it = 0, acc = 0, k = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++k) {
      acc = k & 1;
      mbar_wait(tempty_bar(acc), ((k >> 1) & 1) ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t d = tmem_base + (uint32_t)(acc * 64);
      for (int kb = 0; kb < NKB; ++kb, ++it) {
        const int s = it % TC_STAGES;
        mbar_wait(full_bar(s), (it / TC_STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem + s * TC_STAGE);
          const uint32_t sb = sa + 2 * A_PLANE;
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {  // two K = 16 fp16 steps per 64-byte block
            const uint64_t ahi = umma_desc_sw64(sa + ks * 32), alo = umma_desc_sw64(sa + A_PLANE + ks * 32);
            const uint64_t bhi = umma_desc_sw64(sb + ks * 32), blo = umma_desc_sw64(sb + B_PLANE + ks * 32);
            umma_f16(d, ahi, bhi, id, (kb | ks) != 0);
            umma_f16(d, ahi, blo, id, 1u);
            umma_f16(d, alo, bhi, id, 1u);
          }
          umma_commit(empty_bar(s));
          if (kb == NKB - 1) umma_commit(tfull_bar(acc));
        }
        __syncwarp();
      }
    }
  } else {  // epilogue: warps 2.., TMEM lane quadrant warp & 3, line-entry half eh
    const int ew = warp & 3;
    const int ewi = warp - 2;          // epilogue warp index
    const int eh = ewi >> 2;           // which EPI_SPAN line entries (COL: columns, ROW: rows) of the unit
    const int j0e = eh * EPI_SPAN;
    const int n = p.n;
    const long long ld = p.ld;
    // two staging blocks per quadrant (shared by the quadrant's warps, each
    // touching only its own entries): the Rf block of unit k+1 is loaded while
    // unit k is folded
    float2* bufs[2] = {stage_buf + ew * 32 * 33, stage_buf + (4 + ew) * 32 * 33};
    auto issue_rf = [&](int uu, float2* dstb) {
      int line_, t0_, a_row0_, b_row0_, k0_;
      unit(uu, line_, t0_, a_row0_, b_row0_, k0_);
      const int R0_ = !ROW ? a_row0_ + ew * 32 : line_ * NB;
      const int C0_ = !ROW ? line_ * NB : a_row0_ + ew * 32;
      const bool okt = t0_ + ew < p.h;
      // COL: this warp's columns j0e.. of all 32 rows; ROW: its rows j0e.. of all 32 columns
      // (EPI_SPAN x 32 entries, 32 / EPI_SPAN rows per instruction, coalesced along the rows)
      constexpr int RPI = 32 / EPI_SPAN;  // rows per instruction (COL)
#pragma unroll 4
      for (int it = 0; it < 32 * EPI_SPAN / 32; ++it) {
        int r, c;
        if (!ROW) {
          r = it * RPI + lane / EPI_SPAN;
          c = j0e + lane % EPI_SPAN;
        } else {
          r = j0e + it;
          c = lane;
        }
        const bool ok = okt && R0_ + r < n && C0_ + c < n;
        const float2* src = Rf + (ok ? (size_t)(R0_ + r) * ld + C0_ + c : 0);
        const uint32_t dst = smem_u32(dstb + r * 33 + c);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0)
                     : "memory");
      }
    };
    if ((int)blockIdx.x < units) issue_rf(blockIdx.x, bufs[0]);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    int k = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++k) {
      const int acc = k & 1;
      int line, t0, a_row0, b_row0, k0;
      unit(u, line, t0, a_row0, b_row0, k0);
      // scale exponents: A line of this lane, B lines of the tile (L column / row line * 32 + j)
      const int idx = a_row0 + ew * 32 + lane;  // TMEM lane: COL global row;  ROW global column
      const int ea = idx < n ? line_exp(p.a_max[idx]) : 0;
      const int jl = line * NB + lane;
      __syncwarp();
      // the epilogue scale 2^(e_a + e_b) as a product of two powers of two, one
      // multiply per entry instead of an ldexpf (2^e is exact for line maxima
      // in [2^-127, 2^127), i.e. every complex64 line that is neither
      // subnormal nor within a factor 2 of overflow)
      const int eb = jl < n ? line_exp(max4(p.b_max, (size_t)n, jl)) : 0;
      eb_s[ewi][lane] = ldexpf(1.f, eb);
      eb_x[ewi][lane] = eb;
      const float fa = ldexpf(1.f, ea);
      // a line maximum outside [2^-127, 2^126] makes one factor 0 or inf: then
      // the whole warp scales by the combined 2^(e_a + e_b) instead (one
      // ldexpf per entry), so inf * 0 never turns a finite entry into NaN
      const bool wide = __any_sync(0xffffffffu, ea > 126 || ea < -126 || eb > 126 || eb < -126);
      __syncwarp();
      const int tgt = t0 + ew;  // target tile index along the line
      const bool live = tgt < p.h;
      // this unit's Rf block was prefetched into bufs[k & 1] one unit ahead;
      // start the next unit's now (targets of different units never overlap)
      float2* buf = bufs[k & 1];
      const int R0 = !ROW ? a_row0 + ew * 32 : line * NB;
      const int C0 = !ROW ? line * NB : a_row0 + ew * 32;
      if (u + (int)gridDim.x < units) issue_rf(u + (int)gridDim.x, bufs[(k + 1) & 1]);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      mbar_wait(tfull_bar(acc), (k >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      uint32_t v[2 * EPI_SPAN];  // this warp's line entries (re, im)
#pragma unroll
      for (int qq = 0; qq < 2 * EPI_SPAN / 16; ++qq) {
        uint32_t (&vq)[16] = *reinterpret_cast<uint32_t(*)[16]>(&v[16 * qq]);
        tmem_ld16(tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * 64 + 2 * j0e + 16 * qq), vq);
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      mbar_arrive(tempty_bar(acc));  // the accumulator is in registers: release it to the MMA warp
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // all but the next unit's block
      __syncwarp();
      if (live) {
        if (!ROW) {
          // this lane's accumulator row (R0 + lane), columns j0e.., folded into the
          // staged block, then the block's columns stored row by row
#pragma unroll
          for (int c = 0; c < EPI_SPAN; ++c) {
            const float sc = wide ? ldexpf(1.f, ea + eb_x[ewi][j0e + c]) : fa * eb_s[ewi][j0e + c];
            float2& q = buf[lane * 33 + j0e + c];
            q = make_float2(q.x - __uint_as_float(v[2 * c]) * sc, q.y - __uint_as_float(v[2 * c + 1]) * sc);
          }
          __syncwarp();
          constexpr int RPI = 32 / EPI_SPAN;
          const int cc = j0e + lane % EPI_SPAN;
          if (C0 + cc < n) {
#pragma unroll 4
            for (int it = 0; it < EPI_SPAN; ++it) {
              const int r = it * RPI + lane / EPI_SPAN;
              if (R0 + r < n) Rf[(size_t)(R0 + r) * ld + C0 + cc] = buf[r * 33 + cc];
            }
          }
        } else if (idx < n) {
          // this lane's accumulator column (C0 + lane = idx), rows j0e..
#pragma unroll
          for (int i = 0; i < EPI_SPAN; ++i) {
            const int ri = j0e + i;
            if (R0 + ri < n) {
              const float sc = wide ? ldexpf(1.f, ea + eb_x[ewi][ri]) : fa * eb_s[ewi][ri];
              const float2 q = buf[ri * 33 + lane];
              Rf[(size_t)(R0 + ri) * ld + idx] = make_float2(q.x + __uint_as_float(v[2 * i]) * sc,
                                                             q.y + __uint_as_float(v[2 * i + 1]) * sc);
            }
          }
        }
      }
      __syncwarp();  // buf is refilled by the prefetch two units on
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base),
                              "r"(TC_TMEM_COLS));
  if (threadIdx.x == 0) SR_TL_MARK(g_tl_tc, ROW ? 3 : 2, b, 1);
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline int pitch_h(int n) { return (2 * n + 7) / 8 * 8; }  // fp16 per row, 16-byte multiple

// 3-d map over [2 planes][rows][P] fp16 (logical width 2n), box (32, box_rows, 2), 64-byte swizzle
int make_form_map(CUtensorMap* map, const __half* base, int n, int rows, int P, int box_rows) {
  auto enc = get_encode();
  if (!enc) return SR_ECUDA;
  cuuint64_t dims[3] = {(cuuint64_t)(2 * n), (cuuint64_t)rows, 2};
  cuuint64_t strides[2] = {(cuuint64_t)P * 2, (cuuint64_t)P * 2 * (cuuint64_t)rows};
  cuuint32_t box[3] = {(cuuint32_t)KB_H, (cuuint32_t)box_rows, 2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<__half*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? SR_OK : SR_ECUDA;
}

struct FormLayout {
  size_t t, l, mx, total;
};
FormLayout form_layout(int n) {
  const size_t P = (size_t)pitch_h(n);
  FormLayout f;
  f.t = align_up(2 * (size_t)n * P * 2, 1024);        // one T form: 2 planes x n rows of fp16
  f.l = align_up(2 * (size_t)(2 * n) * P * 2, 1024);  // one L form: 2 planes x 2n rows
  f.mx = align_up((size_t)n * 4 * 10, 1024);          // tmax_r, tmax_c, lmax_c[4], lmax_r[4]
  f.total = 2 * f.t + 2 * f.l + f.mx + 1024;
  return f;
}

}  // namespace

#ifdef SR_TIMELINE
extern "C" int sr_timeline_tc(void* host, int reset) {
  if (reset) {
    static unsigned long long init[8][1024][2];
    for (int k = 0; k < 8; ++k)
      for (int s = 0; s < 1024; ++s) init[k][s][0] = ~0ull, init[k][s][1] = 0;
    return cudaMemcpyToSymbol(g_tl_tc, init, sizeof(init)) == cudaSuccess ? 0 : 4;
  }
  return cudaMemcpyFromSymbol(host, g_tl_tc, sizeof(g_tl_tc)) == cudaSuccess ? 0 : 4;
}
#endif

size_t far_tc_forms_bytes(int n) { return n <= 0 ? 0 : form_layout(n).total; }

int far_tc_prepare(FarTcPlan* plan, int n, const float2* T, long long ld, void* base, cudaStream_t st) {
  const int P = pitch_h(n);
  const FormLayout f = form_layout(n);
  char* p0 = (char*)(((uintptr_t)base + 1023) & ~(uintptr_t)1023);
  plan->n = n;
  plan->P = P;
  plan->tform = (__half*)p0;
  plan->ttform = (__half*)(p0 + f.t);
  plan->lb = (__half*)(p0 + 2 * f.t);
  plan->lc = (__half*)(p0 + 2 * f.t + f.l);
  float* mx = (float*)(p0 + 2 * f.t + 2 * f.l);
  plan->tmax_r = mx;
  plan->tmax_c = mx + n;
  plan->lmax_c = mx + 2 * (size_t)n;
  plan->lmax_r = mx + 6 * (size_t)n;
  if (make_form_map(&plan->a_col, plan->tform, n, n, P, 128) != SR_OK ||
      make_form_map(&plan->a_row, plan->ttform, n, n, P, 128) != SR_OK ||
      make_form_map(&plan->b_col, plan->lb, n, 2 * n, P, 64) != SR_OK ||
      make_form_map(&plan->b_row, plan->lc, n, 2 * n, P, 64) != SR_OK)
    return sr_set_cuda_error(cudaErrorInvalidValue, "cuTensorMapEncodeTiled(solver forms)");
  SR_CUDA_CHECK(cudaMemsetAsync(plan->tmax_r, 0, 2 * (size_t)n * sizeof(float), st));
  const dim3 g(sr_ceil_div(n, NB), sr_ceil_div(n, NB));
  tmax_kernel<<<g, 256, 0, st>>>(n, T, ld, plan->tmax_r, plan->tmax_c);
  SR_LAUNCH_CHECK();
  tforms_kernel<<<g, 256, 0, st>>>(n, T, ld, plan->tmax_r, plan->tmax_c, plan->tform, plan->ttform, P);
  SR_LAUNCH_CHECK();
  static bool configured[SR_MAX_DEVICES] = {};  // function attributes are per device
  int slot = 0;
  if (sr_device_slot(&slot) != SR_OK) return SR_EINVAL;
  if (!configured[slot]) {
    SR_CUDA_CHECK(cudaFuncSetAttribute(far_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM));
    SR_CUDA_CHECK(cudaFuncSetAttribute(far_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM));
    // the whole 228 KB as shared memory: a far CTA (131 KB) leaves room for a
    // critical-path SOLVE CTA on the same SM (a 132 KB carveout would not)
    SR_CUDA_CHECK(cudaFuncSetAttribute(far_tc_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       cudaSharedmemCarveoutMaxShared));
    SR_CUDA_CHECK(cudaFuncSetAttribute(far_tc_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       cudaSharedmemCarveoutMaxShared));
    configured[slot] = true;
  }
  return SR_OK;
}

int far_tc_batch(const FarTcPlan& plan, int N, int b, int h, int first_level, const float2* L, long long ld,
                 float2* Rf, cudaStream_t st) {
  const int n = plan.n;
  SR_CUDA_CHECK(cudaMemsetAsync(plan.lmax_c, 0, 8 * (size_t)n * sizeof(float), st));
  const dim3 gl(BW * b + BW, BW);
  lmax_kernel<<<gl, 256, 0, st>>>(n, N, b, L, ld, plan.lmax_c, plan.lmax_r);
  SR_LAUNCH_CHECK();
  lforms_kernel<<<gl, 256, 0, st>>>(n, N, b, L, ld, plan.lmax_c, plan.lmax_r, plan.lb, plan.lc, plan.P);
  SR_LAUNCH_CHECK();
  const int strips = (h + BW - 1) / BW;
  FarTcArgs a{n, N, b, h, 0, min(BW * b + BW, N), strips, first_level, ld, plan.tmax_r, plan.lmax_c};
  const int grid_c = min(a.lines * strips, 148);
  far_tc_kernel<false><<<grid_c, TC_THREADS, TC_SMEM, st>>>(plan.a_col, plan.b_col, a, Rf);
  SR_LAUNCH_CHECK();
  a.first = N - BW - BW * b;
  a.lines = N - a.first;
  a.a_max = plan.tmax_c;
  a.b_max = plan.lmax_r;
  const int grid_r = min(a.lines * strips, 148);
  far_tc_kernel<true><<<grid_r, TC_THREADS, TC_SMEM, st>>>(plan.a_row, plan.b_row, a, Rf);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

// Low-precision solve of stril(T L - L T) = -E for strictly lower L.
//
// Replaces the reference solver
//   solve_block           /root/reference/pkg/src/ddschur/trisolve.py:243-262
//   _block_solve          trisolve.py:223-240   (recursive halving)
//   _sylvester_tri        trisolve.py:164-196
//   _scalar_solve_inplace trisolve.py:121-145
//   _check_separation     trisolve.py:104-113
// with a blocked wavefront over NB x NB tiles of L.  Tile (I, J), I >= J,
// satisfies
//   T_II L_IJ - L_IJ T_JJ = R_IJ,
//   R_IJ = -E_IJ - sum_{K>I} T_IK L_KJ + sum_{K<J} L_IK T_KJ
// (stril() of both sides when I == J).  Tile (I, J) sits on anti-diagonal
// level (N-1-I) + J and depends only on tiles of lower levels, so launch
// `lev` of the sweep solves every tile of level `lev` (one CTA each).
//
// The contributions of a solved tile (the "source") to the open tiles are
// applied in one of three places, decided by the levels involved.  Levels are
// grouped into batches of BW = 4; a source on level s (batch b = s / 4) feeds
//   * the tiles of level s + 1 inside their SOLVE CTA (the critical path),
//   * the tiles of levels s + 2 .. 4 (b + 1 + FAR_LA) - 1 through the NEAR
//     launch of level s + 1 (rank-NB tile updates, a narrow band of levels),
//   * every tile of level >= 4 (b + 1 + FAR_LA) through the FAR launches of
//     batch b: once the four levels of batch b are solved, their sources for
//     one column (row) of targets are four CONSECUTIVE tiles, so each target
//     receives one rank-4NB update; the FAR launches run on their own stream,
//     overlapped with the next 4 FAR_LA levels of SOLVE / NEAR, and write a
//     second right-hand-side buffer (Rf) so they never race the near band's (Rn).
// (tests/test_trisolve_schedule.py checks on the CPU that these three sets
// apply every (source, target) pair exactly once, after the source is solved
// and before the target is.)
// The far updates carry ~93 % of the n^3/3 complex multiply-adds, as register-
// tiled complex GEMMs on the FP32 (FP64 in dd mode) pipe with cp.async double
// buffering; the running right-hand sides are read and written once per batch
// instead of once per level.
//
// The tile solve is one warp: lane i owns row i, and entry (i, j) is final at
// step (NB-1-i) + j.  Each lane keeps its open entries in a 32-wide register
// window that slides one column per step (fully unrolled, so the slide is
// register renaming); at every step the lanes finalise one entry each
// (multiplying by a reciprocal pivot computed beforehand by the whole CTA),
// exchange the new values with warp shuffles (the column terms) and fold
// their own new value into their later columns through a diagonal-major copy of
// T_JJ (the row terms, conflict-free shared loads).  Clipping is applied at
// finalisation as in the reference (trisolve.py:141-144,192-195), so
// dependants see the clipped zero; any dependency-respecting order gives the
// same L up to rounding.
//
// Templated on the lp type: float2 (FP64 mode, lp = complex64) and double2
// (dd mode, lp = binary64 complex).
#include <stdlib.h>

#include <type_traits>

#include <mutex>

#include "sr_common.cuh"
#include "trisolve_tc.cuh"

namespace {

SR_TL_DECLARE(g_tl_solve)  // kinds: 0 SOLVE, 1 NEAR (slot = level)

#ifndef SR_SOLVE_ONE_WARP
#define SR_SOLVE_ONE_WARP 0  // 1: the earlier single-warp tile solve (A/B builds)
#endif
#ifndef SR_SOLVE_PDL
#define SR_SOLVE_PDL 1  // 0: plain stream-ordered SOLVE launches (A/B builds)
#endif
constexpr int NB = 32;
constexpr int NT = 128;   // NEAR CTAs: 16 x 8 threads, each a 2 x 4 block of the tile
// SOLVE CTAs: 128 threads, 2 x 4 blocks.  (64 threads with 4 x 4 blocks — a
// register footprint that co-resides with a far tensor-core CTA — measured
// slower: 24.8 vs 24.0 ms per n = 8192 solve, 2.69 vs 2.34 ms at n = 2048;
// kept selectable with -DSR_SOLVE_C64_THREADS=64 for the timeline tool.)
template <typename C>
struct SolveShape {
#ifndef SR_SOLVE_C64_THREADS
#define SR_SOLVE_C64_THREADS 128
#endif
  static constexpr int THREADS = sizeof(C) == 8 ? SR_SOLVE_C64_THREADS : 128;
  static constexpr int RPT = NB * NB / (4 * THREADS);  // rows per thread (x 4 columns)
};
constexpr int LD = NB + 1;
constexpr int BW = 4;     // levels per far batch = tiles per far strip = source tiles per far update
#ifndef SR_FAR_LA
#define SR_FAR_LA 1
#endif
constexpr int FAR_LA = SR_FAR_LA;  // batches of slack: the far updates of batch b target levels >= 4 (b + 1 + FAR_LA)
constexpr int FT = 256;   // FAR CTAs

template <typename C>
struct Real;
template <>
struct Real<float2> {
  using T = float;
};
template <>
struct Real<double2> {
  using T = double;
};

template <typename C>
__device__ __forceinline__ C czero() {
  C z;
  z.x = 0;
  z.y = 0;
  return z;
}
template <typename C>
__device__ __forceinline__ void cfma(C& acc, C a, C b) {  // acc += a * b
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
template <typename C>
__device__ __forceinline__ void cfms(C& acc, C a, C b) {  // acc -= a * b
  acc.x = fma(-a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(-a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
__device__ __forceinline__ float2 shfl_down(float2 v, int d) {
  return make_float2(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d));
}
__device__ __forceinline__ double2 shfl_down(double2 v, int d) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d));
}

// Asynchronous copy of a rows x cols block (global rows r0.., cols c0..; r0 or
// c0 may be negative) into shared memory with row pitch `pitch` elements,
// zero-filled outside [0, n) x [0, n).  16-byte copies when the global and the
// shared rows are 16-byte aligned (complex128, or complex64 with an even ld
// and an even pitch), else one element per copy.  The caller commits and waits.
template <typename C>
__device__ __forceinline__ void load_block_async(C* s, int pitch, const C* __restrict__ g, long long ld, int r0,
                                                 int c0, int rows, int cols, int n, int tid, int nthreads) {
  constexpr int EPV = 16 / (int)sizeof(C);  // elements per 16-byte copy
  const bool vec = EPV == 1 || ((ld % 2) == 0 && (pitch % 2) == 0);
  if (vec) {
    const int per_row = cols / EPV;
    for (int idx = tid; idx < rows * per_row; idx += nthreads) {
      const int r = idx / per_row, c = (idx % per_row) * EPV;
      const int gr = r0 + r, gc = c0 + c;
      int valid = (gr >= 0 && gr < n && gc >= 0) ? min(EPV, n - gc) : 0;
      valid = valid < 0 ? 0 : valid;
      const C* src = g + (valid ? (size_t)gr * ld + gc : 0);
      cp_async_16(s + r * pitch + c, src, valid * (int)sizeof(C));
    }
  } else {
    for (int idx = tid; idx < rows * cols; idx += nthreads) {
      const int r = idx / cols, c = idx % cols;
      const int gr = r0 + r, gc = c0 + c;
      const bool ok = gr >= 0 && gr < n && gc >= 0 && gc < n;
      const C* src = g + (ok ? (size_t)gr * ld + gc : 0);
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(s + r * pitch + c);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0));
    }
  }
}

template <typename C, int THREADS = NT>
__device__ __forceinline__ void load_tile_async(C* s, const C* __restrict__ g, long long ld, int r0, int c0, int n) {
  load_block_async<C>(s, LD, g, ld, r0, c0, NB, NB, n, threadIdx.x, THREADS);
}

struct SweepArgs {
  int n, N, lev, lmax;
  long long ld;
};

// acc (RPT x 4 block of the tile per thread: rows RPT ty .., cols 4 tx ..)
// -= A B (col term) / += A B (row term)
template <typename C, bool ADD, int RPT = 2>
__device__ __forceinline__ void tile_mac(C (&acc)[RPT][4], const C* sA, const C* sB, int ty, int tx) {
#pragma unroll 8
  for (int k = 0; k < NB; ++k) {
    C a[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) a[r] = sA[(RPT * ty + r) * LD + k];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const C b = sB[k * LD + 4 * tx + c];
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        if (ADD)
          cfma(acc[r][c], a[r], b);
        else
          cfms(acc[r][c], a[r], b);
      }
    }
  }
}

// 1 / d for the reciprocal pivots: Smith-scaled (no overflow for |d| near the
// range limits), one reciprocal instead of cdiv's four divisions
__device__ __forceinline__ float2 crecip(float2 d) {
  const float s = fmaxf(fabsf(d.x), fabsf(d.y));
  const float is = 1.0f / s;
  const float a = d.x * is, b = d.y * is;
  const float r = is / (a * a + b * b);
  return make_float2(a * r, -b * r);
}
__device__ __forceinline__ double2 crecip(double2 d) {
  const double s = fmax(fabs(d.x), fabs(d.y));
  const double is = 1.0 / s;
  const double a = d.x * is, b = d.y * is;
  const double r = is / (a * a + b * b);
  return make_double2(a * r, -b * r);
}

// In-tile solve by warp 0: T2 X - X T1 = R (strict lower part only when DIAG).
// sP[i][j] = 1 / (T2_ii - T1_jj); sD[d][j] = T1[j][j + d].
template <typename C, bool DIAG>
__device__ __forceinline__ unsigned tile_solve_warp(const C* sT2, const C* sD, const C* sP, const C* sR, C* sX,
                                                    int valid_i, int valid_j, typename Real<C>::T clip) {
  using R = typename Real<C>::T;
  const int i = threadIdx.x & 31;
  const R clip2 = clip * clip;
  unsigned nclip = 0;
  C pend[NB];
  C tr[NB];
#pragma unroll
  for (int d = 0; d < NB; ++d) {
    const int c = i - (NB - 1) + d;  // window at step 0 covers columns i-31 .. i
    pend[d] = (c >= 0) ? sR[i * LD + c] : czero<C>();
    tr[d] = (i + d < NB) ? sT2[i * LD + i + d] : czero<C>();
  }
  // 2 NB steps (the last one is idle for every lane), unrolled by 4 so that
  // most of the window slide becomes register renaming
#pragma unroll 4
  for (int t = 0; t < 2 * NB; ++t) {
    const int j = t - (NB - 1) + i;  // this lane's column at step t
    const bool valid = (j >= 0) && (j < NB) && (i < valid_i) && (j < valid_j) && (!DIAG || i > j);
    C x = czero<C>();
    if (valid) {
      x = cmul(pend[0], sP[i * LD + j]);
      if (clip > 0 && x.x * x.x + x.y * x.y > clip2) {
        x = czero<C>();
        ++nclip;
      }
      sX[i * LD + j] = x;
    }
    // column terms: lane i+d finalised (i+d, j+d); it feeds this lane's (i, j+d)
    // (tr[d] = 0 past the tile edge, so no predicate is needed)
#pragma unroll
    for (int d = 1; d < NB; ++d) {
      const C xv = shfl_down(x, d);
      cfms(pend[d], tr[d], xv);
    }
    // row terms: (i, j) feeds this lane's (i, j+d) through T1[j][j+d]
    // (x = 0 on invalid steps, sD[d][j] = 0 for j + d >= NB)
    {
      const int jc = min(max(j, 0), NB - 1);
#pragma unroll
      for (int d = 1; d < NB; ++d) cfma(pend[d], x, sD[d * NB + jc]);
    }
    // slide the window one column to the right
#pragma unroll
    for (int d = 0; d < NB - 1; ++d) pend[d] = pend[d + 1];
    {
      const int c = t + i + 1;
      pend[NB - 1] = (c < NB) ? sR[i * LD + c] : czero<C>();
    }
  }
  return nclip;
}

// In-tile solve by all four warps of the CTA (same equations and finalisation
// order as tile_solve_warp): lane i owns row i in every warp, warp w owns the
// window positions d = 8w .. 8w+7 (columns j+d of row i).  Per step warp 0
// finalises position 0 and publishes the new values through shared memory;
// after one named barrier every warp folds them into its 8 positions (column
// terms read the new values of rows i+d straight from shared memory, no
// shuffles; row terms as before) and slides its window — the value leaving a
// warp's position 0 is handed to warp w-1's position 7 through a double-
// buffered shared slot that is read after the next step's barrier.  A quarter
// of the multiply-adds per warp and a quarter of the registers (the CTA can
// share an SM with a far tensor-core CTA).
template <typename C, bool DIAG, int NW = 4>
__device__ __forceinline__ unsigned tile_solve_cta(const C* sT2, const C* sD, const C* sP, const C* sR, C* sX,
                                                   C (*xs)[NB], C (*hand)[NW][NB], int valid_i, int valid_j,
                                                   typename Real<C>::T clip) {
  using R = typename Real<C>::T;
  constexpr int W = NB / NW;  // window positions per warp
  const int i = threadIdx.x & 31, w = threadIdx.x >> 5;
  const R clip2 = clip * clip;
  unsigned nclip = 0;
  C pend[W], tr[W];
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const int d = W * w + k;
    const int c = i - (NB - 1) + d;  // window at step 0 covers columns i-31 .. i
    pend[k] = (c >= 0) ? sR[i * LD + c] : czero<C>();
    tr[k] = (i + d < NB) ? sT2[i * LD + i + d] : czero<C>();
  }
#pragma unroll 4
  for (int t = 0; t < 2 * NB - 1; ++t) {
    const int j = t - (NB - 1) + i;  // this lane's column at step t
    if (w == 0) {
      const bool valid = (j >= 0) && (j < NB) && (i < valid_i) && (j < valid_j) && (!DIAG || i > j);
      C x = czero<C>();
      if (valid) {
        x = cmul(pend[0], sP[i * LD + j]);
        if (clip > 0 && x.x * x.x + x.y * x.y > clip2) {
          x = czero<C>();
          ++nclip;
        }
        sX[i * LD + j] = x;
      }
      xs[t & 1][i] = x;
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(NW * 32) : "memory");
    // position W-1: handed over by warp w+1 at the end of the previous step
    // (the last warp: the column entering the window)
    if (t > 0) {
      if (w < NW - 1) {
        pend[W - 1] = hand[(t - 1) & 1][w + 1][i];
      } else {
        const int c = t + i;
        pend[W - 1] = (c < NB) ? sR[i * LD + c] : czero<C>();
      }
    }
    const C xi = xs[t & 1][i];
    const int jc = min(max(j, 0), NB - 1);
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int d = W * w + k;
      if (d == 0) continue;
      // column term: row i+d finalised (i+d, j+d) (tr = 0 past the tile edge)
      const C xv = xs[t & 1][min(i + d, NB - 1)];
      cfms(pend[k], tr[k], xv);
      // row term: (i, j) feeds (i, j+d) through T1[j][j+d] (0 past the edge)
      cfma(pend[k], xi, sD[d * NB + jc]);
    }
    if (w > 0) hand[t & 1][w][i] = pend[0];
#pragma unroll
    for (int k = 0; k < W - 1; ++k) pend[k] = pend[k + 1];
  }
  return nclip;
}

// SOLVE launch of level `lev`: one CTA per tile (M + N - 1 - lev, M).  Folds in
// the level lev-1 sources, adds the two right-hand-side buffers and solves.
template <typename C>
__global__ void __launch_bounds__(SolveShape<C>::THREADS) solve_kernel(SweepArgs p, const C* __restrict__ T, const C* __restrict__ Rn,
                                                   const C* __restrict__ Rf, C* __restrict__ L,
                                                   typename Real<C>::T clip,
                                                   unsigned long long* __restrict__ clipped) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* sR = reinterpret_cast<C*>(smem_raw);  // 9 tiles of NB x LD + one NB x NB
  C* sRf = sR + NB * LD;
  C* s1 = sRf + NB * LD;
  C* s2 = s1 + NB * LD;
  C* s3 = s2 + NB * LD;
  C* s4 = s3 + NB * LD;
  C* sT2 = s4 + NB * LD;
  C* sT1 = sT2 + NB * LD;
  C* sP = sT1 + NB * LD;
  C* sD = sP + NB * LD;
  const int N = p.N, lev = p.lev, n = p.n;
  const long long ld = p.ld;
  const int M = blockIdx.x, I = M + N - 1 - lev;
  const bool has_col = lev >= 1 && M <= lev - 1;
  const bool has_row = lev >= 1 && I >= N - lev;
  const int tid = threadIdx.x;
  if (tid == 0) SR_TL_MARK(g_tl_solve, 0, lev, 0);
  // T_II and T_MM do not depend on the sweep: with a programmatic dependent
  // launch (SR_SOLVE_PDL) this CTA is scheduled while the previous level is
  // still solving, fetches them, and only then waits for that level (and, by
  // the launch's full edges, the NEAR / far updates) before it reads Rn, Rf, L.
  load_tile_async<C, SolveShape<C>::THREADS>(sT2, T, ld, I * NB, I * NB, n);  // T_II
  load_tile_async<C, SolveShape<C>::THREADS>(sT1, T, ld, M * NB, M * NB, n);  // T_MM
  cp_async_commit();
#if SR_SOLVE_PDL
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  // the next level may start its own prologue now (one level ahead at most)
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
  load_tile_async<C, SolveShape<C>::THREADS>(sR, Rn, ld, I * NB, M * NB, n);
  load_tile_async<C, SolveShape<C>::THREADS>(sRf, Rf, ld, I * NB, M * NB, n);
  if (has_col) {
    const int K = M + N - lev;
    load_tile_async<C, SolveShape<C>::THREADS>(s1, T, ld, I * NB, K * NB, n);  // T_IK
    load_tile_async<C, SolveShape<C>::THREADS>(s2, L, ld, K * NB, M * NB, n);  // L_KM
  }
  if (has_row) {
    const int J = I - N + lev;
    load_tile_async<C, SolveShape<C>::THREADS>(s3, L, ld, I * NB, J * NB, n);  // L_IJ
    load_tile_async<C, SolveShape<C>::THREADS>(s4, T, ld, J * NB, M * NB, n);  // T_JM
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  {
    constexpr int RPT = SolveShape<C>::RPT;
    const int ty = tid / 8, tx = tid % 8;  // rows RPT ty .., cols 4tx..4tx+3
    C acc[RPT][4];
#pragma unroll
    for (int a = 0; a < RPT; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int o = (RPT * ty + a) * LD + 4 * tx + c;
        acc[a][c].x = sR[o].x + sRf[o].x;
        acc[a][c].y = sR[o].y + sRf[o].y;
      }
    if (has_col) tile_mac<C, false, RPT>(acc, s1, s2, ty, tx);
    if (has_row) tile_mac<C, true, RPT>(acc, s3, s4, ty, tx);
#pragma unroll
    for (int a = 0; a < RPT; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) sRf[(RPT * ty + a) * LD + 4 * tx + c] = acc[a][c];  // sRf is not read again
    // reciprocal pivots and the diagonal-major copy of T_MM
    for (int idx = tid; idx < NB * NB; idx += SolveShape<C>::THREADS) {
      const int i = idx / NB, j = idx % NB;
      C d;
      d.x = sT2[i * LD + i].x - sT1[j * LD + j].x;
      d.y = sT2[i * LD + i].y - sT1[j * LD + j].y;
      sP[i * LD + j] = crecip(d);
      // idx = dd * NB + jj: sD[dd][jj] = T1[jj][jj + dd]
      sD[idx] = (i + j < NB) ? sT1[j * LD + j + i] : czero<C>();
    }
  }
  __syncthreads();
  const int vi = min(NB, n - I * NB), vj = min(NB, n - M * NB);
  const auto cl = clip;
  unsigned nclip;
#if SR_SOLVE_ONE_WARP
  if (tid >= 32) return;
  if (I == M)
    nclip = tile_solve_warp<C, true>(sT2, sD, sP, sRf, s1, vi, vj, cl);
  else
    nclip = tile_solve_warp<C, false>(sT2, sD, sP, sRf, s1, vi, vj, cl);
  __syncwarp();
  const int gj = M * NB + tid;
  for (int r = 0; r < NB; ++r) {
    const int gi = I * NB + r;
    if (gi < n && gj < n) L[(size_t)gi * ld + gj] = (I == M && r <= tid) ? czero<C>() : s1[r * LD + tid];
  }
#else
  constexpr int NW = SolveShape<C>::THREADS / 32;
  static_assert(NW == 4 || NW == 8, "the CTA tile solve needs four or eight warps");
  __shared__ C xs[2][NB];
  __shared__ C hand[2][NW][NB];
  if (I == M)
    nclip = tile_solve_cta<C, true, NW>(sT2, sD, sP, sRf, s1, xs, hand, vi, vj, cl);
  else
    nclip = tile_solve_cta<C, false, NW>(sT2, sD, sP, sRf, s1, xs, hand, vi, vj, cl);
  __syncthreads();
  {
    const int gj = M * NB + (tid & 31);
    for (int r = tid >> 5; r < NB; r += SolveShape<C>::THREADS / 32) {
      const int gi = I * NB + r;
      if (gi < n && gj < n) L[(size_t)gi * ld + gj] = (I == M && r <= (tid & 31)) ? czero<C>() : s1[r * LD + (tid & 31)];
    }
  }
  if (tid >= 32) return;
#endif
  nclip = __reduce_add_sync(0xffffffffu, nclip);
  if (tid == 0 && nclip) atomicAdd(clipped, (unsigned long long)nclip);
  if (tid == 0) SR_TL_MARK(g_tl_solve, 0, lev, 1);
}

// NEAR launch of level `lev` (sources: the tiles solved at level lev-1): one
// CTA per tile on levels lev+1 .. lmax (blockIdx.y = level - lev - 1,
// blockIdx.x = column M <= level), rank-NB update of Rn in place.
template <typename C>
__global__ void __launch_bounds__(NT) near_kernel(SweepArgs p, const C* __restrict__ T, C* __restrict__ Rn,
                                                  const C* __restrict__ L) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s0 = reinterpret_cast<C*>(smem_raw);  // 5 tiles of NB x LD
  C* s1 = s0 + NB * LD;
  C* s2 = s1 + NB * LD;
  C* s3 = s2 + NB * LD;
  C* s4 = s3 + NB * LD;
  const int N = p.N, lev = p.lev, n = p.n;
  const long long ld = p.ld;
  const int level = lev + 1 + blockIdx.y;
  const int M = blockIdx.x;
  if (M > level) return;
  const int I = M + N - 1 - level;
  const bool has_col = M <= lev - 1;   // source (K, M), K = M + N - lev
  const bool has_row = I >= N - lev;   // source (I, J), J = I - N + lev
  if (!has_col && !has_row) return;
  const int tid = threadIdx.x;
  if (tid == 0) SR_TL_MARK(g_tl_solve, 1, lev, 0);
  load_tile_async(s0, Rn, ld, I * NB, M * NB, n);
  if (has_col) {
    const int K = M + N - lev;
    load_tile_async(s1, T, ld, I * NB, K * NB, n);
    load_tile_async(s2, L, ld, K * NB, M * NB, n);
  }
  if (has_row) {
    const int J = I - N + lev;
    load_tile_async(s3, L, ld, I * NB, J * NB, n);
    load_tile_async(s4, T, ld, J * NB, M * NB, n);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int ty = tid / 8, tx = tid % 8;
  C acc[2][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = s0[(2 * ty + a) * LD + 4 * tx + c];
  if (has_col) tile_mac<C, false>(acc, s1, s2, ty, tx);
  if (has_row) tile_mac<C, true>(acc, s3, s4, ty, tx);
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int gi = I * NB + 2 * ty + a, gj = M * NB + 4 * tx + c;
      if (gi < n && gj < n) Rn[(size_t)gi * ld + gj] = acc[a][c];
    }
  if (tid == 0) SR_TL_MARK(g_tl_solve, 1, lev, 1);
}

struct FarArgs {
  int n, N, beta, h, first;  // h = targets per source line; first = first column (COL) / row (ROW)
  int first_level;           // first target level, 4 (beta + 1 + FAR_LA)
  long long ld;
};

// FAR launch of batch `beta` (sources: the tiles of levels 4b .. 4b+3).
//   COL (ROW = false): blockIdx.y -> column M = first + y (M <= 4b+3); the
//     sources of column M are K = M+N-4b-4 .. M+N-4b-1, the targets its tiles
//     I = M .. M+h-1 (levels >= 4b+8, h = N-4b-8).  CTA = strip of BW target
//     tiles (BW NB x NB rows): Rf[strip, M] -= T[strip, Ks] L[Ks, M].
//   ROW (ROW = true): blockIdx.y -> row I = first + y (I >= N-4b-4); sources
//     J = I-N+1+4b .. I-N+4+4b (J < 0 do not exist: zero tiles), targets
//     M = I-N+4b+9 .. I.  CTA = strip of BW target tiles (BW NB columns):
//     Rf[I, strip] += L[I, Js] T[Js, strip].
// Each source tile is one K-chunk of NB; chunks stream through STAGES shared
// buffers by cp.async while the previous one is multiplied.
template <typename C, bool ROW>
struct FarShape {
  static constexpr int BM = ROW ? NB : BW * NB;   // target rows per CTA
  static constexpr int BN = ROW ? BW * NB : NB;   // target cols per CTA
  static constexpr int AP = NB + (sizeof(C) == 8 ? 2 : 1);  // A pitch: conflict-free column reads
  static constexpr int A_ELEMS = BM * AP;
  static constexpr int B_ELEMS = NB * BN;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
};

template <typename C, bool ROW, int STAGES>
__global__ void __launch_bounds__(FT) far_kernel(FarArgs p, const C* __restrict__ T, const C* __restrict__ L,
                                                 C* __restrict__ Rf) {
  using S = FarShape<C, ROW>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* smem = reinterpret_cast<C*>(smem_raw);
  const int N = p.N, n = p.n, beta = p.beta;
  const long long ld = p.ld;
  const int line = p.first + blockIdx.y;  // M (COL) or I (ROW)
  const int t0 = BW * blockIdx.x;         // first target in the strip (offset along the line)
  // global origin of the target strip and of the first source
  int out_r0, out_c0, src0;
  if (!ROW) {
    const int M = line;
    out_r0 = (M + t0) * NB;
    out_c0 = M * NB;
    src0 = M + N - 4 * beta - 4;  // K of chunk 0
  } else {
    const int I = line;
    out_r0 = I * NB;
    out_c0 = (I - N + 1 + p.first_level + t0) * NB;
    src0 = I - N + 1 + 4 * beta;  // J of chunk 0
  }
  const int tid = threadIdx.x;
  auto chunk_valid = [&](int k) {
    const int s = src0 + k;
    return ROW ? (s >= 0) : (s <= N - 1);
  };
  auto issue = [&](int k) {
    C* sa = smem + (k % STAGES) * S::STAGE;
    C* sb = sa + S::A_ELEMS;
    if (chunk_valid(k)) {
      const int s = src0 + k;
      if (!ROW) {
        load_block_async<C>(sa, S::AP, T, ld, out_r0, s * NB, S::BM, NB, n, tid, FT);  // T[strip, K]
        load_block_async<C>(sb, S::BN, L, ld, s * NB, out_c0, NB, S::BN, n, tid, FT);  // L[K, M]
      } else {
        load_block_async<C>(sa, S::AP, L, ld, out_r0, s * NB, S::BM, NB, n, tid, FT);  // L[I, J]
        load_block_async<C>(sb, S::BN, T, ld, s * NB, out_c0, NB, S::BN, n, tid, FT);  // T[J, strip]
      }
    }
    cp_async_commit();
  };
  // thread -> outputs: rows ra + RS*a, cols cb + CS*q (a, q = 0..3)
  constexpr int CS = ROW ? 32 : 8;
  constexpr int RS = ROW ? 8 : 32;
  const int cb = tid % CS, ra = tid / CS;
  C acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[a][q] = czero<C>();
#pragma unroll
  for (int k = 0; k < STAGES - 1; ++k) issue(k);
#pragma unroll 1
  for (int k = 0; k < BW; ++k) {
    if (k + STAGES - 1 < BW)
      issue(k + STAGES - 1);
    else
      cp_async_commit();  // keep the group count uniform
    cp_async_wait<STAGES - 1>();
    __syncthreads();
    if (chunk_valid(k)) {
      const C* sa = smem + (k % STAGES) * S::STAGE;
      const C* sb = sa + S::A_ELEMS;
#pragma unroll 4
      for (int kk = 0; kk < NB; ++kk) {
        C av[4], bv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = sa[(ra + RS * a) * S::AP + kk];
#pragma unroll
        for (int q = 0; q < 4; ++q) bv[q] = sb[kk * S::BN + cb + CS * q];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int q = 0; q < 4; ++q) cfma(acc[a][q], av[a], bv[q]);
      }
    }
    __syncthreads();  // the stage is refilled by the next issue()
  }
  // epilogue: Rf[target] -= acc (COL) / += acc (ROW), per target tile in the strip
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int r = ra + RS * a;
    const int gi = out_r0 + r;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = cb + CS * q;
      const int tgt = t0 + (ROW ? c / NB : r / NB);  // target index along the line
      const int gj = out_c0 + c;
      if (tgt < p.h && gi < n && gj < n) {
        C v = Rf[(size_t)gi * ld + gj];
        if (ROW) {
          v.x += acc[a][q].x;
          v.y += acc[a][q].y;
        } else {
          v.x -= acc[a][q].x;
          v.y -= acc[a][q].y;
        }
        Rf[(size_t)gi * ld + gj] = v;
      }
    }
  }
}

// Rn = -stril(E) (only the strictly lower part is ever read), Rf = 0, L = 0.
template <typename C>
__global__ void init_kernel(int n, const C* __restrict__ E, C* __restrict__ Rn, C* __restrict__ Rf,
                            C* __restrict__ L, long long ld) {
  for (GridIdx g(n, n); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    const size_t o = (size_t)i * ld + j;
    C r = czero<C>();
    if (i > j) {
      const C e = E[o];
      r.x = -e.x;
      r.y = -e.y;
    }
    Rn[o] = r;
    Rf[o] = czero<C>();
    L[o] = czero<C>();
  }
}

// Exact-duplicate diagonal check (trisolve.py:104-113): flags |= 1 on a hit.
template <typename C>
__global__ void separation_kernel(int n, const C* __restrict__ T, long long ld, int* __restrict__ flags) {
  int i = blockIdx.y * blockDim.y + threadIdx.y;
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || j >= n || j <= i) return;
  C a = T[(size_t)i * ld + i], b = T[(size_t)j * ld + j];
  if (a.x == b.x && a.y == b.y) atomicOr(flags, SR_FLAG_SEPARATION);
}

constexpr int FAR_STAGES = 2;
constexpr int NFAR_EV = 4;

inline size_t r_bytes(int n, long long ld, size_t elt) { return ((size_t)n * ld * elt + 255) & ~(size_t)255; }

// Internal streams and events (created once per lp type): the critical-path
// tile solves, the near band and the far batches; plus the captured graph of
// the last problem (the refinement calls the solver with the same buffers every
// iteration, so the N-level launch sequence is recorded once and replayed).
struct SolveCtx {
  bool ready = false;
  cudaStream_t s_solve, s_near, s_far;
  cudaEvent_t ev_in, ev_s, ev_u, ev_f[NFAR_EV], ev_j;
  // graph of the last (args) seen
  cudaGraphExec_t exec = nullptr;
  unsigned long long kernels = 0;  // kernel nodes in the graph
  const void *t = nullptr, *e = nullptr, *l = nullptr, *ws = nullptr, *clipped = nullptr, *flags = nullptr;
  size_t ws_bytes = 0;
  long long ld = 0;
  int n = -1;
  double clip = 0;
  int calls = 0;  // eager calls with these args before capturing
};

template <typename C>
int ctx_init(SolveCtx& c) {
  if (c.ready) return SR_OK;
  // priorities: the critical-path tile solves first, then the near band, the far batches last
  int prio_lo = 0, prio_hi = 0;
  SR_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  SR_CUDA_CHECK(cudaStreamCreateWithPriority(&c.s_solve, cudaStreamNonBlocking, prio_hi));
  SR_CUDA_CHECK(cudaStreamCreateWithPriority(&c.s_near, cudaStreamNonBlocking, prio_hi + (prio_lo > prio_hi ? 1 : 0)));
  SR_CUDA_CHECK(cudaStreamCreateWithPriority(&c.s_far, cudaStreamNonBlocking, prio_lo));
  SR_CUDA_CHECK(cudaEventCreateWithFlags(&c.ev_in, cudaEventDisableTiming));
  SR_CUDA_CHECK(cudaEventCreateWithFlags(&c.ev_s, cudaEventDisableTiming));
  SR_CUDA_CHECK(cudaEventCreateWithFlags(&c.ev_u, cudaEventDisableTiming));
  SR_CUDA_CHECK(cudaEventCreateWithFlags(&c.ev_j, cudaEventDisableTiming));
  for (int i = 0; i < NFAR_EV; ++i) SR_CUDA_CHECK(cudaEventCreateWithFlags(&c.ev_f[i], cudaEventDisableTiming));
  SR_CUDA_CHECK(cudaFuncSetAttribute(solve_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(C) * (9 * NB * LD + NB * NB))));
  SR_CUDA_CHECK(cudaFuncSetAttribute(near_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(C) * 5 * NB * LD)));
  // one shared-memory carveout (all of it) for every sweep kernel, so SOLVE,
  // NEAR and far CTAs can share an SM whichever launched first
  SR_CUDA_CHECK(cudaFuncSetAttribute(solve_kernel<C>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared));
  SR_CUDA_CHECK(cudaFuncSetAttribute(near_kernel<C>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared));
  SR_CUDA_CHECK(cudaFuncSetAttribute(far_kernel<C, false, FAR_STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(C) * FAR_STAGES * FarShape<C, false>::STAGE)));
  SR_CUDA_CHECK(cudaFuncSetAttribute(far_kernel<C, true, FAR_STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(C) * FAR_STAGES * FarShape<C, true>::STAGE)));
  c.ready = true;
  return SR_OK;
}

// Enqueue one solve.  `origin` is the caller's stream (eager) or the context's
// solve stream under capture; every forked stream is joined back into it.
template <typename C>
int enqueue(SolveCtx& c, int n, const C* t, const C* e, long long ld, C* l, double clip,
            unsigned long long* d_clipped, int* d_flags, void* ws, cudaStream_t origin) {
  const int N = (n + NB - 1) / NB;
  const size_t rb = r_bytes(n, ld, sizeof(C));
  C* Rn = (C*)ws;
  C* Rf = (C*)((char*)ws + rb);
  // complex64 with 16-byte aligned rows: far updates on the tensor cores (trisolve_tc.cu)
  constexpr bool kC64 = std::is_same<C, float2>::value;
  const bool use_tc = kC64 && (ld % 2) == 0 && !getenv("SR_SOLVE_SIMT_FAR");
  FarTcPlan plan;
  {
    const long long total = (long long)n * n;
    const long long blocks = (total + 255) / 256;
    const int grid = (int)(blocks < 148 * 16 ? blocks : 148 * 16);
    init_kernel<C><<<grid, 256, 0, origin>>>(n, e, Rn, Rf, l, ld);
    SR_LAUNCH_CHECK();
  }
  const size_t smem_solve = sizeof(C) * (9 * NB * LD + NB * NB);
  const size_t smem_near = sizeof(C) * 5 * NB * LD;
  const size_t smem_far_col = sizeof(C) * FAR_STAGES * FarShape<C, false>::STAGE;
  const size_t smem_far_row = sizeof(C) * FAR_STAGES * FarShape<C, true>::STAGE;
  cudaStream_t s_solve = c.s_solve, s_near = c.s_near, s_far = c.s_far;
  SR_CUDA_CHECK(cudaEventRecord(c.ev_in, origin));
  if (s_solve != origin) SR_CUDA_CHECK(cudaStreamWaitEvent(s_solve, c.ev_in, 0));
  SR_CUDA_CHECK(cudaStreamWaitEvent(s_near, c.ev_in, 0));
  SR_CUDA_CHECK(cudaStreamWaitEvent(s_far, c.ev_in, 0));
  // off the critical path: the far updates' T forms on the far stream (first
  // read by the far launches of batch 0, after four levels); the separation
  // scan (its flag is read after the join) on the far stream beside the last
  // levels, which have no far targets left and leave most SMs idle
  if constexpr (kC64) {
    if (use_tc) {
      const int rc = far_tc_prepare(&plan, n, t, ld, (char*)ws + 2 * rb, s_far);
      if (rc != SR_OK) return rc;
    }
  }
  const int sep_level = N > 8 ? N - 8 : 0;
  const typename Real<C>::T cl = (typename Real<C>::T)clip;
  for (int lev = 0; lev < N; ++lev) {
    // SOLVE(lev): after NEAR(lev-1) (ev_u) and FAR(lev/4 - 1 - FAR_LA)
    if (lev >= 1) SR_CUDA_CHECK(cudaStreamWaitEvent(s_solve, c.ev_u, 0));
    if (lev % BW == 0 && lev >= BW * (1 + FAR_LA))
      SR_CUDA_CHECK(cudaStreamWaitEvent(s_solve, c.ev_f[(lev / BW - 1 - FAR_LA) % NFAR_EV], 0));
    SweepArgs a{n, N, lev, 0, ld};
#if SR_SOLVE_PDL
    {
      // programmatic edge from SOLVE(lev-1) (same stream); the event waits above stay full edges
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(lev + 1);
      lc.blockDim = dim3(SolveShape<C>::THREADS);
      lc.dynamicSmemBytes = smem_solve;
      lc.stream = s_solve;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      // up to n = 4096 (n = 512 .. 4096 solves 5-6 % faster); at n = 8192 programmatic launches on
      // every level cost 2 % (16.1 vs 15.8 ms: the early-resident CTAs hold shared memory the far and
      // NEAR CTAs want) and on the first 64 / 128 levels only they gain nothing: plain edges there
      at[0].val.programmaticStreamSerializationAllowed = N <= 128 ? 1 : 0;
      lc.attrs = at;
      lc.numAttrs = 1;
      const C* tc = t;
      const C* rn = Rn;
      const C* rf = Rf;
      SR_CUDA_CHECK(cudaLaunchKernelEx(&lc, solve_kernel<C>, a, tc, rn, rf, l, cl, d_clipped));
    }
#else
    solve_kernel<C><<<lev + 1, SolveShape<C>::THREADS, smem_solve, s_solve>>>(a, t, Rn, Rf, l, cl, d_clipped);
#endif
    SR_LAUNCH_CHECK();
    // NEAR(lev): sources of level lev-1 into levels lev+1 .. 4 (b + 1 + FAR_LA) - 1, b = (lev-1)/4
    if (lev >= 1) {
      SR_CUDA_CHECK(cudaStreamWaitEvent(s_near, c.ev_s, 0));  // SOLVE(lev-1)
      const int b = (lev - 1) / BW;
      const int lmax = min(N - 1, BW * (b + 1 + FAR_LA) - 1);
      if (lmax >= lev + 1) {
        a.lmax = lmax;
        dim3 grid(lmax + 1, lmax - lev);
        near_kernel<C><<<grid, NT, smem_near, s_near>>>(a, t, Rn, l);
        SR_LAUNCH_CHECK();
      }
    }
    SR_CUDA_CHECK(cudaEventRecord(c.ev_s, s_solve));
    SR_CUDA_CHECK(cudaEventRecord(c.ev_u, s_near));
    if (lev == sep_level) {
      dim3 b(32, 8), g(sr_ceil_div(n, 32), sr_ceil_div(n, 8));
      separation_kernel<C><<<g, b, 0, s_far>>>(n, t, ld, d_flags);
      SR_LAUNCH_CHECK();
    }
    // FAR(b) once the last level of batch b is solved, if any tile sits on a far target level
#ifndef SR_DIAG_NO_FAR  // timing diagnostic only (tools/solve_bench.py): wrong results without it
    if (lev % BW == BW - 1) {
#else
    if (false) {
#endif
      const int b = lev / BW;
      const int first_level = BW * (b + 1 + FAR_LA);  // first far target level
      const int h = N - first_level;
      if (h >= 1) {
        SR_CUDA_CHECK(cudaStreamWaitEvent(s_far, c.ev_s, 0));
        bool done = false;
        if constexpr (kC64) {
          if (use_tc) {
            const int rc = far_tc_batch(plan, N, b, h, first_level, l, ld, Rf, s_far);
            if (rc != SR_OK) return rc;
            done = true;
          }
        }
        if (!done) {
          FarArgs fa{n, N, b, h, 0, first_level, ld};
          const int strips = (h + BW - 1) / BW;
          fa.first = 0;
          far_kernel<C, false, FAR_STAGES>
              <<<dim3(strips, min(BW * b + BW, N)), FT, smem_far_col, s_far>>>(fa, t, l, Rf);
          SR_LAUNCH_CHECK();
          fa.first = N - BW - BW * b;
          far_kernel<C, true, FAR_STAGES><<<dim3(strips, N - fa.first), FT, smem_far_row, s_far>>>(fa, t, l, Rf);
          SR_LAUNCH_CHECK();
        }
        SR_CUDA_CHECK(cudaEventRecord(c.ev_f[b % NFAR_EV], s_far));
      }
    }
  }
  // join: the near and far streams (already upstream of the last SOLVE, joined
  // explicitly so a capture sees no dangling work), then the solve stream
  SR_CUDA_CHECK(cudaEventRecord(c.ev_j, s_far));
  SR_CUDA_CHECK(cudaStreamWaitEvent(s_solve, c.ev_j, 0));
  SR_CUDA_CHECK(cudaEventRecord(c.ev_j, s_near));
  SR_CUDA_CHECK(cudaStreamWaitEvent(s_solve, c.ev_j, 0));
  if (s_solve != origin) {
    SR_CUDA_CHECK(cudaEventRecord(c.ev_s, s_solve));
    SR_CUDA_CHECK(cudaStreamWaitEvent(origin, c.ev_s, 0));
  }
  return SR_OK;
}

template <typename C>
int solve(int n, const C* t, const C* e, long long ld, C* l, double clip, unsigned long long* d_clipped,
          int* d_flags, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n < 0 || ld < n) return SR_EINVAL;
  if (n == 0) return SR_OK;
  const size_t need = sr_trisolve_workspace_bytes(n, sizeof(C) == 8 ? 1 : 0);
  const size_t rb = r_bytes(n, ld, sizeof(C));
  if (ws_bytes < need || !ws || 2 * rb + (sizeof(C) == 8 ? far_tc_forms_bytes(n) : 0) > need) return SR_EINVAL;
  // one context per (device, lp type); a context serialises its callers
  static SolveCtx ctxs[SR_MAX_DEVICES];
  static std::mutex mus[SR_MAX_DEVICES];
  int slot = 0;
  if (sr_device_slot(&slot) != SR_OK) return SR_EINVAL;
  std::lock_guard<std::mutex> lock(mus[slot]);
  SolveCtx& c = ctxs[slot];
  if (ctx_init<C>(c) != SR_OK) return SR_ECUDA;
  const bool same = c.n == n && c.t == t && c.e == e && c.l == l && c.ld == ld && c.clip == clip &&
                    c.clipped == d_clipped && c.flags == d_flags && c.ws == ws && c.ws_bytes == ws_bytes;
  if (!same) {
    if (c.exec) cudaGraphExecDestroy(c.exec);
    c.exec = nullptr;
    c.n = n, c.t = t, c.e = e, c.l = l, c.ld = ld, c.clip = clip, c.clipped = d_clipped, c.flags = d_flags;
    c.ws = ws, c.ws_bytes = ws_bytes, c.calls = 0;
  }
  // The first call with new arguments runs eagerly; the second records the
  // launch sequence into a CUDA graph, later calls replay it (SR_SOLVE_NO_GRAPH=1: always eager).
  const bool graphs = !getenv("SR_SOLVE_NO_GRAPH");
  if (!graphs || (!c.exec && c.calls == 0)) {
    ++c.calls;
    return enqueue<C>(c, n, t, e, ld, l, clip, d_clipped, d_flags, ws, st);
  }
  SR_CUDA_CHECK(cudaEventRecord(c.ev_in, st));
  SR_CUDA_CHECK(cudaStreamWaitEvent(c.s_solve, c.ev_in, 0));
  if (!c.exec) {
    const unsigned long long k0 = sr_kernel_launches();
    SR_CUDA_CHECK(cudaStreamBeginCapture(c.s_solve, cudaStreamCaptureModeThreadLocal));
    const int rc = enqueue<C>(c, n, t, e, ld, l, clip, d_clipped, d_flags, ws, c.s_solve);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(c.s_solve, &g);
    if (rc != SR_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ce != cudaSuccess) return sr_set_cuda_error(ce, "cudaStreamEndCapture(trisolve)");
    // node priorities as captured (SOLVE > NEAR > far), so the block scheduler
    // keeps preferring the critical path inside the graph too (SR_SOLVE_GRAPH_FLAT=1: off)
    const cudaError_t ie = cudaGraphInstantiateWithFlags(
        &c.exec, g, getenv("SR_SOLVE_GRAPH_FLAT") ? 0 : cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) {
      c.exec = nullptr;
      return sr_set_cuda_error(ie, "cudaGraphInstantiate(trisolve)");
    }
    c.kernels = sr_kernel_launches() - k0;  // counted at capture; replayed by the launch below
  } else {
    sr_count_launches(c.kernels);
  }
  SR_CUDA_CHECK(cudaGraphLaunch(c.exec, c.s_solve));
  SR_CUDA_CHECK(cudaEventRecord(c.ev_s, c.s_solve));
  SR_CUDA_CHECK(cudaStreamWaitEvent(st, c.ev_s, 0));
  return SR_OK;
}

}  // namespace

#ifdef SR_TIMELINE
extern "C" int sr_timeline_solve(void* host, int reset) {
  if (reset) {
    static unsigned long long init[8][1024][2];
    for (int k = 0; k < 8; ++k)
      for (int s = 0; s < 1024; ++s) init[k][s][0] = ~0ull, init[k][s][1] = 0;
    return cudaMemcpyToSymbol(g_tl_solve, init, sizeof(init)) == cudaSuccess ? 0 : 4;
  }
  return cudaMemcpyFromSymbol(host, g_tl_solve, sizeof(g_tl_solve)) == cudaSuccess ? 0 : 4;
}
#endif

extern "C" size_t sr_trisolve_workspace_bytes(int n, int lp_is_c64) {
  const size_t elt = lp_is_c64 ? 8 : 16;
  // two running right-hand sides: Rn (near band) and Rf (far batches); for
  // complex64 also the split operand forms of the tensor-core far updates
  return 2 * r_bytes(n, n + (n & 1), elt) + (lp_is_c64 ? far_tc_forms_bytes(n) : 0) + 256;
}

extern "C" int sr_trisolve_c64(int n, const void* t, const void* e, long long ld, void* l, float clip,
                               unsigned long long* d_clipped, int* d_flags, void* ws, size_t ws_bytes,
                               void* stream) {
  return solve<float2>(n, (const float2*)t, (const float2*)e, ld, (float2*)l, clip, d_clipped, d_flags, ws,
                       ws_bytes, (cudaStream_t)stream);
}

extern "C" int sr_trisolve_c128(int n, const void* t, const void* e, long long ld, void* l, double clip,
                                unsigned long long* d_clipped, int* d_flags, void* ws, size_t ws_bytes,
                                void* stream) {
  return solve<double2>(n, (const double2*)t, (const double2*)e, ld, (double2*)l, clip, d_clipped, d_flags, ws,
                        ws_bytes, (cudaStream_t)stream);
}

// Low-precision solve of stril(T L - L T) = -E for strictly lower L.
//
// Replaces the reference solver
//   solve_block           /root/reference/pkg/src/ddschur/trisolve.py:243-262
//   _block_solve          trisolve.py:223-240   (recursive halving)
//   _sylvester_tri        trisolve.py:164-196
//   _scalar_solve_inplace trisolve.py:121-145
//   _check_separation     trisolve.py:104-113
// with a right-looking blocked wavefront over NB x NB tiles of L.  Tile
// (I, J), I >= J, satisfies
//   T_II L_IJ - L_IJ T_JJ = R_IJ,
//   R_IJ = -E_IJ - sum_{K>I} T_IK L_KJ + sum_{K<J} L_IK T_KJ
// (stril() of both sides when I == J).  Tile (I, J) sits on anti-diagonal
// level (N-1-I) + J and depends only on lower levels.  Launch `lev` of the
// sweep owns every still-open tile that the tiles solved at level lev-1
// contribute to — at most one column term (T_IK L_KJ) and one row term
// (L_IJ T_JM) per tile, so each tile is updated by exactly one CTA and the
// running right-hand side R lives in HBM with no atomics — and the CTAs whose
// tile sits on level `lev` then solve it.  N launches per solve, each fully
// parallel over the open tiles.
//
// The tile solve is one warp: lane i owns row i, and entry (i, j) is final at
// step (NB-1-i) + j.  Each lane keeps its open entries in a 32-wide register
// window that slides one column per step (fully unrolled, so the slide is
// register renaming); at every step the lanes finalise one entry each,
// exchange the new values with warp shuffles (the column terms) and fold
// their own new value into their later columns (the row terms).  Clipping is
// applied at finalisation as in the reference (trisolve.py:141-144,192-195),
// so dependants see the clipped zero; any dependency-respecting order gives
// the same L up to rounding.
//
// Templated on the lp type: float2 (FP64 mode, lp = complex64) and double2
// (dd mode, lp = binary64 complex).
#include "sr_common.cuh"

namespace {

constexpr int NB = 32;
constexpr int NT = 128;  // 16 x 8 threads, each owning a 2 x 4 block of the tile
constexpr int LD = NB + 1;

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

// Load an NB x NB tile (rows r0.., cols c0..) with zero fill outside [0, n).
template <typename C>
__device__ __forceinline__ void load_tile(C* s, const C* __restrict__ g, long long ld, int r0, int c0, int n) {
  for (int idx = threadIdx.x; idx < NB * NB; idx += NT) {
    int r = idx / NB, c = idx % NB;
    int gr = r0 + r, gc = c0 + c;
    s[r * LD + c] = (gr < n && gc < n) ? g[(size_t)gr * ld + gc] : czero<C>();
  }
}

// Same, as asynchronous copies (cp.async, zero-filled outside [0, n)); the
// caller commits and waits once for all the tiles it issued.
template <typename C>
__device__ __forceinline__ void load_tile_async(C* s, const C* __restrict__ g, long long ld, int r0, int c0,
                                                int n) {
  for (int idx = threadIdx.x; idx < NB * NB; idx += NT) {
    const int r = idx / NB, c = idx % NB;
    const int gr = r0 + r, gc = c0 + c;
    const bool ok = gr < n && gc < n;
    const C* src = g + (ok ? (size_t)gr * ld + gc : 0);
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(s + r * LD + c);
    if (sizeof(C) == 16)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0));
    else
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0));
  }
}

struct SweepArgs {
  int n, N, lev, countA;
  long long ld;
};

// In-tile solve by one warp: T2 X - X T1 = R (strict lower part only when diag).
template <typename C, bool DIAG>
__device__ __forceinline__ void tile_solve_warp(const C* sT2, const C* sT1, const C* sR, C* sX, int valid_i,
                                                int valid_j, typename Real<C>::T clip, unsigned int* s_clip) {
  const int i = threadIdx.x & 31;
  C pend[NB];
  C tr[NB];
#pragma unroll
  for (int d = 0; d < NB; ++d) {
    const int c = i - (NB - 1) + d;  // window at step 0 covers columns i-31 .. i
    pend[d] = (c >= 0) ? sR[i * LD + c] : czero<C>();
    tr[d] = (i + d < NB) ? sT2[i * LD + i + d] : czero<C>();
  }
  const C tii = tr[0];
#pragma unroll
  for (int t = 0; t < 2 * NB - 1; ++t) {
    const int j = t - (NB - 1) + i;  // this lane's column at step t
    const bool valid = (j >= 0) && (j < NB) && (i < valid_i) && (j < valid_j) && (!DIAG || i > j);
    C x = czero<C>();
    if (valid) {
      const C tjj = sT1[j * LD + j];
      C piv;
      piv.x = tii.x - tjj.x;
      piv.y = tii.y - tjj.y;
      x = cdiv(pend[0], piv);
      if (clip > 0 && sqrt(x.x * x.x + x.y * x.y) > clip) {
        x = czero<C>();
        if (threadIdx.x < 32) atomicAdd(s_clip, 1u);
      }
      sX[i * LD + j] = x;
    }
    // column terms: lane i+d finalised (i+d, j+d); it feeds this lane's (i, j+d)
#pragma unroll
    for (int d = 1; d < NB; ++d) {
      const C xv = shfl_down(x, d);
      if (i + d < NB) cfms(pend[d], tr[d], xv);
    }
    // row terms: (i, j) feeds this lane's (i, j+d) through T1[j][j+d]
    if (valid) {
#pragma unroll
      for (int d = 1; d < NB; ++d)
        if (j + d < NB) cfma(pend[d], x, sT1[j * LD + j + d]);
    }
    // slide the window one column to the right
#pragma unroll
    for (int d = 0; d < NB - 1; ++d) pend[d] = pend[d + 1];
    {
      const int c = t + i + 1;
      pend[NB - 1] = (c < NB) ? sR[i * LD + c] : czero<C>();
    }
  }
}

// SOLVE = true: one CTA per tile on level `lev` (blockIdx.x = its column M):
//   fold in the level-(lev-1) contributions, then solve the tile (critical path).
// SOLVE = false: one CTA per open tile above level `lev` that level lev-1
//   feeds: fold in the contributions, write R back (bulk work, runs on a
//   second stream concurrently with the SOLVE launch of the same level).
template <typename C, bool SOLVE>
__global__ void __launch_bounds__(NT) sweep_kernel(SweepArgs p, const C* __restrict__ T, C* __restrict__ R,
                                                   C* __restrict__ L, typename Real<C>::T clip,
                                                   unsigned long long* __restrict__ clipped) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s0 = reinterpret_cast<C*>(smem_raw);  // 5 tiles of NB x LD
  C* s1 = s0 + NB * LD;
  C* s2 = s1 + NB * LD;
  C* s3 = s2 + NB * LD;
  C* s4 = s3 + NB * LD;
  __shared__ unsigned int s_clip;
  const int N = p.N, lev = p.lev, n = p.n;
  const long long ld = p.ld;
  // ---- which open tile (I, M) this CTA owns
  int I, M;
  if (SOLVE) {  // tile (M + N - 1 - lev, M) on level lev
    M = blockIdx.x;
    I = M + N - 1 - lev;
  } else if ((int)blockIdx.x < p.countA) {  // region A: M <= lev-1, I in [M, M + N - lev - 1]
    const int h = N - lev;
    M = blockIdx.x / h;
    I = M + blockIdx.x % h;
  } else {  // region B: I = N-lev+r, M in [lev, N-lev+r]
    int rem = blockIdx.x - p.countA, r = 0;
    while (true) {
      const int cnt = N - 2 * lev + r + 1;
      if (cnt > 0) {
        if (rem < cnt) break;
        rem -= cnt;
      }
      ++r;
    }
    M = lev + rem;
    I = N - lev + r;
  }
  const int tlev = (N - 1 - I) + M;
  if (!SOLVE && tlev == lev) return;  // owned by the SOLVE launch
  const bool has_col = lev >= 1 && M <= lev - 1;
  const bool has_row = lev >= 1 && I >= N - lev;
  const int tid = threadIdx.x;
  // ---- load R_IM and the contributing tiles
  load_tile_async(s0, R, ld, I * NB, M * NB, n);
  if (has_col) {
    const int K = M + N - lev;
    load_tile_async(s1, T, ld, I * NB, K * NB, n);  // T_IK
    load_tile_async(s2, L, ld, K * NB, M * NB, n);  // L_KM
  }
  if (has_row) {
    const int J = I - N + lev;
    load_tile_async(s3, L, ld, I * NB, J * NB, n);  // L_IJ
    load_tile_async(s4, T, ld, J * NB, M * NB, n);  // T_JM
  }
  if (SOLVE) {  // the diagonal blocks for the tile solve, behind a separate group
    asm volatile("cp.async.commit_group;\n" ::);
  }
  if (tid == 0) s_clip = 0;
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
  if (has_col || has_row) {
    const int ty = tid / 8, tx = tid % 8;  // rows 2ty..2ty+1, cols 4tx..4tx+3
    C acc[2][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][c] = s0[(2 * ty + a) * LD + 4 * tx + c];
    if (has_col) {
#pragma unroll 8
      for (int k = 0; k < NB; ++k) {
        C a0 = s1[(2 * ty) * LD + k], a1 = s1[(2 * ty + 1) * LD + k];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          C b = s2[k * LD + 4 * tx + c];
          cfms(acc[0][c], a0, b);
          cfms(acc[1][c], a1, b);
        }
      }
    }
    if (has_row) {
#pragma unroll 8
      for (int k = 0; k < NB; ++k) {
        C a0 = s3[(2 * ty) * LD + k], a1 = s3[(2 * ty + 1) * LD + k];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          C b = s4[k * LD + 4 * tx + c];
          cfma(acc[0][c], a0, b);
          cfma(acc[1][c], a1, b);
        }
      }
    }
    if (!SOLVE) {  // still open: write the updated right-hand side back
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int gi = I * NB + 2 * ty + a, gj = M * NB + 4 * tx + c;
          if (gi < n && gj < n) R[(size_t)gi * ld + gj] = acc[a][c];
        }
      return;
    }
    __syncthreads();  // everyone is done reading s0 before it is overwritten
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) s0[(2 * ty + a) * LD + 4 * tx + c] = acc[a][c];
  }
  if (!SOLVE) return;
  // ---- solve the tile: T_II X - X T_MM = R_IM
  __syncthreads();
  load_tile(s1, T, ld, I * NB, I * NB, n);  // T_II
  load_tile(s2, T, ld, M * NB, M * NB, n);  // T_MM
  __syncthreads();
  const int vi = min(NB, n - I * NB), vj = min(NB, n - M * NB);
  // every warp runs the (identical) tile solve: keeping the shuffles outside any
  // thread-dependent branch lets them compile to plain SHFL instead of
  // convergence-barrier sequences; all warps store the same values
  if (I == M)
    tile_solve_warp<C, true>(s1, s2, s0, s3, vi, vj, clip, &s_clip);
  else
    tile_solve_warp<C, false>(s1, s2, s0, s3, vi, vj, clip, &s_clip);
  __syncthreads();
  for (int idx = tid; idx < NB * NB; idx += NT) {
    const int i = idx / NB, j = idx % NB;
    const int gi = I * NB + i, gj = M * NB + j;
    if (gi < n && gj < n) L[(size_t)gi * ld + gj] = (I == M && i <= j) ? czero<C>() : s3[i * LD + j];
  }
  if (tid == 0 && s_clip) atomicAdd(clipped, (unsigned long long)s_clip);
}

// R = -stril(E) (only the strictly lower part is ever read), L = 0.
template <typename C>
__global__ void init_kernel(int n, const C* __restrict__ E, C* __restrict__ R, C* __restrict__ L, long long ld) {
  const long long total = (long long)n * n;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / n), j = (int)(idx % n);
    const C e = E[(size_t)i * ld + j];
    C r;
    r.x = (i > j) ? -e.x : 0;
    r.y = (i > j) ? -e.y : 0;
    R[(size_t)i * ld + j] = r;
    L[(size_t)i * ld + j] = czero<C>();
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

inline int count_b(int N, int lev) {
  int c = 0;
  for (int r = 0; r < lev; ++r) {
    const int cnt = N - 2 * lev + r + 1;
    if (cnt > 0) c += cnt;
  }
  return c;
}

template <typename C>
int solve(int n, const C* t, const C* e, long long ld, C* l, double clip, unsigned long long* d_clipped,
          int* d_flags, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n < 0 || ld < n) return SR_EINVAL;
  if (n == 0) return SR_OK;
  const int N = (n + NB - 1) / NB;
  const size_t need = sr_trisolve_workspace_bytes(n, sizeof(C) == 8 ? 1 : 0);
  if (ws_bytes < need || !ws || (size_t)n * ld * sizeof(C) > need) return SR_EINVAL;
  C* R = (C*)ws;
  {
    const long long total = (long long)n * n;
    const long long blocks = (total + 255) / 256;
    const int grid = (int)(blocks < 148 * 16 ? blocks : 148 * 16);
    init_kernel<C><<<grid, 256, 0, st>>>(n, e, R, l, ld);
    SR_LAUNCH_CHECK();
    dim3 b(32, 8), g(sr_ceil_div(n, 32), sr_ceil_div(n, 8));
    separation_kernel<C><<<g, b, 0, st>>>(n, t, ld, d_flags);
    SR_LAUNCH_CHECK();
  }
  const size_t smem = sizeof(C) * 5 * NB * LD;
  auto ksolve = sweep_kernel<C, true>;
  auto kupd = sweep_kernel<C, false>;
  // Two internal streams (created once): the critical-path tile solves and the
  // bulk right-hand-side updates of each level run concurrently; events order
  // level lev+1 after both launches of level lev.
  static bool configured = false;
  static cudaStream_t s_solve, s_upd;
  static cudaEvent_t ev_in, ev_s, ev_u;
  if (!configured) {
    SR_CUDA_CHECK(cudaFuncSetAttribute(ksolve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SR_CUDA_CHECK(cudaFuncSetAttribute(kupd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SR_CUDA_CHECK(cudaStreamCreateWithFlags(&s_solve, cudaStreamNonBlocking));
    SR_CUDA_CHECK(cudaStreamCreateWithFlags(&s_upd, cudaStreamNonBlocking));
    SR_CUDA_CHECK(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
    SR_CUDA_CHECK(cudaEventCreateWithFlags(&ev_s, cudaEventDisableTiming));
    SR_CUDA_CHECK(cudaEventCreateWithFlags(&ev_u, cudaEventDisableTiming));
    configured = true;
  }
  SR_CUDA_CHECK(cudaEventRecord(ev_in, st));
  SR_CUDA_CHECK(cudaStreamWaitEvent(s_solve, ev_in, 0));
  SR_CUDA_CHECK(cudaStreamWaitEvent(s_upd, ev_in, 0));
  const typename Real<C>::T cl = (typename Real<C>::T)clip;
  for (int lev = 0; lev < N; ++lev) {
    const int countA = lev * (N - lev);
    SweepArgs a{n, N, lev, countA, ld};
    ksolve<<<lev + 1, NT, smem, s_solve>>>(a, t, R, l, cl, d_clipped);
    SR_LAUNCH_CHECK();
    const int grid = lev == 0 ? 0 : countA + count_b(N, lev);
    if (grid > 0) {
      kupd<<<grid, NT, smem, s_upd>>>(a, t, R, l, cl, d_clipped);
      SR_LAUNCH_CHECK();
    }
    SR_CUDA_CHECK(cudaEventRecord(ev_s, s_solve));
    SR_CUDA_CHECK(cudaEventRecord(ev_u, s_upd));
    SR_CUDA_CHECK(cudaStreamWaitEvent(s_solve, ev_u, 0));
    SR_CUDA_CHECK(cudaStreamWaitEvent(s_upd, ev_s, 0));
  }
  SR_CUDA_CHECK(cudaEventRecord(ev_s, s_solve));
  SR_CUDA_CHECK(cudaStreamWaitEvent(st, ev_s, 0));
  return SR_OK;
}

}  // namespace

extern "C" size_t sr_trisolve_workspace_bytes(int n, int lp_is_c64) {
  const size_t elt = lp_is_c64 ? 8 : 16;
  return (size_t)n * (size_t)(n + (n & 1)) * elt + 256;  // the running right-hand side R
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

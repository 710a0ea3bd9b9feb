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
//   T_II L_IJ - L_IJ T_JJ = -E_IJ - sum_{K>I} T_IK L_KJ + sum_{K<J} L_IK T_KJ
// (stril() of both sides when I == J).  Every tile on the anti-diagonal
// level (N-1-I) + J depends only on lower levels, so the sweep is N
// level-synchronous launches.  Inside a launch each tile first forms the
// right-hand side as two skinny products (the off-diagonal updates, split
// over several CTAs when a level has few tiles and reduced in fixed split
// order — deterministic), then one CTA solves the small tile equation by an
// in-tile wavefront: entry (i, j) is finalised at step (NB-1-i) + j, and
// every still-open entry of the CTA folds in the two entries finalised at
// that step (one per row / column neighbour), so a step costs two complex
// FMAs per entry and one barrier.  Clipping is applied at finalisation, as
// in the reference (trisolve.py:141-144,192-195): dependent entries see the
// clipped zero.  Any dependency-respecting order yields the same L up to
// rounding.
//
// Templated on the lp type: float2 (FP64 mode, lp = complex64) and double2
// (dd mode, lp = binary64 complex).
#include "sr_common.cuh"

namespace {

constexpr int NB = 32;
constexpr int NT = 256;  // 16 x 16 threads, each owning a 2 x 2 block of the tile

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
  acc.x += a.x * b.x - a.y * b.y;
  acc.y += a.x * b.y + a.y * b.x;
}
template <typename C>
__device__ __forceinline__ void cfms(C& acc, C a, C b) {  // acc -= a * b
  acc.x -= a.x * b.x - a.y * b.y;
  acc.y -= a.x * b.y + a.y * b.x;
}

// Load an NB x NB tile (rows r0.., cols c0..) with zero fill outside [0, n).
template <typename C>
__device__ __forceinline__ void load_tile(C* s, const C* __restrict__ g, long long ld, int r0, int c0, int n) {
  for (int idx = threadIdx.x; idx < NB * NB; idx += NT) {
    int r = idx / NB, c = idx % NB;
    int gr = r0 + r, gc = c0 + c;
    s[r * (NB + 1) + c] = (gr < n && gc < n) ? g[(size_t)gr * ld + gc] : czero<C>();
  }
}

struct LevelArgs {
  int n, N, level, splits;
  long long ld;
};

// One launch per anti-diagonal level.  grid.x = tiles on the level
// (J = 0..level), grid.y = splits of the update sum.
template <typename C>
__global__ void __launch_bounds__(NT) trisolve_level_kernel(LevelArgs p, const C* __restrict__ T,
                                                            const C* __restrict__ E, C* __restrict__ L,
                                                            C* __restrict__ ws, int* __restrict__ counters,
                                                            typename Real<C>::T clip,
                                                            unsigned long long* __restrict__ clipped) {
  using R = typename Real<C>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* sA = reinterpret_cast<C*>(smem_raw);       // [NB][NB+1]
  C* sB = sA + NB * (NB + 1);                   // [NB][NB+1]
  __shared__ int s_last;
  __shared__ unsigned int s_clip;

  const int J = blockIdx.x;
  const int I = J + (p.N - 1 - p.level);
  const int split = blockIdx.y;
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const int n = p.n;
  const long long ld = p.ld;

  // ---- off-diagonal updates: col terms K = I+1..N-1 (sign -), row terms K = 0..J-1 (sign +)
  const int ncol = p.N - 1 - I, nrow = J, nterms = ncol + nrow;
  const int per = (nterms + p.splits - 1) / p.splits;
  const int t0 = split * per, t1 = min(nterms, t0 + per);
  C acc[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b] = czero<C>();

  for (int term = t0; term < t1; ++term) {
    bool colterm = term < ncol;
    int K = colterm ? I + 1 + term : term - ncol;
    __syncthreads();
    if (colterm) {
      load_tile(sA, T, ld, I * NB, K * NB, n);  // T_IK
      load_tile(sB, L, ld, K * NB, J * NB, n);  // L_KJ
    } else {
      load_tile(sA, L, ld, I * NB, K * NB, n);  // L_IK
      load_tile(sB, T, ld, K * NB, J * NB, n);  // T_KJ
    }
    __syncthreads();
    C part[2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) part[a][b] = czero<C>();
#pragma unroll 8
    for (int k = 0; k < NB; ++k) {
      C a0 = sA[(2 * ty) * (NB + 1) + k], a1 = sA[(2 * ty + 1) * (NB + 1) + k];
      C b0 = sB[k * (NB + 1) + 2 * tx], b1 = sB[k * (NB + 1) + 2 * tx + 1];
      cfma(part[0][0], a0, b0);
      cfma(part[0][1], a0, b1);
      cfma(part[1][0], a1, b0);
      cfma(part[1][1], a1, b1);
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        if (colterm) {
          acc[a][b].x -= part[a][b].x;
          acc[a][b].y -= part[a][b].y;
        } else {
          acc[a][b].x += part[a][b].x;
          acc[a][b].y += part[a][b].y;
        }
      }
  }

  const int tiles = p.level + 1;
  if (p.splits > 1) {
    // publish the partial, last CTA of this tile reduces in split order
    C* mine = ws + ((size_t)split * tiles + J) * NB * NB;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) mine[(2 * ty + a) * NB + 2 * tx + b] = acc[a][b];
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      int prev = atomicAdd(&counters[J], 1);
      s_last = (prev == p.splits - 1);
      if (s_last) counters[J] = 0;  // ready for the next level / call
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        C s = czero<C>();
        for (int q = 0; q < p.splits; ++q) {
          C v = ws[((size_t)q * tiles + J) * NB * NB + (2 * ty + a) * NB + 2 * tx + b];
          s.x += v.x;
          s.y += v.y;
        }
        acc[a][b] = s;
      }
  }

  // ---- tile solve: T_II X - X T_JJ = R,  R = -E_IJ + acc
  C* sT2 = sA;                 // T_II
  C* sT1 = sB;                 // T_JJ
  C* sX = sB + NB * (NB + 1);  // X
  __syncthreads();
  load_tile(sT2, T, ld, I * NB, I * NB, n);
  load_tile(sT1, T, ld, J * NB, J * NB, n);
  if (tid == 0) s_clip = 0;
  for (int idx = tid; idx < NB * NB; idx += NT) sX[(idx / NB) * (NB + 1) + idx % NB] = czero<C>();
  const bool diag = (I == J);
  C r[2][2];
  int stepv[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      int i = 2 * ty + a, j = 2 * tx + b;
      int gi = I * NB + i, gj = J * NB + j;
      bool valid = gi < n && gj < n && (!diag || i > j);
      C e = valid ? E[(size_t)gi * ld + gj] : czero<C>();
      r[a][b].x = acc[a][b].x - e.x;
      r[a][b].y = acc[a][b].y - e.y;
      stepv[a][b] = valid ? (NB - 1 - i) + j : -1;
    }
  __syncthreads();
  const int nsteps = diag ? NB - 1 : 2 * NB - 1;
  for (int s = 0; s < nsteps; ++s) {
    // finalise the entries of anti-diagonal s
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
        if (stepv[a][b] == s) {
          int i = 2 * ty + a, j = 2 * tx + b;
          C t2 = sT2[i * (NB + 1) + i], t1 = sT1[j * (NB + 1) + j];
          C piv;
          piv.x = t2.x - t1.x;
          piv.y = t2.y - t1.y;
          C x = cdiv(r[a][b], piv);
          if (clip > 0 && sqrt(x.x * x.x + x.y * x.y) > clip) {
            x = czero<C>();
            atomicAdd(&s_clip, 1u);
          }
          sX[i * (NB + 1) + j] = x;
        }
    __syncthreads();
    // fold the freshly final neighbours into the open entries
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
        if (stepv[a][b] > s) {
          int i = 2 * ty + a, j = 2 * tx + b;
          int k = NB - 1 - s + j;  // column neighbour (k, j), k > i
          if (k > i && k < NB) cfms(r[a][b], sT2[i * (NB + 1) + k], sX[k * (NB + 1) + j]);
          int k2 = s - (NB - 1 - i);  // row neighbour (i, k2), k2 < j
          if (k2 >= 0 && k2 < j) cfma(r[a][b], sX[i * (NB + 1) + k2], sT1[k2 * (NB + 1) + j]);
        }
  }
  __syncthreads();
  for (int idx = tid; idx < NB * NB; idx += NT) {
    int i = idx / NB, j = idx % NB;
    int gi = I * NB + i, gj = J * NB + j;
    if (gi < n && gj < n) L[(size_t)gi * ld + gj] = (diag && i <= j) ? czero<C>() : sX[i * (NB + 1) + j];
  }
  if (tid == 0 && s_clip) atomicAdd(clipped, (unsigned long long)s_clip);
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

template <typename C>
int solve(int n, const C* t, const C* e, long long ld, C* l, double clip, unsigned long long* d_clipped,
          int* d_flags, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n < 0 || ld < n) return SR_EINVAL;
  if (n == 0) return SR_OK;
  const int N = (n + NB - 1) / NB;
  size_t need = sr_trisolve_workspace_bytes(n, sizeof(C) == 8 ? 1 : 0);
  if (ws_bytes < need || !ws) return SR_EINVAL;
  int* counters = (int*)ws;
  C* part = (C*)((char*)ws + 4096 * sizeof(int) * ((N + 4095) / 4096));
  SR_CUDA_CHECK(cudaMemsetAsync(counters, 0, sizeof(int) * N, st));
  SR_CUDA_CHECK(cudaMemsetAsync(l, 0, sizeof(C) * (size_t)n * ld, st));  // strictly upper tiles stay 0
  {
    dim3 b(32, 8), g(sr_ceil_div(n, 32), sr_ceil_div(n, 8));
    separation_kernel<C><<<g, b, 0, st>>>(n, t, ld, d_flags);
    SR_LAUNCH_CHECK();
  }
  const size_t smem = sizeof(C) * (3 * NB * (NB + 1));
  auto kern = trisolve_level_kernel<C>;
  static bool configured = false;
  if (!configured) {
    SR_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  const int max_ctas = SR_TRISOLVE_MAX_CTAS;
  for (int level = 0; level < N; ++level) {
    int tiles = level + 1;
    int splits = 1;
    if (level >= 4) {
      splits = max(1, min(level / 2, (2 * 148 + tiles - 1) / tiles));
      splits = min(splits, max_ctas / tiles);
      if (splits < 1) splits = 1;
    }
    LevelArgs a{n, N, level, splits, ld};
    kern<<<dim3(tiles, splits), NT, smem, st>>>(a, t, e, l, part, counters, (typename Real<C>::T)clip,
                                                d_clipped);
    SR_LAUNCH_CHECK();
  }
  return SR_OK;
}

}  // namespace

extern "C" size_t sr_trisolve_workspace_bytes(int n, int lp_is_c64) {
  const int N = (n + NB - 1) / NB;
  size_t elt = lp_is_c64 ? 8 : 16;
  return 4096 * sizeof(int) * ((N + 4095) / 4096) + (size_t)SR_TRISOLVE_MAX_CTAS * NB * NB * elt;
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

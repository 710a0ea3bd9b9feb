// Entry guards of the refinement, on the device with no host round trip per
// step:
//
//   sr_power_norm_c64   spectral_norm_estimate (/root/reference/pkg/src/ddschur/
//                       matmul.py:117-142): power iteration on M^H M from the
//                       fixed start 1 + (j mod 7) / 8, stopping when successive
//                       estimates agree to rel_tol or after max_iters; the
//                       NormTooLarge guard of newton_schulz_step
//                       (orthogonal.py:160-166).  The convergence test runs in
//                       the kernels: the host launches steps in groups and reads
//                       one flag per group (one sync for a near-unitary Q^).
//   sr_finite_flag_f64  the finiteness check of _coerce_hp (refine.py:341-350)
//                       as a flag bit, read with the next host sync.
//   sr_phase_perm_scan_f64  the O(n^2) part of _phase_permutation
//                       (refine.py:172-189): is Q a permutation pattern (one
//                       nonzero per row and column), and where.
//
// Arithmetic: the matrix is the complex64 lp downcast; the vectors and every
// sum are FP64 with fixed reduction orders (deterministic).
#include "sr_common.cuh"

namespace {

constexpr int PT = 256;
constexpr int RCH = 64;  // row chunks of the M^H u pass

struct PowerState {
  double est, prev, nw, done, iters, pad[3];
};

__device__ __forceinline__ double block_sum256(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < PT / 32; ++i) s += sh[i];
  return s;  // thread 0
}

// v = (1 + (j mod 7) / 8) / ||.||  (the reference's start vector)
__global__ void power_init_kernel(int n, double2* v, PowerState* st) {
  __shared__ double sh[PT / 32];
  double s = 0.0;
  for (int j = threadIdx.x; j < n; j += PT) {
    const double x = 1.0 + (double)(j % 7) / 8.0;
    s += x * x;
  }
  s = block_sum256(s, sh);
  __shared__ double inv;
  if (threadIdx.x == 0) inv = 1.0 / sqrt(s);
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += PT) v[j] = make_double2((1.0 + (double)(j % 7) / 8.0) * inv, 0.0);
  if (threadIdx.x == 0) *st = PowerState{0.0, 0.0, 0.0, 0.0, 0.0, {0, 0, 0}};
}

// u = M v: one warp per row (coalesced along the row)
__global__ void power_mv_kernel(int n, const float2* __restrict__ m, long long ld, const double2* __restrict__ v,
                                double2* __restrict__ u, const PowerState* st) {
  if (st->done != 0.0) return;
  const int row = (blockIdx.x * PT + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n) return;
  double ar = 0.0, ai = 0.0;
  const float2* r = m + (size_t)row * ld;
  for (int j = lane; j < n; j += 32) {
    const float2 x = r[j];
    const double2 y = v[j];
    ar = fma((double)x.x, y.x, fma(-(double)x.y, y.y, ar));
    ai = fma((double)x.x, y.y, fma((double)x.y, y.x, ai));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ar += __shfl_xor_sync(0xffffffffu, ar, o);
    ai += __shfl_xor_sync(0xffffffffu, ai, o);
  }
  if (lane == 0) u[row] = make_double2(ar, ai);
}

// w_part[c][j] = sum_{i in chunk c} conj(M_ij) u_i  (threads along j: coalesced)
__global__ void power_mhv_kernel(int n, const float2* __restrict__ m, long long ld, const double2* __restrict__ u,
                                 double2* __restrict__ wp, const PowerState* st) {
  if (st->done != 0.0) return;
  const int j = blockIdx.x * PT + threadIdx.x;
  const int c = blockIdx.y;
  const int rows = (n + RCH - 1) / RCH;
  const int i0 = c * rows, i1 = min(n, i0 + rows);
  if (j >= n) return;
  double ar = 0.0, ai = 0.0;
  for (int i = i0; i < i1; ++i) {
    const float2 x = m[(size_t)i * ld + j];
    const double2 y = u[i];
    ar = fma((double)x.x, y.x, fma((double)x.y, y.y, ar));   // conj(x) y
    ai = fma((double)x.x, y.y, fma(-(double)x.y, y.x, ai));
  }
  wp[(size_t)c * n + j] = make_double2(ar, ai);
}

// w = sum of the chunks (fixed order), ||u||, ||w||, v = w / ||w||, the
// convergence test (one block: n is at most a few times 10^4)
__global__ void power_finish_kernel(int n, double2* __restrict__ v, const double2* __restrict__ u,
                                    double2* __restrict__ wp, double rel_tol, PowerState* st) {
  if (st->done != 0.0) return;
  __shared__ double sh[PT / 32];
  __shared__ double s_est, s_nw;
  double su = 0.0, sw = 0.0;
  for (int j = threadIdx.x; j < n; j += PT) {
    const double2 x = u[j];
    su += x.x * x.x + x.y * x.y;
    double wr = 0.0, wi = 0.0;
    for (int c = 0; c < RCH; ++c) {
      const double2 y = wp[(size_t)c * n + j];
      wr += y.x;
      wi += y.y;
    }
    wp[j] = make_double2(wr, wi);  // chunk 0's slot holds w (every chunk of column j read above)
    sw += wr * wr + wi * wi;
  }
  su = block_sum256(su, sh);
  sw = block_sum256(sw, sh);
  if (threadIdx.x == 0) {
    s_est = sqrt(su);
    s_nw = sqrt(sw);
  }
  __syncthreads();
  const double est = s_est, nw = s_nw;
  if (est == 0.0 || nw == 0.0) {  // matmul.py:131-137: return est (0 when u vanishes)
    if (threadIdx.x == 0) {
      st->est = est;
      st->done = 1.0;
      st->iters += 1.0;
    }
    return;
  }
  const double inv = 1.0 / nw;
  for (int j = threadIdx.x; j < n; j += PT) {
    const double2 y = wp[j];
    v[j] = make_double2(y.x * inv, y.y * inv);
  }
  if (threadIdx.x == 0) {
    st->est = est;
    st->iters += 1.0;
    if (fabs(est - st->prev) <= rel_tol * est) st->done = 1.0;
    st->prev = est;
  }
}

__global__ void finite_flag_kernel(int m, int n, const double* __restrict__ re, const double* __restrict__ im,
                                   long long ld, int* flags, int bit) {
  bool bad = false;
  for (GridIdx g(m, n); g.ok(); g.next()) {
    const long long o = (long long)g.i * ld + g.j;
    bad = bad || !isfinite(re[o]) || (im && !isfinite(im[o]));
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, bit);
}

// counts[j] += nonzeros of column j in row chunk blockIdx.y (and row_of_col[j]
// its row; read only when the column's total is one): threads along the
// columns (coalesced), one atomic per thread and chunk
__global__ void perm_cols_kernel(int n, const double* __restrict__ re, const double* __restrict__ im, long long ld,
                                 int* counts, int* row_of_col) {
  const int j = blockIdx.x * PT + threadIdx.x;
  if (j >= n) return;
  const int rows = (n + RCH - 1) / RCH;
  const int i0 = blockIdx.y * rows, i1 = min(n, i0 + rows);
  int c = 0, r = -1;
  for (int i = i0; i < i1; ++i) {
    const bool nz = re[(size_t)i * ld + j] != 0.0 || (im && im[(size_t)i * ld + j] != 0.0);
    if (nz) {
      ++c;
      r = i;
    }
  }
  if (c) {
    atomicAdd(&counts[j], c);
    row_of_col[j] = r;
  }
}

// counts[n + i] = nonzeros of row i: one warp per row
__global__ void perm_rows_kernel(int n, const double* __restrict__ re, const double* __restrict__ im, long long ld,
                                 int* counts) {
  const int row = (blockIdx.x * PT + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n) return;
  int c = 0;
  for (int j0 = 0; j0 < n; j0 += 32) {
    const int j = j0 + lane;
    const bool nz = j < n && (re[(size_t)row * ld + j] != 0.0 || (im && im[(size_t)row * ld + j] != 0.0));
    c += __popc(__ballot_sync(0xffffffffu, nz));
  }
  if (lane == 0) counts[n + row] = c;
}

__global__ void perm_status_kernel(int n, const int* counts, int* status) {
  bool bad = false;
  for (int k = threadIdx.x; k < 2 * n; k += PT) bad = bad || counts[k] != 1;
  const bool any_bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) *status = any_bad ? 0 : 1;
}

}  // namespace

extern "C" size_t sr_power_norm_workspace_bytes(int n) {
  return sizeof(PowerState) + (size_t)(2 + RCH) * (n > 0 ? n : 1) * sizeof(double2) + 256;
}

// Launch up to `steps` power-iteration steps (a group); `first` starts from
// the fixed vector.  st_out (host-visible through a later copy): PowerState
// {est, prev, nw, done, iters}.  The caller reads `done` after each group.
extern "C" int sr_power_norm_c64(int n, const void* m, long long ld, int first, int steps, double rel_tol, void* ws,
                                 size_t ws_bytes, void* stream) {
  if (n <= 0 || ld < n || steps < 1 || !ws || ws_bytes < sr_power_norm_workspace_bytes(n)) return SR_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  PowerState* st = (PowerState*)ws;
  double2* v = (double2*)((char*)ws + sizeof(PowerState));
  double2* u = v + n;
  double2* wp = u + n;
  if (first) {
    power_init_kernel<<<1, PT, 0, s>>>(n, v, st);
    SR_LAUNCH_CHECK();
  }
  const float2* M = (const float2*)m;
  for (int k = 0; k < steps; ++k) {
    power_mv_kernel<<<sr_ceil_div((long long)n * 32, PT), PT, 0, s>>>(n, M, ld, v, u, st);
    SR_LAUNCH_CHECK();
    power_mhv_kernel<<<dim3(sr_ceil_div(n, PT), RCH), PT, 0, s>>>(n, M, ld, u, wp, st);
    SR_LAUNCH_CHECK();
    power_finish_kernel<<<1, PT, 0, s>>>(n, v, u, wp, rel_tol, st);
    SR_LAUNCH_CHECK();
  }
  return SR_OK;
}

extern "C" int sr_finite_flag_f64(int m, int n, const double* re, const double* im, long long ld, int* d_flags,
                                  int bit, void* stream) {
  if (m < 0 || n < 0 || ld < n || !d_flags) return SR_EINVAL;
  if ((long long)m * n == 0) return SR_OK;
  const long long blocks = ((long long)m * n + PT - 1) / PT;
  finite_flag_kernel<<<(int)(blocks < 148 * 8 ? blocks : 148 * 8), PT, 0, (cudaStream_t)stream>>>(m, n, re, im, ld,
                                                                                                   d_flags, bit);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" size_t sr_phase_perm_workspace_bytes(int n) { return (size_t)3 * (n > 0 ? n : 1) * sizeof(int) + 256; }

// d_status = 1 when every row and column of Q holds exactly one nonzero (then
// row_of_col[j] is the row of column j's nonzero), else 0.
extern "C" int sr_phase_perm_scan_f64(int n, const double* re, const double* im, long long ld, int* row_of_col,
                                      int* d_status, void* ws, size_t ws_bytes, void* stream) {
  if (n <= 0 || ld < n || !ws || ws_bytes < sr_phase_perm_workspace_bytes(n)) return SR_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  int* counts = (int*)ws;
  SR_CUDA_CHECK(cudaMemsetAsync(counts, 0, (size_t)n * sizeof(int), s));
  perm_cols_kernel<<<dim3(sr_ceil_div(n, PT), RCH), PT, 0, s>>>(n, re, im, ld, counts, row_of_col);
  SR_LAUNCH_CHECK();
  perm_rows_kernel<<<sr_ceil_div((long long)n * 32, PT), PT, 0, s>>>(n, re, im, ld, counts);
  SR_LAUNCH_CHECK();
  perm_status_kernel<<<1, PT, 0, s>>>(n, counts, d_status);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

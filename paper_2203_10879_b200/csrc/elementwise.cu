// HBM-bound passes of the refinement loop: split + downcast + norms, Sigma
// assembly, skew correction, downcasts.  Every kernel is one coalesced pass
// (row-major, consecutive threads on consecutive columns) with grid-stride
// loops sized to a multiple of the 148 SMs.  Norms use a fixed two-level
// reduction (per-block partials in a fixed slot, then one block sums the
// slots in index order), so a value is bit-reproducible for a given n.
#include "sr_common.cuh"

namespace {

constexpr int RT = 256;                // threads per block
constexpr int RBLOCKS = 148 * 4;       // reduction grid (fixed: deterministic)

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double warp_part[RT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) warp_part[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < RT / 32; ++i) s += warp_part[i];
  return s;  // valid on thread 0
}

// Last block to finish reduces the partials in slot order and writes sqrt.
__device__ __forceinline__ void finish_norm(double mine, double* partials, unsigned int* counter, double* out,
                                            bool squared = false) {
  __shared__ bool last;
  double s = block_sum(mine);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = s;
    __threadfence();
    unsigned int prev = atomicAdd(counter, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double v = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += RT) v += partials[i];
  double tot = block_sum(v);
  if (threadIdx.x == 0) {
    *out = squared ? tot : sqrt(tot);
    *counter = 0u;
  }
}

struct RedWs {
  double* partials;
  unsigned int* counter;
};
inline RedWs red_ws(void* ws) {
  RedWs r;
  r.counter = (unsigned int*)ws;
  r.partials = (double*)((char*)ws + 256);
  return r;
}

// rows x cols block whose first column is global column col0 (the sharded
// driver's column block; the whole matrix: col0 = 0, cols = rows); squared:
// write sum |E|^2 instead of ||E||_F (partials of a cross-rank sum)
__global__ void split_lp_kernel(int rows, int cols, int col0, const double* __restrict__ tr,
                                const double* __restrict__ ti, long long ldt, float2* __restrict__ t_lp,
                                float2* __restrict__ e_lp, long long ld_lp, double* partials, unsigned int* counter,
                                double* out, int squared) {
  double acc = 0.0;
    for (GridIdx g(rows, cols); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    double re = tr[(size_t)i * ldt + j], im = ti[(size_t)i * ldt + j];
    float2 v = make_float2((float)re, (float)im);
    float2 z = make_float2(0.f, 0.f);
    if (i > j + col0) {
      acc += re * re + im * im;
      e_lp[(size_t)i * ld_lp + j] = v;
      t_lp[(size_t)i * ld_lp + j] = z;
    } else {
      e_lp[(size_t)i * ld_lp + j] = z;
      t_lp[(size_t)i * ld_lp + j] = v;
    }
  }
  finish_norm(acc, partials, counter, out, squared != 0);
}

__global__ void fro_norm_kernel(int m, int n, const double* __restrict__ re, const double* __restrict__ im,
                                long long ld, double* partials, unsigned int* counter, double* out) {
  double acc = 0.0;
    for (GridIdx g(m, n); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    double a = re[(size_t)i * ld + j];
    acc += a * a;
    if (im) {
      double b = im[(size_t)i * ld + j];
      acc += b * b;
    }
  }
  finish_norm(acc, partials, counter, out);
}

// ||striu(X)||_F (strict upper triangle): with the split kernel's ||stril||
// it gives the full off-diagonal defect of the Hermitian variant
// (refine.py:130-131, symmetric=True)
__global__ void striu_norm_kernel(int n, const double* __restrict__ re, const double* __restrict__ im, long long ld,
                                  double* partials, unsigned int* counter, double* out) {
  double acc = 0.0;
    for (GridIdx g(n, n); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    if (j > i) {
      const double a = re[(size_t)i * ld + j], b = im ? im[(size_t)i * ld + j] : 0.0;
      acc += a * a + b * b;
    }
  }
  finish_norm(acc, partials, counter, out);
}

// Hermitian variant's solve (_solve_diagonal_correction, refine.py:138-159):
// l_ij = -e_ij / (t_ii - t_jj) on the strict lower part, 0 elsewhere; a zero
// separation sets SR_FLAG_SEPARATION, |l| > clip is zeroed and counted, a
// non-finite quotient sets SR_FLAG_NONFINITE.
template <typename C, typename R>
__global__ void diag_correction_kernel(int n, const C* __restrict__ t, const C* __restrict__ e, long long ld,
                                       C* __restrict__ l, R clip, unsigned long long* clipped, int* flags) {
  unsigned int nclip = 0;
  bool sep = false, bad = false;
    for (GridIdx g(n, n); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    C v;
    v.x = 0;
    v.y = 0;
    if (i > j) {
      const C ti = t[(size_t)i * ld + i], tj = t[(size_t)j * ld + j], ev = e[(size_t)i * ld + j];
      C d;
      d.x = ti.x - tj.x;
      d.y = ti.y - tj.y;
      if (d.x == 0 && d.y == 0) sep = true;
      C me;
      me.x = -ev.x;
      me.y = -ev.y;
      v = cdiv(me, d);
      if (clip > 0 && sqrt(v.x * v.x + v.y * v.y) > clip) {
        v.x = 0;
        v.y = 0;
        ++nclip;
      }
      if (!isfinite(v.x) || !isfinite(v.y)) bad = true;
    }
    l[(size_t)i * ld + j] = v;
  }
  if (sep) atomicOr(flags, SR_FLAG_SEPARATION);
  if (bad) atomicOr(flags, SR_FLAG_NONFINITE);
  if (nclip) atomicAdd(clipped, (unsigned long long)nclip);
}

__global__ void downcast_kernel(int m, int n, const double* __restrict__ re, const double* __restrict__ im,
                                long long ld, float2* __restrict__ out, long long ldo) {
    for (GridIdx g(m, n); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    out[(size_t)i * ldo + j] = make_float2((float)re[(size_t)i * ld + j], (float)im[(size_t)i * ld + j]);
  }
}

__global__ void skew_kernel(int n, const float2* __restrict__ l, long long ld, float2* __restrict__ w, int* flags,
                            double* partials, unsigned int* counter, double* out) {
  double acc = 0.0;
  bool bad = false;
    for (GridIdx g(n, n); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    float2 a = l[(size_t)i * ld + j], b = l[(size_t)j * ld + i];
    // w = l - conj(l^T), in lp (complex64) like l - l.conj().T at refine.py:296
    float2 v = make_float2(a.x - b.x, a.y + b.y);
    w[(size_t)i * ld + j] = v;
    if (!isfinite(a.x) || !isfinite(a.y)) bad = true;
    acc += (double)v.x * v.x + (double)v.y * v.y;
  }
  if (bad) atomicOr(flags, SR_FLAG_NONFINITE);
  finish_norm(acc, partials, counter, out);
}

__global__ void sigma_merged_kernel(int rows, int n, const float2* __restrict__ w, const double* __restrict__ yr,
                                    const double* __restrict__ yi, long long ldy, const float2* __restrict__ yw,
                                    const float2* __restrict__ w2, const float2* __restrict__ w3,
                                    const float2* __restrict__ w2y, const float2* __restrict__ w2yw, long long ldl,
                                    double* __restrict__ sr, double* __restrict__ si, long long lds, double eye) {
    for (GridIdx g(rows, n); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    size_t o = (size_t)i * ldl + j;
    float2 wv = w[o];
    // ((((2I + 2W) - Y) - YW) + W^2) + W^3, left to right (orthogonal.py:191-195)
    double re = (i == j ? eye : 0.0) + 2.0 * (double)wv.x;
    double im = 2.0 * (double)wv.y;
    re = re - yr[(size_t)i * ldy + j];
    im = im - yi[(size_t)i * ldy + j];
    if (yw) {  // null yw (fused form only): X W below the update's error budget
      float2 a = yw[o];
      re = re - (double)a.x;
      im = im - (double)a.y;
    }
    if (w2) {  // null w2 / w3: the fused form, yw already holds YW - W^2 - W^3
      float2 b = w2[o], c = w3[o];
      re = re + (double)b.x;
      im = im + (double)b.y;
      re = re + (double)c.x;
      im = im + (double)c.y;
    }
    if (w2y) {  // restore_full_sigma (orthogonal.py:196-200)
      float2 d = w2y[o], e = w2yw[o];
      re = re + (double)d.x;
      im = im + (double)d.y;
      re = re + (double)e.x;
      im = im + (double)e.y;
    }
    sr[(size_t)i * lds + j] = re;
    si[(size_t)i * lds + j] = im;
  }
}

__global__ void sigma_ns_kernel(int n, const double* __restrict__ gr, const double* __restrict__ gi, long long ldg,
                                double* __restrict__ sr, double* __restrict__ si, long long lds) {
    for (GridIdx g(n, n); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    sr[(size_t)i * lds + j] = (i == j ? 3.0 : 0.0) - gr[(size_t)i * ldg + j];
    si[(size_t)i * lds + j] = -gi[(size_t)i * ldg + j];
  }
}

__global__ void triu_kernel(int n, double* re, double* im, long long ld) {
    for (GridIdx g(n, n); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    if (i > j) {
      re[(size_t)i * ld + j] = 0.0;
      im[(size_t)i * ld + j] = 0.0;
    }
  }
}

// ---- dd mode (hp = double-double planes, lp = complex128) ---------------------

// T^ (hi planes) -> lp T (upper incl. diagonal) and lp E (strictly lower),
// complex128; ||E||_F of the hp values (the lo parts change it by < 2^-52).
__global__ void split_lp_c128_kernel(int n, const double* __restrict__ tr, const double* __restrict__ ti,
                                     long long ldt, double2* __restrict__ t_lp, double2* __restrict__ e_lp,
                                     long long ld_lp, double* partials, unsigned int* counter, double* out) {
  double acc = 0.0;
    for (GridIdx g(n, n); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    const double re = tr[(size_t)i * ldt + j], im = ti[(size_t)i * ldt + j];
    const double2 v = make_double2(re, im), z = make_double2(0.0, 0.0);
    if (i > j) {
      acc += re * re + im * im;
      e_lp[(size_t)i * ld_lp + j] = v;
      t_lp[(size_t)i * ld_lp + j] = z;
    } else {
      e_lp[(size_t)i * ld_lp + j] = z;
      t_lp[(size_t)i * ld_lp + j] = v;
    }
  }
  finish_norm(acc, partials, counter, out);
}

__global__ void skew_c128_kernel(int n, const double2* __restrict__ l, long long ld, double2* __restrict__ w,
                                 int* flags, double* partials, unsigned int* counter, double* out) {
  double acc = 0.0;
  bool bad = false;
    for (GridIdx g(n, n); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    const double2 a = l[(size_t)i * ld + j], b = l[(size_t)j * ld + i];
    const double2 v = make_double2(a.x - b.x, a.y + b.y);  // l - conj(l^T), refine.py:296
    w[(size_t)i * ld + j] = v;
    if (!isfinite(a.x) || !isfinite(a.y)) bad = true;
    acc += v.x * v.x + v.y * v.y;
  }
  if (bad) atomicOr(flags, SR_FLAG_NONFINITE);
  finish_norm(acc, partials, counter, out);
}

__global__ void pack_c128_kernel(int m, int n, const double* __restrict__ re, const double* __restrict__ im,
                                 long long ld, double2* __restrict__ out, long long ldo) {
    for (GridIdx g(m, n); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    out[(size_t)i * ldo + j] = make_double2(re[(size_t)i * ld + j], im[(size_t)i * ld + j]);
  }
}

__device__ __forceinline__ void ew_two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
__device__ __forceinline__ void ew_quick_two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  e = b - (s - a);
}
// accurate dd sum (dd.py:96-104): (ah, al) + (bh, bl)
__device__ __forceinline__ void ew_dd_add(double& ah, double& al, double bh, double bl) {
  double s1, s2, t1, t2;
  ew_two_sum(ah, bh, s1, s2);
  ew_two_sum(al, bl, t1, t2);
  s2 += t1;
  ew_quick_two_sum(s1, s2, s1, s2);
  s2 += t2;
  ew_quick_two_sum(s1, s2, ah, al);
}

// Sigma' = S - 2I of merged_update in double-double, summed left to right as
// the reference does (orthogonal.py:191-200); the binary64 terms are exact
// embeddings: ((((2W) - Y) - YW) + W^2) + W^3 [+ W^2 Y + W^2 Y W] (+ 2I when
// with_identity).
__global__ void sigma_merged_dd_kernel(int n, const double2* __restrict__ w, const double* __restrict__ yrh,
                                       const double* __restrict__ yih, const double* __restrict__ yrl,
                                       const double* __restrict__ yil, long long ldy, const double2* __restrict__ yw,
                                       const double2* __restrict__ w2, const double2* __restrict__ w3,
                                       const double2* __restrict__ w2y, const double2* __restrict__ w2yw,
                                       long long ldl, double* __restrict__ srh, double* __restrict__ sih,
                                       double* __restrict__ srl, double* __restrict__ sil, long long lds,
                                       double eye) {
    for (GridIdx g(n, n); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    const size_t o = (size_t)i * ldl + j, oy = (size_t)i * ldy + j;
    const double2 wv = w[o];
    double rh = (i == j ? eye : 0.0), rl = 0.0, ih = 0.0, il = 0.0;
    ew_dd_add(rh, rl, 2.0 * wv.x, 0.0);
    ew_dd_add(ih, il, 2.0 * wv.y, 0.0);
    ew_dd_add(rh, rl, -yrh[oy], -yrl[oy]);
    ew_dd_add(ih, il, -yih[oy], -yil[oy]);
    const double2 a = yw[o], b = w2[o], c = w3[o];
    ew_dd_add(rh, rl, -a.x, 0.0);
    ew_dd_add(ih, il, -a.y, 0.0);
    ew_dd_add(rh, rl, b.x, 0.0);
    ew_dd_add(ih, il, b.y, 0.0);
    ew_dd_add(rh, rl, c.x, 0.0);
    ew_dd_add(ih, il, c.y, 0.0);
    if (w2y) {  // restore_full_sigma (orthogonal.py:196-200)
      const double2 d = w2y[o], e = w2yw[o];
      ew_dd_add(rh, rl, d.x, 0.0);
      ew_dd_add(ih, il, d.y, 0.0);
      ew_dd_add(rh, rl, e.x, 0.0);
      ew_dd_add(ih, il, e.y, 0.0);
    }
    const size_t os = (size_t)i * lds + j;
    srh[os] = rh;
    srl[os] = rl;
    sih[os] = ih;
    sil[os] = il;
  }
}

inline int ew_grid(long long total) {
  long long b = (total + RT - 1) / RT;
  return (int)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

}  // namespace

extern "C" size_t sr_reduce_workspace_bytes(void) { return 256 + sizeof(double) * RBLOCKS; }

extern "C" int sr_split_lp_c64(int n, const double* that_re, const double* that_im, long long ldt, void* t_lp,
                               void* e_lp, long long ld_lp, double* d_norm_e, void* ws, size_t ws_bytes,
                               void* stream) {
  if (n < 0 || !ws || ws_bytes < sr_reduce_workspace_bytes()) return SR_EINVAL;
  RedWs r = red_ws(ws);
  split_lp_kernel<<<RBLOCKS, RT, 0, (cudaStream_t)stream>>>(n, n, 0, that_re, that_im, ldt, (float2*)t_lp,
                                                             (float2*)e_lp, ld_lp, r.partials, r.counter,
                                                             d_norm_e, 0);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_fro_norm_f64(int m, int n, const double* re, const double* im, long long ld, double* d_out,
                               void* ws, size_t ws_bytes, void* stream) {
  if (m < 0 || n < 0 || !ws || ws_bytes < sr_reduce_workspace_bytes()) return SR_EINVAL;
  RedWs r = red_ws(ws);
  fro_norm_kernel<<<RBLOCKS, RT, 0, (cudaStream_t)stream>>>(m, n, re, im, ld, r.partials, r.counter, d_out);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_striu_norm_f64(int n, const double* re, const double* im, long long ld, double* d_out, void* ws,
                                 size_t ws_bytes, void* stream) {
  if (n < 0 || !ws || ws_bytes < sr_reduce_workspace_bytes()) return SR_EINVAL;
  RedWs r = red_ws(ws);
  striu_norm_kernel<<<RBLOCKS, RT, 0, (cudaStream_t)stream>>>(n, re, im, ld, r.partials, r.counter, d_out);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_diag_correction_c64(int n, const void* t, const void* e, long long ld, void* l, float clip,
                                      unsigned long long* d_clipped, int* d_flags, void* stream) {
  if (n < 0 || ld < n) return SR_EINVAL;
  if (n == 0) return SR_OK;
  diag_correction_kernel<float2, float><<<ew_grid((long long)n * n), RT, 0, (cudaStream_t)stream>>>(
      n, (const float2*)t, (const float2*)e, ld, (float2*)l, clip, d_clipped, d_flags);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_diag_correction_c128(int n, const void* t, const void* e, long long ld, void* l, double clip,
                                       unsigned long long* d_clipped, int* d_flags, void* stream) {
  if (n < 0 || ld < n) return SR_EINVAL;
  if (n == 0) return SR_OK;
  diag_correction_kernel<double2, double><<<ew_grid((long long)n * n), RT, 0, (cudaStream_t)stream>>>(
      n, (const double2*)t, (const double2*)e, ld, (double2*)l, clip, d_clipped, d_flags);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_downcast_c64(int m, int n, const double* re, const double* im, long long ld, void* out,
                               long long ld_out, void* stream) {
  if (m < 0 || n < 0) return SR_EINVAL;
  if ((long long)m * n == 0) return SR_OK;
  downcast_kernel<<<ew_grid((long long)m * n), RT, 0, (cudaStream_t)stream>>>(m, n, re, im, ld, (float2*)out,
                                                                              ld_out);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_skew_c64(int n, const void* l, long long ld, void* w, double* d_norm_w, int* d_flags, void* ws,
                           size_t ws_bytes, void* stream) {
  if (n < 0 || !ws || ws_bytes < sr_reduce_workspace_bytes()) return SR_EINVAL;
  RedWs r = red_ws(ws);
  skew_kernel<<<RBLOCKS, RT, 0, (cudaStream_t)stream>>>(n, (const float2*)l, ld, (float2*)w, d_flags, r.partials,
                                                         r.counter, d_norm_w);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

// X = Y - W - W^2 in complex64: the A operand of the fused lp product
// X W = YW - W^2 - W^3 (one product instead of YW, W^3)
__global__ void fused_lp_operand_kernel(int n, int cols, const double* __restrict__ yr, const double* __restrict__ yi,
                                        long long ldy, const float2* __restrict__ w, const float2* __restrict__ w2,
                                        long long ldl, float2* __restrict__ x) {
    for (GridIdx g(n, cols); g.ok(); g.next()) {
    const int i = g.i, j = g.j;
    const size_t o = (size_t)i * ldl + j, oy = (size_t)i * ldy + j;
    const float2 a = w[o], b = w2 ? w2[o] : make_float2(0.f, 0.f);  // null w2: W^2 below the update's error budget
    x[o] = make_float2((float)(yr[oy] - (double)a.x - (double)b.x), (float)(yi[oy] - (double)a.y - (double)b.y));
  }
}

extern "C" int sr_fused_lp_operand_c64(int n, const double* y_re, const double* y_im, long long ldy, const void* w,
                                       const void* w2, long long ld_lp, void* x, void* stream) {
  if (n < 0 || !y_re || !y_im || !w || !x) return SR_EINVAL;
  if (n == 0) return SR_OK;
  fused_lp_operand_kernel<<<ew_grid((long long)n * n), RT, 0, (cudaStream_t)stream>>>(
      n, n, y_re, y_im, ldy, (const float2*)w, (const float2*)w2, ld_lp, (float2*)x);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

// column-block forms for the sharded driver (sharded.py): rows x cols blocks,
// the block's first column is global column col0
extern "C" int sr_split_lp_block_c64(int rows, int cols, int col0, const double* that_re, const double* that_im,
                                     long long ldt, void* t_lp, void* e_lp, long long ld_lp, double* d_sq_e,
                                     void* ws, size_t ws_bytes, void* stream) {
  if (rows < 0 || cols < 0 || col0 < 0 || !ws || ws_bytes < sr_reduce_workspace_bytes()) return SR_EINVAL;
  RedWs r = red_ws(ws);
  split_lp_kernel<<<RBLOCKS, RT, 0, (cudaStream_t)stream>>>(rows, cols, col0, that_re, that_im, ldt, (float2*)t_lp,
                                                             (float2*)e_lp, ld_lp, r.partials, r.counter, d_sq_e,
                                                             1);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_fused_lp_operand_block_c64(int rows, int cols, const double* y_re, const double* y_im,
                                             long long ldy, const void* w, const void* w2, long long ld_lp, void* x,
                                             void* stream) {
  if (rows < 0 || cols < 0 || !y_re || !y_im || !w || !x) return SR_EINVAL;
  if ((long long)rows * cols == 0) return SR_OK;
  fused_lp_operand_kernel<<<ew_grid((long long)rows * cols), RT, 0, (cudaStream_t)stream>>>(
      rows, cols, y_re, y_im, ldy, (const float2*)w, (const float2*)w2, ld_lp, (float2*)x);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_sigma_merged_f64(int n, int cols, const void* w, const double* y_re, const double* y_im,
                                   long long ldy, const void* yw, const void* w2, const void* w3, const void* w2y,
                                   const void* w2yw, long long ld_lp, double* s_re, double* s_im, long long lds,
                                   int with_identity, void* stream) {
  if (n < 0 || cols < 0 || (w2y == nullptr) != (w2yw == nullptr) || (w2 == nullptr) != (w3 == nullptr))
    return SR_EINVAL;
  if (!w2 && w2y) return SR_EINVAL;  // the fused form has no restore_full_sigma terms
  if (!yw && w2) return SR_EINVAL;   // only the fused form may drop its lp term
  if (with_identity && cols != n) return SR_EINVAL;
  if ((long long)n * cols == 0) return SR_OK;
  sigma_merged_kernel<<<ew_grid((long long)n * cols), RT, 0, (cudaStream_t)stream>>>(
      n, cols, (const float2*)w, y_re, y_im, ldy, (const float2*)yw, (const float2*)w2, (const float2*)w3,
      (const float2*)w2y, (const float2*)w2yw, ld_lp, s_re, s_im, lds, with_identity ? 2.0 : 0.0);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_sigma_ns_f64(int n, const double* g_re, const double* g_im, long long ldg, double* s_re,
                               double* s_im, long long lds, void* stream) {
  if (n < 0) return SR_EINVAL;
  if (n == 0) return SR_OK;
  sigma_ns_kernel<<<ew_grid((long long)n * n), RT, 0, (cudaStream_t)stream>>>(n, g_re, g_im, ldg, s_re, s_im, lds);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_triu_inplace_f64(int n, double* re, double* im, long long ld, void* stream) {
  if (n < 0) return SR_EINVAL;
  if (n == 0) return SR_OK;
  triu_kernel<<<ew_grid((long long)n * n), RT, 0, (cudaStream_t)stream>>>(n, re, im, ld);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_split_lp_c128(int n, const double* that_re, const double* that_im, long long ldt, void* t_lp,
                                void* e_lp, long long ld_lp, double* d_norm_e, void* ws, size_t ws_bytes,
                                void* stream) {
  if (n < 0 || !ws || ws_bytes < sr_reduce_workspace_bytes()) return SR_EINVAL;
  RedWs r = red_ws(ws);
  split_lp_c128_kernel<<<RBLOCKS, RT, 0, (cudaStream_t)stream>>>(n, that_re, that_im, ldt, (double2*)t_lp,
                                                                  (double2*)e_lp, ld_lp, r.partials, r.counter,
                                                                  d_norm_e);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_skew_c128(int n, const void* l, long long ld, void* w, double* d_norm_w, int* d_flags, void* ws,
                            size_t ws_bytes, void* stream) {
  if (n < 0 || !ws || ws_bytes < sr_reduce_workspace_bytes()) return SR_EINVAL;
  RedWs r = red_ws(ws);
  skew_c128_kernel<<<RBLOCKS, RT, 0, (cudaStream_t)stream>>>(n, (const double2*)l, ld, (double2*)w, d_flags,
                                                              r.partials, r.counter, d_norm_w);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_pack_c128(int m, int n, const double* re, const double* im, long long ld, void* out,
                            long long ld_out, void* stream) {
  if (m < 0 || n < 0) return SR_EINVAL;
  if ((long long)m * n == 0) return SR_OK;
  pack_c128_kernel<<<ew_grid((long long)m * n), RT, 0, (cudaStream_t)stream>>>(m, n, re, im, ld, (double2*)out,
                                                                               ld_out);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_sigma_merged_dd(int n, const void* w, const double* y_re_hi, const double* y_im_hi,
                                  const double* y_re_lo, const double* y_im_lo, long long ldy, const void* yw,
                                  const void* w2, const void* w3, const void* w2y, const void* w2yw, long long ld_lp,
                                  double* s_re_hi, double* s_im_hi, double* s_re_lo, double* s_im_lo, long long lds,
                                  int with_identity, void* stream) {
  if (n < 0 || (w2y == nullptr) != (w2yw == nullptr)) return SR_EINVAL;
  if (n == 0) return SR_OK;
  sigma_merged_dd_kernel<<<ew_grid((long long)n * n), RT, 0, (cudaStream_t)stream>>>(
      n, (const double2*)w, y_re_hi, y_im_hi, y_re_lo, y_im_lo, ldy, (const double2*)yw, (const double2*)w2,
      (const double2*)w3, (const double2*)w2y, (const double2*)w2yw, ld_lp, s_re_hi, s_im_hi, s_re_lo, s_im_lo,
      lds, with_identity ? 2.0 : 0.0);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

// Double-double container operations of the boundary (the reference's
// DDMatrix arithmetic and matrix-core helpers), BIT-IDENTICAL to the
// reference's numpy / numba kernels:
//
//   sr_dd_add         DDMatrix.__add__ / __sub__   ddmatrix.py:114-126 -> dd.add / dd.sub (dd.py:96-114)
//   sr_dd_scale       DDMatrix.scale(float)        ddmatrix.py:138-147 -> dd.mul_d (dd.py:127-132)
//   sr_stril_split_f64 stril_extract               ddmatrix.py:190-209 (pure masking)
//   sr_fro_norm_dd    frobenius_norm               ddmatrix.py:216-251 (dd squares, the fixed
//                                                  pairwise tree over column-major order, dd sqrt)
//
// Every product goes through __dmul_rn / every sum through __dadd_rn, so
// nvcc never contracts a*b+c into an FMA: each operation rounds exactly
// where the reference's does.  two_prod's error term is the EXACT error of
// the product in both (Dekker's split in the reference, an FMA here), so it
// is the same double.  One real plane per launch; complex matrices call twice.
#include "sr_common.cuh"

namespace {

struct dd {
  double h, l;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dadd_rn(s, -a);
  const double e = __dadd_rn(__dadd_rn(a, -__dadd_rn(s, -bb)), __dadd_rn(b, -bb));
  return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  return {s, __dadd_rn(b, -__dadd_rn(s, -a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  const double p = __dmul_rn(a, b);
  return {p, __fma_rn(a, b, -p)};  // the exact error of fl(a b) (= Dekker's, barring over/underflow)
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {  // dd.py:96-104
  dd s = two_sum(a.h, b.h);
  const dd t = two_sum(a.l, b.l);
  s.l = __dadd_rn(s.l, t.h);
  s = quick_two_sum(s.h, s.l);
  s.l = __dadd_rn(s.l, t.l);
  return quick_two_sum(s.h, s.l);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {  // dd.py:117-124
  dd p = two_prod(a.h, b.h);
  const double cross = __dadd_rn(__dmul_rn(a.h, b.l), __dmul_rn(a.l, b.h));
  p.l = __dadd_rn(p.l, __dadd_rn(cross, __dmul_rn(a.l, b.l)));
  return quick_two_sum(p.h, p.l);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {  // dd.py:127-132
  dd p = two_prod(a.h, b);
  p.l = __dadd_rn(p.l, __dmul_rn(a.l, b));
  return quick_two_sum(p.h, p.l);
}
__device__ __forceinline__ dd dd_sqrt(dd a) {  // dd.py:149-164
  if (a.h == 0.0) return {0.0, 0.0};
  if (a.h < 0.0) return {__longlong_as_double(0x7ff8000000000000ll), __longlong_as_double(0x7ff8000000000000ll)};
  const double r = __dsqrt_rn(a.h);
  const dd s = two_prod(r, r);
  const dd d = dd_add(a, {-s.h, -s.l});  // sub(a, s) == add(a, -s) bit for bit
  const double corr = __ddiv_rn(d.h, __dmul_rn(2.0, r));
  return quick_two_sum(r, corr);
}

constexpr int ET = 256;

__global__ void dd_add_kernel(int m, int n, const double* __restrict__ xh, const double* __restrict__ xl,
                              long long ldx, const double* __restrict__ yh, const double* __restrict__ yl,
                              long long ldy, double sy, double* __restrict__ zh, double* __restrict__ zl,
                              long long ldz) {
  const long long total = (long long)m * n;
  for (long long k = blockIdx.x * (long long)ET + threadIdx.x; k < total; k += (long long)gridDim.x * ET) {
    const long long i = k / n, j = k % n;
    const dd x = {xh[i * ldx + j], xl[i * ldx + j]};
    const dd y = {sy * yh[i * ldy + j], sy * yl[i * ldy + j]};  // sy = +-1: exact
    const dd z = dd_add(x, y);
    zh[i * ldz + j] = z.h;
    zl[i * ldz + j] = z.l;
  }
}

__global__ void dd_scale_kernel(int m, int n, const double* __restrict__ xh, const double* __restrict__ xl,
                                long long ldx, double s, double* __restrict__ zh, double* __restrict__ zl,
                                long long ldz) {
  const long long total = (long long)m * n;
  for (long long k = blockIdx.x * (long long)ET + threadIdx.x; k < total; k += (long long)gridDim.x * ET) {
    const long long i = k / n, j = k % n;
    const dd z = dd_mul_d({xh[i * ldx + j], xl[i * ldx + j]}, s);
    zh[i * ldz + j] = z.h;
    zl[i * ldz + j] = z.l;
  }
}

__global__ void stril_split_kernel(int m, int n, const double* __restrict__ src, long long lds,
                                   double* __restrict__ e, long long lde, double* __restrict__ t, long long ldt) {
  const long long total = (long long)m * n;
  for (long long k = blockIdx.x * (long long)ET + threadIdx.x; k < total; k += (long long)gridDim.x * ET) {
    const long long i = k / n, j = k % n;
    const double v = src[i * lds + j];
    const bool low = i > j;
    if (e) e[i * lde + j] = low ? v : 0.0;
    if (t) t[i * ldt + j] = low ? 0.0 : v;
  }
}

// One level group of the reference's pairwise tree (_pairwise_dd_sum,
// ddmatrix.py:216-226): aligned chunks of CH = 2^11 consecutive entries are
// reduced exactly as the global tree reduces them (pairs (2i, 2i+1), an odd
// trailing entry carried), so chaining launches reproduces the global tree.
constexpr int CH = 2048;

// leaf pass: entry f (column-major index over rows x cols) -> |z_f|^2 in dd,
// v_mul(re)+v_mul(im) then v_add (ddmatrix.py:240-243)
__device__ __forceinline__ dd square_entry(long long f, int rows, const double* rh, const double* rl,
                                           const double* ih, const double* il, long long ld) {
  const long long r = f % rows, c = f / rows;
  const long long o = r * ld + c;
  const dd re = {rh[o], rl ? rl[o] : 0.0};
  const dd im = {ih ? ih[o] : 0.0, il ? il[o] : 0.0};
  return dd_add(dd_mul(re, re), dd_mul(im, im));
}

__global__ void __launch_bounds__(1024) tree_kernel(long long len, int leaf, int rows, const double* rh,
                                                    const double* rl, const double* ih, const double* il,
                                                    long long ld, const double* in_h, const double* in_l,
                                                    double* out_h, double* out_l) {
  // ping-pong buffers: the first level halves the chunk, so the second buffer needs CH / 2
  __shared__ double ah[CH], al[CH], bh[CH / 2], bl[CH / 2];
  double* sh[2] = {ah, bh};
  double* sl[2] = {al, bl};
  const long long base = (long long)blockIdx.x * CH;
  int c = (int)(len - base < CH ? len - base : CH);
  for (int i = threadIdx.x; i < c; i += blockDim.x) {
    dd v;
    if (leaf) v = square_entry(base + i, rows, rh, rl, ih, il, ld);
    else v = {in_h[base + i], in_l[base + i]};
    sh[0][i] = v.h;
    sl[0][i] = v.l;
  }
  __syncthreads();
  int cur = 0;
  while (c > 1) {
    const int m = c >> 1;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      const dd s = dd_add({sh[cur][2 * i], sl[cur][2 * i]}, {sh[cur][2 * i + 1], sl[cur][2 * i + 1]});
      sh[cur ^ 1][i] = s.h;
      sl[cur ^ 1][i] = s.l;
    }
    if ((c & 1) && threadIdx.x == 0) {
      sh[cur ^ 1][m] = sh[cur][c - 1];
      sl[cur ^ 1][m] = sl[cur][c - 1];
    }
    c = m + (c & 1);
    cur ^= 1;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out_h[blockIdx.x] = sh[cur][0];
    out_l[blockIdx.x] = sl[cur][0];
  }
}

__global__ void sqrt_kernel(const double* h, const double* l, double* out) {
  const dd r = dd_sqrt({h[0], l[0]});
  out[0] = r.h;
  out[1] = r.l;
}

inline int grid_for(long long total) {
  const long long b = (total + ET - 1) / ET;
  return (int)(b < 148 * 8 ? (b > 0 ? b : 1) : 148 * 8);
}

}  // namespace

extern "C" int sr_dd_add(int m, int n, const double* xh, const double* xl, long long ldx, const double* yh,
                         const double* yl, long long ldy, int negate_y, double* zh, double* zl, long long ldz,
                         void* stream) {
  if (m < 0 || n < 0 || ldx < n || ldy < n || ldz < n) return SR_EINVAL;
  if ((long long)m * n == 0) return SR_OK;
  dd_add_kernel<<<grid_for((long long)m * n), ET, 0, (cudaStream_t)stream>>>(m, n, xh, xl, ldx, yh, yl, ldy,
                                                                           negate_y ? -1.0 : 1.0, zh, zl, ldz);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_dd_scale(int m, int n, const double* xh, const double* xl, long long ldx, double s, double* zh,
                           double* zl, long long ldz, void* stream) {
  if (m < 0 || n < 0 || ldx < n || ldz < n) return SR_EINVAL;
  if ((long long)m * n == 0) return SR_OK;
  dd_scale_kernel<<<grid_for((long long)m * n), ET, 0, (cudaStream_t)stream>>>(m, n, xh, xl, ldx, s, zh, zl, ldz);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_stril_split_f64(int m, int n, const double* src, long long lds, double* e, long long lde,
                                  double* t, long long ldt, void* stream) {
  if (m < 0 || n < 0 || lds < n || (e && lde < n) || (t && ldt < n)) return SR_EINVAL;
  if ((long long)m * n == 0) return SR_OK;
  stril_split_kernel<<<grid_for((long long)m * n), ET, 0, (cudaStream_t)stream>>>(m, n, src, lds, e, lde, t, ldt);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" size_t sr_fro_norm_dd_workspace_bytes(long long entries) {
  // two ping-pong partial arrays (hi, lo) of ceil(entries / 2048) doubles each
  const long long p = (entries + CH - 1) / CH + 1;
  return (size_t)(4 * p) * sizeof(double) + 256;
}

extern "C" int sr_fro_norm_dd(int rows, int cols, const double* rh, const double* rl, const double* ih,
                              const double* il, long long ld, double* d_out, void* ws, size_t ws_bytes,
                              void* stream) {
  const long long len = (long long)rows * cols;
  if (rows < 0 || cols < 0 || ld < cols || !d_out) return SR_EINVAL;
  if (!ws || ws_bytes < sr_fro_norm_dd_workspace_bytes(len)) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (len == 0) {
    SR_CUDA_CHECK(cudaMemsetAsync(d_out, 0, 2 * sizeof(double), st));
    return SR_OK;
  }
  const long long p = (len + CH - 1) / CH + 1;
  double* bufs[2][2] = {{(double*)ws, (double*)ws + p}, {(double*)ws + 2 * p, (double*)ws + 3 * p}};
  long long cur_len = len;
  int which = 0;
  bool leaf = true;
  do {
    const long long blocks = (cur_len + CH - 1) / CH;
    const double* in_h = leaf ? nullptr : bufs[which ^ 1][0];
    const double* in_l = leaf ? nullptr : bufs[which ^ 1][1];
    tree_kernel<<<(unsigned)blocks, 1024, 0, st>>>(cur_len, leaf ? 1 : 0, rows, rh, rl, ih, il, ld, in_h, in_l,
                                                   bufs[which][0], bufs[which][1]);
    SR_LAUNCH_CHECK();
    leaf = false;
    cur_len = blocks;
    which ^= 1;
  } while (cur_len > 1);
  sqrt_kernel<<<1, 1, 0, st>>>(bufs[which ^ 1][0], bufs[which ^ 1][1], d_out);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

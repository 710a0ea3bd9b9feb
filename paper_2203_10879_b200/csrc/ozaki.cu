// Ozaki-II emulated complex products: operand encoding and CRT decoding.
//
// An FP64 (or complex64) product C = op(A) B is evaluated exactly on
// integers (Ozaki, Uchino, Imamura — "Ozaki scheme II", CRT variant):
//   1. scale   every row of op(A) and every column of B by a power of two so
//              its largest entry is below 2^beta, round to integers A', B'
//              (for beta = 60 every entry within 2^-7 of its row / column
//              maximum is represented exactly — no quantisation at all);
//   2. encode  the residues A' mod p_l, B' mod p_l (symmetric, int8) for the
//              pairwise-coprime moduli p_1..p_r <= 256 of the plan, K-major;
//   3. multiply on the tensor cores: R_l = A'_l B'_l mod p_l (oz_gemm.cu);
//   4. decode  C' from its residues by the Chinese remainder theorem in
//              exact FP64 chunk arithmetic, then unscale:
//              C = alpha * C' * 2^-(rho_i + sigma_j) + shift * I + add_scale * X.
// Because every integer product and sum is exact, the result is independent
// of the summation order and its only error is the operand rounding of step 1
// plus one final rounding — unlike a K-long FP64 accumulation chain, whose
// noise on stril(Q^H A Q) grows like sqrt(K).
//
// This replaces, in FP64 mode, the reference's hp product
//   matmul_hp (/root/reference/pkg/src/ddschur/matmul.py:52-81) and lp product
//   matmul_lp (matmul.py:84-110); the reference ships an Ozaki-I variant for
//   dd (matmul.py:151-212) which this generalises to CRT residues on int8
//   tensor cores.
#include "sr_common.cuh"

namespace {

constexpr int MAXMOD = 32;
constexpr int MAXCHUNK = 4;

__device__ __forceinline__ void load_src(const double* re, const double* im, int c64, size_t off, double& vr,
                                         double& vi) {
  if (c64) {
    float2 v = reinterpret_cast<const float2*>(re)[off];
    vr = v.x;
    vi = v.y;
  } else {
    vr = re[off];
    vi = im ? im[off] : 0.0;
  }
}

struct EncodeParams {
  int rows_out, K, transposed, conj, layout, beta, nmod, src_c64;
  long long ld, kpitch;
  int moduli[MAXMOD];
  double inv[MAXMOD];
};

// ---- exponents: e_i with max_k |op(X)[i,k]| < 2^e_i -------------------------
__global__ void exps_direct_kernel(int rows, int cols, const double* __restrict__ re, const double* __restrict__ im,
                                   long long ld, int c64, int* __restrict__ e) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  double m = 0.0;
  for (int k = lane; k < cols; k += 32) {
    double vr, vi;
    load_src(re, im, c64, (size_t)warp * ld + k, vr, vi);
    m = fmax(m, fmax(fabs(vr), fabs(vi)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) {
    int ex = 0;
    if (m > 0.0) frexp(m, &ex);
    e[warp] = ex;
  }
}

__global__ void exps_transposed_kernel(int rows, int cols, const double* __restrict__ re,
                                       const double* __restrict__ im, long long ld, int c64, int* __restrict__ e) {
  // one thread per column j, rows split over blockDim.y partial maxima
  __shared__ double part[8][33];
  const int j = blockIdx.x * 32 + threadIdx.x;
  double m = 0.0;
  if (j < cols)
    for (int i = threadIdx.y; i < rows; i += 8) {
      double vr, vi;
      load_src(re, im, c64, (size_t)i * ld + j, vr, vi);
      m = fmax(m, fmax(fabs(vr), fabs(vi)));
    }
  part[threadIdx.y][threadIdx.x] = m;
  __syncthreads();
  if (threadIdx.y == 0 && j < cols) {
    for (int y = 1; y < 8; ++y) m = fmax(m, part[y][threadIdx.x]);
    int ex = 0;
    if (m > 0.0) frexp(m, &ex);
    e[j] = ex;
  }
}

// Symmetric residue of an integer-valued double a (|a| < 2^62) modulo p, in
// [-floor(p/2), ceil(p/2) - 1].  Two exact fma reductions: the first quotient
// estimate is within a few units, the second reduction is then exact.
__device__ __forceinline__ double res_f64(double a, double p, double inv, double hi) {
  double r = fma(-rint(a * inv), p, a);  // exact, |r| < 8p
  r = fma(-rint(r * inv), p, r);         // exact, |r| <= p/2
  if (r > hi) r -= p;
  return r;
}

// ---- encode: residue planes [nmod][planes][rows_out][kpitch] -------------------
// layout 0: A operand (re, im);  1: B operand (-im, re, im);  2: B operand (re)
constexpr int ETI = 64, ETK = 32;  // tile: 64 output rows x 32 k
__global__ void __launch_bounds__(256) encode_kernel(const __grid_constant__ EncodeParams p,
                                                     const double* __restrict__ re, const double* __restrict__ im,
                                                     const int* __restrict__ exps, int8_t* __restrict__ out) {
  __shared__ double s_re[ETI][ETK + 1];
  __shared__ double s_im[ETI][ETK + 1];
  const int i0 = blockIdx.y * ETI, k0 = blockIdx.x * ETK;
  const int tid = threadIdx.x;
  // stage the source tile as s[i_local][k_local] = op(X)[i0 + i][k0 + k]
  for (int idx = tid; idx < ETI * ETK; idx += 256) {
    double vr = 0.0, vi = 0.0;
    if (p.transposed) {
      int a = idx / ETI, b = idx % ETI;  // coalesced along the source row (i)
      int k = k0 + a, i = i0 + b;        // source X[k][i]
      if (k < p.K && i < p.rows_out) load_src(re, im, p.src_c64, (size_t)k * p.ld + i, vr, vi);
      s_re[b][a] = vr;
      s_im[b][a] = vi;
    } else {
      int a = idx / ETK, b = idx % ETK;  // coalesced along the source row (k)
      int i = i0 + a, k = k0 + b;        // source X[i][k]
      if (k < p.K && i < p.rows_out) load_src(re, im, p.src_c64, (size_t)i * p.ld + k, vr, vi);
      s_re[a][b] = vr;
      s_im[a][b] = vi;
    }
  }
  __syncthreads();
  const int planes = p.layout == 0 ? 2 : (p.layout == 1 ? 3 : 1);
  const long long plane_stride = (long long)p.rows_out * p.kpitch;
  const long long mod_stride = plane_stride * planes;
  // each thread: one output row i, 4 consecutive k -> one 32-bit word per (modulus, plane)
  for (int g = tid; g < ETI * (ETK / 4); g += 256) {
    const int il = g / (ETK / 4), kl = (g % (ETK / 4)) * 4;
    const int i = i0 + il, k = k0 + kl;
    if (i >= p.rows_out || k >= p.K) continue;
    const int sh = p.beta - exps[i];
    double ar[4], ai[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      double xr = s_re[il][kl + e], xi = s_im[il][kl + e];
      if (p.conj) xi = -xi;
      ar[e] = rint(ldexp(xr, sh));  // exact integers (|.| <= 2^beta)
      ai[e] = rint(ldexp(xi, sh));
    }
    int8_t* dst = out + (size_t)i * p.kpitch + k;
    for (int l = 0; l < p.nmod; ++l) {
      const double pm = (double)p.moduli[l], inv = p.inv[l];
      const double hi = (double)(((p.moduli[l] + 1) >> 1) - 1);
      uint32_t wr = 0, wi = 0, wn = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int rr = (int)res_f64(ar[e], pm, inv, hi);
        const int ri = (int)res_f64(ai[e], pm, inv, hi);
        int rn = -ri;
        if (rn > (int)hi) rn -= p.moduli[l];
        wr |= (uint32_t)(rr & 0xFF) << (8 * e);
        wi |= (uint32_t)(ri & 0xFF) << (8 * e);
        wn |= (uint32_t)(rn & 0xFF) << (8 * e);
      }
      int8_t* dm = dst + (size_t)l * mod_stride;
      if (p.layout == 0) {
        *reinterpret_cast<uint32_t*>(dm) = wr;
        *reinterpret_cast<uint32_t*>(dm + plane_stride) = wi;
      } else if (p.layout == 1) {
        *reinterpret_cast<uint32_t*>(dm) = wn;
        *reinterpret_cast<uint32_t*>(dm + plane_stride) = wr;
        *reinterpret_cast<uint32_t*>(dm + 2 * plane_stride) = wi;
      } else {
        *reinterpret_cast<uint32_t*>(dm) = wr;
      }
    }
  }
}

// ---- decode -----------------------------------------------------------------
struct DecodeParams {
  int M, N, nmod, nchunk, beta_a, beta_b, out_kind, has_add;
  long long res_pitch, res_plane, res_mod, ld_out, ld_add;
  double alpha, shift, add_scale;
  double w[MAXMOD][MAXCHUNK];  // CRT weights, chunk j in units of 2^off[j]
  double pc[MAXCHUNK];         // modulus product P in the same chunks
  int off[MAXCHUNK];
  double inv_p;                // 1 / P
};

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
__device__ __forceinline__ void dd_add_d(double& hi, double& lo, double b) {
  double s, e;
  two_sum(hi, b, s, e);
  e += lo;
  hi = s + e;
  lo = e - (hi - s);
}

// CRT finish: S[j] = sum_l x_l w_lj (exact chunk sums) -> double-double value
__device__ __forceinline__ void crt_finish(const DecodeParams& p, const double (&S)[MAXCHUNK], double& hi,
                                           double& lo) {
  double approx = ldexp(S[0], p.off[0]);
  if (p.nchunk > 1) approx += ldexp(S[1], p.off[1]);
  const double k = rint(approx * p.inv_p);
  hi = 0.0;
  lo = 0.0;
#pragma unroll
  for (int j = 0; j < MAXCHUNK; ++j) {
    if (j >= p.nchunk) break;
    const double t = fma(-k, p.pc[j], S[j]);  // exact integer
    dd_add_d(hi, lo, ldexp(t, p.off[j]));
  }
}

// one thread: row i, columns j0..j0+3, both planes
__global__ void __launch_bounds__(256) decode_kernel(const __grid_constant__ DecodeParams p,
                                                     const int8_t* __restrict__ res, const int* __restrict__ ea,
                                                     const int* __restrict__ eb, const double* __restrict__ add_re,
                                                     const double* __restrict__ add_im, void* __restrict__ out_re,
                                                     double* __restrict__ out_im) {
  const int ngrp = (p.N + 3) >> 2;
  const long long total = (long long)p.M * ngrp;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / ngrp), j0 = (int)(idx % ngrp) * 4;
    const int rho = p.beta_a - ea[i];
#pragma unroll 1
    for (int plane = 0; plane < 2; ++plane) {
      double S[4][MAXCHUNK];
#pragma unroll
      for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int j = 0; j < MAXCHUNK; ++j) S[e][j] = 0.0;
      const int8_t* r = res + (size_t)plane * p.res_plane + (size_t)i * p.res_pitch + j0;
#pragma unroll 4
      for (int l = 0; l < p.nmod; ++l) {
        // int8 -> double without I2F: the byte with its sign bit flipped is
        // x + 128 in [0, 255]; as the low word of 0x4338000000000000 it reads
        // 1.5 * 2^52 + x + 128, so one DADD recovers x exactly.
        const uint32_t w4 = *reinterpret_cast<const uint32_t*>(r + (size_t)l * p.res_mod) ^ 0x80808080u;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const double x = __hiloint2double(0x43380000, (w4 >> (8 * e)) & 0xFF) - 6755399441055872.0;
#pragma unroll
          for (int j = 0; j < MAXCHUNK; ++j) S[e][j] = fma(x, p.w[l][j], S[e][j]);  // exact: < 2^52
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = j0 + e;
        if (j >= p.N) break;
        double hi, lo;
        crt_finish(p, S[e], hi, lo);
        const int sc = -(rho + (p.beta_b - eb[j]));
        hi = ldexp(hi, sc) * p.alpha;
        lo = ldexp(lo, sc) * p.alpha;
        if (plane == 0 && i == j && p.shift != 0.0) dd_add_d(hi, lo, p.shift);
        if (p.has_add) {
          const double av = plane == 0 ? add_re[(size_t)i * p.ld_add + j] : add_im[(size_t)i * p.ld_add + j];
          dd_add_d(hi, lo, p.add_scale * av);
        }
        const double v = hi + lo;
        if (p.out_kind == 0) {
          if (plane == 0)
            ((double*)out_re)[(size_t)i * p.ld_out + j] = v;
          else
            out_im[(size_t)i * p.ld_out + j] = v;
        } else {
          float* o = reinterpret_cast<float*>(out_re) + 2 * ((size_t)i * p.ld_out + j);
          o[plane] = (float)v;
        }
      }
    }
  }
}

}  // namespace

extern "C" int sr_oz_exponents(int rows, int cols, const void* src, const double* im, long long ld, int src_c64,
                               int transposed, int* exps, void* stream) {
  const double* re = (const double*)src;
  if (rows < 0 || cols < 0 || !re || !exps) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (!transposed) {
    if (rows == 0) return SR_OK;
    exps_direct_kernel<<<sr_ceil_div((long long)rows * 32, 256), 256, 0, st>>>(rows, cols, re, im, ld, src_c64, exps);
  } else {
    if (cols == 0) return SR_OK;
    exps_transposed_kernel<<<sr_ceil_div(cols, 32), dim3(32, 8), 0, st>>>(rows, cols, re, im, ld, src_c64, exps);
  }
  SR_LAUNCH_CHECK();
  return SR_OK;
}

extern "C" int sr_oz_encode(int rows_out, int K, const void* src, const double* im, long long ld, int src_c64,
                            int transposed, int conj, int layout, const int* exps, int beta, int nmod,
                            const int* moduli, void* out, long long kpitch, void* stream) {
  const double* re = (const double*)src;
  if (rows_out <= 0 || K <= 0 || nmod <= 0 || nmod > MAXMOD || layout < 0 || layout > 2) return SR_EINVAL;
  if (beta < 1 || beta > 61 || (kpitch & 15) || kpitch < K) return SR_EINVAL;
  EncodeParams p;
  memset(&p, 0, sizeof(p));
  p.rows_out = rows_out;
  p.K = K;
  p.transposed = transposed;
  p.conj = conj;
  p.layout = layout;
  p.beta = beta;
  p.nmod = nmod;
  p.ld = ld;
  p.kpitch = kpitch;
  p.src_c64 = src_c64;
  for (int l = 0; l < nmod; ++l) {
    if (moduli[l] < 129 || moduli[l] > 256) return SR_EINVAL;
    p.moduli[l] = moduli[l];
    p.inv[l] = 1.0 / moduli[l];
  }
  // K padding columns of the residue planes must read as zero
  const int planes = layout == 0 ? 2 : (layout == 1 ? 3 : 1);
  if (kpitch > K)
    SR_CUDA_CHECK(cudaMemsetAsync(out, 0, (size_t)nmod * planes * rows_out * kpitch, (cudaStream_t)stream));
  dim3 grid(sr_ceil_div(K, ETK), sr_ceil_div(rows_out, ETI));
  encode_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(p, re, im, exps, (int8_t*)out);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

// table: [nmod][4] weights, [4] P chunks, [4] offsets (as doubles), inv_p  (9 + 4*nmod doubles)
extern "C" int sr_oz_decode(int M, int N, int nmod, int nchunk, const double* table, const void* res,
                            long long res_pitch, const int* exps_a, int beta_a, const int* exps_b, int beta_b,
                            double alpha, double shift, const double* add_re, const double* add_im, long long ld_add,
                            double add_scale, int out_kind, void* out_re, double* out_im, long long ld_out,
                            void* stream) {
  if (M <= 0 || N <= 0 || nmod <= 0 || nmod > MAXMOD || nchunk < 1 || nchunk > MAXCHUNK) return SR_EINVAL;
  if (out_kind == 0 && !out_im) return SR_EINVAL;
  DecodeParams p;
  memset(&p, 0, sizeof(p));
  p.M = M;
  p.N = N;
  p.nmod = nmod;
  p.nchunk = nchunk;
  p.beta_a = beta_a;
  p.beta_b = beta_b;
  p.out_kind = out_kind;
  p.has_add = add_re != nullptr;
  p.res_pitch = res_pitch;
  p.res_plane = res_pitch * M;
  p.res_mod = p.res_plane * 2;
  p.ld_out = ld_out;
  p.ld_add = ld_add;
  p.alpha = alpha;
  p.shift = shift;
  p.add_scale = add_scale;
  for (int l = 0; l < nmod; ++l)
    for (int j = 0; j < MAXCHUNK; ++j) p.w[l][j] = table[l * MAXCHUNK + j];
  for (int j = 0; j < MAXCHUNK; ++j) {
    p.pc[j] = table[nmod * MAXCHUNK + j];
    p.off[j] = (int)table[nmod * MAXCHUNK + MAXCHUNK + j];
  }
  p.inv_p = table[nmod * MAXCHUNK + 2 * MAXCHUNK];
  if (res_pitch & 3) return SR_EINVAL;
  const long long total = (long long)M * ((N + 3) / 4);
  int grid = (int)((total + 255) / 256);
  if (grid > 148 * 16) grid = 148 * 16;
  decode_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(p, (const int8_t*)res, exps_a, exps_b, add_re, add_im,
                                                        out_re, out_im);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

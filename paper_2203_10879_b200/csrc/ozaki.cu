// Ozaki-II emulated complex products: operand encoding and CRT decoding.
//
// A product C = op(A) B is evaluated exactly on integers (Ozaki, Uchino,
// Imamura — "Ozaki scheme II", CRT variant):
//   1. scale   every row of op(A) and every column of B by a power of two so
//              its largest entry is below 2^beta, round to integers A', B'
//              (FP64 mode, beta = 60: every entry within 2^-7 of its row or
//              column maximum is represented exactly; dd mode, beta = 104);
//   2. encode  the residues A' mod p_l, B' mod p_l (symmetric, int8) for the
//              pairwise-coprime moduli p_1..p_r <= 256 of the plan, K-major;
//   3. multiply on the tensor cores: R_l = A'_l B'_l mod p_l (oz_gemm.cu);
//   4. decode  C' from its residues by the Chinese remainder theorem in
//              exact FP64 chunk arithmetic (carry-normalised, so the final
//              double-double sum has no cancellation), then unscale:
//              C = alpha * C' * 2^-(rho_i + sigma_j) + shift * I + add_scale * X.
// Every integer product and sum is exact, so the result is independent of
// the summation order; its only errors are the operand rounding of step 1
// and one final rounding — unlike a K-long FP64 accumulation chain, whose
// noise on stril(Q^H A Q) grows like sqrt(K).
//
// Matrix kinds (SR_MAT_*, include/sr.h): planar FP64 (the FP64-mode hp type),
// interleaved complex64 (FP64-mode lp), interleaved complex128 (dd-mode lp),
// planar double-double (dd-mode hp, four planes re_hi, im_hi, re_lo, im_lo).
//
// This replaces matmul_hp / matmul_lp
// (/root/reference/pkg/src/ddschur/matmul.py:52-110) and generalises the
// reference's own Ozaki-I dd product (_ozaki_gemm_hp, matmul.py:151-212).
#include "sr_common.cuh"
#include "tc_common.cuh"

namespace {

constexpr int MAXMOD = 32;
constexpr int MAXCHUNK = 6;  // 40-bit CRT chunks: modulus products up to 240 bits
constexpr int MAXDIG = 10;   // 11-bit digits: integers up to 2^109
constexpr int EXP_FLOOR = -1074;  // below every finite double's exponent: all-zero rows/columns

// x * 2^e without the libm ldexp (~15 instructions): two exact power-of-two
// multiplies (the split keeps both factors in the normal range).
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }
__device__ __forceinline__ double scale2(double x, int e) {
  const int e1 = e / 2;
  return (x * pow2(e1)) * pow2(e - e1);
}

struct Src {
  const double* re;
  const double* im;
  const double* re_lo;
  const double* im_lo;
  int kind;
};

// element (re, im) [+ (re_lo, im_lo) for dd] at linear offset off
template <int KIND>
__device__ __forceinline__ void load_elem(const Src& s, size_t off, double& vr, double& vi, double& lr,
                                          double& li) {
  lr = li = 0.0;
  if (KIND == SR_MAT_C64) {
    const float2 v = reinterpret_cast<const float2*>(s.re)[off];
    vr = v.x;
    vi = v.y;
  } else if (KIND == SR_MAT_C128) {
    const double2 v = reinterpret_cast<const double2*>(s.re)[off];
    vr = v.x;
    vi = v.y;
  } else {
    vr = s.re[off];
    vi = s.im ? s.im[off] : 0.0;
    if (KIND == SR_MAT_DD) {
      lr = s.re_lo[off];
      li = s.im_lo[off];
    }
  }
}

// ---- exponents: e_i with max_k |op(X)[i,k]| < 2^e_i (dd: of the hi parts) ----
// With rmax != null also r_i = ||op(X)[i, :]||_2 2^-e_i (the line's 2-norm in
// units of its power-of-two scale) and rmax = max_i r_i (atomicMax on the bits
// of a non-negative double): the CRT bound of a product (ozaki.fit_plan).
__device__ __forceinline__ void atomic_max_nonneg(double* a, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(a), (unsigned long long)__double_as_longlong(v));
}

template <int KIND>
__global__ void exps_direct_kernel(int rows, int cols, Src s, long long ld, int* __restrict__ e,
                                   double* __restrict__ rmax) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  double m = 0.0, ss = 0.0;
  for (int k = lane; k < cols; k += 32) {
    double vr, vi, lr, li;
    load_elem<KIND>(s, (size_t)warp * ld + k, vr, vi, lr, li);
    m = fmax(m, fmax(fabs(vr), fabs(vi)));
    ss = fma(vr, vr, fma(vi, vi, ss));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  if (lane == 0) {
    int ex = EXP_FLOOR;
    if (m > 0.0) frexp(m, &ex);
    e[warp] = ex;
    if (rmax && m > 0.0) atomic_max_nonneg(rmax, sqrt(ss) * scale2(1.0, -ex));
  }
}

__global__ void exps_fill_kernel(int n, int* __restrict__ e) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) e[i] = EXP_FLOOR;
}

// rmax -> a pinned host word by a plain store over the bus (UVA): no copy
// engine, so the read never queues behind a large device-to-host copy
__global__ void publish_kernel(const double* __restrict__ src, volatile double* dst) {
  *dst = *src;
  __threadfence_system();
}

// column bound: r_j = sqrt(ss_j) 2^-e_j, rmax = max_j r_j
__global__ void bound_finish_kernel(int cols, const double* __restrict__ ss, const int* __restrict__ e,
                                    double* __restrict__ rmax) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < cols && e[j] > EXP_FLOOR) atomic_max_nonneg(rmax, sqrt(ss[j]) * scale2(1.0, -e[j]));
}

// per-column maxima over a chunk of rows per block (grid.y), merged with an
// integer atomicMax on the exponent (frexp's exponent is monotone in |x|);
// with ss != null also the columns' sums of squares (atomicAdd: a bound only)
template <int KIND>
__global__ void exps_transposed_kernel(int rows, int cols, Src s, long long ld, int rows_per_block,
                                       int* __restrict__ e, double* __restrict__ ssum) {
  __shared__ double part[8][33];
  __shared__ double psq[8][33];
  const int j = blockIdx.x * 32 + threadIdx.x;
  const int r0 = blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  double m = 0.0, ss = 0.0;
  if (j < cols)
    for (int i = r0 + threadIdx.y; i < r1; i += 8) {
      double vr, vi, lr, li;
      load_elem<KIND>(s, (size_t)i * ld + j, vr, vi, lr, li);
      m = fmax(m, fmax(fabs(vr), fabs(vi)));
      ss = fma(vr, vr, fma(vi, vi, ss));
    }
  part[threadIdx.y][threadIdx.x] = m;
  psq[threadIdx.y][threadIdx.x] = ss;
  __syncthreads();
  if (threadIdx.y == 0 && j < cols) {
    for (int y = 1; y < 8; ++y) {
      m = fmax(m, part[y][threadIdx.x]);
      ss += psq[y][threadIdx.x];
    }
    if (m > 0.0) {
      int ex = 0;
      frexp(m, &ex);
      atomicMax(&e[j], ex);
    }
    if (ssum && ss > 0.0) atomicAdd(&ssum[j], ss);
  }
}

// ---- encode: residue planes [nmod][planes][rows_out][kpitch] -------------------
// layout 0: A operand (re, im);  1: B operand (-im, re, im);  2: B operand (re);
// 3: both roles of one matrix X read column-wise (transposed): the A operand
//    of X^H (re, -im) into out and the B operand of X (-im, re, im) into out2,
//    sharing the residue computation (Q^H and Q of every measurement);
// 4: Gaussian planes (re + iota im, re - iota im) mod p, iota^2 = -1 mod p, for
//    either role: a complex product mod p is then two independent real
//    products (oz_gemm.cu, gauss mode).  The conjugate swaps the two planes, so
//    the B operand of X is also the A operand of X^H (planes swapped).
struct EncodeParams {
  int rows_out, K, transposed, conj, layout, beta, nmod, ndig;
  long long ld, kpitch;
  int8_t* out2;
  float pf[MAXMOD], invf[MAXMOD], hif[MAXMOD], lof[MAXMOD];
  float pow2[MAXMOD][MAXDIG];  // 2^(11 c) mod p, symmetric
  int pi[MAXMOD];              // the moduli as ints
  int wb[MAXMOD][2];           // 2^(8 c) mod p, c = 0..7, symmetric int8, packed 4 per word
  int c64[MAXMOD];             // 2^64 mod p, symmetric
  uint32_t bm[MAXMOD];         // Barrett multiplier floor(2^32 / p) + 1
  int off0[MAXMOD], off1[MAXMOD];  // positive shift (a multiple of p), and it minus 2^64 mod p
  int wgp[MAXMOD][2], wgm[MAXMOD][2];  // layout 4: +-iota 2^(8 c) mod p, symmetric int8, packed 4 per word
  int cgp[MAXMOD];                 // layout 4: iota 2^64 mod p, symmetric
  int offg[MAXMOD];                // layout 4: a multiple of p above four byte dot products, minus lo
  int offb[MAXMOD], offi[MAXMOD];  // layout 4: offg - (2^63 mod p), -(iota 2^63 mod p) (sign-bit-flipped bytes)
};

// balanced 11-bit digits of an integer-valued double (error-free, top-down)
template <int ND>
__device__ __forceinline__ void digits(double a, float (&d)[ND]) {
#pragma unroll
  for (int c = ND - 1; c >= 0; --c) {
    const double sc = (double)(1ull << (11 * (c % 5))) * (c >= 5 ? 36028797018963968.0 : 1.0);  // 2^(11c)
    const double q = rint(a * (1.0 / sc));
    a = fma(-q, sc, a);
    d[c] = (float)q;
  }
}

__device__ __forceinline__ int dp4a_us(uint32_t a, int b, int c) {  // unsigned bytes . signed bytes + c
  int d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// the residue words of 4 consecutive k of row i, modulus l, in the layout's planes
__device__ __forceinline__ void store_planes(const EncodeParams& p, int8_t* dst, int l, long long mod_stride,
                                             long long mod_stride2, long long plane_stride, int i, int k,
                                             uint32_t wr, uint32_t wi, uint32_t wn) {
  int8_t* dm = dst + (size_t)l * mod_stride;
  if (p.layout == 0) {
    *reinterpret_cast<uint32_t*>(dm) = wr;
    *reinterpret_cast<uint32_t*>(dm + plane_stride) = wi;
  } else if (p.layout == 1) {
    *reinterpret_cast<uint32_t*>(dm) = wn;
    *reinterpret_cast<uint32_t*>(dm + plane_stride) = wr;
    *reinterpret_cast<uint32_t*>(dm + 2 * plane_stride) = wi;
  } else if (p.layout == 4) {
    *reinterpret_cast<uint32_t*>(dm) = wr;  // (phi+, phi-) passed in wr, wi
    *reinterpret_cast<uint32_t*>(dm + plane_stride) = wi;
  } else if (p.layout == 3) {
    *reinterpret_cast<uint32_t*>(dm) = wr;  // A operand of X^H: (re, -im)
    *reinterpret_cast<uint32_t*>(dm + plane_stride) = wn;
    int8_t* d2 = p.out2 + (size_t)l * mod_stride2 + (size_t)i * p.kpitch + k;  // B operand of X
    *reinterpret_cast<uint32_t*>(d2) = wn;
    *reinterpret_cast<uint32_t*>(d2 + plane_stride) = wr;
    *reinterpret_cast<uint32_t*>(d2 + 2 * plane_stride) = wi;
  } else {
    *reinterpret_cast<uint32_t*>(dm) = wr;
  }
}

template <int KIND>
__global__ void __launch_bounds__(256) encode_kernel(const __grid_constant__ EncodeParams p, Src s,
                                                     const int* __restrict__ exps, int8_t* __restrict__ out) {
  constexpr bool DD = KIND == SR_MAT_DD;
  constexpr int ETI = DD ? 32 : 64, ETK = 32;  // tile: ETI output rows x 32 k
  constexpr int ND = DD ? MAXDIG : 6;          // beta <= 61 needs 6 digits, dd up to 10
  __shared__ double s_re[ETI][ETK + 1];
  __shared__ double s_im[ETI][ETK + 1];
  __shared__ double s_rl[DD ? ETI : 1][ETK + 1];
  __shared__ double s_il[DD ? ETI : 1][ETK + 1];
  const int i0 = blockIdx.y * ETI, k0 = blockIdx.x * ETK;
  const int tid = threadIdx.x;
  // stage the source tile as s[i_local][k_local] = op(X)[i0 + i][k0 + k]
  for (int idx = tid; idx < ETI * ETK; idx += 256) {
    double vr = 0.0, vi = 0.0, lr = 0.0, li = 0.0;
    int il, kl;
    if (p.transposed) {
      const int a = idx / ETI, b = idx % ETI;  // coalesced along the source row (i)
      const int k = k0 + a, i = i0 + b;        // source X[k][i]
      if (k < p.K && i < p.rows_out) load_elem<KIND>(s, (size_t)k * p.ld + i, vr, vi, lr, li);
      il = b;
      kl = a;
    } else {
      const int a = idx / ETK, b = idx % ETK;  // coalesced along the source row (k)
      const int i = i0 + a, k = k0 + b;        // source X[i][k]
      if (k < p.K && i < p.rows_out) load_elem<KIND>(s, (size_t)i * p.ld + k, vr, vi, lr, li);
      il = a;
      kl = b;
    }
    s_re[il][kl] = vr;
    s_im[il][kl] = vi;
    if (DD) {
      s_rl[il][kl] = lr;
      s_il[il][kl] = li;
    }
  }
  __syncthreads();
  const int planes = p.layout == 0 || p.layout == 3 || p.layout == 4 ? 2 : (p.layout == 1 ? 3 : 1);
  const long long plane_stride = (long long)p.rows_out * p.kpitch;
  const long long mod_stride = plane_stride * planes;
  const long long mod_stride2 = plane_stride * 3;  // layout 3: out2 holds the 3 B planes
  // each thread: one output row i, 4 consecutive k -> one 32-bit word per (modulus, plane)
  for (int g = tid; g < ETI * (ETK / 4); g += 256) {
    const int il = g / (ETK / 4), kl = (g % (ETK / 4)) * 4;
    const int i = i0 + il, k = k0 + kl;
    if (i >= p.rows_out || k >= p.K) continue;
    const int sh = p.beta - exps[i];
    int8_t* dst = out + (size_t)i * p.kpitch + k;
    if constexpr (!DD) {
      // |scaled| <= 2^61: exact int64.  Its two's-complement bytes u_c give
      // x mod p = sum_c u_c (2^(8c) mod p) - [x < 0] (2^64 mod p): two byte dot
      // products (dp4a) per value and modulus, one reduction
      uint32_t lo_r[4], hi_r[4], lo_i[4], hi_i[4];
      bool ng_r[4], ng_i[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        double xi = s_im[il][kl + e];
        if (p.conj) xi = -xi;
        const long long a = __double2ll_rn(scale2(s_re[il][kl + e], sh));
        const long long b = __double2ll_rn(scale2(xi, sh));
        lo_r[e] = (uint32_t)a;
        hi_r[e] = (uint32_t)((unsigned long long)a >> 32);
        lo_i[e] = (uint32_t)b;
        hi_i[e] = (uint32_t)((unsigned long long)b >> 32);
        ng_r[e] = a < 0;
        ng_i[e] = b < 0;
      }
      const bool need_neg = p.layout == 1 || p.layout == 3;  // planes with -im
      if (p.layout == 4) {
        // Gaussian planes straight from the bytes: phi+- = re +- iota im mod p.
        // With the sign bit flipped, the bytes u_c of x + 2^63 are unsigned, so
        // x mod p = sum_c u_c (2^(8c) mod p) - (2^63 mod p) for either sign: four
        // byte dot products (dp4a) per modulus, the 2^63 terms folded into the
        // per-modulus offsets (offb: real part, offi: imaginary part), one
        // Barrett reduction per plane (0 <= v < 2^21)
        uint32_t hr[4], hm[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          hr[e] = hi_r[e] ^ 0x80000000u;
          hm[e] = hi_i[e] ^ 0x80000000u;
        }
        int8_t* dm = dst;
        for (int l = 0; l < p.nmod; ++l, dm += mod_stride) {
          const int pm = p.pi[l];
          const uint32_t bm = p.bm[l];
          const int lo = -(pm >> 1);
          const int w0 = p.wb[l][0], w1 = p.wb[l][1];
          const int gp0 = p.wgp[l][0], gp1 = p.wgp[l][1];
          const int ob = p.offb[l], oi = p.offi[l];
          int rp[4], rm[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int base = dp4a_us(hr[e], w1, dp4a_us(lo_r[e], w0, ob));
            const int vp = dp4a_us(hm[e], gp1, dp4a_us(lo_i[e], gp0, base + oi));
            // the -iota weights are the negated +iota ones (symmetric residues,
            // odd p), so phi- = 2 base - phi+ exactly (both stay in [0, 2^21):
            // the offset exceeds the sixteen byte products and the 2^63 terms)
            const int vm = 2 * base - vp;
            // v < 2^21: umulhi(v, floor(2^32 / p) + 1) is exactly floor(v / p)
            // (the multiplier's excess times v stays below 2^32), so v - q p is
            // already in [0, p)
            rp[e] = vp - (int)__umulhi((uint32_t)vp, bm) * pm + lo;
            rm[e] = vm - (int)__umulhi((uint32_t)vm, bm) * pm + lo;
          }
          const uint32_t wp = __byte_perm(__byte_perm(rp[0], rp[1], 0x0040), __byte_perm(rp[2], rp[3], 0x0040), 0x5410);
          const uint32_t wm = __byte_perm(__byte_perm(rm[0], rm[1], 0x0040), __byte_perm(rm[2], rm[3], 0x0040), 0x5410);
          *reinterpret_cast<uint32_t*>(dm) = wp;
          *reinterpret_cast<uint32_t*>(dm + plane_stride) = wm;
        }
        continue;
      }
      for (int l = 0; l < p.nmod; ++l) {
        const int pm = p.pi[l];
        const uint32_t bm = p.bm[l];
        const int lo = -(pm >> 1);
        const int w0 = p.wb[l][0], w1 = p.wb[l][1], o0 = p.off0[l], c64 = p.c64[l];
        int rr[4], ri[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          // v = byte dot products + a positive multiple of p - lo (- 2^64 mod p when
          // negative): 0 <= v < 2^20; u = v mod p by Barrett, r = u + lo symmetric
          const int vr = dp4a_us(hi_r[e], w1, dp4a_us(lo_r[e], w0, o0 - (int)ng_r[e] * c64));
          const int vi = dp4a_us(hi_i[e], w1, dp4a_us(lo_i[e], w0, o0 - (int)ng_i[e] * c64));
          // v < 2^20: the Barrett quotient is exact, v - q p is in [0, p)
          rr[e] = vr - (int)__umulhi((uint32_t)vr, bm) * pm + lo;
          ri[e] = vi - (int)__umulhi((uint32_t)vi, bm) * pm + lo;
        }
        // pack the four low bytes per plane (two byte permutes each)
        const uint32_t wr = __byte_perm(__byte_perm(rr[0], rr[1], 0x0040), __byte_perm(rr[2], rr[3], 0x0040), 0x5410);
        const uint32_t wi = __byte_perm(__byte_perm(ri[0], ri[1], 0x0040), __byte_perm(ri[2], ri[3], 0x0040), 0x5410);
        // -im: per-byte two's-complement negation is the symmetric residue of
        // -x for every modulus (odd p: |r| <= 127; p = 256: -(-128) wraps to
        // -128, the representative of 128)
        const uint32_t wn = need_neg ? __vneg4(wi) : 0u;
        store_planes(p, dst, l, mod_stride, mod_stride2, plane_stride, i, k, wr, wi, wn);
      }
      continue;
    }
    // dd operands (beta up to 106): exact 11-bit digit expansions of hi and lo
    float dr[4][ND], di[4][ND];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      double xr = s_re[il][kl + e], xi = s_im[il][kl + e];
      if (p.conj) xi = -xi;
      digits<ND>(rint(scale2(xr, sh)), dr[e]);  // exact integers, |.| <= 2^beta
      digits<ND>(rint(scale2(xi, sh)), di[e]);
      if (DD) {  // + the rounded lo part: digit-wise sum, still exact in FP32
        double lr = s_rl[il][kl + e], li = s_il[il][kl + e];
        if (p.conj) li = -li;
        float er[ND], ei[ND];
        digits<ND>(rint(scale2(lr, sh)), er);
        digits<ND>(rint(scale2(li, sh)), ei);
#pragma unroll
        for (int c = 0; c < ND; ++c) {
          dr[e][c] += er[c];
          di[e][c] += ei[c];
        }
      }
    }
    for (int l = 0; l < p.nmod; ++l) {
      const float pm = p.pf[l], inv = p.invf[l], hi = p.hif[l], lo = p.lof[l];
      uint32_t wr = 0, wi = 0, wn = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        // residue = sum_c digit_c * (2^(11c) mod p), exact in FP32 (|.| < 2^22), then one reduction
        float vr = 0.f, vi = 0.f;
#pragma unroll
        for (int c = 0; c < ND; ++c) {
          if (c < p.ndig) {
            vr = fmaf(dr[e][c], p.pow2[l][c], vr);
            vi = fmaf(di[e][c], p.pow2[l][c], vi);
          }
        }
        const float qr = (vr * inv + 12582912.f) - 12582912.f;  // round-to-nearest, |.| < 2^22
        const float qi = (vi * inv + 12582912.f) - 12582912.f;
        float rr = fmaf(-qr, pm, vr);
        float ri = fmaf(-qi, pm, vi);
        rr = rr > hi ? rr - pm : (rr < lo ? rr + pm : rr);
        ri = ri > hi ? ri - pm : (ri < lo ? ri + pm : ri);
        float rn = -ri;
        rn = rn > hi ? rn - pm : rn;
        // the low byte of (r + 1.5 * 2^23) is r in two's complement
        wr |= (__float_as_uint(rr + 12582912.f) & 0xFFu) << (8 * e);
        wi |= (__float_as_uint(ri + 12582912.f) & 0xFFu) << (8 * e);
        wn |= (__float_as_uint(rn + 12582912.f) & 0xFFu) << (8 * e);
      }
      store_planes(p, dst, l, mod_stride, mod_stride2, plane_stride, i, k, wr, wi, wn);
    }
  }
}

// ---- decode -----------------------------------------------------------------
struct DecodeParams {
  int M, N, nmod, nchunk, beta_a, beta_b, hermitian, diag_col0;
  long long res_pitch, res_plane, res_mod, ld_out, ld_add;
  double alpha, shift, add_scale;
  double w[MAXMOD][MAXCHUNK];  // CRT weights, chunk j in units of 2^off[j]
  double pc[MAXCHUNK];         // modulus product P in the same chunks
  double offv[MAXCHUNK];       // 2^off[j]
  double cw[MAXCHUNK], icw[MAXCHUNK];  // 2^(off[j-1]-off[j]) and its inverse
  double inv_p;                // 1 / P
  double snap, inv_snap;       // truncated CRT (nchunk below the plan's): grid of the lowest kept chunk
  double w_im[MAXMOD][MAXCHUNK];  // gauss: weights of the imaginary part (w holds the real part's)
};

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
__device__ __forceinline__ void quick_two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  e = b - (s - a);
}
// (hi, lo) += b
__device__ __forceinline__ void dd_add_d(double& hi, double& lo, double b) {
  double s, e;
  two_sum(hi, b, s, e);
  e += lo;
  quick_two_sum(s, e, hi, lo);
}
// (hi, lo) += (bh, bl), the accurate dd sum of the reference (dd.py:96-104)
__device__ __forceinline__ void dd_add_dd(double& hi, double& lo, double bh, double bl) {
  double s1, s2, t1, t2;
  two_sum(hi, bh, s1, s2);
  two_sum(lo, bl, t1, t2);
  s2 += t1;
  quick_two_sum(s1, s2, s1, s2);
  s2 += t2;
  quick_two_sum(s1, s2, hi, lo);
}

// CRT finish: S[j] = sum_l x_l w_lj (exact chunk sums) -> double-double value
template <int NC>
__device__ __forceinline__ void crt_finish(const DecodeParams& p, const double (&S)[NC], double& hi, double& lo) {
  double approx = S[0] * p.offv[0];
  if (NC > 1) approx += S[1] * p.offv[1];
  const double k = rint(approx * p.inv_p);
  double t[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) t[j] = fma(-k, p.pc[j], S[j]);  // exact integers
  // carry-normalise from the bottom chunk up so that |t_j| <= 2^(width_j - 1)
  // for j >= 1: the double-double sum below then has no cancellation
#pragma unroll
  for (int j = NC - 1; j >= 1; --j) {
    const double c = rint(t[j] * p.icw[j]);
    t[j] = fma(-c, p.cw[j], t[j]);
    t[j - 1] += c;
  }
  // truncated CRT (OzPlan.decode_chunks): C' is known to < snap / 2 in units
  // of the lowest kept chunk, so round it to that grid — an exact C' on the
  // grid (0, I I = I, small integers) comes out exact, lo parts included
  if (p.snap > 0.0) t[NC - 1] = rint(t[NC - 1] * p.inv_snap) * p.snap;
  hi = t[0] * p.offv[0];
  lo = 0.0;
#pragma unroll
  for (int j = 1; j < NC; ++j) dd_add_d(hi, lo, t[j] * p.offv[j]);
}

struct Dst {
  double* re;
  double* im;
  double* re_lo;
  double* im_lo;
};

// CRT finish, unscale, shift / add and the one rounding of entry (i, j),
// output plane pl (0 = re, 1 = im)
template <int NC, int OUT, int ADD>
__device__ __forceinline__ void finish_store(const DecodeParams& p, const double (&S)[NC], int i, int j, int rho,
                                             int sigma, int pl, const Src& add, const Dst& out) {
  double hi, lo;
  crt_finish<NC>(p, S, hi, lo);
  const int sc = -(rho + sigma);
  hi = scale2(hi, sc) * p.alpha;
  lo = scale2(lo, sc) * p.alpha;
  if (pl == 0 && i == j + p.diag_col0 && p.shift != 0.0) dd_add_d(hi, lo, p.shift);
  const size_t oa = (size_t)i * p.ld_add + j;
  if (ADD == SR_MAT_F64) dd_add_d(hi, lo, p.add_scale * (pl == 0 ? add.re[oa] : add.im[oa]));
  if (ADD == SR_MAT_DD)
    dd_add_dd(hi, lo, p.add_scale * (pl == 0 ? add.re[oa] : add.im[oa]),
              p.add_scale * (pl == 0 ? add.re_lo[oa] : add.im_lo[oa]));
  const size_t o = (size_t)i * p.ld_out + j;
  if (OUT == SR_MAT_F64) {
    (pl == 0 ? out.re : out.im)[o] = hi + lo;
  } else if (OUT == SR_MAT_DD) {
    quick_two_sum(hi, lo, hi, lo);
    (pl == 0 ? out.re : out.im)[o] = hi;
    (pl == 0 ? out.re_lo : out.im_lo)[o] = lo;
  } else if (OUT == SR_MAT_C64) {
    reinterpret_cast<float*>(out.re)[2 * o + pl] = (float)(hi + lo);
  } else {
    out.re[2 * o + pl] = hi + lo;
  }
}

// Lean CRT finish for FP64 / complex64 outputs of the Gaussian products (both
// the SIMT and the tensor-core decode use it, so they agree bit for bit):
// t_j = S_j - k P_j exact, the bottom chunk snapped as in crt_finish (no carry
// normalisation needed), then V = t_0 2^o0 + t_1 2^o1 (+ t_2 2^o2 ...) as an exact
// two_sum of the top pair plus the rest, unscaled, shifted / added with one
// more exact two_sum, and rounded once: correctly rounded up to a rare double
// rounding (error < 0.5 ulp + 2^-80 relative), exact whenever the result is
// representable (zeros, I I = I, small integers), ~35 FP64 instructions per
// entry and plane instead of ~120 for the double-double finish.
// rint for |x| < 2^51 on the FP64 pipe (two DADDs; FRND.F64 runs on the
// narrow XU pipe, which the decode's three roundings per entry saturated):
// round-to-nearest-even like rint
__device__ __forceinline__ double rint_small(double x) {
  return __dsub_rn(__dadd_rn(x, 6755399441055744.0), 6755399441055744.0);
}

template <int NC, int ADD>
__device__ __forceinline__ double crt_lean(const DecodeParams& p, const double (&S)[NC], int i, int j, int sc,
                                           int pl, double x) {
  double approx = S[0] * p.offv[0];
  if (NC > 1) approx += S[1] * p.offv[1];
  const double k = rint_small(approx * p.inv_p);
  double t[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) t[c] = fma(-k, p.pc[c], S[c]);  // exact integers
  // snap (truncated CRT): the chunks above the bottom one are multiples of its
  // 2^40 units, so rounding the bottom chunk to the grid rounds C' to it
  // whether or not the chunks are carry-normalised (two_sum below needs no
  // ordering of its operands)
  if (p.snap > 0.0) t[NC - 1] = rint_small(t[NC - 1] * p.inv_snap) * p.snap;
  double s, e = 0.0;
  if (NC > 1)
    two_sum(t[0] * p.offv[0], t[1] * p.offv[1], s, e);
  else
    s = t[0] * p.offv[0];
#pragma unroll
  for (int c = 2; c < NC; ++c) e = fma(t[c], p.offv[c], e);
  const bool shifted = pl == 0 && p.shift != 0.0 && i == j + p.diag_col0;
  if (ADD != SR_MAT_F64 && !shifted) return scale2(s + e, sc) * p.alpha;  // one rounding, then exact scaling
  // unscale (exact) and alpha (a power of two), then + shift / + X with one more exact two_sum
  s = scale2(s, sc) * p.alpha;
  e = scale2(e, sc) * p.alpha;
  if (shifted) {
    double s2, e2;
    two_sum(s, p.shift, s2, e2);
    s = s2;
    e += e2;
  }
  if (ADD == SR_MAT_F64) {
    double s2, e2;
    two_sum(s, p.add_scale * x, s2, e2);
    s = s2;
    e += e2;
  }
  return s + e;
}

// one thread: row i, columns j0..j0+3, both planes.  (re, im) residues: one
// pass per plane.  G: the residue planes are Gaussian (phi+, phi-) =
// (re + iota im, re - iota im) mod p; re = (phi+ + phi-)/2 and
// im = (phi+ - phi-)/(2 iota) mod p, the constant factors folded into the CRT
// weights (w: real part, w_im: imaginary part), so the decode forms phi+ +-
// phi- in integers (|.| <= 240: the chunk sums stay below 2^53 for <= 32
// moduli) and accumulates both planes in ONE pass over the residues.  With
// four or six chunks a thread takes two columns instead of four (two
// accumulator sets of four columns: 150 registers, 3.4 vs 3.1 ms for an
// n = 8192 hp decode).
template <int NC, int OUT, int ADD, bool G = false>
// (Gaussian: at most 80 registers, three CTAs per SM — 2.68 -> 2.48 ms for an
// n = 8192 hp decode despite a few spilled words)
__global__ void __launch_bounds__(256, G ? 3 : 1) decode_kernel(const __grid_constant__ DecodeParams p,
                                                     const int8_t* __restrict__ res, const int* __restrict__ ea,
                                                     const int* __restrict__ eb, Src add, Dst out) {
  constexpr bool ONE = G;                    // both Gaussian planes in one pass
  constexpr int CPT = (G && NC > 2) ? 2 : 4;  // columns per thread
  const int ngrp = (p.N + CPT - 1) / CPT;
  // idx = i ngrp + jg stepped by the grid stride without a 64-bit division per
  // entry group (its I2F / MUFU / F2I sequence runs on the narrow XU pipe)
  const long long start = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int sq = (int)(stride / ngrp), sr = (int)(stride % ngrp);
  int i = (int)(start / ngrp), jg = (int)(start % ngrp);
  for (; i < p.M; i += sq, jg += sr) {
    if (jg >= ngrp) {
      jg -= ngrp;
      if (++i >= p.M) break;
    }
    const int j0 = jg * CPT;
    if (p.hermitian && (j0 >> 7) > (i >> 7)) continue;  // upper GEMM tile: mirrored afterwards
    const int rho = p.beta_a - ea[i];
#pragma unroll 1
    for (int plane = 0; plane < (ONE ? 1 : 2); ++plane) {
      double S[CPT][NC], S2[ONE ? CPT : 1][NC];
#pragma unroll
      for (int e = 0; e < CPT; ++e)
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          S[e][j] = 0.0;
          if (ONE) S2[e][j] = 0.0;
        }
      const double(*W)[MAXCHUNK] = (G && plane == 1) ? p.w_im : p.w;
      const int8_t* r = res + (size_t)(G ? 0 : plane) * p.res_plane + (size_t)i * p.res_pitch + j0;
      // residue words in groups of 8 moduli (8 loads in flight, bounded registers)
#pragma unroll 1
      for (int l0 = 0; l0 < p.nmod; l0 += 8) {
        uint32_t wv[8], wm[8];
#pragma unroll
        for (int g = 0; g < 8; ++g)
          if (l0 + g < p.nmod) {
            if (CPT == 4) {
              wv[g] = *reinterpret_cast<const uint32_t*>(r + (size_t)(l0 + g) * p.res_mod);
              if (G) wm[g] = *reinterpret_cast<const uint32_t*>(r + p.res_plane + (size_t)(l0 + g) * p.res_mod);
            } else {
              wv[g] = *reinterpret_cast<const uint16_t*>(r + (size_t)(l0 + g) * p.res_mod);
              wm[g] = *reinterpret_cast<const uint16_t*>(r + p.res_plane + (size_t)(l0 + g) * p.res_mod);
            }
          }
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          if (l0 + g >= p.nmod) break;
          if (G) {
#pragma unroll
            for (int e = 0; e < CPT; ++e) {
              // phi+ +- phi- in integers, one exact conversion each (the low word
              // of 1.5 * 2^52 carries x + 2^31)
              const int bp = (int)(int8_t)(wv[g] >> (8 * e)), bn = (int)(int8_t)(wm[g] >> (8 * e));
              if (ONE) {
                const double xr = __hiloint2double(0x43380000, (bp + bn) ^ 0x80000000) - 6755401588539392.0;
                const double xi = __hiloint2double(0x43380000, (bp - bn) ^ 0x80000000) - 6755401588539392.0;
#pragma unroll
                for (int j = 0; j < NC; ++j) {
                  S[e][j] = fma(xr, p.w[l0 + g][j], S[e][j]);  // exact: < 2^53
                  S2[e][j] = fma(xi, p.w_im[l0 + g][j], S2[e][j]);
                }
              } else {
                const int xs = plane == 0 ? bp + bn : bp - bn;
                const double x = __hiloint2double(0x43380000, xs ^ 0x80000000) - 6755401588539392.0;
#pragma unroll
                for (int j = 0; j < NC; ++j) S[e][j] = fma(x, W[l0 + g][j], S[e][j]);  // exact: < 2^53
              }
            }
          } else {
            // int8 -> double without I2F: the byte with its sign bit flipped is
            // x + 128 in [0, 255]; as the low word of 0x4338000000000000 it reads
            // 1.5 * 2^52 + x + 128, so one DADD recovers x exactly.
            const uint32_t w4 = wv[g] ^ 0x80808080u;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const double x = __hiloint2double(0x43380000, (w4 >> (8 * e)) & 0xFF) - 6755399441055872.0;
#pragma unroll
              for (int j = 0; j < NC; ++j) S[e][j] = fma(x, p.w[l0 + g][j], S[e][j]);  // exact: < 2^52
            }
          }
        }
      }
#pragma unroll
      for (int e = 0; e < CPT; ++e) {
        const int j = j0 + e;
        if (j >= p.N) break;
        const int sigma = p.beta_b - eb[j];
        if (G && (OUT == SR_MAT_F64 || OUT == SR_MAT_C64) && (ADD < 0 || ADD == SR_MAT_F64)) {
          const size_t oa = (size_t)i * p.ld_add + j;
          const double xr = ADD == SR_MAT_F64 ? add.re[oa] : 0.0, xi = ADD == SR_MAT_F64 ? add.im[oa] : 0.0;
          const double vr = crt_lean<NC, ADD>(p, S[e], i, j, -(rho + sigma), 0, xr);
          const double vi = crt_lean<NC, ADD>(p, S2[e], i, j, -(rho + sigma), 1, xi);
          const size_t o = (size_t)i * p.ld_out + j;
          if (OUT == SR_MAT_F64) {
            out.re[o] = vr;
            out.im[o] = vi;
          } else {
            reinterpret_cast<float2*>(out.re)[o] = make_float2((float)vr, (float)vi);
          }
          continue;
        }
        finish_store<NC, OUT, ADD>(p, S[e], i, j, rho, sigma, plane, add, out);
        if (ONE) finish_store<NC, OUT, ADD>(p, S2[e], i, j, rho, sigma, 1, add, out);
      }
    }
  }
}

// Hermitian products are computed on the lower 128 x 128 tiles only; fill the
// strictly-upper tiles with the conjugate transpose (smem-tiled, coalesced).
// planes: (re, im) or dd (re, im, re_lo, im_lo); imaginary planes are negated
// (Hermitian, sign = 1) or the real planes are (skew-Hermitian, sign = -1).
__global__ void __launch_bounds__(256) mirror_kernel(int n, Dst d, int nplanes, long long ld, double sign) {
  __shared__ double t[32][33];
  const int bi = blockIdx.y, bj = blockIdx.x;  // destination 32-tile (bi, bj), bj > bi
  if ((bj >> 2) <= (bi >> 2)) return;           // only strictly-upper 128-tiles
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int q = 0; q < nplanes; ++q) {
    double* pl = q == 0 ? d.re : (q == 1 ? d.im : (q == 2 ? d.re_lo : d.im_lo));
    const double s2 = (q & 1) ? -sign : sign;  // sign * conj: re -> sign*re, im -> -sign*im
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {  // read source tile (bj, bi), coalesced
      const int si = bj * 32 + r, sj = bi * 32 + tx;
      if (si < n && sj < n) t[r][tx] = pl[(size_t)si * ld + sj];
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
      const int di = bi * 32 + r, dj = bj * 32 + tx;
      if (di < n && dj < n) pl[(size_t)di * ld + dj] = s2 * t[tx][r];
    }
  }
}

// Same for an interleaved lp output (complex64 / complex128).
template <typename CT>
__global__ void __launch_bounds__(256) mirror_lp_kernel(int n, CT* d, long long ld, float sign) {
  __shared__ CT t[32][33];
  const int bi = blockIdx.y, bj = blockIdx.x;
  if ((bj >> 2) <= (bi >> 2)) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int si = bj * 32 + r, sj = bi * 32 + tx;
    if (si < n && sj < n) t[r][tx] = d[(size_t)si * ld + sj];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int di = bi * 32 + r, dj = bj * 32 + tx;
    if (di < n && dj < n) {
      CT v = t[tx][r];
      v.x = sign * v.x;
      v.y = -sign * v.y;
      d[(size_t)di * ld + dj] = v;
    }
  }
}

// ---- tensor-core CRT decode (Gaussian residues) -----------------------------
// The decode's chunk sums S_j = sum_l (phi+_l + phi-_l) w_lj (real part) and
// sum_l (phi+_l - phi-_l) w'_lj (imaginary part) are a tiny integer matrix
// product per output entry: K = 2 nmod residue slots (phi+, phi- of every
// modulus) against 6 balanced base-256 digits of every kept 40-bit weight
// chunk.  One tcgen05 kind::i8 MMA (M = 128 output entries, N = 2 planes x NC
// chunks x 6 digits, K = 32 or 64) forms all digit sums T exactly (|T| < 2^20,
// int32 in TMEM); the epilogue recombines S_j = sum_d T_d 256^d exactly in
// FP64 (|S_j| < 2^53) and runs the same CRT finish as decode_kernel, so the
// result is bit-identical to it.  The A operand is the residue buffer itself,
// read MN-major: a 4-d TMA box (128 columns, 1 row, 2 planes, 32 moduli, the
// moduli beyond nmod zero-filled) lands as 64 slot rows of 128 bytes in the
// canonical 128-byte-swizzled MN-major layout.  The SIMT decode spent ~8 FP64
// instructions per (entry, modulus) on these sums (~150 of its ~300 per
// entry); here they cost 5 per (entry, chunk, plane).
#ifndef SR_DTC_TB  // measured at n = 8192 (hp decode): (2, 4, 1) 1.07 ms, (4, 2, 2) 1.44, (2, 5, 1) 1.11, (1, 6, 1) 1.77
#define SR_DTC_TB 2
#define SR_DTC_NG 4
#define SR_DTC_TPL 1
#endif
constexpr int DTC_TB = SR_DTC_TB;               // 128-column tiles per work unit (one row)
constexpr int DTC_NG = SR_DTC_NG;               // epilogue warpgroups, one TMEM accumulator (unit) each
constexpr int DTC_TPL = SR_DTC_TPL;             // tiles an epilogue lane finishes at once
constexpr int DTC_THREADS = 64 + 128 * DTC_NG;  // warp 0 TMA, warp 1 MMA, then the epilogue groups
#ifndef SR_DTC_STAGES
#define SR_DTC_STAGES 4
#endif
constexpr int DTC_STAGES = SR_DTC_STAGES;       // ring slots of one unit each
constexpr int DTC_TILE = 64 * 128;              // 64 slot rows x 128 output columns (bytes)
constexpr int DTC_UNIT = DTC_TB * DTC_TILE;
constexpr int DTC_DIGITS = 6;                   // balanced base-256 digits of a 40-bit weight chunk
constexpr int DTC_BROWS = 48;                   // MMA N rows of the weight image (2 planes x <= 4 chunks x 6 digits)
constexpr int DTC_BBYTES = DTC_BROWS * 64;
#ifndef SR_DTC_TCOLS
#define SR_DTC_TCOLS 64
#endif
constexpr int DTC_TCOLS = SR_DTC_TCOLS;         // TMEM columns per tile accumulator (>= the MMA N)
constexpr int DTC_ACC_COLS = DTC_TCOLS * DTC_TB;  // one unit's accumulators
constexpr int DTC_TMEM_COLS = DTC_ACC_COLS * DTC_NG <= 32 ? 32 : DTC_ACC_COLS * DTC_NG <= 64 ? 64 : DTC_ACC_COLS * DTC_NG <= 128 ? 128 : DTC_ACC_COLS * DTC_NG <= 256 ? 256 : 512;
constexpr int DTC_SMEM = 1024 + DTC_STAGES * DTC_UNIT + DTC_BBYTES + 256;

struct DecodeTcArgs {
  int tiles_n;     // 128-column tiles per output row
  int units_n;     // units per output row
  int rows;        // output rows
  int herm;        // Hermitian: only tiles of the lower 128 x 128 GEMM tiles
  int kmma;        // K = 32 MMAs per tile (2 nmod slots)
  int tile_bytes;  // bytes the TMA box writes per tile (2 nmod slot rows x 128)
  uint32_t idesc;  // instruction descriptor
  alignas(16) int8_t bimg[DTC_BBYTES];  // weight digits, [N rows][64 slots], K-major, 64-byte swizzle
};

// UMMA descriptor, MN-major, 128-byte swizzle: 128 bytes along M per row, 8-row
// groups of K 1024 B apart (one 128-element atom along M, so LBO is unused)
__device__ __forceinline__ uint64_t umma_desc_mn_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(DTC_TILE >> 4) << 16;  // LBO: stride between 128-element M atoms (unused for M = 128)
  d |= (uint64_t)(1024 >> 4) << 32;      // SBO: 8 K rows x 128 B
  d |= (uint64_t)1 << 46;                // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void umma_i8_mn(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// exact int32 -> double (|x| < 2^31) without the conversion pipe
__device__ __forceinline__ double i2d_exact(int x) {
  return __hiloint2double(0x43380000, x ^ 0x80000000) - 6755401588539392.0;
}

// S = sum_d T[d] 256^d, exact (|T| < 2^20, |S| < 2^53): digit pairs in int32
// (|u| < 2^29), the low two pairs as an int64 below 2^45 converted with the
// 1.5 * 2^52 bias, the top pair with the int32 bias, one FMA
__device__ __forceinline__ double digits_to_chunk(const uint32_t* T) {
  const int u0 = (int)T[0] + ((int)T[1] << 8), u1 = (int)T[2] + ((int)T[3] << 8), u2 = (int)T[4] + ((int)T[5] << 8);
  const long long lo = ((long long)u1 << 16) + (long long)u0;
  const double dlo = __longlong_as_double(lo + 0x4338000000000000LL) - 6755399441055744.0;
  return fma(i2d_exact(u2), 4294967296.0, dlo);
}

// one unit = DTC_TB column tiles of row i; tile b valid when inside the matrix
// and (Hermitian) inside the lower 128 x 128 GEMM tiles
__device__ __forceinline__ int unit_mask_at(const DecodeTcArgs& t, int i, int r, int& jt0) {
  jt0 = r * DTC_TB;
  const int hi = t.herm ? min(t.tiles_n, (i >> 7) + 1) : t.tiles_n;
  const int nv = max(0, min(DTC_TB, hi - jt0));
  return (1 << nv) - 1;
}

// a CTA's units u = blockIdx.x + k grid as (row i, unit r in the row), stepped
// without integer divisions (their I2F / MUFU.RCP / F2I sequences ran on the
// narrow XU pipe of every epilogue warp: 12 % XU issue in the decode)
struct UnitIt {
  int u, i, r;
  int gq, gr;  // grid = gq units_n + gr
  __device__ __forceinline__ void init(const DecodeTcArgs& t, int u0, int grid) {
    u = u0;
    i = u0 / t.units_n;
    r = u0 - i * t.units_n;
    gq = grid / t.units_n;
    gr = grid - gq * t.units_n;
  }
  __device__ __forceinline__ void step(const DecodeTcArgs& t, int grid) {
    u += grid;
    i += gq;
    r += gr;
    if (r >= t.units_n) {
      r -= t.units_n;
      ++i;
    }
  }
  __device__ __forceinline__ int mask(const DecodeTcArgs& t, int& row, int& jt0) const {
    row = i;
    return unit_mask_at(t, i, r, jt0);
  }
};

// Persistent, warp-specialised, one CTA per SM.  The TMA warp streams units
// (DTC_TB x 128 output columns of one row: one 4-d box of 2 nmod slot rows per
// tile) through a 4-slot ring; a single thread issues each tile's MMAs (K = 32
// per MMA, descriptors as offsets of per-CTA bases) into a DTC_TCOLS-column
// slice of one of DTC_NG TMEM accumulators; the DTC_NG epilogue warpgroups
// take the units round-robin, each lane finishing one entry per tile while
// the operands of its group's next unit (exponents, X) load.  Measured
// (tools/crt_bench.py, n = 8192 hp decode): the memory / MMA path alone runs at
// 0.61 ms (5.9 TB/s); the FP64 finish is latency-bound, so the split of TMEM
// into four groups of two tiles (16 epilogue warps) beats two groups of four
// (1.07 vs 1.44 ms).
template <int NC, int OUT, int ADD>
__global__ void __launch_bounds__(DTC_THREADS, 1)
    decode_tc_kernel(const __grid_constant__ CUtensorMap map, const __grid_constant__ DecodeParams p,
                     const __grid_constant__ DecodeTcArgs t, const int* __restrict__ ea,
                     const int* __restrict__ eb, Src add, Dst out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* bsm = smem + DTC_STAGES * DTC_UNIT;
  uint64_t* bars = (uint64_t*)(bsm + DTC_BBYTES);  // full[S], empty[S], tfull[NG], tempty[NG]; tmem slot
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * DTC_STAGES + 2 * DTC_NG);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (DTC_STAGES + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * DTC_STAGES + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * DTC_STAGES + DTC_NG + a); };

  // the weight image, and zeros in the slot rows the TMA boxes never write (K padding)
  for (int x = threadIdx.x; x < DTC_BBYTES / 16; x += DTC_THREADS)
    reinterpret_cast<int4*>(bsm)[x] = reinterpret_cast<const int4*>(t.bimg)[x];
  const int pad16 = (DTC_TILE - t.tile_bytes) / 16;
  for (int x = threadIdx.x; x < DTC_STAGES * DTC_TB * pad16; x += DTC_THREADS) {
    const int tile = x / pad16, o = x - tile * pad16;
    reinterpret_cast<int4*>(smem + tile * DTC_TILE + t.tile_bytes)[o] = make_int4(0, 0, 0, 0);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes read by the async proxy
  if (threadIdx.x == 0) {
    for (int s = 0; s < DTC_STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < DTC_NG; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&map) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(DTC_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  const int total = t.rows * t.units_n;
  const int grid = gridDim.x;

  if (warp == 0) {
    if (lane == 0) {
      int k = 0;
      UnitIt it;
      for (it.init(t, blockIdx.x, grid); it.u < total; it.step(t, grid)) {
        int i, jt0;
        const int m = it.mask(t, i, jt0);
        if (!m) continue;
        const int s = k % DTC_STAGES;
        if (k >= DTC_STAGES) mbar_wait(empty_bar(s), ((k / DTC_STAGES) - 1) & 1);
        mbar_expect_tx(full_bar(s), __popc(m) * t.tile_bytes);
        for (int b = 0; b < DTC_TB; ++b)
          if (m >> b & 1)
            tma_load_4d(smem_u32(smem + s * DTC_UNIT + b * DTC_TILE), &map, full_bar(s), (jt0 + b) * 128, i, 0, 0);
        ++k;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // single-thread MMA issuer: descriptors are offsets of per-CTA bases
      const uint64_t bd0 = umma_desc_sw64(smem_u32(bsm));
      const uint64_t ad0 = umma_desc_mn_sw128(smem_u32(smem));
      const uint32_t idesc = t.idesc;
      const bool two = t.kmma > 1;
      int k = 0;
      UnitIt it;
      for (it.init(t, blockIdx.x, grid); it.u < total; it.step(t, grid)) {
        int i, jt0;
        const int m = it.mask(t, i, jt0);
        if (!m) continue;
        const int s = k % DTC_STAGES, g = k % DTC_NG, r = k / DTC_NG;
        mbar_wait(tempty_bar(g), (r & 1) ^ 1);
        mbar_wait(full_bar(s), (k / DTC_STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t d0 = tmem_base + (uint32_t)(g * DTC_ACC_COLS);
        const uint64_t as = ad0 + (uint64_t)((s * DTC_UNIT) >> 4);
#pragma unroll
        for (int b = 0; b < DTC_TB; ++b) {
          if (m >> b & 1) {  // K = 32 slots per MMA: 32 rows of the A tile (4 KB), 32 bytes of a B row
            umma_i8_mn(d0 + b * DTC_TCOLS, as + (uint64_t)((b * DTC_TILE) >> 4), bd0, idesc, 0u);
            if (two) umma_i8_mn(d0 + b * DTC_TCOLS, as + (uint64_t)((b * DTC_TILE + 4096) >> 4), bd0 + 2, idesc, 1u);
          }
        }
        umma_commit(empty_bar(s));
        umma_commit(tfull_bar(g));
        ++k;
      }
    }
  } else {
    const int g = (warp - 2) >> 2;  // epilogue group: this CTA's live units k = g, g + NG, ...
    const int q = warp & 3;         // TMEM lane quadrant = output columns 32 q .. 32 q + 31 of each tile
    struct Pre {
      int i, m, jt0, rho;
      int sigma[DTC_TB];
      double xr[DTC_TB], xi[DTC_TB];
    };
    // the unit after u among this group's units (NG live units on)
    auto next_unit = [&](UnitIt u, int steps) {
      for (int c = 0; c < steps;) {
        u.step(t, grid);
        if (u.u >= total) return u;
        int i, jt0;
        if (u.mask(t, i, jt0)) ++c;
      }
      return u;
    };
    auto prefetch = [&](const UnitIt& u, Pre& r) {
      r.m = 0;
      if (u.u >= total) return;
      r.m = u.mask(t, r.i, r.jt0);
      r.rho = p.beta_a - __ldg(ea + r.i);
#pragma unroll
      for (int b = 0; b < DTC_TB; ++b) {
        const int j = (r.jt0 + b) * 128 + q * 32 + lane;
        if ((r.m >> b & 1) && j < p.N) {
          r.sigma[b] = p.beta_b - __ldg(eb + j);
          if (ADD == SR_MAT_F64) {
            const size_t oa = (size_t)r.i * p.ld_add + j;
            r.xr[b] = add.re[oa];
            r.xi[b] = add.im[oa];
          }
        }
      }
    };
    UnitIt u;
    u.init(t, blockIdx.x, grid);
    {
      int i, jt0;
      if (u.u < total && !u.mask(t, i, jt0)) u = next_unit(u, 1);
    }
    u = next_unit(u, g);  // this group's first unit
    // two operand sets, software-pipelined: the loads for a unit are issued a
    // whole unit of work before their first use
    auto process = [&](const Pre& cur, int r) {
      mbar_wait(tfull_bar(g), r & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(g * DTC_ACC_COLS);
#pragma unroll
      for (int b0 = 0; b0 < DTC_TB; b0 += DTC_TPL) {
        uint32_t v[DTC_TPL][48];
#pragma unroll
        for (int h = 0; h < DTC_TPL; ++h) {
          tmem_ld16(ta + (b0 + h) * DTC_TCOLS, *reinterpret_cast<uint32_t(*)[16]>(&v[h][0]));
          tmem_ld16(ta + (b0 + h) * DTC_TCOLS + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[h][16]));
          if (2 * NC * DTC_DIGITS > 32) tmem_ld16(ta + (b0 + h) * DTC_TCOLS + 32, *reinterpret_cast<uint32_t(*)[16]>(&v[h][32]));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (b0 + DTC_TPL >= DTC_TB) {  // the whole accumulator is in registers: release it to the MMA warp
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
          mbar_arrive(tempty_bar(g));
        }
#pragma unroll
        for (int h = 0; h < DTC_TPL; ++h) {
          const int b = b0 + h;
          const int j = (cur.jt0 + b) * 128 + q * 32 + lane;
          if (!((cur.m >> b & 1) && j < p.N)) continue;
#ifdef SR_DTC_NOFINISH  // A/B diagnostic: the memory / MMA path without the FP64 finish
          if (OUT == SR_MAT_F64) {
            const size_t o = (size_t)cur.i * p.ld_out + j;
            out.re[o] = (double)(int)(v[h][0] + v[h][5] + v[h][11]);
            out.im[o] = (double)(int)(v[h][17] + v[h][23] + v[h][29]);
          }
          continue;
#endif
          double hv[2];
#pragma unroll
          for (int pl = 0; pl < 2; ++pl) {
            double S[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) S[c] = digits_to_chunk(&v[h][(pl * NC + c) * DTC_DIGITS]);
            hv[pl] = crt_lean<NC, ADD>(p, S, cur.i, j, -(cur.rho + cur.sigma[b]), pl,
                                       ADD == SR_MAT_F64 ? (pl == 0 ? cur.xr[b] : cur.xi[b]) : 0.0);
          }
          const size_t o = (size_t)cur.i * p.ld_out + j;
          if (OUT == SR_MAT_F64) {
            out.re[o] = hv[0];
            out.im[o] = hv[1];
          } else {
            reinterpret_cast<float2*>(out.re)[o] = make_float2((float)hv[0], (float)hv[1]);
          }
        }
      }
    };
    Pre A, B;
    prefetch(u, A);
    UnitIt ub = next_unit(u, DTC_NG);
    prefetch(ub, B);
    for (int r = 0; u.u < total; r += 2) {
      process(A, r);
      const UnitIt ua = next_unit(ub, DTC_NG);
      prefetch(ua, A);
      if (ub.u >= total) break;
      process(B, r + 1);
      const UnitIt ub2 = next_unit(ua, DTC_NG);
      prefetch(ub2, B);
      u = ua;
      ub = ub2;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(DTC_TMEM_COLS));
}

// decode path selection (sr_oz_set_options): 1 = tensor-core decode where it applies
int g_decode_tc = 1;

// weight digit image + TMA map; false when the tensor-core decode does not apply
bool decode_tc_prepare(const DecodeParams& p, const double* table, int nchunk, const void* res,
                       long long res_pitch, int hermitian, DecodeTcArgs* t, CUtensorMap* map) {
  // nchunk 2 (the lp products): the SIMT decode is as fast (0.84 vs 0.91 ms at n = 8192)
  if (!g_decode_tc || nchunk < 3 || nchunk > 4 || p.nmod > 32 || (res_pitch & 15) ||
      ((uintptr_t)res & 15))
    return false;
  auto enc = get_encode();
  if (!enc) return false;
  memset(t, 0, sizeof(*t));
  t->tiles_n = (p.N + 127) / 128;
  t->units_n = (t->tiles_n + DTC_TB - 1) / DTC_TB;
  t->rows = p.M;
  t->tile_bytes = 2 * p.nmod * 128;
  t->herm = hermitian != 0;
  t->kmma = (2 * p.nmod + 31) / 32;
  const int ncols = 2 * nchunk * DTC_DIGITS <= 32 ? 32 : 48;
  // D = S32, A = B = S8, A MN-major, B K-major, M = 128
  t->idesc = (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(ncols >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const int nmod = p.nmod;
  const double* w_im = table + nmod * MAXCHUNK + 2 * MAXCHUNK + 1;
  for (int pl = 0; pl < 2; ++pl)
    for (int c = 0; c < nchunk; ++c)
      for (int l = 0; l < nmod; ++l)
        for (int g = 0; g < 2; ++g) {  // slot 2 l + g: phi+ (g = 0), phi- (g = 1)
          long long w = (long long)(pl == 0 ? table[l * MAXCHUNK + c] : w_im[l * MAXCHUNK + c]);
          if (pl == 1 && g == 1) w = -w;  // im = (phi+ - phi-) / (2 iota)
          const int slot = 2 * l + g;
          for (int d = 0; d < DTC_DIGITS; ++d) {
            long long r = w & 255;
            if (r >= 128) r -= 256;
            w = (w - r) >> 8;
            const int n = (pl * nchunk + c) * DTC_DIGITS + d;
            const int off = n * 64 + ((((slot >> 4) ^ ((n >> 1) & 3)) << 4) | (slot & 15));
            t->bimg[off] = (int8_t)r;
          }
          if (w != 0) return false;  // not a 40-bit chunk
        }
  cuuint64_t dims[4] = {(cuuint64_t)p.N, (cuuint64_t)p.M, 2, (cuuint64_t)nmod};
  cuuint64_t strides[3] = {(cuuint64_t)res_pitch, (cuuint64_t)(res_pitch * p.M), (cuuint64_t)(2 * res_pitch * p.M)};
  cuuint32_t box[4] = {128, 1, 2, (cuuint32_t)nmod};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(res), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int NC, int OUT, int ADD>
int launch_decode_tc(cudaStream_t st, const CUtensorMap& map, const DecodeParams& p, const DecodeTcArgs& t,
                     const int* ea, const int* eb, Src add, Dst out) {
  static bool configured[SR_MAX_DEVICES] = {};
  int slot = 0;
  if (sr_device_slot(&slot) != SR_OK) return SR_EINVAL;
  if (!configured[slot]) {
    SR_CUDA_CHECK(cudaFuncSetAttribute(decode_tc_kernel<NC, OUT, ADD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       DTC_SMEM));
    configured[slot] = true;
  }
  long long units = (long long)t.rows * t.units_n;
  int grid = (int)std::min<long long>(units, 148LL);
  decode_tc_kernel<NC, OUT, ADD><<<grid, DTC_THREADS, DTC_SMEM, st>>>(map, p, t, ea, eb, add, out);
  return SR_OK;
}

template <int NC>
int dispatch_gauss_tc(int out_kind, int add_kind, cudaStream_t st, const CUtensorMap& map, const DecodeParams& p,
                      const DecodeTcArgs& t, const int* ea, const int* eb, Src add, Dst out) {
  if (add_kind >= 0 && add_kind != SR_MAT_F64) return SR_EINVAL;
  if (out_kind == SR_MAT_F64)
    return add_kind == SR_MAT_F64 ? launch_decode_tc<NC, SR_MAT_F64, SR_MAT_F64>(st, map, p, t, ea, eb, add, out)
                                  : launch_decode_tc<NC, SR_MAT_F64, -1>(st, map, p, t, ea, eb, add, out);
  if (out_kind == SR_MAT_C64 && add_kind < 0) return launch_decode_tc<NC, SR_MAT_C64, -1>(st, map, p, t, ea, eb, add, out);
  return SR_EINVAL;
}

template <int NC, int OUT, int ADD>
void launch_decode(int grid, cudaStream_t st, const DecodeParams& p, const int8_t* res, const int* ea,
                   const int* eb, Src add, Dst out) {
  decode_kernel<NC, OUT, ADD><<<grid, 256, 0, st>>>(p, res, ea, eb, add, out);
}

// Gaussian residues: FP64-mode outputs only (planar FP64 or complex64; + FP64 X)
template <int NC>
int dispatch_gauss(int out_kind, int add_kind, int grid, cudaStream_t st, const DecodeParams& p, const int8_t* res,
                   const int* ea, const int* eb, Src add, Dst out) {
  if (add_kind >= 0 && add_kind != SR_MAT_F64) return SR_EINVAL;
  const bool with_add = add_kind == SR_MAT_F64;
  if (out_kind == SR_MAT_F64) {
    if (with_add)
      decode_kernel<NC, SR_MAT_F64, SR_MAT_F64, true><<<grid, 256, 0, st>>>(p, res, ea, eb, add, out);
    else
      decode_kernel<NC, SR_MAT_F64, -1, true><<<grid, 256, 0, st>>>(p, res, ea, eb, add, out);
  } else if (out_kind == SR_MAT_C64 && !with_add) {
    decode_kernel<NC, SR_MAT_C64, -1, true><<<grid, 256, 0, st>>>(p, res, ea, eb, add, out);
  } else {
    return SR_EINVAL;
  }
  return SR_OK;
}

template <int NC, int OUT>
int dispatch_add(int add_kind, int grid, cudaStream_t st, const DecodeParams& p, const int8_t* res, const int* ea,
                 const int* eb, Src add, Dst out) {
  if (add_kind < 0)
    launch_decode<NC, OUT, -1>(grid, st, p, res, ea, eb, add, out);
  else if (add_kind == SR_MAT_F64)
    launch_decode<NC, OUT, SR_MAT_F64>(grid, st, p, res, ea, eb, add, out);
  else if (add_kind == SR_MAT_DD)
    launch_decode<NC, OUT, SR_MAT_DD>(grid, st, p, res, ea, eb, add, out);
  else
    return SR_EINVAL;
  return SR_OK;
}

template <int NC>
int dispatch_out(int out_kind, int add_kind, int grid, cudaStream_t st, const DecodeParams& p, const int8_t* res,
                 const int* ea, const int* eb, Src add, Dst out) {
  switch (out_kind) {
    case SR_MAT_F64:
      return dispatch_add<NC, SR_MAT_F64>(add_kind, grid, st, p, res, ea, eb, add, out);
    case SR_MAT_C64:
      return dispatch_add<NC, SR_MAT_C64>(add_kind, grid, st, p, res, ea, eb, add, out);
    case SR_MAT_C128:
      return dispatch_add<NC, SR_MAT_C128>(add_kind, grid, st, p, res, ea, eb, add, out);
    case SR_MAT_DD:
      return dispatch_add<NC, SR_MAT_DD>(add_kind, grid, st, p, res, ea, eb, add, out);
  }
  return SR_EINVAL;
}

}  // namespace

namespace {
int exponents_launch(int rows, int cols, int kind, const void* re, const double* im, long long ld, int transposed,
                     int* exps, double* ss_work, double* rmax, cudaStream_t st) {
  if (rows < 0 || cols < 0 || !re || !exps || kind < 0 || kind > SR_MAT_DD) return SR_EINVAL;
  Src s{(const double*)re, im, nullptr, nullptr, kind};
  if (kind == SR_MAT_DD) kind = SR_MAT_F64;  // the hi parts decide the scale
  if (rmax) SR_CUDA_CHECK(cudaMemsetAsync(rmax, 0, sizeof(double), st));
  if (!transposed) {
    if (rows == 0) return SR_OK;
    const int grid = sr_ceil_div((long long)rows * 32, 256);
    if (kind == SR_MAT_F64) exps_direct_kernel<SR_MAT_F64><<<grid, 256, 0, st>>>(rows, cols, s, ld, exps, rmax);
    if (kind == SR_MAT_C64) exps_direct_kernel<SR_MAT_C64><<<grid, 256, 0, st>>>(rows, cols, s, ld, exps, rmax);
    if (kind == SR_MAT_C128) exps_direct_kernel<SR_MAT_C128><<<grid, 256, 0, st>>>(rows, cols, s, ld, exps, rmax);
  } else {
    if (cols == 0) return SR_OK;
    exps_fill_kernel<<<sr_ceil_div(cols, 256), 256, 0, st>>>(cols, exps);
    SR_LAUNCH_CHECK();
    double* ssum = rmax ? ss_work : nullptr;
    if (ssum) SR_CUDA_CHECK(cudaMemsetAsync(ssum, 0, (size_t)cols * sizeof(double), st));
    const int rpb = 256;
    dim3 g(sr_ceil_div(cols, 32), sr_ceil_div(rows, rpb));
    if (kind == SR_MAT_F64)
      exps_transposed_kernel<SR_MAT_F64><<<g, dim3(32, 8), 0, st>>>(rows, cols, s, ld, rpb, exps, ssum);
    if (kind == SR_MAT_C64)
      exps_transposed_kernel<SR_MAT_C64><<<g, dim3(32, 8), 0, st>>>(rows, cols, s, ld, rpb, exps, ssum);
    if (kind == SR_MAT_C128)
      exps_transposed_kernel<SR_MAT_C128><<<g, dim3(32, 8), 0, st>>>(rows, cols, s, ld, rpb, exps, ssum);
    if (ssum) {
      SR_LAUNCH_CHECK();
      bound_finish_kernel<<<sr_ceil_div(cols, 256), 256, 0, st>>>(cols, ssum, exps, rmax);
    }
  }
  SR_LAUNCH_CHECK();
  return SR_OK;
}
}  // namespace

extern "C" int sr_oz_exponents(int rows, int cols, int kind, const void* re, const double* im, long long ld,
                               int transposed, int* exps, void* stream) {
  return exponents_launch(rows, cols, kind, re, im, ld, transposed, exps, nullptr, nullptr, (cudaStream_t)stream);
}

extern "C" int sr_oz_exponents_bound(int rows, int cols, int kind, const void* re, const double* im, long long ld,
                                     int transposed, int* exps, double* ss_work, double* rmax, double* host_rmax,
                                     void* stream) {
  if (!rmax || (transposed && !ss_work)) return SR_EINVAL;
  const int rc = exponents_launch(rows, cols, kind, re, im, ld, transposed, exps, ss_work, rmax, (cudaStream_t)stream);
  if (rc != SR_OK || !host_rmax) return rc;
  publish_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(rmax, host_rmax);
  SR_LAUNCH_CHECK();
  return SR_OK;
}

namespace {
int encode_launch(int rows_out, int K, int kind, const void* re, const double* im, const double* re_lo,
                  const double* im_lo, long long ld, int transposed, int conj, int layout, const int* exps, int beta,
                  int nmod, const int* moduli, void* out, void* out2, long long kpitch, cudaStream_t st) {
  if (rows_out <= 0 || K <= 0 || nmod <= 0 || nmod > MAXMOD || layout < 0 || layout > 4) return SR_EINVAL;
  if (layout == 4 && kind == SR_MAT_DD) return SR_EINVAL;
  if (kind < 0 || kind > SR_MAT_DD || (kind == SR_MAT_DD && (!re_lo || !im_lo || !im))) return SR_EINVAL;
  const int max_beta = kind == SR_MAT_DD ? 106 : 61;
  if (beta < 1 || beta > max_beta || (kpitch & 15) || kpitch < K) return SR_EINVAL;
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
  p.out2 = (int8_t*)out2;
  p.ndig = (beta + 2 + 10) / 11;  // digits covering |a| <= 2^beta plus a carry
  if (p.ndig > MAXDIG) p.ndig = MAXDIG;
  for (int l = 0; l < nmod; ++l) {
    const int m = moduli[l];
    if (m < 3 || m > 256) return SR_EINVAL;
    p.pf[l] = (float)m;
    p.invf[l] = 1.0f / (float)m;
    p.hif[l] = (float)(((m + 1) >> 1) - 1);
    p.lof[l] = (float)(-(m >> 1));
    long long pw = 1;
    for (int c = 0; c < MAXDIG; ++c) {
      long long r = pw % m;
      if (r > ((m + 1) >> 1) - 1) r -= m;
      p.pow2[l][c] = (float)r;
      pw = (pw << 11) % m;
    }
    p.pi[l] = m;
    auto sym = [m](long long r) { r %= m; return r > ((m + 1) >> 1) - 1 ? r - m : r; };
    long long pb = 1;  // 2^(8c) mod m
    uint32_t words[2] = {0, 0};
    for (int c = 0; c < 8; ++c) {
      words[c / 4] |= ((uint32_t)(sym(pb) & 0xFF)) << (8 * (c % 4));
      pb = (pb << 8) % m;
    }
    p.wb[l][0] = (int)words[0];
    p.wb[l][1] = (int)words[1];
    p.c64[l] = (int)sym(pb);  // after 8 steps pb = 2^64 mod m
    p.bm[l] = (uint32_t)((1ull << 32) / (unsigned long long)m + 1);
    const int shift = (8 * 255 * 128 + 256 + m - 1) / m * m;  // > |byte dot products| + |2^64 mod m|
    p.off0[l] = shift + (m >> 1);  // + (-lo): the residue comes out in [0, m), then shifted by lo
    p.off1[l] = 0;
    if (layout == 4) {
      int io = 0;
      for (int x = 1; x < m && !io; ++x)
        if ((x * x + 1) % m == 0) io = x;
      if (!io || !(m & 1)) return SR_EINVAL;  // needs an odd modulus with a square root of -1
      long long pg = 1;  // 2^(8c) mod m
      uint32_t wp[2] = {0, 0}, wm[2] = {0, 0};
      for (int c = 0; c < 8; ++c) {
        wp[c / 4] |= ((uint32_t)(sym(io * pg) & 0xFF)) << (8 * (c % 4));
        wm[c / 4] |= ((uint32_t)(sym(m - io * pg % m) & 0xFF)) << (8 * (c % 4));
        pg = (pg << 8) % m;
      }
      p.wgp[l][0] = (int)wp[0];
      p.wgp[l][1] = (int)wp[1];
      p.wgm[l][0] = (int)wm[0];
      p.wgm[l][1] = (int)wm[1];
      p.cgp[l] = (int)sym(io * pg);  // pg = 2^64 mod m here
      const int bound = 16 * 255 * (m >> 1) + 2 * (m >> 1);  // |16 byte products| + |corrections|
      p.offg[l] = (bound + m - 1) / m * m + (m >> 1);        // a multiple of m above it, then -lo
      long long p63 = 1;
      for (int c = 0; c < 63; ++c) p63 = (p63 * 2) % m;  // 2^63 mod m
      p.offb[l] = p.offg[l] - (int)sym(p63);
      p.offi[l] = -(int)sym(io * p63);
    }
  }
  // K padding columns of the residue planes must read as zero
  const int planes = layout == 0 || layout == 3 || layout == 4 ? 2 : (layout == 1 ? 3 : 1);
  if (kpitch > K) {
    SR_CUDA_CHECK(cudaMemsetAsync(out, 0, (size_t)nmod * planes * rows_out * kpitch, st));
    if (out2) SR_CUDA_CHECK(cudaMemsetAsync(out2, 0, (size_t)nmod * 3 * rows_out * kpitch, st));
  }
  Src s{(const double*)re, im, re_lo, im_lo, kind};
  const int eti = kind == SR_MAT_DD ? 32 : 64;
  dim3 grid(sr_ceil_div(K, 32), sr_ceil_div(rows_out, eti));
  switch (kind) {
    case SR_MAT_F64:
      encode_kernel<SR_MAT_F64><<<grid, 256, 0, st>>>(p, s, exps, (int8_t*)out);
      break;
    case SR_MAT_C64:
      encode_kernel<SR_MAT_C64><<<grid, 256, 0, st>>>(p, s, exps, (int8_t*)out);
      break;
    case SR_MAT_C128:
      encode_kernel<SR_MAT_C128><<<grid, 256, 0, st>>>(p, s, exps, (int8_t*)out);
      break;
    default:
      encode_kernel<SR_MAT_DD><<<grid, 256, 0, st>>>(p, s, exps, (int8_t*)out);
  }
  SR_LAUNCH_CHECK();
  return SR_OK;
}
}  // namespace

extern "C" int sr_oz_encode(int rows_out, int K, int kind, const void* re, const double* im, const double* re_lo,
                            const double* im_lo, long long ld, int transposed, int conj, int layout,
                            const int* exps, int beta, int nmod, const int* moduli, void* out, long long kpitch,
                            void* stream) {
  if (layout == 3) return SR_EINVAL;  // the dual layout has its own entry (two outputs)
  return encode_launch(rows_out, K, kind, re, im, re_lo, im_lo, ld, transposed, conj, layout, exps, beta, nmod,
                       moduli, out, nullptr, kpitch, (cudaStream_t)stream);
}

extern "C" int sr_oz_encode_dual(int rows_out, int K, int kind, const void* re, const double* im,
                                 const double* re_lo, const double* im_lo, long long ld, const int* exps, int beta,
                                 int nmod, const int* moduli, void* out_ah, void* out_b, long long kpitch,
                                 void* stream) {
  if (!out_ah || !out_b) return SR_EINVAL;
  return encode_launch(rows_out, K, kind, re, im, re_lo, im_lo, ld, 1, 0, 3, exps, beta, nmod, moduli, out_ah,
                       out_b, kpitch, (cudaStream_t)stream);
}

// table (host): [nmod][6] CRT weights, [6] modulus-product chunks, [6] chunk
// offsets (as doubles), 1/P
namespace {
int decode_launch(int M, int N, int nmod, int nchunk, const double* table, const void* res, long long res_pitch,
                  const int* exps_a, int beta_a, const int* exps_b, int beta_b, double alpha, double shift,
                  int add_kind, const double* add_re, const double* add_im, const double* add_re_lo,
                  const double* add_im_lo, long long ld_add, double add_scale, int out_kind, void* out_re,
                  double* out_im, double* out_re_lo, double* out_im_lo, long long ld_out, int hermitian,
                  int diag_col0, bool gauss, void* stream) {
  if (gauss && hermitian < 0) return SR_EINVAL;  // Hermitian only (the GEMM's transpose shortcut)
  if (M <= 0 || N <= 0 || nmod <= 0 || nmod > MAXMOD || nchunk < 1 || nchunk > MAXCHUNK) return SR_EINVAL;
  if (res_pitch & 3) return SR_EINVAL;
  if (out_kind < 0 || out_kind > SR_MAT_DD) return SR_EINVAL;
  if ((out_kind == SR_MAT_F64 || out_kind == SR_MAT_DD) && !out_im) return SR_EINVAL;
  if (out_kind == SR_MAT_DD && (!out_re_lo || !out_im_lo)) return SR_EINVAL;
  if (add_kind >= 0 && !add_re) return SR_EINVAL;
  if (hermitian != 0 && (M != N || add_kind >= 0 || (hermitian != 1 && hermitian != -1))) return SR_EINVAL;
  DecodeParams p;
  memset(&p, 0, sizeof(p));
  p.M = M;
  p.N = N;
  p.nmod = nmod;
  p.nchunk = nchunk;
  p.beta_a = beta_a;
  p.beta_b = beta_b;
  p.hermitian = hermitian;
  p.diag_col0 = diag_col0;
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
  int off[MAXCHUNK];
  for (int j = 0; j < MAXCHUNK; ++j) {
    p.pc[j] = table[nmod * MAXCHUNK + j];
    off[j] = (int)table[nmod * MAXCHUNK + MAXCHUNK + j];
    p.offv[j] = ldexp(1.0, off[j]);
  }
  for (int j = 1; j < MAXCHUNK; ++j) {
    p.cw[j] = ldexp(1.0, off[j - 1] - off[j]);
    p.icw[j] = ldexp(1.0, -(off[j - 1] - off[j]));
  }
  p.inv_p = table[nmod * MAXCHUNK + 2 * MAXCHUNK];
  // fewer chunks than the plan holds: the dropped weight tails and the dropped
  // tail of k P move C' by less than 2 nmod 256 units of the lowest kept
  // chunk; snap to twice that grid
  bool truncated = false;
  for (int l = 0; l < nmod; ++l)
    for (int j = nchunk; j < MAXCHUNK; ++j) truncated = truncated || table[l * MAXCHUNK + j] != 0.0;
  if (truncated) {
    int bits = 10;  // 4 * 256
    while ((1 << (bits - 9)) < nmod) ++bits;
    p.snap = ldexp(1.0, bits);
    p.inv_snap = ldexp(1.0, -bits);
  }
  if (gauss)
    for (int l = 0; l < nmod; ++l)
      for (int j = 0; j < MAXCHUNK; ++j) p.w_im[l][j] = table[nmod * MAXCHUNK + 2 * MAXCHUNK + 1 + l * MAXCHUNK + j];
  const long long total = (long long)M * ((N + 3) / 4);
  int grid = (int)((total + 255) / 256);
  if (grid > 148 * 16) grid = 148 * 16;
  cudaStream_t st = (cudaStream_t)stream;
  Src add{add_re, add_im, add_re_lo, add_im_lo, add_kind};
  Dst out{(double*)out_re, out_im, out_re_lo, out_im_lo};
  int rc;
  static thread_local DecodeTcArgs tca;  // host staging of the kernel argument (3 KB)
  CUtensorMap tmap;
  if (gauss && decode_tc_prepare(p, table, nchunk, res, res_pitch, hermitian, &tca, &tmap)) {
    rc = nchunk == 2   ? dispatch_gauss_tc<2>(out_kind, add_kind, st, tmap, p, tca, exps_a, exps_b, add, out)
         : nchunk == 3 ? dispatch_gauss_tc<3>(out_kind, add_kind, st, tmap, p, tca, exps_a, exps_b, add, out)
                       : dispatch_gauss_tc<4>(out_kind, add_kind, st, tmap, p, tca, exps_a, exps_b, add, out);
  } else if (gauss) {
    const int8_t* r8 = (const int8_t*)res;
    // nchunk: the top CRT chunks the output's precision needs (OzPlan.decode_chunks)
    rc = nchunk <= 2    ? dispatch_gauss<2>(out_kind, add_kind, grid, st, p, r8, exps_a, exps_b, add, out)
         : nchunk == 3  ? dispatch_gauss<3>(out_kind, add_kind, grid, st, p, r8, exps_a, exps_b, add, out)
         : nchunk == 4  ? dispatch_gauss<4>(out_kind, add_kind, grid, st, p, r8, exps_a, exps_b, add, out)
                        : dispatch_gauss<6>(out_kind, add_kind, grid, st, p, r8, exps_a, exps_b, add, out);
  } else {
  switch (nchunk) {
    case 1:
    case 2:
      rc = dispatch_out<2>(out_kind, add_kind, grid, st, p, (const int8_t*)res, exps_a, exps_b, add, out);
      break;
    case 3:
      rc = dispatch_out<3>(out_kind, add_kind, grid, st, p, (const int8_t*)res, exps_a, exps_b, add, out);
      break;
    case 4:
      rc = dispatch_out<4>(out_kind, add_kind, grid, st, p, (const int8_t*)res, exps_a, exps_b, add, out);
      break;
    default:
      rc = dispatch_out<6>(out_kind, add_kind, grid, st, p, (const int8_t*)res, exps_a, exps_b, add, out);
  }
  }
  if (rc != SR_OK) return rc;
  SR_LAUNCH_CHECK();
  if (hermitian) {
    dim3 g(sr_ceil_div(N, 32), sr_ceil_div(M, 32));
    if (out_kind == SR_MAT_C64)
      mirror_lp_kernel<float2><<<g, 256, 0, st>>>(M, (float2*)out_re, ld_out, (float)hermitian);
    else if (out_kind == SR_MAT_C128)
      mirror_lp_kernel<double2><<<g, 256, 0, st>>>(M, (double2*)out_re, ld_out, (float)hermitian);
    else
      mirror_kernel<<<g, 256, 0, st>>>(M, out, out_kind == SR_MAT_DD ? 4 : 2, ld_out, (double)hermitian);
    SR_LAUNCH_CHECK();
  }
  return SR_OK;
}
}  // namespace

extern "C" int sr_oz_decode(int M, int N, int nmod, int nchunk, const double* table, const void* res,
                            long long res_pitch, const int* exps_a, int beta_a, const int* exps_b, int beta_b,
                            double alpha, double shift, int add_kind, const double* add_re, const double* add_im,
                            const double* add_re_lo, const double* add_im_lo, long long ld_add, double add_scale,
                            int out_kind, void* out_re, double* out_im, double* out_re_lo, double* out_im_lo,
                            long long ld_out, int hermitian, int diag_col0, void* stream) {
  return decode_launch(M, N, nmod, nchunk, table, res, res_pitch, exps_a, beta_a, exps_b, beta_b, alpha, shift,
                       add_kind, add_re, add_im, add_re_lo, add_im_lo, ld_add, add_scale, out_kind, out_re, out_im,
                       out_re_lo, out_im_lo, ld_out, hermitian, diag_col0, false, stream);
}

extern "C" int sr_oz_decode_gauss(int M, int N, int nmod, int nchunk, const double* table, const void* res,
                                  long long res_pitch, const int* exps_a, int beta_a, const int* exps_b, int beta_b,
                                  double alpha, double shift, int add_kind, const double* add_re,
                                  const double* add_im, long long ld_add, double add_scale, int out_kind,
                                  void* out_re, double* out_im, long long ld_out, int hermitian, int diag_col0,
                                  void* stream) {
  return decode_launch(M, N, nmod, nchunk, table, res, res_pitch, exps_a, beta_a, exps_b, beta_b, alpha, shift,
                       add_kind, add_re, add_im, nullptr, nullptr, ld_add, add_scale, out_kind, out_re, out_im,
                       nullptr, nullptr, ld_out, hermitian, diag_col0, true, stream);
}

// Ozaki path options (tests / A-B tools).  key 0: tensor-core CRT decode of
// Gaussian residues (1, default) or the SIMT decode_kernel (0).  Returns the
// previous value, or -1 for an unknown key.
extern "C" int sr_oz_config(int key, int value) {
  if (key == 0) {
    const int old = g_decode_tc;
    if (value >= 0) g_decode_tc = value ? 1 : 0;
    return old;
  }
  return -1;
}

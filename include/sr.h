/*
 * libsr — B200-native Schur-refinement kernels, C ABI.
 *
 * The drop-in boundary for the hot path of the reference package `ddschur`
 * (/root/reference/pkg/src/ddschur): `refine_template` and the operators it
 * calls.  The reference's "FFI" is Python calling its numba kernels with
 * caller-allocated output planes and no error path
 * (matmul.py:71-77 -> _numba_kernels.gemm_hp / gemm_lp).  Every entry below
 * replaces one such call site (cited per entry).  Conventions:
 *   - plain device pointers, sizes and leading dimensions (in elements);
 *     row-major storage, element (i, j) at i*ld + j;
 *   - hp complex matrices are planar (separate re / im float64 planes),
 *     lp complex matrices interleaved (complex64 = 8-byte float2 pairs,
 *     complex128 = 16-byte double2 pairs);
 *   - the caller (PyTorch on the Python side) owns every buffer; the library
 *     allocates nothing per call; workspaces are caller-provided;
 *   - all work is stream-ordered on `stream` (a cudaStream_t); results that
 *     are scalars (norms, flags, counts) are written to device memory;
 *   - every entry returns an int status: SR_OK or an SR_E* code; the message
 *     of the last failure is available from sr_last_error().
 * No entry has a CPU fallback: without a CUDA device they return SR_ECUDA.
 */
#ifndef SR_H_
#define SR_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (Python maps them onto the reference's exception classes:
   ValueError, SeparationError, NonFiniteError — trisolve.py:50-55) */
#define SR_OK 0
#define SR_EINVAL 1
#define SR_ESEPARATION 2
#define SR_ENONFINITE 3
#define SR_ECUDA 4

/* device flag bits written by the solver / norm kernels */
#define SR_FLAG_SEPARATION 1
#define SR_FLAG_NONFINITE 2

/* op(A) selector: A or its conjugate transpose (matmul.py:64, trans_a) */
#define SR_OP_N 0
#define SR_OP_C 1

#define SR_TRISOLVE_MAX_CTAS 1184 /* 8 x 148 SMs: cap on tiles x splits per level */

int sr_version(void);
const char* sr_last_error(void);
/* number of kernels this process has launched through libsr (bench evidence) */
unsigned long long sr_kernel_launches(void);

/* hp product in FP64 mode: C = alpha * op(A) * B, then C_ii += diag_shift.
   Replaces matmul_hp (matmul.py:52-81) -> gemm_hp (_numba_kernels.py:18-46).
   b_im == NULL means B is real (config 3's real A in Q^H A).  lda/ldb/ldc
   even and planes 16-byte aligned. */
int sr_zgemm_f64(int op_a, int m, int n, int k, double alpha, double diag_shift, const double* a_re,
                 const double* a_im, long long lda, const double* b_re, const double* b_im, long long ldb,
                 double* c_re, double* c_im, long long ldc, void* stream);

/* lp product in FP64 mode (complex64): C = op(A) * B.
   Replaces matmul_lp (matmul.py:84-110) -> gemm_lp (_numba_kernels.py:49-69). */
int sr_cgemm_c64(int op_a, int m, int n, int k, const void* a, long long lda, const void* b, long long ldb,
                 void* c, long long ldc, void* stream);

/* Split T^ into lp T (upper incl. diagonal) and lp E (strictly lower), both
   complex64, and ||E||_F of the hp values into *d_norm_e (FP64).
   Replaces stril_extract (ddmatrix.py:190-209) + frobenius_norm (216-251)
   + the .to_lp() downcasts at refine.py:263-264,284. */
int sr_split_lp_c64(int n, const double* that_re, const double* that_im, long long ldt, void* t_lp, void* e_lp,
                    long long ld_lp, double* d_norm_e, void* ws, size_t ws_bytes, void* stream);

/* ||M||_F of a planar FP64 matrix (frobenius_norm, ddmatrix.py:229-251):
   fixed-shape two-level reduction, deterministic for a given n. */
int sr_fro_norm_f64(int m, int n, const double* re, const double* im, long long ld, double* d_out, void* ws,
                    size_t ws_bytes, void* stream);

/* complex64 copy of a planar FP64 matrix (DDMatrix.to_lp / y.to_lp(),
   orthogonal.py:187). */
int sr_downcast_c64(int m, int n, const double* re, const double* im, long long ld, void* out, long long ld_out,
                    void* stream);

/* lp solve of stril(T L - L T) = -E (solve_block, trisolve.py:243-262).
   clip <= 0 disables clipping; *d_clipped accumulates the clip count;
   *d_flags |= SR_FLAG_SEPARATION on an exactly repeated diagonal. */
size_t sr_trisolve_workspace_bytes(int n, int lp_is_c64);
int sr_trisolve_c64(int n, const void* t, const void* e, long long ld, void* l, float clip,
                    unsigned long long* d_clipped, int* d_flags, void* ws, size_t ws_bytes, void* stream);
int sr_trisolve_c128(int n, const void* t, const void* e, long long ld, void* l, double clip,
                     unsigned long long* d_clipped, int* d_flags, void* ws, size_t ws_bytes, void* stream);

/* Hermitian variant (refine_symmetric, refine.py:409-438).
   ||striu(X)||_F of planar FP64 X (with the split's ||stril|| the full
   off-diagonal defect, refine.py:130-131).  The lp solve collapses to
   l_ij = -e_ij / (t_ii - t_jj) on the strict lower part
   (_solve_diagonal_correction, refine.py:138-159): clip <= 0 disables
   clipping, *d_clipped accumulates, *d_flags gets SR_FLAG_SEPARATION on a
   zero separation and SR_FLAG_NONFINITE on a non-finite quotient. */
int sr_striu_norm_f64(int n, const double* re, const double* im, long long ld, double* d_out, void* ws,
                      size_t ws_bytes, void* stream);
int sr_diag_correction_c64(int n, const void* t, const void* e, long long ld, void* l, float clip,
                           unsigned long long* d_clipped, int* d_flags, void* stream);
int sr_diag_correction_c128(int n, const void* t, const void* e, long long ld, void* l, double clip,
                            unsigned long long* d_clipped, int* d_flags, void* stream);

/* W = L - L^H (complex64), ||W||_F into *d_norm_w, SR_FLAG_NONFINITE into
   *d_flags when L holds a non-finite entry (refine.py:296-297 and
   _check_finite, trisolve.py:116-118). */
int sr_skew_c64(int n, const void* l, long long ld, void* w, double* d_norm_w, int* d_flags, void* ws,
                size_t ws_bytes, void* stream);

/* Sigma of the merged Newton-Schulz update (merged_update,
   orthogonal.py:191-201), planar FP64, summed left to right:
   S = ((((2I + 2W) - Y) - YW) + W^2) + W^3 [+ W^2 Y + W^2 Y W].
   w, yw, w2, w3 (and optional w2y, w2yw, NULL to skip) are complex64;
   w2 = w3 = NULL: yw holds the fused product YW - W^2 - W^3 (yw = NULL too:
   that product lies below the update's error budget and is left out).
   with_identity = 0 drops the 2I term (S' = S - 2I, used by the Ozaki path,
   which forms Q S / 2 = Q + Q S' / 2 exactly).  n rows x cols columns (a
   column block of S' in the sharded driver; cols == n with the identity). */
int sr_sigma_merged_f64(int n, int cols, const void* w, const double* y_re, const double* y_im, long long ldy,
                        const void* yw, const void* w2, const void* w3, const void* w2y, const void* w2yw,
                        long long ld_lp, double* s_re, double* s_im, long long lds, int with_identity,
                        void* stream);

/* X = Y - W - W^2 (complex64 out; Y planar FP64, W and W^2 complex64): the A
   operand of the fused lp product X W = YW - W^2 - W^3, passed as `yw` to
   sr_sigma_merged_f64 with w2 = w3 = NULL (merged_update, orthogonal.py:191-195,
   with two lp products instead of three).  w2 = NULL: X = Y - W (the W^3
   term lies below the update's error budget). */
int sr_fused_lp_operand_c64(int n, const double* y_re, const double* y_im, long long ldy, const void* w,
                            const void* w2, long long ld_lp, void* x, void* stream);

/* Sigma of the entry Newton-Schulz step: S = 3I - G (orthogonal.py:167-168). */
int sr_sigma_ns_f64(int n, const double* g_re, const double* g_im, long long ldg, double* s_re, double* s_im,
                    long long lds, void* stream);

/* Zero the strictly lower triangle in place (upper part of the last T^,
   refine.py:324). */
int sr_triu_inplace_f64(int n, double* re, double* im, long long ld, void* stream);

/* ---- dd mode (hp = double-double planes, lp = complex128) ---- */

/* sr_split_lp_c64 for dd mode: lp T, E complex128 from the hi planes of T^,
   ||E||_F into *d_norm_e (stril_extract + frobenius_norm + to_lp). */
int sr_split_lp_c128(int n, const double* that_re, const double* that_im, long long ldt, void* t_lp, void* e_lp,
                     long long ld_lp, double* d_norm_e, void* ws, size_t ws_bytes, void* stream);

/* sr_skew_c64 for complex128 (refine.py:296-297). */
int sr_skew_c128(int n, const void* l, long long ld, void* w, double* d_norm_w, int* d_flags, void* ws,
                 size_t ws_bytes, void* stream);

/* interleaved complex128 copy of a planar FP64 pair (DDMatrix.to_lp,
   ddmatrix.py:84-86, applied to the hi planes). */
int sr_pack_c128(int m, int n, const double* re, const double* im, long long ld, void* out, long long ld_out,
                 void* stream);

/* Sigma of merged_update in double-double (orthogonal.py:191-201); w, yw,
   w2, w3 (w2y, w2yw optional) complex128, Y and S dd planes. */
int sr_sigma_merged_dd(int n, const void* w, const double* y_re_hi, const double* y_im_hi, const double* y_re_lo,
                       const double* y_im_lo, long long ldy, const void* yw, const void* w2, const void* w3,
                       const void* w2y, const void* w2yw, long long ld_lp, double* s_re_hi, double* s_im_hi,
                       double* s_re_lo, double* s_im_lo, long long lds, int with_identity, void* stream);

/* bytes of reduction workspace the norm kernels need */
size_t sr_reduce_workspace_bytes(void);

/* ---- Ozaki-II emulated products on the int8 tensor cores (csrc/ozaki.cu,
   csrc/oz_gemm.cu).  Replace matmul_hp / matmul_lp (matmul.py:52-110) in
   FP64 mode; generalise the reference's Ozaki-I dd path (matmul.py:151-212).
   Sources are planar FP64 (src_c64 = 0; im may be NULL for a real matrix) or
   interleaved complex64 (src_c64 = 1; im unused). */

/* matrix kinds of the Ozaki entry points */
#define SR_MAT_F64 0  /* planar FP64 (re, im); im == NULL: real */
#define SR_MAT_C64 1  /* interleaved complex64 (re) */
#define SR_MAT_C128 2 /* interleaved complex128 (re) */
#define SR_MAT_DD 3   /* planar double-double: re = re_hi, im = im_hi, re_lo, im_lo */

/* exps[i] = e with max_k |op(X)[i,k]| < 2^e (dd: of the hi parts); op(X) = X
   (transposed = 0: per row) or X^T (transposed = 1: per column). */
int sr_oz_exponents(int rows, int cols, int kind, const void* re, const double* im, long long ld, int transposed,
                    int* exps, void* stream);

/* sr_oz_exponents plus the lines' CRT bound: rmax (one double, device) =
   max_i ||op(X)[i, :]||_2 2^-exps[i], so that an integer-scaled line
   round(op(X)[i, :] 2^(beta - exps[i])) has 2-norm <= 2^beta rmax +
   sqrt(2K)/2 (Cauchy-Schwarz then bounds every entry of a product, which lets
   the Python plan drop moduli: ozaki.fit_plan).  ss_work: cols doubles of
   workspace when transposed (column sums of squares).  host_rmax (optional):
   pinned host memory that also receives rmax, stored by a kernel (no copy
   engine).  No reference counterpart (the reference's Ozaki path,
   matmul.py:151-212, sizes its slices from the worst case). */
int sr_oz_exponents_bound(int rows, int cols, int kind, const void* re, const double* im, long long ld,
                          int transposed, int* exps, double* ss_work, double* rmax, double* host_rmax,
                          void* stream);

/* Residue planes [nmod][planes][rows_out][kpitch] (int8, K-major) of
   round(op(X) * 2^(beta - exps[i])) modulo moduli[l] (3..256, pairwise
   coprime; host array).  op(X)[i][k] = X[i][k], or X[k][i] when transposed;
   conj negates the imaginary part.  layout 0: (re, im) A operand;
   1: (-im, re, im) complex B operand; 2: (re) real B operand; 4: Gaussian
   planes (re + iota im, re - iota im) mod p for either role (see below).
   beta <= 61 (<= 106 for SR_MAT_DD). */
int sr_oz_encode(int rows_out, int K, int kind, const void* re, const double* im, const double* re_lo,
                 const double* im_lo, long long ld, int transposed, int conj, int layout, const int* exps, int beta,
                 int nmod, const int* moduli, void* out, long long kpitch, void* stream);

/* Both operand roles of one matrix X (rows_out = columns of X, K = rows of X,
   scaled per column of X by exps): the A operand of X^H, layout 0 of the
   conjugate (re, -im), into out_ah and the B operand of X, layout 1, into out_b
   — one residue computation for the Q^H / Q pair of every measurement
   (refine.py:259,265).  Same kpitch for both. */
int sr_oz_encode_dual(int rows_out, int K, int kind, const void* re, const double* im, const double* re_lo,
                      const double* im_lo, long long ld, const int* exps, int beta, int nmod, const int* moduli,
                      void* out_ah, void* out_b, long long kpitch, void* stream);

/* R_l = A_l B_l^T mod p_l on tcgen05 (kind::i8), out [nmod][2][M][out_pitch]
   int8 (re, im).  a_planes = 2; b_planes = 3 (complex B) or 1 (real B).
   moduli is a host array; num_sms <= 0 means 148.  lower_only (M == N):
   skip the 128 x 128 tiles above the diagonal (Hermitian products such as
   Q^H Q, whose upper part the decode mirrors). */
int sr_oz_gemm_i8(int M, int N, int K, int nmod, const int* moduli, const void* a, int a_planes,
                  long long a_kpitch, const void* b, int b_planes, long long b_kpitch, void* out,
                  long long out_pitch, int lower_only, int num_sms, void* stream);

/* CRT decode of the residues into C = alpha * C' * 2^-(rho_i + sigma_j)
   + shift * I + add_scale * X (X of add_kind SR_MAT_F64 or SR_MAT_DD, or
   add_kind < 0 for none), with rho_i = beta_a - exps_a[i], sigma_j =
   beta_b - exps_b[j], rounded once into out_kind (any SR_MAT_*).  table
   (host): [nmod][6] CRT weights, [6] modulus-product chunks, [6] chunk
   offsets, 1/P.  hermitian = 1 / -1: the residues hold only the lower
   128-tiles (sr_oz_gemm_i8 with lower_only); the strictly upper tiles are
   written as the conjugate transpose (Hermitian C, 1) or its negative
   (skew-Hermitian C, -1); M == N, no add, any out_kind.
   diag_col0: the shift lands on entries (i, j) with i == j + diag_col0
   (column blocks of a sharded product). */
int sr_oz_decode(int M, int N, int nmod, int nchunk, const double* table, const void* res, long long res_pitch,
                 const int* exps_a, int beta_a, const int* exps_b, int beta_b, double alpha, double shift,
                 int add_kind, const double* add_re, const double* add_im, const double* add_re_lo,
                 const double* add_im_lo, long long ld_add, double add_scale, int out_kind, void* out_re,
                 double* out_im, double* out_re_lo, double* out_im_lo, long long ld_out, int hermitian,
                 int diag_col0, void* stream);

/* ---- Gaussian-CRT complex products (FP64 mode).  Moduli p with a square
   root iota of -1 (odd, every prime factor = 1 mod 4) split Z[i]/p into two
   copies of Z/p: x + iy -> (x + iota y, x - iota y).  A complex product mod p
   is then two independent REAL products, C+ = A+ B+^T and C- = A- B-^T, half
   the tensor-core work of (re, im) planes.  Operands: sr_oz_encode layout 4
   (planes phi+, phi-; the conjugate swaps them, so the B operand of X is the
   A operand of X^H with a_swap = 1).  Replace the same matmul_hp / matmul_lp
   call sites (matmul.py:52-110) as the entries above. */

/* R[l][g] = A[l][g ^ sa] B[l][b_planes == 2 ? g ^ sb : 0]^T mod p_l, g = 0, 1,
   with sa = a_swap & 1, sb = (a_swap >> 1) & 1 (swapped planes read the
   operand as its conjugate; b_planes = 1: a real B operand, layout 2).  herm = +1 / -1 (M == N,
   b_planes == 2, C Hermitian / skew-Hermitian): only plane 0 is multiplied and
   plane 1 is written as +-(plane 0)^T, since C- = +-C+^T.  Valid when the
   INTEGER product is (skew-)Hermitian: row i of A and column i of B scaled
   alike (Q^H Q from one encoding of Q; W W for skew-Hermitian W). */
int sr_oz_gemm_i8_gauss(int M, int N, int K, int nmod, const int* moduli, const void* a, int a_swap,
                        long long a_kpitch, const void* b, int b_planes, long long b_kpitch, void* out,
                        long long out_pitch, int herm, int num_sms, void* stream);

/* sr_oz_decode for Gaussian residue planes: table = the sr_oz_decode table
   with the weights of the real part (w_l (p_l+1)/2 mod P), followed by
   [nmod][6] weights of the imaginary part (w_l (2 iota_l)^-1 mod P).
   out_kind SR_MAT_F64 (add: none or SR_MAT_F64) or SR_MAT_C64 (no add).
   hermitian = 1 (C Hermitian, no add): only the lower 128-tiles are decoded,
   the strictly upper ones written as their conjugate transpose. */
int sr_oz_decode_gauss(int M, int N, int nmod, int nchunk, const double* table, const void* res,
                       long long res_pitch, const int* exps_a, int beta_a, const int* exps_b, int beta_b,
                       double alpha, double shift, int add_kind, const double* add_re, const double* add_im,
                       long long ld_add, double add_scale, int out_kind, void* out_re, double* out_im,
                       long long ld_out, int hermitian, int diag_col0, void* stream);

/* Ozaki path options (no reference counterpart: implementation switches for
   tests and A/B tools).  key 0: 1 (default) = Gaussian decodes with nchunk
   2..4 and nmod <= 32 run the tensor-core CRT decode (the digit sums of the
   CRT weights as one tcgen05 kind::i8 MMA per 128 outputs), 0 = the SIMT
   decode; both give bit-identical results.  value < 0 only queries.
   Returns the previous value, -1 for an unknown key. */
int sr_oz_config(int key, int value);


/* ---- double-double container operations (csrc/dd_ops.cu), bit-identical to
   the reference's numpy / numba kernels for finite operands.  One real plane
   (hi, lo) per call; row-major with leading dimensions. */

/* z = x + y (negate_y = 0) or x - y (negate_y = 1) in dd: DDMatrix.__add__ /
   __sub__ (ddmatrix.py:114-126 -> dd.add / dd.sub, dd.py:96-114). */
int sr_dd_add(int m, int n, const double* xh, const double* xl, long long ldx, const double* yh,
              const double* yl, long long ldy, int negate_y, double* zh, double* zl, long long ldz, void* stream);

/* z = s x (s a binary64 scalar): DDMatrix.scale(float) (ddmatrix.py:138-147 -> dd.mul_d, dd.py:127-132). */
int sr_dd_scale(int m, int n, const double* xh, const double* xl, long long ldx, double s, double* zh,
                double* zl, long long ldz, void* stream);

/* e = strictly lower part of src, t = the rest (either may be NULL):
   stril_extract (ddmatrix.py:190-209), pure masking. */
int sr_stril_split_f64(int m, int n, const double* src, long long lds, double* e, long long lde, double* t,
                       long long ldt, void* stream);

/* d_out[0..1] = (hi, lo) of the dd Frobenius norm of a complex dd matrix
   (rl, ih, il may be NULL = zero planes): frobenius_norm (ddmatrix.py:216-251) —
   dd squares, the reference's fixed pairwise tree over COLUMN-MAJOR order,
   dd sqrt.  ws: sr_fro_norm_dd_workspace_bytes(rows * cols) bytes. */
size_t sr_fro_norm_dd_workspace_bytes(long long entries);
int sr_fro_norm_dd(int rows, int cols, const double* rh, const double* rl, const double* ih, const double* il,
                   long long ld, double* d_out, void* ws, size_t ws_bytes, void* stream);

/* C = op(A) B in double-double with FMA error-free transformations on the
   FP64 pipe (csrc/ddgemm_fma.cu): the measured alternative to the Ozaki-II
   dd products for gemm_hp (_numba_kernels.py:18-46, dd.py:53-180); planar
   row-major dd planes, op_a = SR_OP_N or SR_OP_C. */
int sr_zgemm_dd_fma(int op_a, int m, int n, int k, const double* a_rh, const double* a_rl, const double* a_ih,
                    const double* a_il, long long lda, const double* b_rh, const double* b_rl, const double* b_ih,
                    const double* b_il, long long ldb, double* c_rh, double* c_rl, double* c_ih, double* c_il,
                    long long ldc, void* stream);

/* Column-block forms for the sharded driver (sharded.py): a rows x cols block
   of T^ whose first column is global column col0 is split into lp T, E blocks
   (the strict-lower mask in global indices) and *d_sq_e = sum |E|^2 (a partial
   of the cross-rank sum); X = Y - W - W^2 for a rows x cols block. */
int sr_split_lp_block_c64(int rows, int cols, int col0, const double* that_re, const double* that_im,
                          long long ldt, void* t_lp, void* e_lp, long long ld_lp, double* d_sq_e, void* ws,
                          size_t ws_bytes, void* stream);
int sr_fused_lp_operand_block_c64(int rows, int cols, const double* y_re, const double* y_im, long long ldy,
                                  const void* w, const void* w2, long long ld_lp, void* x, void* stream);

/* ---- entry guards (csrc/guards.cu) ---- */

/* Power iteration on M^H M for the spectral-norm guard of newton_schulz_step
   (spectral_norm_estimate, matmul.py:117-142; orthogonal.py:160-166): M is
   the n x n complex64 lp downcast (ld in elements), vectors and sums FP64.
   Launches `steps` iterations (first = 1: from the reference's fixed start
   vector); the convergence test runs on the device and later steps of a
   group exit at once.  ws starts with five doubles {est, prev, ||w||, done,
   iterations} the caller copies back after each group. */
size_t sr_power_norm_workspace_bytes(int n);
int sr_power_norm_c64(int n, const void* m, long long ld, int first, int steps, double rel_tol, void* ws,
                      size_t ws_bytes, void* stream);

/* *d_flags |= bit when a planar FP64 matrix (im may be NULL) has a
   non-finite entry: the finiteness check of _coerce_hp (refine.py:341-350). */
int sr_finite_flag_f64(int m, int n, const double* re, const double* im, long long ld, int* d_flags, int bit,
                       void* stream);

/* *d_status = 1 when every row and column of the n x n planar matrix holds
   exactly one nonzero (row_of_col[j]: the row of column j's nonzero), else 0:
   the O(n^2) scan of _phase_permutation (refine.py:172-189). */
size_t sr_phase_perm_workspace_bytes(int n);
int sr_phase_perm_scan_f64(int n, const double* re, const double* im, long long ld, int* row_of_col, int* d_status,
                           void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SR_H_ */

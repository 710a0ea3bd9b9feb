// Tensor-core (tcgen05 kind::f16, scaled two-piece FP16) far updates of the complex64 lp
// solver — see trisolve_tc.cu.  Internal interface between trisolve.cu (the
// wavefront driver) and trisolve_tc.cu; not part of the C ABI.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stddef.h>

struct FarTcPlan {
  CUtensorMap a_col, b_col, a_row, b_row;  // T, LB (COL) and T^T, LC (ROW) operand forms
  __half* tform;                           // [2][n][P]   hi / lo of row-scaled T (re, im interleaved)
  __half* ttform;                          // [2][n][P]   hi / lo of row-scaled T^T
  __half* lb;                              // [2][2n][P]  rows 2c, 2c+1: conj(L[:, c]), i conj(L[:, c])
  __half* lc;                              // [2][2n][P]  rows 2i, 2i+1: conj(L[i, :]), i conj(L[i, :])
  float *tmax_r, *tmax_c;                  // [n] row / column maxima of T
  float *lmax_c, *lmax_r;                  // [4][n] column / row maxima of the batch's L tiles, per level
  int n, P;
};

// bytes of the four operand forms at size n (0 when the tensor-core path does not apply)
size_t far_tc_forms_bytes(int n);
// carve the forms out of `base`, encode the tensor maps, launch the T / T^T split
int far_tc_prepare(FarTcPlan* plan, int n, const float2* T, long long ld, void* base, cudaStream_t st);
// batch b: split the L tiles of levels 4b .. 4b+3, then the COL and ROW far updates of Rf
int far_tc_batch(const FarTcPlan& plan, int N, int b, int h, int first_level, const float2* L, long long ld,
                 float2* Rf, cudaStream_t st);

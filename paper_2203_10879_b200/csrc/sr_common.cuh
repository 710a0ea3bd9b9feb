// Shared helpers for the sm_100a Schur-refinement kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sr.h"

#define SR_CUDA_CHECK(expr)                                        \
  do {                                                             \
    cudaError_t _e = (expr);                                       \
    if (_e != cudaSuccess) return sr_set_cuda_error(_e, #expr);    \
  } while (0)

int sr_set_cuda_error(cudaError_t e, const char* what);
void sr_count_launch();
void sr_count_launches(unsigned long long k);  // kernels replayed from a CUDA graph
extern "C" unsigned long long sr_kernel_launches(void);

// after every kernel launch: count it (sr_kernel_launches) and surface launch errors
#define SR_LAUNCH_CHECK()                       \
  do {                                          \
    sr_count_launch();                          \
    SR_CUDA_CHECK(cudaGetLastError());          \
  } while (0)

static inline int sr_ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// Library state that belongs to a device (unit-counter pools, cached unit
// tables, solver streams / graphs, one-time kernel attributes) lives in
// per-device slots: a process may drive several GPUs (or switch devices)
// and each device gets its own.  The slot index is the CURRENT device.
constexpr int SR_MAX_DEVICES = 16;
static inline int sr_device_slot(int* slot) {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= SR_MAX_DEVICES) return SR_EINVAL;
  *slot = d;
  return SR_OK;
}

struct cf32 {
  float x, y;
};

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a / b with the reference's semantics (numpy complex division; Smith's scaling
// keeps |b| near the overflow threshold finite).
__device__ __forceinline__ float2 cdiv(float2 a, float2 b) {
  float s = fabsf(b.x) + fabsf(b.y);
  float ars = a.x / s, ais = a.y / s, brs = b.x / s, bis = b.y / s;
  float d = brs * brs + bis * bis;
  return make_float2((ars * brs + ais * bis) / d, (ais * brs - ars * bis) / d);
}
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  double s = fabs(b.x) + fabs(b.y);
  double ars = a.x / s, ais = a.y / s, brs = b.x / s, bis = b.y / s;
  double d = brs * brs + bis * bis;
  return make_double2((ars * brs + ais * bis) / d, (ais * brs - ars * bis) / d);
}

__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem, int src_bytes) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Kernel timeline for diagnostics (tools/solve_timeline.py builds with
// -DSR_TIMELINE): per (kind, slot) the earliest CTA start and the latest CTA
// end in %globaltimer ns.  Compiled out of the product library.
#ifdef SR_TIMELINE
#define SR_TL_DECLARE(name) __device__ unsigned long long name[8][1024][2];
#define SR_TL_MARK(name, kind, slot, end)                                              \
  do {                                                                                  \
    unsigned long long t_;                                                              \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                             \
    if (end) atomicMax(&name[(kind)][(slot)&1023][1], t_);                              \
    else atomicMin(&name[(kind)][(slot)&1023][0], t_);                                  \
  } while (0)
#else
#define SR_TL_DECLARE(name)
#define SR_TL_MARK(name, kind, slot, end) \
  do {                                    \
  } while (0)
#endif

// (row, column) of a grid-stride loop over a rows x cols matrix, stepped
// without a 64-bit division per element (its I2F / MUFU / F2I sequence runs
// on the narrow XU pipe and made the lighter passes issue-bound); every thread
// visits the same entries in the same order as a flat idx loop would
struct GridIdx {
  int i, j, rows, cols, sq, sr;
  __device__ __forceinline__ GridIdx(int rows_, int cols_) : rows(rows_), cols(cols_) {
    const long long start = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    if (cols <= 0) {
      i = rows;
      j = sq = sr = 0;
      return;
    }
    i = (int)(start / cols);
    j = (int)(start % cols);
    sq = (int)(stride / cols);
    sr = (int)(stride % cols);
  }
  __device__ __forceinline__ bool ok() const { return i < rows; }
  __device__ __forceinline__ void next() {
    i += sq;
    j += sr;
    if (j >= cols) {
      j -= cols;
      ++i;
    }
  }
};

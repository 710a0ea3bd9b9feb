// Microbenchmark: legacy warp-level mma.sync throughput on sm_100a
// (tf32 m16n8k8, bf16 m16n8k16, int8 m16n8k32) against FFMA.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tf32_kernel(float* out, int iters) {
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(1.0f - i * 1e-3f);
  float c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void bf16_kernel(float* out, int iters) {
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3f803f80u + threadIdx.x;
  for (int i = 0; i < 2; ++i) b[i] = 0x3f803f80u;
  float c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void i8_kernel(float* out, int iters) {
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x01010101u + threadIdx.x;
  for (int i = 0; i < 2; ++i) b[i] = 0x01010101u;
  int c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  int s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}

__global__ void ffma_kernel(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9f + i;
  const float b = 0.999999f, c = 1e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b, c);
  }
  float s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d\n", p.name, p.multiProcessorCount);
  float* d;
  cudaMalloc(&d, 1 << 26);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  for (int threads : {128, 256, 512}) {
    const int blocks = sms * (2048 / threads);
    const int iters = 4000;
    float ms;
    double warps = (double)blocks * threads / 32;
#define RUN(K, FLOPS_PER_WARP_ITER, NAME)                                   \
    K<<<blocks, threads>>>(d, 10);                                          \
    cudaEventRecord(e0);                                                    \
    K<<<blocks, threads>>>(d, iters);                                       \
    cudaEventRecord(e1);                                                    \
    cudaEventSynchronize(e1);                                               \
    cudaEventElapsedTime(&ms, e0, e1);                                      \
    printf("%-28s threads=%d: %8.1f TFLOP/s\n", NAME, threads, (FLOPS_PER_WARP_ITER) * iters * warps / ms / 1e9);
    RUN(ffma_kernel, 2.0 * 128 * 32, "FFMA");
    RUN(tf32_kernel, 8.0 * 2 * 16 * 8 * 8, "mma.sync tf32 m16n8k8");
    RUN(bf16_kernel, 8.0 * 2 * 16 * 8 * 16, "mma.sync bf16 m16n8k16");
    RUN(i8_kernel, 8.0 * 2 * 16 * 8 * 32, "mma.sync s8 m16n8k32 (TOPS)");
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

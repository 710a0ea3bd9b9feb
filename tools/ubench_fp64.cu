// Microbenchmark: FP64 pipe throughput on sm_100a (DFMA vs DMMA shapes).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma1684_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0, b = 1.0;
  double c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - i * 1e-3;
  double c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma_kernel(float* out, int iters) {
  float a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9f + i;
  const float b = 0.999999f, c = 1e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b, c);
  }
  float s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s SMs %d clock(kHz) %d\n", p.name, p.multiProcessorCount, p.clockRate);
  double* d; cudaMalloc(&d, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * (2048 / threads);
    int iters = 2000;
    // DFMA: per thread per iter 128 fma
    dfma_kernel<<<blocks, threads>>>(d, 10);
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 128 * iters * (double)blocks * threads;
    printf("DFMA threads=%d: %.2f TFLOP/s\n", threads, fl / ms / 1e9);
    ffma_kernel<<<blocks, threads>>>((float*)d, 10);
    cudaEventRecord(e0); ffma_kernel<<<blocks, threads>>>((float*)d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA threads=%d: %.2f TFLOP/s\n", threads, fl / ms / 1e9);
    // DMMA 884: per warp per iter 8 mma * 8*8*4*2 flops
    dmma884_kernel<<<blocks, threads>>>(d, 10);
    cudaEventRecord(e0); dmma884_kernel<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 8.0 * 512 * iters * (double)blocks * threads / 32;
    printf("DMMA m8n8k4 threads=%d: %.2f TFLOP/s\n", threads, fl / ms / 1e9);
    dmma1684_kernel<<<blocks, threads>>>(d, 10);
    cudaEventRecord(e0); dmma1684_kernel<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 8.0 * 1024 * iters * (double)blocks * threads / 32;
    printf("DMMA m16n8k4 threads=%d: %.2f TFLOP/s\n", threads, fl / ms / 1e9);
    dmma16816_kernel<<<blocks, threads>>>(d, 10);
    cudaEventRecord(e0); dmma16816_kernel<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 4.0 * 4096 * iters * (double)blocks * threads / 32;
    printf("DMMA m16n8k16 threads=%d: %.2f TFLOP/s\n", threads, fl / ms / 1e9);
  }
  cudaError_t err = cudaGetLastError(); printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}

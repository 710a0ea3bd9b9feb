// Probe: does tcgen05.mma .kind::i8 honour the instruction descriptor's
// negate-B bit (bit 14)?  A and B are all ones (so the shared-memory layout
// is irrelevant), K = 32: D = 32 without negation, -32 with it.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2203_10879_b200/csrc \
//      tools/ubench_negate.cu -o tools/ubench_negate -lcuda
#include <cstdio>

#include "tc_common.cuh"

__global__ void probe(uint32_t neg_bits, int* out) {
  __shared__ __align__(1024) int8_t sa[128 * 64];
  __shared__ __align__(1024) int8_t sb[128 * 64];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    sa[i] = 1;
    sb[i] = 1;
  }
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) mbar_init(smem_u32(&bar), 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t d = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24) | neg_bits;
    const uint64_t ad = umma_desc_sw64(smem_u32(sa)), bd = umma_desc_sw64(smem_u32(sb));
    asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 0;\n" ::"r"(d), "l"(ad), "l"(bd), "r"(idesc));
    umma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t v[16];
  tmem_ld16(d + ((uint32_t)(warp * 32) << 16), v);
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  if ((threadIdx.x & 31) == 0 && warp == 0) out[0] = (int)v[0];
  if ((threadIdx.x & 31) == 5 && warp == 3) out[1] = (int)v[7];
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(d));
}

int main() {
  int* out;
  cudaMalloc(&out, 8);
  const uint32_t variants[3] = {0u, 1u << 14, 1u << 13};
  const char* names[3] = {"plain", "negate B (bit 14)", "negate A (bit 13)"};
  for (int k = 0; k < 3; ++k) {
    cudaMemset(out, 0x7f, 8);
    probe<<<1, 128>>>(variants[k], out);
    cudaError_t e = cudaDeviceSynchronize();
    int h[2] = {0, 0};
    if (e == cudaSuccess) cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    printf("%-20s: %s D = %d, %d\n", names[k], cudaGetErrorString(e), h[0], h[1]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}

// Microbenchmark: tcgen05.mma kind::i8 issue-rate ceiling on sm_100a with the
// operands already in shared memory (no TMA), to separate the MMA pipe's own
// limit from the operand-feed limit of oz_gemm_kernel.
//   variant 0: cta_group::1, M=128, N=256, SWIZZLE_64B  (oz_gemm's complex MMAs)
//   variant 1: cta_group::1, M=128, N=256, SWIZZLE_128B
//   variant 2: cta_group::1, M=128, N=128, SWIZZLE_64B  (oz_gemm's real-B MMAs)
//   variant 3: cta_group::2, M=256, N=256, SWIZZLE_64B  (CTA pair)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_umma tools/ubench_umma.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr, int sw128) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((sw128 ? 1024 : 512) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(sw128 ? 2 : 4) << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <int V>
__global__ void __launch_bounds__(128, 1) umma_loop(int iters, unsigned long long* cycles, const uint8_t* gsrc,
                                                     unsigned long long* bulk_bytes) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  constexpr int CG = (V == 3) ? 2 : 1;
  constexpr bool BULK = (V >= 4);
  __shared__ __align__(8) uint64_t bbar[4];
  __shared__ volatile int stop;
  constexpr int N = (V == 2) ? 128 : 256;
  (void)BULK;
  constexpr int SW128 = (V == 1);
  const int warp = threadIdx.x >> 5;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bbar[i])));
    stop = 0;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_slot;
  unsigned long long t0 = clock64();
  if (BULK && threadIdx.x == 32) {
    // load generator: 4 x 24 KB bulk copies in flight from an L2-resident buffer into smem [96K, 192K)
    unsigned long long bytes = 0;
    uint32_t ph[4] = {0, 0, 0, 0};
    const uint32_t dst0 = smem_u32(smem) + 96 * 1024;
    for (int k = 0; !stop; ++k) {
      const int s = k & 3;
      if (k >= 4) {
        asm volatile("{\n.reg .pred P1;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D1;\nbra W1;\nD1:\n}\n" ::"r"(
                         smem_u32(&bbar[s])), "r"(ph[s]) : "memory");
        ph[s] ^= 1;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bbar[s])), "r"(24576) : "memory");
      const uint8_t* src = gsrc + ((size_t)((blockIdx.x * 7 + k) & 255) * 24576);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       dst0 + s * 24576), "l"(src), "r"(24576), "r"(smem_u32(&bbar[s])) : "memory");
      bytes += 24576;
      if (V == 5 && k > iters) break;
    }
    for (int s2 = 0; s2 < 4; ++s2) {  // drain the copies still in flight
      asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D2;\nbra W2;\nD2:\n}\n" ::"r"(
                       smem_u32(&bbar[s2])), "r"(ph[s2]) : "memory");
    }
    bulk_bytes[blockIdx.x] = bytes;
  }
  if (threadIdx.x == 0 && rank == 0 && V != 5) {
    const uint32_t base = smem_u32(smem);
    constexpr uint32_t id = idesc_i8(CG == 2 ? 256 : 128, N);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        // A: 4 rotating 16 KB regions, B: 2 rotating regions after them (like the stage ring)
        const uint32_t sa = base + (uint32_t)((j & 3) * 8192) + (uint32_t)((j >> 2) & 1) * 32;
        const uint32_t sb = base + 32768 + (uint32_t)((j & 1) * 8192) + (uint32_t)((j >> 1) & 1) * 32;
        const uint64_t ad = desc(sa, SW128), bd = desc(sb, SW128);
        const uint32_t d = tmem + (uint32_t)((j & 1) * 256 * (N == 256 ? 1 : 0));
        if (CG == 1)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                       "l"(ad), "l"(bd), "r"(id), "r"(1));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                       "l"(ad), "l"(bd), "r"(id), "r"(1));
      }
    }
    if (CG == 1)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                       smem_u32(&bar)), "h"((uint16_t)3) : "memory");
  }
  if (threadIdx.x == 0 && V != 5) {
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
            smem_u32(&bar)) : "memory");
    cycles[blockIdx.x] = clock64() - t0;
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (warp == 0) {
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

template <int V>
void run(const char* name, int iters) {
  const int grid = 148;
  unsigned long long* cyc;
  cudaMalloc(&cyc, grid * sizeof(unsigned long long));
  unsigned long long* bb;
  cudaMalloc(&bb, grid * sizeof(unsigned long long));
  cudaMemset(bb, 0, grid * sizeof(unsigned long long));
  uint8_t* gsrc;
  cudaMalloc(&gsrc, 256 * 24576 + 4096);
  const size_t smem = 200 * 1024 + 1024;
  cudaFuncSetAttribute(umma_loop<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = (V == 3) ? 2 : 1;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, umma_loop<V>, iters / 10, cyc, (const uint8_t*)gsrc, bb);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, umma_loop<V>, iters, cyc, (const uint8_t*)gsrc, bb);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const int M = (V == 3) ? 256 : 128, N = (V == 2) ? 128 : 256;
  const int ctas_issuing = (V == 3) ? grid / 2 : grid;
  const double ops = 2.0 * M * N * 32 * 8.0 * iters * ctas_issuing * reps;
  const double mmas = 8.0 * iters;
  unsigned long long hb[148];
  cudaMemcpy(hb, bb, sizeof(hb), cudaMemcpyDeviceToHost);
  double bsum = 0;
  for (int i = 0; i < grid; ++i) bsum += (double)hb[i];
  printf("%-44s %8.1f TOP/s  %7.1f cycles/MMA (CTA 0)  bulk(last rep) %.2f TB/s  err=%s\n", name,
         V == 5 ? 0.0 : ops / (ms * 1e-3) / 1e12, (double)h[0] / mmas, bsum / (ms * 1e-3 / reps) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
  cudaFree(bb);
  cudaFree(gsrc);
}

// L2 -> SM bulk-copy throughput vs bytes in flight: SLOTS copies of CHUNK bytes
// outstanding per CTA, source = a src_bytes buffer (L2-resident when small).
template <int SLOTS, int CHUNK>
__global__ void __launch_bounds__(32, 1) bulk_loop(int iters, const uint8_t* gsrc, size_t src_chunks) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bbar[SLOTS];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < SLOTS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bbar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  uint32_t ph[SLOTS];
  for (int i = 0; i < SLOTS; ++i) ph[i] = 0;
  const uint32_t dst0 = smem_u32(smem_raw);
  for (int k = 0; k < iters; ++k) {
    const int s = k % SLOTS;
    if (k >= SLOTS) {
      asm volatile("{\n.reg .pred P1;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D1;\nbra W1;\nD1:\n}\n" ::"r"(
                       smem_u32(&bbar[s])), "r"(ph[s]) : "memory");
      ph[s] ^= 1;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bbar[s])), "r"(CHUNK) : "memory");
    const uint8_t* src = gsrc + ((size_t)(blockIdx.x * 131 + k * 7) % src_chunks) * CHUNK;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     dst0 + s * CHUNK), "l"(src), "r"(CHUNK), "r"(smem_u32(&bbar[s])) : "memory");
  }
  for (int s2 = 0; s2 < SLOTS; ++s2)
    asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D2;\nbra W2;\nD2:\n}\n" ::"r"(
                     smem_u32(&bbar[s2])), "r"(ph[s2]) : "memory");
}

template <int SLOTS, int CHUNK>
void run_bulk(size_t src_bytes) {
  uint8_t* g;
  cudaMalloc(&g, src_bytes + CHUNK);
  cudaMemset(g, 1, src_bytes);
  const size_t chunks = src_bytes / CHUNK;
  const int smem = SLOTS * CHUNK;
  cudaFuncSetAttribute(bulk_loop<SLOTS, CHUNK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = (int)(((size_t)2 << 30) / 148 / CHUNK);
  bulk_loop<SLOTS, CHUNK><<<148, 32, smem>>>(iters / 10, g, chunks);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bulk_loop<SLOTS, CHUNK><<<148, 32, smem>>>(iters, g, chunks);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("bulk %2d x %6d B in flight (%3d KB), src %5zu MB: %6.2f TB/s  err=%s\n", SLOTS, CHUNK, SLOTS * CHUNK / 1024,
         src_bytes >> 20, 148.0 * iters * CHUNK / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(g);
}

int main() {
  const int iters = 20000;
  run<0>("cg1 M128 N256 SW64", iters);
  run<1>("cg1 M128 N256 SW128", iters);
  run<2>("cg1 M128 N128 SW64", iters);
  run<3>("cg2 M256 N256 SW64 (pair)", iters);
  run<4>("cg1 M128 N256 SW64 + bulk loads", iters);
  run<5>("bulk loads only (24 KB x4 in flight)", iters);
  run<0>("cg1 M128 N256 SW64 (again)", iters);
  for (size_t src : {(size_t)16 << 20, (size_t)1 << 30}) {
    run_bulk<2, 16384>(src);
    run_bulk<4, 16384>(src);
    run_bulk<8, 16384>(src);
    run_bulk<12, 16384>(src);
    run_bulk<4, 40960>(src);
    run_bulk<5, 40960>(src);
    run_bulk<16, 8192>(src);
    run_bulk<24, 8192>(src);
  }
  return 0;
}

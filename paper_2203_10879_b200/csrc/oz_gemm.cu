// Modular int8 GEMM on the 5th-generation tensor cores (tcgen05, kind::i8).
//
// The engine of the Ozaki-II emulated FP64 / FP32 complex products (see
// ozaki.cu and DESIGN.md §Ozaki): for every modulus p_l of the plan it
// computes the residue matrix
//     R_l = (A_l B_l^T) mod p_l            (complex: 4M, fused in one tile)
// from int8 residue operands that ozaki.cu's encoder wrote K-major.
// Every product is exact (|A_l|,|B_l| <= 128, int32 accumulation of K <= 2^17
// terms), so the result is independent of the summation order.
//
// Complex tile trick: the B stage holds three 128-row planes in the order
// [-B_im | B_re | B_im], so the two N = 256 MMAs
//     D[:, 0:256] += A_re x [B_re | B_im]^T
//     D[:, 0:256] += A_im x [-B_im | B_re]^T
// leave D = [C_re | C_im] in one 256-column TMEM accumulator.
//
// Kernel shape: persistent, one CTA per SM, warp-specialised —
//   warp 0     TMA producer (4-d tensor maps, 64-byte swizzle, 5-stage ring)
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5  epilogue: tcgen05.ld -> mod p -> int8 residues -> global
// with two 256-column TMEM accumulators so the epilogue of tile i overlaps
// the MMAs of tile i+1.  Tiles are rasterised in groups of 16 M-tiles and
// handed out from a global counter, so the units in flight are one contiguous
// window of the raster and their shared operand panels hit in the 126 MB L2.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "sr_common.cuh"
#include "tc_common.cuh"

namespace {

constexpr int TM = 128, TN = 128, TK = 64;  // tile: 128 rows x 128 cols, 64-byte k blocks
constexpr int MAX_STAGES = 12;                // ring slots (2-SM: complex 6 x 32 KB, real 12 x 16 KB)
constexpr int SMEM_RING = 200 * 1024;
constexpr int PLANE_BYTES = TM * TK;        // 8 KB per 128-row, 64-byte plane
// epilogue warps: 16 (four per TMEM lane quadrant, splitting the 16-column
// chunks) for wide units, whose epilogue does not overlap the MMAs (config-3
// refinement 0.354 -> 0.341 s against 8, interleaved A/B); 4 for the
// double-buffered narrow units (8 measured 10 % slower on Hermitian products)
constexpr int MAX_EPI_WARPS = 16;
#ifndef SR_OZ_DIAG_NO_TRANSPOSE
#define SR_OZ_DIAG_NO_TRANSPOSE 0  // timing diagnostic only: Hermitian products without the C- = C+^T write
#endif
constexpr int NUM_THREADS = 64 + 32 * MAX_EPI_WARPS;  // launch bound; the block has 64 + 32 p.epi threads
// M-tiles per rasterisation group (complex products; the stacked real ones use
// twice as many — their M is 2n).  Measured with the dynamic unit queue at
// n = 8192, 17 moduli: DRAM reads per hp launch 30 / 17.7 / 31.7 / 132 GB for
// groups of 8 / 16 / 32 / 64 (operands 5.4 GB), 26.9 ms at 16.
constexpr int GROUP_M = 16;
constexpr int MAX_MODULI = 32;
constexpr int QD = 16;        // work-unit queue depth (producer -> MMA / epilogue, rank 0 -> rank 1)
constexpr int SMEM_TAIL = 1024;  // barriers, unit queues, TMEM slot
constexpr int XPOSE_WARP_BYTES = 16 * 32;  // per epilogue warp: the 32 x 16 transposed-write tile

struct OzParams {
  int M, N, K, nmod;
  int a_planes, b_planes;
  int tiles_m, tiles_n;
  int lower_only;               // Hermitian product: only tiles with nt <= mt
  int group_m;                  // work units per rasterisation group (L2 reuse of the A panel)
  int real;                     // real x real product, 256-column tiles, one N = 256 MMA per k-step
  const int* table;             // lower_only: the units of one modulus that hold a lower tile, in raster
  int units_per_mod;            //   order (mp | nt << 16), so every cluster gets only real work
  int stages;                   // ring slots in use
  int gauss;                    // Gaussian planes: tile plane g = mt / tpp (real product of A plane g ^ a_swap
  int a_swap, b_gplane, tpp;    //   with B plane g ^ b_swap, or B plane 0 when b_gplane = 0), output plane g
  int b_swap;
  int wide;                     // TWO && real: a unit is N = 512 (two N = 256 MMAs per k-block into both TMEM
                                //   accumulators): the pair's A tile is read once per 512 B rows, 25 % less
                                //   L2->SM ingest per MAC; the epilogue then drains both accumulators
  int epi;                      // epilogue warps (4 or 8)
  int kstep;                    // 2-SM real products: 64-byte k-blocks per ring slot (MMAs per barrier round trip)
  int herm;                     // gauss, Hermitian (+1) / skew (-1) C: only plane 0 is computed, and the
                                //   epilogue also writes herm * its transpose as plane 1 (C- = +-C+^T)
  long long out_pitch;          // bytes between output rows
  long long out_plane;          // bytes between output planes (re / im)
  long long out_mod;            // bytes between moduli
  int moduli[MAX_MODULI];
  float inv[MAX_MODULI];
  uint32_t bm[MAX_MODULI];      // Barrett multiplier floor(2^32 / p) + 1
  uint32_t roff[MAX_MODULI];    // a multiple of p above |accumulator|, + p/2 (symmetric residue)
};

__device__ __forceinline__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ int ld_volatile_shared(const int* p) {
  int v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

// cta_group::2 variants: the TMA completes on the pair leader's mbarrier (a
// shared::cluster address), the MMA spans both CTAs (M = 256), its commit
// arrives on the barrier at the same offset in every CTA of the mask.
__device__ __forceinline__ void tma_load_4d_2sm(uint32_t dst, const CUtensorMap* map, uint32_t cluster_bar, int c0,
                                                int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(cluster_bar)
      : "memory");
}
__device__ __forceinline__ void umma_i8_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_2sm(uint32_t bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          bar),
      "h"(cta_mask)
      : "memory");
}

__device__ __forceinline__ void decode_tile(const OzParams& p, int t, int& l, int& mt, int& nt) {
  const int per_mod = p.tiles_m * p.tiles_n;
  const int G = p.group_m;
  l = t / per_mod;
  int r = t - l * per_mod;
  const int group = r / (G * p.tiles_n);
  const int first_m = group * G;
  const int gm = min(G, p.tiles_m - first_m);
  const int in = r - group * G * p.tiles_n;
  mt = first_m + in % gm;
  nt = in / gm;
}


// CM = 1: one CTA per tile.  CM = 2: clusters of two CTAs own vertically
// adjacent M-tiles with the same N-tile; each CTA TMA-loads half the rows of
// the shared B tile and multicasts it to both, halving the per-SM L2->SM
// operand traffic (the L1TEX->XBAR request path is the measured limiter,
// profiles/r1_oz_gemm_ncu.md).  A stage slot is refilled only after both
// CTAs' MMAs released it (empty barriers count the two multicast commits).
// TWO (CM = 2): one M = 256 MMA per pair (tcgen05 cta_group::2) issued by the
// leader; each CTA holds its 128 A rows and HALF of the N = 256 B operand, so
// an SM ingests 32 KB per complex k-block instead of 40 (B planes: leader
// [B_re, -B_im], peer [B_im, B_re]: the pair's two MMAs read [B_re | B_im] and
// [-B_im | B_re]) and 16 KB instead of 24 for the stacked real products.
template <int CM, bool TWO = false>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                   const __grid_constant__ OzParams p, int8_t* __restrict__ out, int* __restrict__ counter) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int a_bytes = p.a_planes * PLANE_BYTES;
  // real: one 256-row B plane (TWO: this CTA's 128 rows); complex: 3 planes (TWO: 2)
  const int b_bytes = TWO ? (p.real ? (p.wide ? 2 : 1) : 2) * PLANE_BYTES : (p.real ? 2 : p.b_planes) * PLANE_BYTES;
  // 2-SM real products carry two 64-byte k-blocks per ring slot (four MMAs per
  // barrier round trip, like the complex products): with one k-block per slot
  // the issuer's per-slot overhead left the tensor pipe ~45 % idle
  const int kstep = (TWO && p.real) ? p.kstep : 1;
  const int stage_bytes = kstep * (a_bytes + b_bytes);
  const int STAGES = p.stages;
  const int tn = p.real ? (p.wide ? 4 : 2) * TN : TN;
  uint64_t* bars = (uint64_t*)(smem + SMEM_RING);
  // bars: full[MAX_STAGES], empty[MAX_STAGES], tfull[2], tempty[2], qfull[QD], qempty[QD],
  // pfull[QD], pempty[QD]; then the unit queues unitq[QD], peerq[QD] and the tmem base slot
  int* unitq = (int*)(bars + 2 * MAX_STAGES + 4 + 4 * QD);
  int* peerq = unitq + QD;
  uint32_t* tmem_slot = (uint32_t*)(peerq + QD);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (MAX_STAGES + s); };
  auto tfull_bar = [&](int b) { return bar0 + 8u * (2 * MAX_STAGES + b); };
  auto tempty_bar = [&](int b) { return bar0 + 8u * (2 * MAX_STAGES + 2 + b); };
  // work-unit queue: the producer pushes every unit it fetched to the MMA and
  // epilogue warps (qfull / qempty); in a pair, rank 0 fetches and hands the
  // unit to rank 1's producer (pfull / pempty, arrived across the cluster)
  auto qfull_bar = [&](int s) { return bar0 + 8u * (2 * MAX_STAGES + 4 + s); };
  auto qempty_bar = [&](int s) { return bar0 + 8u * (2 * MAX_STAGES + 4 + QD + s); };
  auto pfull_bar = [&](int s) { return bar0 + 8u * (2 * MAX_STAGES + 4 + 2 * QD + s); };
  auto pempty_bar = [&](int s) { return bar0 + 8u * (2 * MAX_STAGES + 4 + 3 * QD + s); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), TWO ? 1 : CM);  // TWO: the leader's commit arrives in both CTAs
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull_bar(b), 1);
      mbar_init(tempty_bar(b), TWO ? 2 * p.epi : 32 * p.epi);  // TWO: one arrive per epilogue warp of both CTAs
    }
    for (int q = 0; q < QD; ++q) {
      mbar_init(qfull_bar(q), 1);
      mbar_init(qempty_bar(q), 1 + p.epi);  // the MMA thread + one lane per epilogue warp
      mbar_init(pfull_bar(q), 1);
      mbar_init(pempty_bar(q), CM > 1 ? CM - 1 : 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&tmap_a) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&tmap_b) : "memory");
  }
  if (warp == 1) {
    if (TWO) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (CM > 1) cluster_sync();  // peers' barriers are initialised before any multicast
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  // work units: tiles (CM = 1) or vertical tile pairs (CM = 2), in raster
  // order, handed out dynamically (one global counter per launch) so the
  // units in flight always form one contiguous window of the raster: the
  // operand panels they share are read within microseconds of each other
  // and hit in L2, however much the clusters drift apart
  const int crank = CM > 1 ? (int)cluster_ctarank() : 0;
  OzParams pu = p;
  pu.tiles_m = (p.tiles_m + CM - 1) / CM;
  const int total_tiles = p.table ? p.nmod * p.units_per_mod : p.nmod * pu.tiles_m * p.tiles_n;
  const int kblocks = (p.K + TK - 1) / TK;
  // a Hermitian (lower_only) unit is skipped only when every tile of it is
  // strictly upper, so both CTAs of a cluster run identical pipelines
  auto unit = [&](int t, int& l, int& mt, int& nt) -> bool {
    int mp;
    if (p.table) {
      l = t / p.units_per_mod;
      const int v = __ldg(p.table + (t - l * p.units_per_mod));
      mp = v & 0xFFFF;
      nt = v >> 16;
      mt = mp * CM + crank;
      return true;
    }
    decode_tile(pu, t, l, mp, nt);
    mt = mp * CM + crank;
    return !(p.lower_only && nt > mp * CM + CM - 1);
  };

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // the next unit is fetched one unit ahead, so the atomic's round trip
      // overlaps the current unit's loads
      int t_next = (CM == 1 || crank == 0) ? atomicAdd(counter, 1) : 0;
      for (int v = 0;; ++v) {
        const int qs = v % QD;
        const uint32_t qph = (uint32_t)(v / QD) & 1u;
        int t;
        if (CM == 1) {
          t = t_next;
          if (t < total_tiles) t_next = atomicAdd(counter, 1);
        } else if (crank == 0) {
          t = t_next;
          if (t < total_tiles) t_next = atomicAdd(counter, 1);
          if (v >= QD) mbar_wait_cluster(pempty_bar(qs), qph ^ 1);  // every peer has taken unit v - QD
#pragma unroll
          for (int r = 1; r < CM; ++r) {
            st_cluster_u32(mapa_u32(smem_u32(peerq + qs), r), t);
            mbar_arrive_cluster(mapa_u32(pfull_bar(qs), r));
          }
        } else {
          mbar_wait_cluster(pfull_bar(qs), qph);
          t = ld_volatile_shared(peerq + qs);
          mbar_arrive_cluster(mapa_u32(pempty_bar(qs), 0));
        }
        if (v >= QD) mbar_wait(qempty_bar(qs), qph ^ 1);
        unitq[qs] = t;
        mbar_arrive(qfull_bar(qs));  // release: the unit is visible to the waiting warps
        if (t >= total_tiles) break;
        int l, mt, nt;
        if (!unit(t, l, mt, nt)) continue;
        int arow = mt * TM, apl = 0, bpl = 0;
        if (p.gauss) {
          const int g = mt / p.tpp;
          arow = (mt - g * p.tpp) * TM;
          apl = g ^ p.a_swap;
          bpl = p.b_gplane ? (g ^ p.b_swap) : 0;
        }
        for (int kb = 0; kb < kblocks; kb += kstep) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          uint8_t* st = smem + stage * stage_bytes;
          if (TWO) {
            // both CTAs' bytes complete on the leader's full barrier
            const uint32_t fb = mapa_u32(full_bar(stage), 0);
            if (crank == 0) mbar_expect_tx(full_bar(stage), 2 * stage_bytes);
            if (p.real) {
              // [A kb, A kb+1 | B kb, B kb+1]; a k-block past K is zero-filled by the TMA.
              // wide: B kb = [rows of the first N = 256 half | of the second], this CTA's 128 of each
              for (int h = 0; h < kstep; ++h) {
                tma_load_4d_2sm(smem_u32(st + h * a_bytes), &tmap_a, fb, (kb + h) * TK, arow, apl, l);
                tma_load_4d_2sm(smem_u32(st + kstep * a_bytes + h * b_bytes), &tmap_b, fb, (kb + h) * TK,
                                nt * tn + crank * TN, bpl, l);
                if (p.wide)
                  tma_load_4d_2sm(smem_u32(st + kstep * a_bytes + h * b_bytes + PLANE_BYTES), &tmap_b, fb,
                                  (kb + h) * TK, nt * tn + 2 * TN + crank * TN, bpl, l);
              }
            } else {
              tma_load_4d_2sm(smem_u32(st), &tmap_a, fb, kb * TK, arow, apl, l);
              // encoded B planes: 0 = -im, 1 = re, 2 = im
              tma_load_4d_2sm(smem_u32(st + a_bytes), &tmap_b, fb, kb * TK, nt * TN, crank == 0 ? 1 : 2, l);
              tma_load_4d_2sm(smem_u32(st + a_bytes + PLANE_BYTES), &tmap_b, fb, kb * TK, nt * TN,
                              crank == 0 ? 0 : 1, l);
            }
          } else {
          mbar_expect_tx(full_bar(stage), stage_bytes);
          tma_load_4d(smem_u32(st), &tmap_a, full_bar(stage), kb * TK, arow, apl, l);
          if (CM == 1) {
            tma_load_4d(smem_u32(st + a_bytes), &tmap_b, full_bar(stage), kb * TK, nt * tn, bpl, l);
          } else if (p.real) {
            // this CTA's 128 of the tile's 256 B rows, multicast to the pair
            tma_load_4d_mc(smem_u32(st + a_bytes + crank * (2 * PLANE_BYTES / CM)), &tmap_b, full_bar(stage),
                           kb * TK, nt * tn + crank * (tn / CM), bpl, l, (uint16_t)((1 << CM) - 1));
          } else {
            // this CTA's half of every B plane, multicast to the pair
            for (int pl = 0; pl < p.b_planes; ++pl)
              tma_load_4d_mc(smem_u32(st + a_bytes + pl * PLANE_BYTES + crank * (PLANE_BYTES / CM)), &tmap_b,
                             full_bar(stage), kb * TK, nt * TN + crank * (TN / CM), pl, l, (uint16_t)((1 << CM) - 1));
          }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const bool cplx = (p.b_planes == 3);
    const uint32_t id256 = idesc_i8(128, 256), id128 = idesc_i8(128, 128);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int v = 0;; ++v) {
      const int qs = v % QD;
      mbar_wait(qfull_bar(qs), (uint32_t)(v / QD) & 1u);
      const int t = ld_volatile_shared(unitq + qs);
      __syncwarp();
      if (lane == 0) mbar_arrive(qempty_bar(qs));
      if (t >= total_tiles) break;
      {
        int l, mt, nt;
        if (!unit(t, l, mt, nt)) continue;
      }
      if (TWO && crank != 0) continue;  // the pair's MMAs are issued by the leader
      if (TWO)
        mbar_wait_cluster(tempty_bar(acc), acc_phase ^ 1);
      else
        mbar_wait(tempty_bar(acc), acc_phase ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t d = tmem_base + (uint32_t)(acc * 256);
      for (int kb = 0; kb < kblocks; kb += kstep) {
        mbar_wait(full_bar(stage), phase);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem + stage * stage_bytes);
          const uint32_t sb = sa + a_bytes;
          if (TWO) {
            const uint32_t id = idesc_i8(256, 256);
            // descriptors as 16-byte offsets of the stage's base descriptor (the
            // start-address field is the low 14 bits; every address stays below
            // 256 KB): a handful of adds per MMA instead of a descriptor build
            const uint64_t ds = umma_desc_sw64(sa);
            if (p.real) {
              for (int h = 0; h < kstep; ++h)
#pragma unroll
                for (int ks = 0; ks < TK / 32; ++ks) {
                  const uint64_t ad = ds + (uint64_t)((h * a_bytes + ks * 32) >> 4);
                  const uint64_t bd = ds + (uint64_t)((kstep * a_bytes + h * b_bytes + ks * 32) >> 4);
                  umma_i8_2sm(d, ad, bd, id, (kb | h | ks) != 0);
                  if (p.wide)  // the second N = 256 half into the other accumulator (d = base)
                    umma_i8_2sm(d + 256, ad, bd + (uint64_t)(PLANE_BYTES >> 4), id, (kb | h | ks) != 0);
                }
            } else {
#pragma unroll
              for (int ks = 0; ks < TK / 32; ++ks) {
                const uint32_t acc_flag = (kb | ks) != 0;
                const uint64_t ad = ds + (uint64_t)((ks * 32) >> 4), bd = ds + (uint64_t)((a_bytes + ks * 32) >> 4);
                umma_i8_2sm(d, ad, bd, id, acc_flag);
                umma_i8_2sm(d, ad + (uint64_t)(PLANE_BYTES >> 4), bd + (uint64_t)(PLANE_BYTES >> 4), id, 1u);
              }
            }
            umma_commit_2sm(empty_bar(stage), 3);
            if (kb + kstep >= kblocks) umma_commit_2sm(tfull_bar(acc), 3);
          } else {
#pragma unroll
          for (int ks = 0; ks < TK / 32; ++ks) {
            const uint32_t acc_flag = (kb | ks) != 0;
            const uint64_t are = umma_desc_sw64(sa + ks * 32);
            const uint64_t aim = umma_desc_sw64(sa + (p.real ? 0 : PLANE_BYTES) + ks * 32);
            if (p.real) {
              umma_i8(d, are, umma_desc_sw64(sb + ks * 32), id256, acc_flag);
            } else if (cplx) {
              const uint64_t b1 = umma_desc_sw64(sb + PLANE_BYTES + ks * 32);  // [B_re | B_im]
              const uint64_t b2 = umma_desc_sw64(sb + ks * 32);                // [-B_im | B_re]
              umma_i8(d, are, b1, id256, acc_flag);
              umma_i8(d, aim, b2, id256, 1u);
            } else {
              const uint64_t b = umma_desc_sw64(sb + ks * 32);
              umma_i8(d, are, b, id128, acc_flag);
              umma_i8(d + 128, aim, b, id128, acc_flag);
            }
          }
          if (CM == 1)
            umma_commit(empty_bar(stage));
          else
            umma_commit_mc(empty_bar(stage), (uint16_t)((1 << CM) - 1));  // release the slot in every CTA
          if (kb == kblocks - 1) umma_commit(tfull_bar(acc));
          }
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (!p.wide) acc ^= 1;  // wide: every unit uses both accumulators (acc stays 0)
      if (acc == 0) acc_phase ^= 1;
    }
  } else {
    // ---------------- epilogue: TMEM -> residues -> global ----------------
    // p.epi warps: lane quadrant ew = warp & 3; with 8, the two warps of a quadrant
    // take alternate 16-column chunks.  Residues by an integer Barrett step
    // (no conversions: the float quotient's I2F / F2I ran on the narrow XU pipe),
    // the next chunk's TMEM load in flight while this one is reduced.  With wide
    // units the epilogue does not overlap the MMAs, so its length is tensor-pipe
    // idle time.
    const int ew = warp & 3;  // TMEM lane quadrant this warp may access
    const int half = (warp - 2) >> 2;  // 0 .. p.epi / 4 - 1
    const int CSTEP = p.epi >> 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int v = 0;; ++v) {
      const int qs = v % QD;
      mbar_wait(qfull_bar(qs), (uint32_t)(v / QD) & 1u);
      const int t = ld_volatile_shared(unitq + qs);
      __syncwarp();
      if (lane == 0) mbar_arrive(qempty_bar(qs));
      if (t >= total_tiles) break;
      int l, mt, nt;
      if (!unit(t, l, mt, nt)) continue;
      const int pm = p.moduli[l];
      const uint32_t bm = p.bm[l], roff = p.roff[l];
      const int hp = pm >> 1;
      mbar_wait(tfull_bar(acc), acc_phase);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      int g = 0, row = mt * TM + ew * 32 + lane;
      if (p.gauss) {
        g = mt / p.tpp;
        row = (mt - g * p.tpp) * TM + ew * 32 + lane;
      }
      int8_t* base = out + (size_t)l * p.out_mod + (size_t)g * p.out_plane + (size_t)row * p.out_pitch;
      const int nchunks = p.wide ? 32 : 16;
      const uint32_t tbase = tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * 256);
      // symmetric residue of the accumulator v: u = v + roff in [0, 2^32),
      // q = umulhi(u, bm) is floor(u / p) or one more, r = u - q p in [-p, p)
      auto red = [&](uint32_t vv) -> int {
        const uint32_t u = vv + roff;
        const int r = (int)(u - __umulhi(u, bm) * (uint32_t)pm);
        return r - hp + ((r >> 31) & pm);
      };
      // Hermitian products: per-warp staging for the transposed write (below)
      uint8_t* xs = smem + SMEM_RING + SMEM_TAIL + (warp - 2) * XPOSE_WARP_BYTES;
      const int row0 = row - lane;  // the warp's first row
      auto emit = [&](const uint32_t (&vc)[16], int chunk) {
        const int plane = p.real ? 0 : chunk >> 3;
        const int col0 = nt * tn + (p.real ? chunk : (chunk & 7)) * 16;
        int r[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) r[e] = red(vc[e]);
        uint32_t packed[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          packed[q] = __byte_perm(__byte_perm(r[q * 4], r[q * 4 + 1], 0x0040),
                                  __byte_perm(r[q * 4 + 2], r[q * 4 + 3], 0x0040), 0x5410);
        if (p.herm && !SR_OZ_DIAG_NO_TRANSPOSE) {
          // C- = herm * C+^T: the warp's 32 rows x 16 columns go down columns
          // row0 .. row0 + 31 of plane 1 — transposed through shared memory so
          // each lane stores 16 contiguous bytes of one target row (16 byte
          // stores per lane straight to global cost ~2 ms per n = 8192 product)
          __syncwarp();  // the previous chunk's reads of xs are done
#pragma unroll
          for (int e = 0; e < 16; ++e) xs[e * 32 + lane] = (int8_t)(p.herm < 0 ? -r[e] : r[e]);
          __syncwarp();
          const uint4 tv = *reinterpret_cast<const uint4*>(xs + (lane >> 1) * 32 + (lane & 1) * 16);
          const int tcol = col0 + (lane >> 1), trow = row0 + (lane & 1) * 16;
          if (tcol < p.N && trow < p.M) {
            int8_t* tdst = out + (size_t)l * p.out_mod + p.out_plane + (size_t)tcol * p.out_pitch + trow;
            if (trow + 16 <= p.M) {
              *reinterpret_cast<uint4*>(tdst) = tv;
            } else {
              const uint32_t w[4] = {tv.x, tv.y, tv.z, tv.w};
              for (int e = 0; e < 16 && trow + e < p.M; ++e) tdst[e] = (int8_t)((w[e >> 2] >> (8 * (e & 3))) & 0xFF);
            }
          }
        }
        if (row < p.M) {
          int8_t* dst = base + (size_t)plane * p.out_plane + col0;
          if (col0 + 16 <= p.N) {
            *reinterpret_cast<uint4*>(dst) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
          } else {
            for (int e = 0; e < 16 && col0 + e < p.N; ++e) dst[e] = (int8_t)((packed[e >> 2] >> (8 * (e & 3))) & 0xFF);
          }
        }
      };
      uint32_t va[16], vb[16];
      int chunk = half;
      tmem_ld16(tbase + (uint32_t)(chunk * 16), va);
#pragma unroll 1
      for (; chunk < nchunks; chunk += 2 * CSTEP) {
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");  // va = chunk
        if (chunk + CSTEP < nchunks) tmem_ld16(tbase + (uint32_t)((chunk + CSTEP) * 16), vb);
        emit(va, chunk);
        if (chunk + CSTEP >= nchunks) break;
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");  // vb = chunk + CSTEP
        if (chunk + 2 * CSTEP < nchunks) tmem_ld16(tbase + (uint32_t)((chunk + 2 * CSTEP) * 16), va);
        emit(vb, chunk + CSTEP);
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      if (TWO) {
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_u32(tempty_bar(acc), 0));  // the leader's barrier
      } else {
        mbar_arrive(tempty_bar(acc));
      }
      if (!p.wide) acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (CM > 1) cluster_sync();  // no CTA leaves while its peer may still multicast into it
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 1) {
    if (TWO)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem_base));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem_base));
  }
}

// 4-d map over [nmod][planes][rows][kpitch] int8, box (64, 128, planes, 1).
int make_map(CUtensorMap* map, const void* base, int K, int rows, int planes, int nmod, long long kpitch,
             int box_rows, int box_planes) {
  auto enc = get_encode();
  if (!enc) return SR_ECUDA;
  cuuint64_t dims[4] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)planes, (cuuint64_t)nmod};
  cuuint64_t strides[3] = {(cuuint64_t)kpitch, (cuuint64_t)(kpitch * rows), (cuuint64_t)(kpitch * rows * planes)};
  cuuint32_t box[4] = {(cuuint32_t)TK, (cuuint32_t)box_rows, (cuuint32_t)box_planes, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? SR_OK : SR_ECUDA;
}

// Unit table of a lower_only product (cached per shape): units (mp, nt) with
// at least one tile on or below the diagonal, in decode_tile's raster order.
// Per-device launch state (sr_device_slot): the unit-table cache, the pool of
// zeroed unit counters and the one-time shared-memory attributes.
struct OzDevState {
  std::mutex mu;
  std::map<std::tuple<int, int, int, int>, std::pair<int*, int>> tables;
  int* counters = nullptr;
  unsigned launch_seq = 0;
  bool configured = false;
};
OzDevState g_oz_dev[SR_MAX_DEVICES];

const int* lower_table(OzDevState& ds, int tiles_mp, int tiles_n, int cm, int group, int* count) {
  auto& cache = ds.tables;
  const auto key = std::make_tuple(tiles_mp, tiles_n, cm, group);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *count = it->second.second;
    return it->second.first;
  }
  std::vector<int> v;
  for (int first = 0; first < tiles_mp; first += group) {
    const int gm = std::min(group, tiles_mp - first);
    for (int nt = 0; nt < tiles_n; ++nt)
      for (int mp = first; mp < first + gm; ++mp)
        if (nt <= mp * cm + cm - 1) v.push_back(mp | (nt << 16));
  }
  int* d = nullptr;
  if (cudaMalloc(&d, v.size() * sizeof(int)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  cache[key] = std::make_pair(d, (int)v.size());
  *count = (int)v.size();
  return d;
}

int gemm_launch(int M, int N, int K, int nmod, const int* moduli, const void* a, int a_planes, long long a_kpitch,
                const void* b, int b_planes, long long b_kpitch, void* out, long long out_pitch, int lower_only,
                int num_sms, void* stream, bool gauss, int a_swap, int herm) {
  if (M <= 0 || N <= 0 || K <= 0 || nmod <= 0 || nmod > MAX_MODULI) return SR_EINVAL;
  if (lower_only && M != N) return SR_EINVAL;
  if (gauss) {
    if (a_planes != 2 || (b_planes != 1 && b_planes != 2) || lower_only) return SR_EINVAL;
    if (herm != 0 && (M != N || b_planes != 2 || (herm != 1 && herm != -1))) return SR_EINVAL;
  } else if (a_planes != 2 || (b_planes != 1 && b_planes != 3)) {
    return SR_EINVAL;
  }
  if ((a_kpitch | b_kpitch | out_pitch) & 15) return SR_EINVAL;
  if (K > (1 << 16)) return SR_EINVAL;  // 2K terms of |x| <= 2^14: int32 accumulation stays exact
  if (((uintptr_t)a | (uintptr_t)b | (uintptr_t)out) & 15) return SR_EINVAL;
  int slot = 0;
  if (sr_device_slot(&slot) != SR_OK) return SR_EINVAL;
  OzDevState& ds = g_oz_dev[slot];
  std::lock_guard<std::mutex> lock(ds.mu);
  OzParams p;
  memset(&p, 0, sizeof(p));
  // complex x real: [C_re; C_im] = [A_re; A_im] B^T is one real product with
  // 2M stacked rows (the A planes and the output planes are stacked row blocks)
  const bool real = gauss || (b_planes == 1 && !lower_only && !getenv("SR_OZ_NO_REAL"));
  p.M = (real && !gauss) ? 2 * M : M;
  p.N = N;
  p.K = K;
  p.nmod = nmod;
  p.real = real ? 1 : 0;
  p.a_planes = real ? 1 : a_planes;
  p.b_planes = b_planes;
  p.tiles_m = (p.M + TM - 1) / TM;
  const int planes_out = herm ? 1 : 2;
  if (gauss) {
    p.gauss = 1;
    p.a_swap = a_swap & 1;        // bit 0: A planes swapped (X^H from X's B operand)
    p.b_swap = (a_swap >> 1) & 1;  // bit 1: B planes swapped
    p.b_gplane = b_planes == 2 ? 1 : 0;
    p.herm = herm;
    p.tpp = p.tiles_m;
    p.tiles_m = planes_out * p.tpp;
  }
  p.tiles_n = (N + (real ? 2 * TN : TN) - 1) / (real ? 2 * TN : TN);  // (wide: recomputed below)
  p.lower_only = lower_only;
  p.out_pitch = out_pitch;
  p.out_plane = out_pitch * M;
  p.out_mod = out_pitch * M * 2;
  // 2-SM MMAs (cta_group::2) for CTA pairs unless SR_OZ_2SM=0
  const bool two_sm = !(getenv("SR_OZ_2SM") && atoi(getenv("SR_OZ_2SM")) == 0);
  {
    const int stage_bytes = (p.a_planes + (real ? 2 : b_planes)) * PLANE_BYTES;
    p.stages = SMEM_RING / stage_bytes;
    if (p.stages > MAX_STAGES) p.stages = MAX_STAGES;
    if (getenv("SR_OZ_STAGES")) p.stages = std::max(2, std::min(p.stages, atoi(getenv("SR_OZ_STAGES"))));
  }
  for (int i = 0; i < nmod; ++i) {
    if (moduli[i] < 3 || moduli[i] > 256) return SR_EINVAL;
    p.moduli[i] = moduli[i];
    p.inv[i] = 1.0f / (float)moduli[i];
    // |accumulator| <= 2 K (p/2)^2 (two MMAs per k for the (re, im) planes); the
    // offset keeps v + roff in [0, 2^32) for the Barrett step
    const unsigned long long m = (unsigned long long)moduli[i];
    const unsigned long long vmax = 2ull * (unsigned long long)K * (m / 2) * (m / 2);
    const unsigned long long off = (vmax / m + 1) * m + m / 2;
    if (off + vmax >= (1ull << 32)) return SR_EINVAL;  // K beyond 2^16
    p.bm[i] = (uint32_t)((1ull << 32) / m + 1);
    p.roff[i] = (uint32_t)off;
  }
  int grid = num_sms > 0 ? num_sms : 148;
  // clusters of two CTAs sharing the B tile whenever there are M-tile pairs to share
  int cm = (p.tiles_m >= 2 && grid >= 2 && !getenv("SR_OZ_NO_CLUSTER")) ? 2 : 1;
  if (getenv("SR_OZ_CM")) cm = atoi(getenv("SR_OZ_CM"));
  if (cm != 1 && cm != 2 && cm != 4) cm = 2;
  if (p.tiles_m < cm) cm = 1;
  if (gauss && cm == 4) cm = 2;
  if (gauss && cm == 2 && (p.tpp & 1)) {  // a CTA pair never straddles two planes
    p.tpp += 1;
    p.tiles_m = planes_out * p.tpp;
  }
  const bool two = two_sm && cm == 2;
  // wide units (N = 512) for the 2-SM real products: 18-20 % faster at
  // n = K = 8192 (tools/oz_wide_ab.py, interleaved A/B), but the epilogue of a
  // wide unit is not overlapped with MMAs, so short K (15-22 % slower at 2048)
  // stays narrow.  Hermitian products: wide since their transposed write is
  // staged through shared memory (7.6-8.1 vs 8.8-9.0 ms narrow at n = 8192).
  // SR_OZ_WIDE=0 / 1 forces either.
  bool wide = two && real && K >= 4096;
  const char* wide_env = getenv("SR_OZ_WIDE");
  if (wide_env && *wide_env && strcmp(wide_env, "auto") != 0) wide = two && real && atoi(wide_env) != 0;
  p.wide = wide ? 1 : 0;
  p.epi = (wide && !getenv("SR_OZ_EPI4")) ? (getenv("SR_OZ_EPI") ? atoi(getenv("SR_OZ_EPI")) : 16) : 4;
  if (p.epi != 4 && p.epi != 8 && p.epi != 16) p.epi = 8;
  if (p.wide) p.tiles_n = (N + 4 * TN - 1) / (4 * TN);
  const int tiles = nmod * p.tiles_m * p.tiles_n;
  if (two) {  // per CTA: its A rows and half of the pair's B operand (real: two k-blocks per slot)
    // narrow real products: four k-blocks per slot (eight MMAs per barrier round trip, like the wide ones)
    p.kstep = real ? ((p.wide || getenv("SR_OZ_KSTEP2")) ? 2 : 4) : 1;
    p.stages = std::min(MAX_STAGES, SMEM_RING / ((real ? p.kstep : 1) *
                                                 (p.a_planes + (real ? (p.wide ? 2 : 1) : 2)) * PLANE_BYTES));
    if (getenv("SR_OZ_STAGES")) p.stages = std::max(2, std::min(p.stages, atoi(getenv("SR_OZ_STAGES"))));
  }
  p.group_m = (getenv("SR_OZ_GROUP_M") ? atoi(getenv("SR_OZ_GROUP_M")) : (real ? 2 : 1) * GROUP_M) / cm;
  if (p.group_m < 1) p.group_m = 1;
  if (lower_only && !getenv("SR_OZ_NO_COMPACT")) {
    const int tiles_mp = (p.tiles_m + cm - 1) / cm;
    p.table = lower_table(ds, tiles_mp, p.tiles_n, cm, p.group_m, &p.units_per_mod);
    if (!p.table) return sr_set_cuda_error(cudaErrorMemoryAllocation, "oz_gemm lower-unit table");
  }
  if (grid > tiles) grid = tiles;
  grid -= grid % cm;
  if (grid < cm) grid = cm;
  CUtensorMap ma, mb;
  const int rc_a = gauss ? make_map(&ma, a, K, M, 2, nmod, a_kpitch, TM, 1)
                         : make_map(&ma, a, K, p.M, p.a_planes, nmod, a_kpitch, TM, p.a_planes);
  if (rc_a != SR_OK) return sr_set_cuda_error(cudaErrorInvalidValue, "cuTensorMapEncodeTiled(A)");
  if (make_map(&mb, b, K, N, b_planes, nmod, b_kpitch, two ? TN : (real ? 2 * TN : TN) / cm,
               (cm == 1 && !two && !gauss) ? b_planes : 1) != SR_OK)
    return sr_set_cuda_error(cudaErrorInvalidValue, "cuTensorMapEncodeTiled(B)");
  const size_t smem = 1024 + (size_t)SMEM_RING + SMEM_TAIL + (herm ? (size_t)MAX_EPI_WARPS * XPOSE_WARP_BYTES : 0);
  // one zeroed unit counter per launch (a pool, so launches on different
  // streams never share one)
  constexpr int NCOUNTERS = 256;
  if (!ds.counters && cudaMalloc(&ds.counters, NCOUNTERS * 32 * sizeof(int)) != cudaSuccess)
    return sr_set_cuda_error(cudaErrorMemoryAllocation, "oz_gemm unit counters");
  int* counter = ds.counters + 32 * (ds.launch_seq++ % NCOUNTERS);  // 128-byte apart
  SR_CUDA_CHECK(cudaMemsetAsync(counter, 0, sizeof(int), (cudaStream_t)stream));
  if (!ds.configured) {
    SR_CUDA_CHECK(cudaFuncSetAttribute(oz_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    SR_CUDA_CHECK(cudaFuncSetAttribute(oz_gemm_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    SR_CUDA_CHECK(
        cudaFuncSetAttribute(oz_gemm_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    SR_CUDA_CHECK(cudaFuncSetAttribute(oz_gemm_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    ds.configured = true;
  }
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(64 + 32 * p.epi);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = cm;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  if (cm == 4) {
    // persistent clusters: never more than can be co-resident
    int ncl = 0;
    cfg.gridDim = dim3(cm);
    SR_CUDA_CHECK(cudaOccupancyMaxActiveClusters(&ncl, oz_gemm_kernel<4>, &cfg));
    if (ncl > 0 && ncl * cm < grid) grid = ncl * cm;
    cfg.gridDim = dim3(grid);
    SR_CUDA_CHECK(cudaLaunchKernelEx(&cfg, oz_gemm_kernel<4>, ma, mb, p, (int8_t*)out, counter));
  } else if (two)
    SR_CUDA_CHECK(cudaLaunchKernelEx(&cfg, oz_gemm_kernel<2, true>, ma, mb, p, (int8_t*)out, counter));
  else if (cm == 2)
    SR_CUDA_CHECK(cudaLaunchKernelEx(&cfg, oz_gemm_kernel<2>, ma, mb, p, (int8_t*)out, counter));
  else
    SR_CUDA_CHECK(cudaLaunchKernelEx(&cfg, oz_gemm_kernel<1>, ma, mb, p, (int8_t*)out, counter));
  SR_LAUNCH_CHECK();
  return SR_OK;
}
}  // namespace

extern "C" int sr_oz_gemm_i8(int M, int N, int K, int nmod, const int* moduli, const void* a, int a_planes,
                             long long a_kpitch, const void* b, int b_planes, long long b_kpitch, void* out,
                             long long out_pitch, int lower_only, int num_sms, void* stream) {
  return gemm_launch(M, N, K, nmod, moduli, a, a_planes, a_kpitch, b, b_planes, b_kpitch, out, out_pitch, lower_only,
                     num_sms, stream, false, 0, 0);
}

extern "C" int sr_oz_gemm_i8_gauss(int M, int N, int K, int nmod, const int* moduli, const void* a, int a_swap,
                                   long long a_kpitch, const void* b, int b_planes, long long b_kpitch, void* out,
                                   long long out_pitch, int herm, int num_sms, void* stream) {
  return gemm_launch(M, N, K, nmod, moduli, a, 2, a_kpitch, b, b_planes, b_kpitch, out, out_pitch, 0, num_sms, stream,
                     true, a_swap, herm);
}

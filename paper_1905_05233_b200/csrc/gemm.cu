// gemm.cu -- K3: the Winograd-domain channel reduction on the 5th-generation
// tensor cores (the Hadamard product, summed over input
// channels, "dominates the execution time" of DNN Winograd convolution):
//
//     M_p[k][t] = sum_{(q, u) in sched(p)} sum_c U_u[k][c] * V_q[t][c]
//
// SUBSOLVER lowering: sched(p) = {(p, p)} -- mu^2 independent GEMMs.
// RESIDUE lowering:   sched(p) = the block-pair units of output point p (the
// "2x2-block polynomial product mod m_i" contracting C x |I| x |J|).
//
// Design (sm_100a): persistent, warp-specialised, one CTA per SM.
//   warp 0      TMA producer: A = V_q tile [128 t x BK c], B = U_u tile
//               [BN k x BK c], both K-major with the 128-byte swizzle, into a
//               STAGES-deep mbarrier ring.
//   warp 1      MMA issuer (one thread): tcgen05.mma.cta_group::1, M = 128,
//               N = BN, fp32 accumulators in TMEM (2 x BN columns, double
//               buffered so the epilogue of item i overlaps the MMAs of i+1).
//               kind::f16 for fp16/bf16; fp32 runs three kind::tf32 products
//               hi*hi + hi*lo + lo*hi per K step (hi/lo planes made by K1/K2).
//   warps 4..7  epilogue: tcgen05.ld 32x32b (TMEM lane = tile t) into
//               registers, st.shared into a [32 k][128 t] staging buffer
//               (conflict-free: a warp writes 128 contiguous bytes per k), then
//               one thread TMA-stores the box to M[p][k0:k0+32][t0:t0+128]
//               (cp.async.bulk.tensor, clipped at the ragged edges).  The
//               accumulator is released to the MMA warp as soon as its last
//               columns are in registers.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "device.cuh"
#include "geometry.hpp"
#include "tmap.hpp"
#include "gemm_common.cuh"

namespace wino {

// M element of the epilogue store: 0 = fp32 (reading R1), 1 = fp16, 2 = bf16
// (reading M3: the fp32 accumulator rounded once to the layer dtype, RNE)
template <int MT>
__device__ __forceinline__ void epi_put(float* buf, int idx, float v) {
  if constexpr (MT == 0) buf[idx] = v;
  else if constexpr (MT == 1) reinterpret_cast<__half*>(buf)[idx] = __float2half_rn(v);
  else reinterpret_cast<__nv_bfloat16*>(buf)[idx] = __float2bfloat16_rn(v);
}

template <bool kTF32, int BN, int STAGES, int MT = 0>
__global__ void __launch_bounds__(256, 1)
    domain_gemm_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmU,
                       const __grid_constant__ CUtensorMap tmM, int T, int K, int Cp, int nMB, int nNB, int Q, int S,
                       uint32_t idesc, const __grid_constant__ GemmSched gs, int mb0, int TBv) {
  using Cfg = GemmCfg<kTF32, BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned for the 128-byte swizzle atoms; offsetting the shared array keeps
  // a shared-space pointer (STS / LDS, no generic stores and CTA-wide MEMBARs)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* epi = reinterpret_cast<float*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::EPI_BUFS * Cfg::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmV);
    tma_prefetch(&tmU);
    tma_prefetch(&tmM);
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    for (int a = 0; a < 2; ++a) mbar_init(&tfull[a], 1), mbar_init(&tempty[a], 4);
    fence_barrier_init();
    fence_proxy_async_shared();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int nItems = Q * nMB * nNB;
  const int KB = Cp / Cfg::BK;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int item = blockIdx.x; item < nItems; item += gridDim.x) {
        const int nb = item % nNB, mb = (item / nNB) % nMB, p = item / (nNB * nMB);
        for (int pr = gs.off[p]; pr < gs.off[p + 1]; ++pr) {
          const int qi = gs.in_pt[pr], sl = gs.slab[pr];
          for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
            uint8_t* base = smem + stage * Cfg::STAGE_BYTES;
            tma_load_3d(base, &tmV, &full[stage], 0, 0, ((mb0 + mb) * KB + kb) * Q + qi);   // blocked V: one 16 KB block
            if constexpr (kTF32)
              tma_load_3d(base + Cfg::A_BYTES, &tmV, &full[stage], 0, 0, ((TBv + mb0 + mb) * KB + kb) * Q + qi);
            uint8_t* bb = base + Cfg::NPL * Cfg::A_BYTES;
            tma_load_3d(bb, &tmU, &full[stage], kb * Cfg::BK, nb * BN, sl);
            if constexpr (kTF32) tma_load_3d(bb + Cfg::B_BYTES, &tmU, &full[stage], kb * Cfg::BK, nb * BN, sl + S);
            if (++stage == STAGES) stage = 0, phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int item = blockIdx.x; item < nItems; item += gridDim.x) {
        const int p = item / (nNB * nMB);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        int step = 0;
        for (int pr = gs.off[p]; pr < gs.off[p + 1]; ++pr) {
          for (int kb = 0; kb < KB; ++kb, ++step) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t a0 = smem_u32(smem + stage * Cfg::STAGE_BYTES);
            const uint32_t b0 = a0 + Cfg::NPL * Cfg::A_BYTES;
#pragma unroll
            for (int k = 0; k < Cfg::BK / Cfg::UK; ++k) {
              const uint32_t koff = k * Cfg::UK * Cfg::ES;  // 32 bytes
              mma_ss<kTF32>(d_tmem, umma_desc_sw128(a0 + koff), umma_desc_sw128(b0 + koff), idesc,
                            (step | k) != 0);
              if constexpr (kTF32) {
                mma_ss<true>(d_tmem, umma_desc_sw128(a0 + koff), umma_desc_sw128(b0 + Cfg::B_BYTES + koff), idesc, 1);
                mma_ss<true>(d_tmem, umma_desc_sw128(a0 + Cfg::A_BYTES + koff), umma_desc_sw128(b0 + koff), idesc, 1);
              }
            }
            mma_commit(&empty[stage]);
            if (++stage == STAGES) stage = 0, phase ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
        if (++acc == 2) acc = 0, acc_phase ^= 1;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // -------------------------------------------------- epilogue
    const int wq = warp & 3;
    const bool storer = (warp == 4 && lane == 0);
    int acc = 0, chunk = 0;
    uint32_t acc_phase = 0;
    for (int item = blockIdx.x; item < nItems; item += gridDim.x) {
      const int nb = item % nNB, mb = (item / nNB) % nMB, p = item / (nNB * nMB);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int j0 = 0; j0 < BN; j0 += 32) {
        float v[32];
        tmem_ld32(tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN + j0, v);
        if (j0 + 32 == BN) {  // accumulator fully read: hand it back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        if (nb * BN + j0 >= K) continue;                 // columns past K (uniform branch)
        float* buf = epi + (chunk % Cfg::EPI_BUFS) * (Cfg::EPI_BYTES / 4);
        if (storer) bulk_wait_read<Cfg::EPI_BUFS - 1>();   // the store that last read `buf` is done
        named_bar_sync(1, 128);
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) epi_put<MT>(buf, jj * kBM + wq * 32 + lane, v[jj]);
        fence_proxy_async_shared();
        named_bar_sync(1, 128);
        if (storer) {
          tma_store_3d(&tmM, buf, mb * kBM, nb * BN + j0, p);
          bulk_commit();
        }
        ++chunk;
      }
      if (++acc == 2) acc = 0, acc_phase ^= 1;
    }
    if (storer) bulk_wait_all();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ CTA-pair variant
// The same GEMM with cta_group::2: a cluster of two CTAs (one TPC) owns a
// [256 t x 256 k] output tile of one point.  CTA r loads its own A block (V, tiles
// [256 mb2 + 128 r, +128)) and half of B (U rows k in [256 nb + 128 r, +128)); the
// leader's single MMA thread issues M = 256, N = 256 MMAs that read both CTAs'
// shared memory, and each CTA's TMEM receives its own 128 tile rows x 256 k.
// Per SM that is 32 KB of operands per 128 x 256 x 64 step instead of 48 KB
// (B is no longer loaded by both SMs): K3 at one CTA per SM is bound by the
// SM's L2 ingress together with its fp32 M egress.
//   barriers: full[s] (leader: 2 arrivals + both CTAs' bytes), empty[s] (each CTA,
//   multicast MMA commit), tfull[a] (each CTA, multicast commit), tempty[a]
//   (leader: 4 epilogue warps x 2 CTAs, remote arrives from the peer).
template <bool kTF32, int STAGES, int EPI, int EC = 32>
struct PairCfg {
  static constexpr int ES = kTF32 ? 4 : 2;
  static constexpr int BK = 128 / ES;
  static constexpr int UK = kTF32 ? 8 : 16;
  static constexpr int NPL = kTF32 ? 2 : 1;
  static constexpr int BN = 256;                    // k per pair tile (N of the MMA)
  static constexpr int A_BYTES = kBM * 128;         // 128 t rows x 128 B
  static constexpr int B_BYTES = (BN / 2) * 128;    // this CTA's 128 k rows
  static constexpr int STAGE_BYTES = NPL * (A_BYTES + B_BYTES);
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int EPI_COLS = EC;               // k columns per M store box
  static constexpr int EPI_BYTES = EC * kBM * 4;
  static constexpr int EPI_BUFS = EPI;
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BUFS * EPI_BYTES + 1024 + 256;
  static_assert(EPI_BUFS >= 2 && SMEM <= 227 * 1024 && (EC == 16 || EC == 32), "shared memory");
};

// L2 eviction-priority policy (createpolicy) for the streamed fp32 M stores
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_store_3d_hint(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                                  uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4}], [%1], %5;" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
      : "memory");
}

template <bool kTF32, int STAGES, int EPI, bool kHint, int EC, int MT = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    domain_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmU,
                            const __grid_constant__ CUtensorMap tmM, int T, int K, int Cp, int nMB2, int nNB, int Q,
                            int S, uint32_t idesc, const __grid_constant__ GemmSched gs, int mb0, int TBv) {
  using Cfg = PairCfg<kTF32, STAGES, EPI, EC>;
  constexpr int BN = Cfg::BN;
  extern __shared__ uint8_t smem_raw[];
  // the same offset in both CTAs (the MMA addresses the peer's operands by the leader's offsets)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* epi = reinterpret_cast<float*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::EPI_BUFS * Cfg::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmV);
    tma_prefetch(&tmU);
    tma_prefetch(&tmM);
    // full: (leader) its own expect_tx arrival + the peer's arrival, both CTAs' bytes;
    // tempty: (leader) 4 epilogue warps x 2 CTAs
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 2), mbar_init(&empty[s], 1);
    for (int a = 0; a < 2; ++a) mbar_init(&tfull[a], 1), mbar_init(&tempty[a], 8);
    fence_barrier_init();
    fence_proxy_async_shared();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int nItems = Q * nMB2 * nNB;
  const int KB = Cp / Cfg::BK;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int item = cl; item < nItems; item += ncl) {
        const int nb = item % nNB, mb2 = (item / nNB) % nMB2, p = item / (nNB * nMB2);
        const int mb = mb0 + 2 * mb2 + (int)rank;   // this CTA's 128-tile block
        const int k0 = nb * BN + (int)rank * (BN / 2);
        for (int pr = gs.off[p]; pr < gs.off[p + 1]; ++pr) {
          const int qi = gs.in_pt[pr], sl = gs.slab[pr];
          for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t fb = mapa_rank(&full[stage], 0);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * Cfg::STAGE_BYTES);
            else mbar_arrive_cluster(fb);
            uint8_t* base = smem + stage * Cfg::STAGE_BYTES;
            tma_load_3d_pair(base, &tmV, fb, 0, 0, (mb * KB + kb) * Q + qi);
            if constexpr (kTF32) tma_load_3d_pair(base + Cfg::A_BYTES, &tmV, fb, 0, 0, ((TBv + mb) * KB + kb) * Q + qi);
            uint8_t* bb = base + Cfg::NPL * Cfg::A_BYTES;
            tma_load_3d_pair(bb, &tmU, fb, kb * Cfg::BK, k0, sl);
            if constexpr (kTF32) tma_load_3d_pair(bb + Cfg::B_BYTES, &tmU, fb, kb * Cfg::BK, k0, sl + S);
            if (++stage == STAGES) stage = 0, phase ^= 1;
          }
        }
      }
      // drain: every stage released by the leader's MMAs (all multicast arrivals
      // on this CTA's barriers have landed before the CTA may exit)
      for (int s = 0; s < STAGES; ++s) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (++stage == STAGES) stage = 0, phase ^= 1;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ------------------------------------------------ MMA issuer (leader only)
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int item = cl; item < nItems; item += ncl) {
        const int p = item / (nNB * nMB2);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        int step = 0;
        for (int pr = gs.off[p]; pr < gs.off[p + 1]; ++pr) {
          for (int kb = 0; kb < KB; ++kb, ++step) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t a0 = smem_u32(smem + stage * Cfg::STAGE_BYTES);
            const uint32_t b0 = a0 + Cfg::NPL * Cfg::A_BYTES;
#pragma unroll
            for (int k = 0; k < Cfg::BK / Cfg::UK; ++k) {
              const uint32_t koff = k * Cfg::UK * Cfg::ES;  // 32 bytes
              mma_ss_pair<kTF32>(d_tmem, umma_desc_sw128(a0 + koff), umma_desc_sw128(b0 + koff), idesc,
                                 (step | k) != 0);
              if constexpr (kTF32) {
                mma_ss_pair<true>(d_tmem, umma_desc_sw128(a0 + koff), umma_desc_sw128(b0 + Cfg::B_BYTES + koff),
                                  idesc, 1);
                mma_ss_pair<true>(d_tmem, umma_desc_sw128(a0 + Cfg::A_BYTES + koff), umma_desc_sw128(b0 + koff),
                                  idesc, 1);
              }
            }
            mma_commit_pair(&empty[stage]);
            if (++stage == STAGES) stage = 0, phase ^= 1;
          }
        }
        mma_commit_pair(&tfull[acc]);
        if (++acc == 2) acc = 0, acc_phase ^= 1;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // -------------------------------------------------- epilogue (both CTAs)
    const int wq = warp & 3;
    const bool storer = (warp == 4 && lane == 0);
    uint64_t pol = 0;
    if constexpr (kHint) pol = l2_evict_first();
    int acc = 0, chunk = 0;
    uint32_t acc_phase = 0;
    for (int item = cl; item < nItems; item += ncl) {
      const int nb = item % nNB, mb2 = (item / nNB) % nMB2, p = item / (nNB * nMB2);
      const int t0 = (2 * mb2 + (int)rank) * kBM;   // relative to mb0 * 128 (M holds this slice)
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int j0 = 0; j0 < BN; j0 += 32) {
        float v[32];
        tmem_ld32(tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN + j0, v);
        if (j0 + 32 == BN) {  // accumulator fully read: hand it back to the leader's MMA thread
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_rank(&tempty[acc], 0));
        }
        if (nb * BN + j0 >= K || t0 >= T) continue;   // columns past K, tile block past the slice (uniform)
#pragma unroll
        for (int h = 0; h < 32; h += EC) {
          float* buf = epi + (chunk % Cfg::EPI_BUFS) * (Cfg::EPI_BYTES / 4);
          if (storer) bulk_wait_read<Cfg::EPI_BUFS - 1>();
          named_bar_sync(1, 128);
#pragma unroll
          for (int jj = 0; jj < EC; ++jj) epi_put<MT>(buf, jj * kBM + wq * 32 + lane, v[h + jj]);
          fence_proxy_async_shared();
          named_bar_sync(1, 128);
          if (storer) {
            if constexpr (kHint) tma_store_3d_hint(&tmM, buf, t0, nb * BN + j0 + h, p, pol);
            else tma_store_3d(&tmM, buf, t0, nb * BN + j0 + h, p);
            bulk_commit();
          }
          ++chunk;
        }
      }
      if (++acc == 2) acc = 0, acc_phase ^= 1;
    }
    if (storer) bulk_wait_all();
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ CTA pair, resident U
// The CTA-pair GEMM with the B operand kept in shared memory.  A work unit is one
// (point p, 256-wide k block nb) and a range of 256-tile blocks: each CTA loads its
// 128 k rows of U_p for ALL Cp channels once (Cp <= 512: 8 swizzled 16 KB boxes,
// 128 KB) and then streams only V through a 4-stage ring, so a CTA receives 16 KB
// of operands per 128 x 256 x 64 step instead of 32 KB (the per-SM L2 ingress
// that bounds the streamed-B kernel).  SUBSOLVER (identity
// schedule), 16-bit operands.  Same accumulation order per output element as the
// other K3 kernels (k blocks ascending, 16-element MMA steps): identical bits.
//   barriers: as domain_gemm_pair_kernel, plus ufull (leader: 2 arrivals + both
//   CTAs' U bytes) and uempty (each CTA, multicast commit after a unit's MMAs).
template <int STAGES, int MT>
struct UresCfg {
  static constexpr int BK = 64, UK = 16, BN = 256;
  static constexpr int A_BYTES = kBM * 128;
  static constexpr int UBLK = 128 * 128;             // one k block of this CTA's 128 U rows
  static constexpr int U_BYTES = 8 * UBLK;           // Cp <= 512
  static constexpr int EPI_BYTES = 32 * kBM * 4;
  static constexpr int SMEM = U_BYTES + STAGES * A_BYTES + 2 * EPI_BYTES + 1024 + 256;
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

template <int STAGES, int MT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    domain_gemm_ures_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmU,
                            const __grid_constant__ CUtensorMap tmM, int T, int K, int Cp, int nMB2, int nNB, int Q,
                            int nSplit, uint32_t idesc, int mb0) {
  using Cfg = UresCfg<STAGES, MT>;
  constexpr int BN = Cfg::BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ures = smem;
  uint8_t* astg = smem + Cfg::U_BYTES;
  float* epi = reinterpret_cast<float*>(astg + STAGES * Cfg::A_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(epi) + 2 * Cfg::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ufull = tempty + 2;
  uint64_t* uempty = ufull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(uempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmV);
    tma_prefetch(&tmU);
    tma_prefetch(&tmM);
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 2), mbar_init(&empty[s], 1);
    for (int a = 0; a < 2; ++a) mbar_init(&tfull[a], 1), mbar_init(&tempty[a], 8);
    mbar_init(ufull, 2), mbar_init(uempty, 1);
    fence_barrier_init();
    fence_proxy_async_shared();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, 2 * BN);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int KB = Cp / Cfg::BK;
  const int nWork = Q * nNB * nSplit;
  // work w: unit (p, nb) = w / nSplit, tile-block-pair range [lo, hi) of split w % nSplit
  auto work = [&](int w, int& p, int& nb, int& lo, int& hi) {
    const int u = w / nSplit, sp = w % nSplit;
    p = u / nNB, nb = u % nNB;
    lo = (int)((long long)nMB2 * sp / nSplit), hi = (int)((long long)nMB2 * (sp + 1) / nSplit);
  };

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0, uphase = 0;
      for (int w = cl; w < nWork; w += ncl) {
        int p, nb, lo, hi;
        work(w, p, nb, lo, hi);
        if (lo >= hi) continue;
        // this CTA's 128 U rows of (p, nb), every k block, once per unit
        mbar_wait(uempty, uphase ^ 1);
        const uint32_t ub = mapa_rank(ufull, 0);
        if (rank == 0) mbar_arrive_expect_tx(ufull, 2 * KB * Cfg::UBLK);
        else mbar_arrive_cluster(ub);
        const int k0 = nb * BN + (int)rank * (BN / 2);
        for (int kb = 0; kb < KB; ++kb) tma_load_3d_pair(ures + kb * Cfg::UBLK, &tmU, ub, kb * Cfg::BK, k0, p);
        uphase ^= 1;
        for (int mb2 = lo; mb2 < hi; ++mb2) {
          const int mb = mb0 + 2 * mb2 + (int)rank;
          for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t fb = mapa_rank(&full[stage], 0);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * Cfg::A_BYTES);
            else mbar_arrive_cluster(fb);
            tma_load_3d_pair(astg + stage * Cfg::A_BYTES, &tmV, fb, 0, 0, (mb * KB + kb) * Q + p);
            if (++stage == STAGES) stage = 0, phase ^= 1;
          }
        }
      }
      for (int s = 0; s < STAGES; ++s) {   // drain: every multicast arrival has landed
        mbar_wait(&empty[stage], phase ^ 1);
        if (++stage == STAGES) stage = 0, phase ^= 1;
      }
      mbar_wait(uempty, uphase ^ 1);
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ------------------------------------------------ MMA issuer (leader only)
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0, uphase = 0;
      for (int w = cl; w < nWork; w += ncl) {
        int p, nb, lo, hi;
        work(w, p, nb, lo, hi);
        if (lo >= hi) continue;
        mbar_wait(ufull, uphase);
        uphase ^= 1;
        tc_fence_after();
        const uint32_t u0 = smem_u32(ures);
        for (int mb2 = lo; mb2 < hi; ++mb2) {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t a0 = smem_u32(astg + stage * Cfg::A_BYTES);
            const uint32_t b0 = u0 + kb * Cfg::UBLK;
#pragma unroll
            for (int k = 0; k < Cfg::BK / Cfg::UK; ++k) {
              const uint32_t koff = k * Cfg::UK * 2;   // 32 bytes
              mma_ss_pair<false>(d_tmem, umma_desc_sw128(a0 + koff), umma_desc_sw128(b0 + koff), idesc,
                                 (kb | k) != 0);
            }
            mma_commit_pair(&empty[stage]);
            if (++stage == STAGES) stage = 0, phase ^= 1;
          }
          mma_commit_pair(&tfull[acc]);
          if (++acc == 2) acc = 0, acc_phase ^= 1;
        }
        mma_commit_pair(uempty);   // the unit's MMAs (all readers of U) are done
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // -------------------------------------------------- epilogue (both CTAs)
    const int wq = warp & 3;
    const bool storer = (warp == 4 && lane == 0);
    int acc = 0, chunk = 0;
    uint32_t acc_phase = 0;
    for (int w = cl; w < nWork; w += ncl) {
      int p, nb, lo, hi;
      work(w, p, nb, lo, hi);
      for (int mb2 = lo; mb2 < hi; ++mb2) {
        const int t0 = (2 * mb2 + (int)rank) * kBM;
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
#pragma unroll 1
        for (int j0 = 0; j0 < BN; j0 += 32) {
          float v[32];
          tmem_ld32(tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN + j0, v);
          if (j0 + 32 == BN) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_rank(&tempty[acc], 0));
          }
          if (nb * BN + j0 >= K || t0 >= T) continue;
          float* buf = epi + (chunk & 1) * (Cfg::EPI_BYTES / 4);
          if (storer) bulk_wait_read<1>();
          named_bar_sync(1, 128);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) epi_put<MT>(buf, jj * kBM + wq * 32 + lane, v[jj]);
          fence_proxy_async_shared();
          named_bar_sync(1, 128);
          if (storer) {
            tma_store_3d(&tmM, buf, t0, nb * BN + j0, p);
            bulk_commit();
          }
          ++chunk;
        }
        if (++acc == 2) acc = 0, acc_phase ^= 1;
      }
    }
    if (storer) bulk_wait_all();
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 2 * BN);
  }
}

// ------------------------------------------------------------------ host side

template <bool kTF32, int STAGES, int EPI, bool kHint, int EC = 32, int MT = 0>
static wino_status launch_gemm_pair(const CUtensorMap& tv, const CUtensorMap& tu, const CUtensorMap& tm, const Geo& g,
                                    const GemmSched& gs, uint32_t fmt, int mb0, int nT, cudaStream_t st) {
  using Cfg = PairCfg<kTF32, STAGES, EPI, EC>;
  auto kern = domain_gemm_pair_kernel<kTF32, STAGES, EPI, kHint, EC, MT>;
  WINO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int nMB2 = (nT + 2 * kBM - 1) / (2 * kBM), nNB = (g.K + Cfg::BN - 1) / Cfg::BN;
  const int items = g.Q * nMB2 * nNB;
  DevState* ds = dev_state();
  if (!ds) return WINO_E_CUDA;
  if (ds->pair_clusters == 0) {   // co-resident clusters of two (every config runs one CTA per SM)
    cudaLaunchConfig_t qc = {};
    qc.gridDim = dim3(2 * (ds->sms / 2), 1, 1);
    qc.blockDim = dim3(256, 1, 1);
    qc.dynamicSmemBytes = Cfg::SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
    qc.attrs = at, qc.numAttrs = 1;
    int ncl = 0;
    WINO_CUDA_CHECK(cudaOccupancyMaxActiveClusters(&ncl, kern, &qc));
    ds->pair_clusters = ncl > 0 ? ncl : 1;
  }
  const int ncl = items < ds->pair_clusters ? items : ds->pair_clusters;
  kern<<<2 * ncl, 256, Cfg::SMEM, st>>>(tv, tu, tm, nT, g.K, g.Cp, nMB2, nNB, g.Q, g.S,
                                        make_idesc(fmt, 2 * kBM, Cfg::BN), gs, mb0, g.TB);
  WINO_LAUNCH_CHECK();
  return WINO_OK;
}

template <bool kTF32, int BN, int STAGES, int MT = 0>
static wino_status launch_gemm(const CUtensorMap& tv, const CUtensorMap& tu, const CUtensorMap& tm, const Geo& g,
                               const GemmSched& gs, uint32_t fmt, int mb0, int nT, cudaStream_t st) {
  using Cfg = GemmCfg<kTF32, BN, STAGES>;
  auto kern = domain_gemm_kernel<kTF32, BN, STAGES, MT>;
  // (a per-device attribute: set on every launch, it is a cheap host call)
  WINO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int nMB = (nT + kBM - 1) / kBM, nNB = (g.K + BN - 1) / BN;
  const int items = g.Q * nMB * nNB;
  const int grid = items < num_sms() ? items : num_sms();
  kern<<<grid, 256, Cfg::SMEM, st>>>(tv, tu, tm, nT, g.K, g.Cp, nMB, nNB, g.Q, g.S,
                                     make_idesc(fmt, kBM, BN), gs, mb0, g.TB);
  WINO_LAUNCH_CHECK();
  return WINO_OK;
}

template <int STAGES, int MT>
static wino_status launch_gemm_ures(const CUtensorMap& tv, const CUtensorMap& tu, const CUtensorMap& tm,
                                    const Geo& g, uint32_t fmt, int mb0, int nT, cudaStream_t st) {
  using Cfg = UresCfg<STAGES, MT>;
  auto kern = domain_gemm_ures_kernel<STAGES, MT>;
  WINO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int nMB2 = (nT + 2 * kBM - 1) / (2 * kBM), nNB = (g.K + Cfg::BN - 1) / Cfg::BN;
  DevState* ds = dev_state();
  if (!ds) return WINO_E_CUDA;
  if (ds->ures_clusters == 0) {
    cudaLaunchConfig_t qc = {};
    qc.gridDim = dim3(2 * (ds->sms / 2), 1, 1);
    qc.blockDim = dim3(256, 1, 1);
    qc.dynamicSmemBytes = Cfg::SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
    qc.attrs = at, qc.numAttrs = 1;
    int ncl = 0;
    WINO_CUDA_CHECK(cudaOccupancyMaxActiveClusters(&ncl, kern, &qc));
    ds->ures_clusters = ncl > 0 ? ncl : 1;
  }
  // units (p, nb); split each unit's tile-block range so every cluster has work
  const int units = g.Q * nNB;
  int nSplit = (ds->ures_clusters + units - 1) / units;
  if (nSplit > nMB2) nSplit = nMB2;
  if (nSplit < 1) nSplit = 1;
  const int works = units * nSplit;
  const int ncl = works < ds->ures_clusters ? works : ds->ures_clusters;
  kern<<<2 * ncl, 256, Cfg::SMEM, st>>>(tv, tu, tm, nT, g.K, g.Cp, nMB2, nNB, g.Q, nSplit,
                                        make_idesc(fmt, 2 * kBM, Cfg::BN), mb0);
  WINO_LAUNCH_CHECK();
  return WINO_OK;
}

// Resident-U CTA-pair K3, opt-in (WINO_URES=1): 16-bit SUBSOLVER layers with the
// identity schedule, K > 128 and Cp <= 512.  Measured slower than the streamed-U
// pair kernel on cfg5 lin4 (266 vs 240 us fp32 M, 217 vs 198 us 16-bit M): halving
// the per-SM operand ingress does not pay for its shallower (4 x 16 KB) A ring and
// the per-unit U reload bubbles.
static bool ures_enabled() {
  const char* e = getenv("WINO_URES");
  return e && *e == '1';
}
static bool identity_sched(const GemmSched& gs) {
  if (gs.npairs != gs.Q) return false;
  for (int p = 0; p < gs.Q; ++p)
    if (gs.off[p] != p || gs.in_pt[p] != p || gs.slab[p] != p) return false;
  return true;
}

// The CTA-pair K3 is the default for 16-bit layers with K > 128 (WINO_PAIR=0 selects
// the one-CTA kernel, for comparison).
static bool pair_enabled() {
  const char* e = getenv("WINO_PAIR");   // read per call (tests compare both kernels in one process)
  return !(e && *e == '0');
}

// M_xi for the tiles [mb0 * 128, mb0 * 128 + nT) of V (all of them by default) into
// M [Q][K][Tpm] with Tpm = nT rounded up to 32 (chunked layers: an L2-sized slice);
// M is fp32, or the layer dtype for 16-bit layers when the algorithm stores M in
// the dtype (wino_set_m_storage, reading M3)
template <int MT>
static wino_status launch_domain_gemm_16(const CUtensorMap& tv, const CUtensorMap& tu, const CUtensorMap& tm,
                                         const void* U, const Geo& g, const wino_algo* al, CUtensorMapDataType cdt,
                                         uint32_t fmt, int BN, int mb0, int nT, cudaStream_t st) {
  const uint32_t BK = 128 / (uint32_t)g.es;
  if (BN == 256 && nT > kBM && pair_enabled() && ures_enabled() && g.Cp <= 512 && identity_sched(al->gs)) {
    CUtensorMap tu2;
    if (!make_map3(&tu2, cdt, g.es, U, g.Cp, g.K, (uint64_t)g.S * g.planes, BK, 128)) {
      set_last_error("cuTensorMapEncodeTiled failed");
      return WINO_E_CUDA;
    }
    return launch_gemm_ures<4, MT>(tv, tu2, tm, g, fmt, mb0, nT, st);
  }
  if (BN == 256 && nT > kBM && pair_enabled()) {
    CUtensorMap tu2;   // B boxes of 128 k rows: each CTA of the pair loads half of the 256-wide tile
    if (!make_map3(&tu2, cdt, g.es, U, g.Cp, g.K, (uint64_t)g.S * g.planes, BK, 128)) {
      set_last_error("cuTensorMapEncodeTiled failed");
      return WINO_E_CUDA;
    }
    // 6 stages + 2 epilogue buffers: 237 us on cfg5 lin4 bf16 (5 + 4: 248; 4 + 6: 262;
    // 3 + 8: 296; 16-column store boxes or an evict-first L2 hint on the M stores: +-2)
    return launch_gemm_pair<false, 6, 2, false, 32, MT>(tv, tu2, tm, g, al->gs, fmt, mb0, nT, st);
  }
  if (BN == 256) return launch_gemm<false, 256, 4, MT>(tv, tu, tm, g, al->gs, fmt, mb0, nT, st);   // 3 stages + 4 epilogue buffers: 8 % slower
  if (BN == 128) return launch_gemm<false, 128, 6, MT>(tv, tu, tm, g, al->gs, fmt, mb0, nT, st);
  return launch_gemm<false, 64, 8, MT>(tv, tu, tm, g, al->gs, fmt, mb0, nT, st);
}

wino_status run_domain_gemm(const void* V, const void* U, const Geo& g, const wino_algo* al, wino_dtype dt,
                            void* M, cudaStream_t st, int mb0, int nT) {
  if (nT < 0) nT = g.T;
  const int Tpm = (nT + 31) / 32 * 32;
  const bool tf32 = dt == WINO_F32;
  CUtensorMapDataType cdt = dt == WINO_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                            : dt == WINO_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                             : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const bool m16 = m_in_dtype(al, dt);
  int BN = tf32 ? (g.K > 64 ? 128 : 64) : (g.K > 128 ? 256 : (g.K > 64 ? 128 : 64));
  const uint32_t BK = 128 / (uint32_t)g.es;
  CUtensorMap tv, tu, tm;
  if (!make_map3(&tv, cdt, g.es, V, BK, kBM, (uint64_t)g.planes * g.Q * g.TB * (g.Cp / BK), BK, kBM) ||
      !make_map3(&tu, cdt, g.es, U, g.Cp, g.K, (uint64_t)g.S * g.planes, BK, BN) ||
      !make_map3(&tm, m16 ? cdt : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, m16 ? 2 : 4, M, nT, g.K, g.Q, kBM, 32, false,
                 Tpm)) {
    set_last_error("cuTensorMapEncodeTiled failed (driver entry point unavailable or bad geometry)");
    return WINO_E_CUDA;
  }
  // UMMA operand formats: kind::f16 F16 = 0, BF16 = 1; kind::tf32 TF32 = 2.
  const uint32_t fmt = dt == WINO_F16 ? 0u : dt == WINO_BF16 ? 1u : 2u;
  if (tf32) {
    if (g.K > 128 && nT > kBM && pair_enabled()) {
      CUtensorMap tu2;
      if (!make_map3(&tu2, cdt, g.es, U, g.Cp, g.K, (uint64_t)g.S * g.planes, BK, 128)) {
        set_last_error("cuTensorMapEncodeTiled failed");
        return WINO_E_CUDA;
      }
      return launch_gemm_pair<true, 3, 2, false>(tv, tu2, tm, g, al->gs, fmt, mb0, nT, st);
    }
    if (BN == 128) return launch_gemm<true, 128, 3>(tv, tu, tm, g, al->gs, fmt, mb0, nT, st);
    return launch_gemm<true, 64, 4>(tv, tu, tm, g, al->gs, fmt, mb0, nT, st);
  }
  if (!m16) return launch_domain_gemm_16<0>(tv, tu, tm, U, g, al, cdt, fmt, BN, mb0, nT, st);
  if (dt == WINO_F16) return launch_domain_gemm_16<1>(tv, tu, tm, U, g, al, cdt, fmt, BN, mb0, nT, st);
  return launch_domain_gemm_16<2>(tv, tu, tm, U, g, al, cdt, fmt, BN, mb0, nT, st);
}

}  // namespace wino

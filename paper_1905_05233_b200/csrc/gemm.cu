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
#include <cstdlib>
#include <string>

#include "device.cuh"
#include "geometry.hpp"
#include "tmap.hpp"

namespace wino {

constexpr int kBM = 128;

template <bool kTF32, int BN, int STAGES, int EPI = 0>
struct GemmCfg {
  static constexpr int ES = kTF32 ? 4 : 2;
  static constexpr int BK = 128 / ES;   // elements per 128-byte swizzled row
  static constexpr int UK = kTF32 ? 8 : 16;
  static constexpr int NPL = kTF32 ? 2 : 1;
  static constexpr int A_BYTES = kBM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = NPL * (A_BYTES + B_BYTES);
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int EPI_BYTES = 32 * kBM * 4;   // one [32 k][128 t] fp32 box
  // as many epilogue staging buffers (TMA stores in flight) as shared memory allows, 2..4
  static constexpr int EPI_FREE = (227 * 1024 - STAGES * STAGE_BYTES - 1024 - 256) / EPI_BYTES;
  static constexpr int EPI_BUFS = EPI ? EPI : (EPI_FREE > 4 ? 4 : (EPI_FREE < 2 ? 2 : EPI_FREE));
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BUFS * EPI_BYTES + 1024 + 256;
};

template <bool kTF32, int BN, int STAGES>
__global__ void __launch_bounds__(256, 1)
    domain_gemm_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmU,
                       const __grid_constant__ CUtensorMap tmM, int T, int K, int Cp, int nMB, int nNB, int Q, int S,
                       uint32_t idesc, const __grid_constant__ GemmSched gs) {
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
            tma_load_3d(base, &tmV, &full[stage], 0, 0, (qi * nMB + mb) * KB + kb);   // blocked V: one 16 KB block
            if constexpr (kTF32)
              tma_load_3d(base + Cfg::A_BYTES, &tmV, &full[stage], 0, 0, ((qi + Q) * nMB + mb) * KB + kb);
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
        for (int jj = 0; jj < 32; ++jj) buf[jj * kBM + wq * 32 + lane] = v[jj];
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

// ------------------------------------------------------------------ fused K3 + K4
// Same warp-specialised tcgen05 pipeline, plus the output transform done from
// L2: items are ordered tile-block (mb) major, so the Q * nNB point-GEMMs of a
// 128-tile block finish close together; after an item's M boxes are stored
// the storer publishes it on the block's counter (release), and four extra
// "fixup" warps (8..15) of the CTAs pick the fixup items (mb, 32-channel
// slice ks) of completed blocks, read M from L2 (ld.global.cg), apply
// Y = A^T M A and store y, then discard the consumed M lines from L2
// (discard.global.L2, no write-back).  M thus lives in L2 only (written and
// read once there) instead of crossing HBM twice.  All CTAs are co-resident
// (cooperative launch, one CTA per SM), so the fixup warps' waits always end.
struct FuseArgs {
  float AT[kMaxM][kMaxDomain];
  int D, Q;             // domain, output points (= D * D)
  int K, T, Tp, Ho, Wo, th, tw;
  int nKS;              // 32-channel slices of K
  int need;             // point-GEMM items per tile block (= Q * nNB)
  void* y;
  const float* M;       // the M workspace (for the L2 discards)
  int* done;            // [nMB] point-GEMM items stored, per tile block (zeroed before the launch)
  int* fixed;           // [nMB] fixup items finished, per tile block (zeroed before the launch)
  int lag;              // the producer starts tile block mb only once block mb - lag is fully fixed up
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// Output transform of one (tile t, channel k) from the TMA-staged M piece
// fb[q][128 t] (all Q points of channel k for the 128-tile block): Y = A^T M A,
// same fp32 operation order as K4 (output_transform_nchw).
template <int DT, int M, int D>
__device__ __forceinline__ void fixup_point(const float* fb, const FuseArgs& fa, int t, int tl, int k) {
  using Tr = DType<DT>;
  using TT = typename Tr::T;
  const int tj = t % fa.tw, rest = t / fa.tw;
  const int ti = rest % fa.th, n = rest / fa.th;
  float Y[M][M];
#pragma unroll
  for (int p = 0; p < M; ++p)
#pragma unroll
    for (int q = 0; q < M; ++q) Y[p][q] = 0.f;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    float v[D];
#pragma unroll
    for (int j = 0; j < D; ++j) v[j] = fb[(i * D + j) * kBM + tl];
    float Z[M];
#pragma unroll
    for (int q = 0; q < M; ++q) {
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < D; ++j) acc = fmaf(v[j], fa.AT[q][j], acc);
      Z[q] = acc;
    }
#pragma unroll
    for (int p = 0; p < M; ++p)
#pragma unroll
      for (int q = 0; q < M; ++q) Y[p][q] = fmaf(fa.AT[p][i], Z[q], Y[p][q]);
  }
  TT* dst = reinterpret_cast<TT*>(fa.y) + (((size_t)n * fa.K + k) * fa.Ho + (size_t)ti * M) * fa.Wo + (size_t)tj * M;
#pragma unroll
  for (int p = 0; p < M; ++p) {
    if (ti * M + p >= fa.Ho) break;
    store_tile_row<Tr, M>(dst + (size_t)p * fa.Wo, Y[p], fa.Wo - tj * M);
  }
}

constexpr int kFuseStages = 3;   // GEMM stages of the fused kernel (room for the M pieces)
template <int BN>
using FusedCfg = GemmCfg<false, BN, kFuseStages, 2>;
// shared memory of the fused kernel: GEMM stages + 2 epilogue boxes + barriers,
// then two M pieces of Q x 128 fp32 (one channel of every point for a 128-tile block)
template <int BN>
constexpr int fused_smem(int Q) { return FusedCfg<BN>::SMEM + 128 + 2 * Q * kBM * 4; }

template <int BN, int STAGES, int DT, int MO, int DO>
__global__ void __launch_bounds__(384, 1)
    domain_gemm_fused_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmU,
                             const __grid_constant__ CUtensorMap tmM, const __grid_constant__ CUtensorMap tmMl,
                             int T, int K, int Cp, int nMB, int nNB, int Q, int S, uint32_t idesc,
                             const __grid_constant__ GemmSched gs, const __grid_constant__ FuseArgs fa) {
  using Cfg = GemmCfg<false, BN, STAGES, 2>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned for the 128-byte swizzle atoms; offsetting the shared array keeps
  // a shared-space pointer (STS / LDS, no generic stores and CTA-wide MEMBARs)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* epi = reinterpret_cast<float*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::EPI_BUFS * Cfg::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ffull = tempty + 2;    // [2] M piece landed (TMA)
  uint64_t* fempty = ffull + 2;    // [2] M piece consumed (128 fixup threads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fempty + 2);
  float* fbuf = reinterpret_cast<float*>(smem + Cfg::SMEM - 1024 + 128);   // 2 x [Q][128] fp32

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmV);
    tma_prefetch(&tmU);
    tma_prefetch(&tmM);
    tma_prefetch(&tmMl);
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    for (int a = 0; a < 2; ++a) mbar_init(&tfull[a], 1), mbar_init(&tempty[a], 4);
    for (int a = 0; a < 2; ++a) mbar_init(&ffull[a], 1), mbar_init(&fempty[a], kBM);
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
  // item -> (mb slowest, then output point p, then nb)
  auto decode = [&](int item, int& mb, int& p, int& nb) {
    nb = item % nNB;
    p = (item / nNB) % Q;
    mb = item / (nNB * Q);
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int item = blockIdx.x; item < nItems; item += gridDim.x) {
        int mb, p, nb;
        decode(item, mb, p, nb);
        // backpressure: keep at most `lag` tile blocks of M in flight in L2
        if (mb >= fa.lag)
          while (ld_acquire(fa.fixed + mb - fa.lag) < fa.nKS) __nanosleep(128);
        for (int pr = gs.off[p]; pr < gs.off[p + 1]; ++pr) {
          const int qi = gs.in_pt[pr], sl = gs.slab[pr];
          for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
            uint8_t* base = smem + stage * Cfg::STAGE_BYTES;
            tma_load_3d(base, &tmV, &full[stage], 0, 0, (qi * nMB + mb) * KB + kb);   // blocked V: one 16 KB block
            tma_load_3d(base + Cfg::A_BYTES, &tmU, &full[stage], kb * Cfg::BK, nb * BN, sl);
            if (++stage == STAGES) stage = 0, phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int item = blockIdx.x; item < nItems; item += gridDim.x) {
        int mb, p, nb;
        decode(item, mb, p, nb);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        int step = 0;
        for (int pr = gs.off[p]; pr < gs.off[p + 1]; ++pr) {
          for (int kb = 0; kb < KB; ++kb, ++step) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t a0 = smem_u32(smem + stage * Cfg::STAGE_BYTES);
            const uint32_t b0 = a0 + Cfg::A_BYTES;
#pragma unroll
            for (int k = 0; k < Cfg::BK / Cfg::UK; ++k) {
              const uint32_t koff = k * Cfg::UK * Cfg::ES;
              mma_ss<false>(d_tmem, umma_desc_sw128(a0 + koff), umma_desc_sw128(b0 + koff), idesc, (step | k) != 0);
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
  } else if (warp >= 4 && warp < 8) {
    // -------------------------------------------------- epilogue: TMEM -> SMEM -> TMA store, then publish
    const int wq = warp & 3;
    const bool storer = (warp == 4 && lane == 0);
    int acc = 0, chunk = 0;
    uint32_t acc_phase = 0;
    for (int item = blockIdx.x; item < nItems; item += gridDim.x) {
      int mb, p, nb;
      decode(item, mb, p, nb);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int j0 = 0; j0 < BN; j0 += 32) {
        float v[32];
        tmem_ld32(tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN + j0, v);
        if (j0 + 32 == BN) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        if (nb * BN + j0 >= K) continue;
        float* buf = epi + (chunk % Cfg::EPI_BUFS) * (Cfg::EPI_BYTES / 4);
        if (storer) bulk_wait_read<Cfg::EPI_BUFS - 1>();
        named_bar_sync(1, 128);
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) buf[jj * kBM + wq * 32 + lane] = v[jj];
        fence_proxy_async_shared();
        named_bar_sync(1, 128);
        if (storer) {
          tma_store_3d(&tmM, buf, mb * kBM, nb * BN + j0, p);
          bulk_commit();
        }
        ++chunk;
      }
      if (++acc == 2) acc = 0, acc_phase ^= 1;
      if (storer) {
        // the item's M boxes are in memory: publish them to the fixup warps
        bulk_wait_all();
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __threadfence();
        red_release_add(fa.done + mb, 1);
      }
    }
    if (storer) bulk_wait_all();
  } else if (warp >= 8) {
    // -------------------------------------------------- fixup warps: output transform from L2
    // Fixup item (mb, ks): channels [32 ks, 32 ks + 32) of tile block mb.  One
    // thread streams the item's M pieces (all Q points of one channel k, 128
    // tiles: a {128, 1, Q} TMA box of M) through two shared-memory buffers;
    // thread tl computes tile mb*128 + tl.  Consumed M lines are discarded
    // from L2 (no write-back), and the block's `fixed` counter releases the
    // producer's backpressure.
    const int tl = threadIdx.x - 256;
    const bool issuer = tl == 0;
    const int nFix = nMB * fa.nKS;
    const uint32_t piece_bytes = (uint32_t)fa.Q * kBM * 4;
    const size_t qs = (size_t)fa.K * fa.Tp;
    int piece = 0;   // running piece counter (buffer = piece & 1, use = piece >> 1)
    for (int f = blockIdx.x; f < nFix; f += gridDim.x) {
      const int mb = f / fa.nKS, ks = f % fa.nKS;
      const int k0 = ks * 32, nk = min(fa.K, k0 + 32) - k0;
      if (issuer) {
        while (ld_acquire(fa.done + mb) < fa.need) __nanosleep(256);
        asm volatile("fence.proxy.async.global;" ::: "memory");
        for (int j = 0; j < 2 && j < nk; ++j) {
          const int pc = piece + j, b = pc & 1;
          if (pc >= 2) mbar_wait(&fempty[b], (uint32_t)(((pc >> 1) - 1) & 1));
          mbar_arrive_expect_tx(&ffull[b], piece_bytes);
          tma_load_3d(fbuf + (size_t)b * fa.Q * kBM, &tmMl, &ffull[b], mb * kBM, k0 + j, 0);
        }
      }
      for (int j = 0; j < nk; ++j, ++piece) {
        const int b = piece & 1;
        mbar_wait(&ffull[b], (uint32_t)((piece >> 1) & 1));
        const float* fb = fbuf + (size_t)b * fa.Q * kBM;
        // the piece is in shared memory: its L2 lines (Q rows x 512 B) can go
        for (int l = tl; l < fa.Q * 4; l += kBM)
          discard_l2(fa.M + (size_t)(l >> 2) * qs + (size_t)(k0 + j) * fa.Tp + (size_t)mb * kBM + (l & 3) * 32);
        const int t = mb * kBM + tl;
        if (t < fa.T) fixup_point<DT, MO, DO>(fb, fa, t, tl, k0 + j);
        mbar_arrive(&fempty[b]);
        if (issuer && j + 2 < nk) {
          const int pc = piece + 2;
          mbar_wait(&fempty[b], (uint32_t)(((pc >> 1) - 1) & 1));
          mbar_arrive_expect_tx(&ffull[b], piece_bytes);
          tma_load_3d(fbuf + (size_t)b * fa.Q * kBM, &tmMl, &ffull[b], mb * kBM, k0 + j + 2, 0);
        }
      }
      named_bar_sync(2, kBM);
      if (issuer) {
        __threadfence();
        red_release_add(fa.fixed + mb, 1);
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <bool kTF32, int BN, int STAGES>
static wino_status launch_gemm(const CUtensorMap& tv, const CUtensorMap& tu, const CUtensorMap& tm, const Geo& g,
                               const GemmSched& gs, uint32_t fmt, cudaStream_t st) {
  using Cfg = GemmCfg<kTF32, BN, STAGES>;
  auto kern = domain_gemm_kernel<kTF32, BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    WINO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    attr = true;
  }
  const int nMB = (g.T + kBM - 1) / kBM, nNB = (g.K + BN - 1) / BN;
  const int items = g.Q * nMB * nNB;
  const int grid = items < num_sms() ? items : num_sms();
  kern<<<grid, 256, Cfg::SMEM, st>>>(tv, tu, tm, g.T, g.K, g.Cp, nMB, nNB, g.Q, g.S,
                                     make_idesc(fmt, kBM, BN), gs);
  WINO_LAUNCH_CHECK();
  return WINO_OK;
}

template <int DT, int MO, int DO>
static wino_status launch_fused(const CUtensorMap& tv, const CUtensorMap& tu, const CUtensorMap& tm, const Geo& g,
                                const wino_algo* al, uint32_t fmt, const float* M, void* y, int* done, cudaStream_t st) {
  constexpr int BN = 256, STAGES = kFuseStages;
  auto kern = domain_gemm_fused_kernel<BN, STAGES, DT, MO, DO>;
  const int smem = fused_smem<BN>(g.Q);
  WINO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int nMB = (g.T + kBM - 1) / kBM, nNB = (g.K + BN - 1) / BN;
  // M pieces for the fixup warps: box {128 t, 1 k, Q points} of M [Q][K][Tp]
  CUtensorMap tml;
  {
    const uint64_t dims[3] = {(uint64_t)g.Tp, (uint64_t)g.K, (uint64_t)g.Q};
    const uint64_t str[2] = {(uint64_t)g.Tp * 4, (uint64_t)g.K * g.Tp * 4};
    const uint32_t box[3] = {(uint32_t)kBM, 1, (uint32_t)g.Q};
    if (!make_map(&tml, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, M, dims, str, box, false)) {
      set_last_error("cuTensorMapEncodeTiled failed for the fused M pieces");
      return WINO_E_CUDA;
    }
  }
  FuseArgs fa{};
  for (int q = 0; q < al->m; ++q)
    for (int j = 0; j < al->D; ++j) fa.AT[q][j] = al->xp.AT[q][j];
  fa.D = al->D, fa.Q = g.Q, fa.K = g.K, fa.T = g.T, fa.Tp = g.Tp, fa.Ho = g.Ho, fa.Wo = g.Wo, fa.th = g.th,
  fa.tw = g.tw, fa.nKS = (g.K + 31) / 32, fa.need = al->gs.Q * nNB, fa.y = y, fa.M = M, fa.done = done;
  fa.fixed = done + nMB;
  {
    // tile blocks of M (Q * K * 128 * 4 bytes each) allowed in flight
    const size_t blk = (size_t)g.Q * g.K * kBM * 4;
    int lag = (int)((40u << 20) / (blk ? blk : 1));
    fa.lag = lag < 2 ? 2 : lag;
    if (const char* e = getenv("WINO_FUSED_LAG")) fa.lag = atoi(e);
  }
  WINO_CUDA_CHECK(cudaMemsetAsync(done, 0, sizeof(int) * 2 * nMB, st));
  const int items = al->gs.Q * nMB * nNB;
  int grid = items < num_sms() ? items : num_sms();
  if (grid < 1) grid = 1;
  const uint32_t idesc = make_idesc(fmt, kBM, BN);
  int T = g.T, K = g.K, Cp = g.Cp, Q = al->gs.Q, S = g.S;
  int nMBv = nMB, nNBv = nNB;
  void* args[] = {(void*)&tv, (void*)&tu, (void*)&tm, (void*)&tml, &T, &K, &Cp, (void*)&nMBv, (void*)&nNBv, &Q, &S,
                  (void*)&idesc, (void*)&al->gs, (void*)&fa};
  // cooperative launch: every CTA is resident (the fixup warps wait on other CTAs' items)
  WINO_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(384), args, smem, st));
  WINO_LAUNCH_CHECK();
  return WINO_OK;
}

template <int DT, int MO>
static wino_status fused_d(int doff, const CUtensorMap& tv, const CUtensorMap& tu, const CUtensorMap& tm, const Geo& g,
                           const wino_algo* al, uint32_t fmt, const float* M, void* y, int* done, cudaStream_t st) {
  switch (doff) {
    case 0: return launch_fused<DT, MO, MO + 2>(tv, tu, tm, g, al, fmt, M, y, done, st);
    case 1: return launch_fused<DT, MO, MO + 3>(tv, tu, tm, g, al, fmt, M, y, done, st);
    default: return launch_fused<DT, MO, MO + 4>(tv, tu, tm, g, al, fmt, M, y, done, st);
  }
}
template <int DT>
static wino_status fused_m(int m, int doff, const CUtensorMap& tv, const CUtensorMap& tu, const CUtensorMap& tm,
                           const Geo& g, const wino_algo* al, uint32_t fmt, const float* M, void* y, int* done,
                           cudaStream_t st) {
  switch (m) {
    case 2: return fused_d<DT, 2>(doff, tv, tu, tm, g, al, fmt, M, y, done, st);
    case 3: return fused_d<DT, 3>(doff, tv, tu, tm, g, al, fmt, M, y, done, st);
    case 4: return fused_d<DT, 4>(doff, tv, tu, tm, g, al, fmt, M, y, done, st);
    case 5: return fused_d<DT, 5>(doff, tv, tu, tm, g, al, fmt, M, y, done, st);
    case 6: return fused_d<DT, 6>(doff, tv, tu, tm, g, al, fmt, M, y, done, st);
    case 7: return fused_d<DT, 7>(doff, tv, tu, tm, g, al, fmt, M, y, done, st);
    default: return fused_d<DT, 8>(doff, tv, tu, tm, g, al, fmt, M, y, done, st);
  }
}

// Fused K3 + K4 (16-bit dtypes, K > 128, NCHW output).  Returns WINO_E_UNSUPPORTED
// (without launching) when the configuration is not covered.
wino_status run_domain_gemm_fused(const void* V, const void* U, const Geo& g, const wino_algo* al, wino_dtype dt,
                                  float* M, void* y, int* done, cudaStream_t st) {
  const int doff = al->D - al->m - 2;
  if (dt == WINO_F32 || g.K <= 128 || al->m < 2 || al->m > 8 || doff < 0 || doff > 2) return WINO_E_UNSUPPORTED;
  if (fused_smem<256>(g.Q) > 227 * 1024) return WINO_E_UNSUPPORTED;   // the M pieces must fit (Q <= 49)
  CUtensorMapDataType cdt = dt == WINO_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  constexpr int BN = 256;
  const uint32_t BK = 128 / (uint32_t)g.es;
  CUtensorMap tv, tu, tm;
  if (!make_map3(&tv, cdt, g.es, V, BK, kBM, (uint64_t)g.planes * g.Q * g.TB * (g.Cp / BK), BK, kBM) ||
      !make_map3(&tu, cdt, g.es, U, g.Cp, g.K, (uint64_t)g.S * g.planes, BK, BN) ||
      !make_map3(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, g.T, g.K, g.Q, kBM, 32, false, g.Tp)) {
    set_last_error("cuTensorMapEncodeTiled failed (driver entry point unavailable or bad geometry)");
    return WINO_E_CUDA;
  }
  const uint32_t fmt = dt == WINO_F16 ? 0u : 1u;
  return dt == WINO_F16 ? fused_m<WINO_F16>(al->m, doff, tv, tu, tm, g, al, fmt, M, y, done, st)
                        : fused_m<WINO_BF16>(al->m, doff, tv, tu, tm, g, al, fmt, M, y, done, st);
}

wino_status run_domain_gemm(const void* V, const void* U, const Geo& g, const wino_algo* al, wino_dtype dt,
                            float* M, cudaStream_t st) {
  const bool tf32 = dt == WINO_F32;
  CUtensorMapDataType cdt = dt == WINO_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                            : dt == WINO_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                             : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  int BN = tf32 ? (g.K > 64 ? 128 : 64) : (g.K > 128 ? 256 : (g.K > 64 ? 128 : 64));
  const uint32_t BK = 128 / (uint32_t)g.es;
  CUtensorMap tv, tu, tm;
  if (!make_map3(&tv, cdt, g.es, V, BK, kBM, (uint64_t)g.planes * g.Q * g.TB * (g.Cp / BK), BK, kBM) ||
      !make_map3(&tu, cdt, g.es, U, g.Cp, g.K, (uint64_t)g.S * g.planes, BK, BN) ||
      !make_map3(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, g.T, g.K, g.Q, kBM, 32, false, g.Tp)) {
    set_last_error("cuTensorMapEncodeTiled failed (driver entry point unavailable or bad geometry)");
    return WINO_E_CUDA;
  }
  // UMMA operand formats: kind::f16 F16 = 0, BF16 = 1; kind::tf32 TF32 = 2.
  const uint32_t fmt = dt == WINO_F16 ? 0u : dt == WINO_BF16 ? 1u : 2u;
  if (tf32) {
    if (BN == 128) return launch_gemm<true, 128, 3>(tv, tu, tm, g, al->gs, fmt, st);
    return launch_gemm<true, 64, 4>(tv, tu, tm, g, al->gs, fmt, st);
  }
  if (BN == 256) return launch_gemm<false, 256, 4>(tv, tu, tm, g, al->gs, fmt, st);   // 3 stages + 4 epilogue buffers: 8 % slower
  if (BN == 128) return launch_gemm<false, 128, 6>(tv, tu, tm, g, al->gs, fmt, st);
  return launch_gemm<false, 64, 8>(tv, tu, tm, g, al->gs, fmt, st);
}

}  // namespace wino

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
  int dbg;              // timing experiments only (WINO_FUSED_DBG): 1 no wait, 2 no fixup math, 4 no discard, 8 no fixup loads
  int lag;              // work-list distance, in tile blocks, from a block's GEMM items to its fixups
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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

// Time-multiplexed persistent K3 + K4.  One ordered work list holds the
// point-GEMM items of each 128-tile block mb (Q * nNB of them) and, LAG blocks
// later, the block's fixup items (mb, 32-channel slice ks).  CTA c runs list
// positions c, c + G, ... in order.  GEMM items use the warp-specialised
// tcgen05 pipeline (producer / MMA / epilogue, which publishes each stored
// item on done[mb]); at a fixup item every warp of the CTA meets at a barrier
// (so the GEMM pipeline is drained) and the whole CTA turns into an output
// transform: the 192 KB of stage memory becomes a ring of NB M pieces
// ({128 t, 1 k, Q points} TMA boxes read from L2), two 128-thread halves apply
// Y = A^T M A to alternate channels, store y and discard the consumed M lines
// from L2 -- so M is written to and read from L2 only.  A fixup waits only for
// GEMM items earlier in the list, and all CTAs are resident (cooperative
// launch), so the smallest pending list position always makes progress.

template <int BN, int STAGES, int DT, int MO, int DO>
__global__ void __launch_bounds__(256, 1)
    domain_gemm_fused_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmU,
                             const __grid_constant__ CUtensorMap tmM, const __grid_constant__ CUtensorMap tmMl,
                             int T, int K, int Cp, int nMB, int nNB, int Q, int S, uint32_t idesc,
                             const __grid_constant__ GemmSched gs, const __grid_constant__ FuseArgs fa) {
  using Cfg = GemmCfg<false, BN, STAGES, 2>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* epi = reinterpret_cast<float*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::EPI_BUFS * Cfg::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ffull = tempty + 2;   // [kMaxPieces] M piece landed (TMA)
  constexpr int kMaxPieces = 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ffull + kMaxPieces);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const uint32_t piece_bytes = (uint32_t)fa.Q * kBM * 4;
  int NB = (STAGES * Cfg::STAGE_BYTES) / (int)piece_bytes;   // M pieces that fit in the stage memory
  NB = (NB > kMaxPieces ? kMaxPieces : NB) & ~1;              // even: buffer b belongs to half b & 1
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmV);
    tma_prefetch(&tmU);
    tma_prefetch(&tmM);
    tma_prefetch(&tmMl);
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    for (int a = 0; a < 2; ++a) mbar_init(&tfull[a], 1), mbar_init(&tempty[a], 4);
    for (int b = 0; b < kMaxPieces; ++b) mbar_init(&ffull[b], 1);
    fence_barrier_init();
    fence_proxy_async_shared();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int KB = Cp / Cfg::BK;
  const int IP = Q * nNB, nKS = fa.nKS, SEC = IP + nKS;
  const int L = fa.lag < nMB ? fa.lag : nMB;
  const int A_end = L * IP, B_end = A_end + (nMB - L) * SEC, LEN = B_end + L * nKS;
  // list position -> GEMM item (mb, p, nb) or fixup item (mb, ks)
  auto decode = [&](int w, bool& isF, int& mb, int& p, int& nb, int& ks) {
    int r;
    if (w < A_end) {
      isF = false, mb = w / IP, r = w % IP;
    } else if (w < B_end) {
      const int u = w - A_end, sct = u / SEC;
      r = u % SEC;
      if (r < IP) isF = false, mb = L + sct;
      else isF = true, mb = sct, ks = r - IP;
    } else {
      const int u = w - B_end;
      isF = true, mb = (nMB - L) + u / nKS, ks = u % nKS;
    }
    if (!isF) p = r / nNB, nb = r % nNB;
  };

  // role state carried across list positions
  int pstage = 0, mstage = 0, acc_m = 0, acc_e = 0, chunk = 0;
  uint32_t pphase = 0, mphase = 0, accph_m = 0, accph_e = 0;
  int piece = 0;   // running M-piece counter (fixups)
  const int wq = warp & 3;
  const bool storer = (warp == 4 && lane == 0);

  for (int w = blockIdx.x; w < LEN; w += gridDim.x) {
    bool isF;
    int mb, p = 0, nb = 0, ks = 0;
    decode(w, isF, mb, p, nb, ks);
    if (!isF) {
      if (warp == 0) {
        if (lane == 0) {
          fence_proxy_async_shared();   // a fixup may have read the stage memory through the generic proxy
          for (int pr = gs.off[p]; pr < gs.off[p + 1]; ++pr) {
            const int qi = gs.in_pt[pr], sl = gs.slab[pr];
            for (int kb = 0; kb < KB; ++kb) {
              mbar_wait(&empty[pstage], pphase ^ 1);
              mbar_arrive_expect_tx(&full[pstage], Cfg::STAGE_BYTES);
              uint8_t* base = smem + pstage * Cfg::STAGE_BYTES;
              tma_load_3d(base, &tmV, &full[pstage], 0, 0, (mb * KB + kb) * fa.Q + qi);
              tma_load_3d(base + Cfg::A_BYTES, &tmU, &full[pstage], kb * Cfg::BK, nb * BN, sl);
              if (++pstage == STAGES) pstage = 0, pphase ^= 1;
            }
          }
        }
        __syncwarp();
      } else if (warp == 1) {
        if (lane == 0) {
          mbar_wait(&tempty[acc_m], accph_m ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc_m * BN;
          int step = 0;
          for (int pr = gs.off[p]; pr < gs.off[p + 1]; ++pr) {
            for (int kb = 0; kb < KB; ++kb, ++step) {
              mbar_wait(&full[mstage], mphase);
              tc_fence_after();
              const uint32_t a0 = smem_u32(smem + mstage * Cfg::STAGE_BYTES);
              const uint32_t b0 = a0 + Cfg::A_BYTES;
#pragma unroll
              for (int k = 0; k < Cfg::BK / Cfg::UK; ++k) {
                const uint32_t koff = k * Cfg::UK * Cfg::ES;
                mma_ss<false>(d_tmem, umma_desc_sw128(a0 + koff), umma_desc_sw128(b0 + koff), idesc, (step | k) != 0);
              }
              mma_commit(&empty[mstage]);
              if (++mstage == STAGES) mstage = 0, mphase ^= 1;
            }
          }
          mma_commit(&tfull[acc_m]);
          if (++acc_m == 2) acc_m = 0, accph_m ^= 1;
        }
        __syncwarp();
      } else if (warp >= 4) {
        mbar_wait(&tfull[acc_e], accph_e);
        tc_fence_after();
#pragma unroll 1
        for (int j0 = 0; j0 < BN; j0 += 32) {
          float v[32];
          tmem_ld32(tmem_base + ((uint32_t)(wq * 32) << 16) + acc_e * BN + j0, v);
          if (j0 + 32 == BN) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc_e]);
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
        if (++acc_e == 2) acc_e = 0, accph_e ^= 1;
        if (storer) {
          bulk_wait_all();   // the item's M boxes are in memory: publish them
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __threadfence();
          red_release_add(fa.done + mb, 1);
        }
      }
    } else {
      // ---------------------------------------------------------------- fixup item
      __syncthreads();   // every warp is past its earlier items: the stage memory is free
      if (tid == 0) {
        if (!(fa.dbg & 1))
          while (ld_acquire(fa.done + mb) < fa.need) __nanosleep(128);
        asm volatile("fence.proxy.async.global;" ::: "memory");
        fence_proxy_async_shared();
      }
      __syncthreads();
      const int k0 = ks * 32, nk = min(fa.K, k0 + 32) - k0;
      const int half = tid >> 7, tl = tid & (kBM - 1);
      float* ring = reinterpret_cast<float*>(smem);
      const size_t qs = (size_t)fa.K * fa.Tp;
      // each half's thread 0 streams the pieces of its channels j = half, half + 2, ...
      if (tl == 0 && !(fa.dbg & 8))
        for (int j = half, n = 0; j < nk && n < NB / 2; j += 2, ++n) {
          const int pc = piece + j, b = pc % NB;
          mbar_arrive_expect_tx(&ffull[b], piece_bytes);
          tma_load_3d(ring + (size_t)b * fa.Q * kBM, &tmMl, &ffull[b], mb * kBM, k0 + j, 0);
        }
      for (int j = half; j < nk; j += 2) {
        const int pc = piece + j, b = pc % NB;
        if (!(fa.dbg & 8)) mbar_wait(&ffull[b], (uint32_t)((pc / NB) & 1));
        const float* fb = ring + (size_t)b * fa.Q * kBM;
        for (int l = tl; l < fa.Q * 4; l += kBM)   // lines past Tp belong to the next channel's row: keep them
          if (mb * kBM + (l & 3) * 32 < fa.Tp && !(fa.dbg & 4))
            discard_l2(fa.M + (size_t)(l >> 2) * qs + (size_t)(k0 + j) * fa.Tp + (size_t)mb * kBM + (l & 3) * 32);
        const int t = mb * kBM + tl;
        if (t < fa.T && !(fa.dbg & 2)) fixup_point<DT, MO, DO>(fb, fa, t, tl, k0 + j);
        named_bar_sync(2 + half, kBM);   // this half is done with buffer b
        const int jn = j + NB;            // the next piece of this half that maps to buffer b
        if (tl == 0 && jn < nk && !(fa.dbg & 8)) {
          fence_proxy_async_shared();
          mbar_arrive_expect_tx(&ffull[b], piece_bytes);
          tma_load_3d(ring + (size_t)b * fa.Q * kBM, &tmMl, &ffull[b], mb * kBM, k0 + jn, 0);
        }
      }
      piece += nk;
      __syncthreads();   // fixup done: the stage memory goes back to the GEMM
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
                               const GemmSched& gs, uint32_t fmt, int mb0, int nT, cudaStream_t st) {
  using Cfg = GemmCfg<kTF32, BN, STAGES>;
  auto kern = domain_gemm_kernel<kTF32, BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    WINO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    attr = true;
  }
  const int nMB = (nT + kBM - 1) / kBM, nNB = (g.K + BN - 1) / BN;
  const int items = g.Q * nMB * nNB;
  const int grid = items < num_sms() ? items : num_sms();
  kern<<<grid, 256, Cfg::SMEM, st>>>(tv, tu, tm, nT, g.K, g.Cp, nMB, nNB, g.Q, g.S,
                                     make_idesc(fmt, kBM, BN), gs, mb0, g.TB);
  WINO_LAUNCH_CHECK();
  return WINO_OK;
}

template <int DT, int MO, int DO>
static wino_status launch_fused(const CUtensorMap& tv, const CUtensorMap& tu, const CUtensorMap& tm, const Geo& g,
                                const wino_algo* al, uint32_t fmt, const float* M, void* y, int* done, cudaStream_t st) {
  constexpr int BN = 256, STAGES = 4;
  auto kern = domain_gemm_fused_kernel<BN, STAGES, DT, MO, DO>;
  const int smem = GemmCfg<false, BN, STAGES, 2>::SMEM;
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
    // list distance (in tile blocks) between a block's GEMM items and its fixups
    fa.lag = 2;
    if (const char* e = getenv("WINO_FUSED_LAG")) fa.lag = atoi(e) < 1 ? 1 : atoi(e);
    if (const char* e = getenv("WINO_FUSED_DBG")) fa.dbg = atoi(e);
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
  WINO_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(256), args, smem, st));
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
  if ((4 * GemmCfg<false, 256, 4>::STAGE_BYTES) / (g.Q * kBM * 4) < 2) return WINO_E_UNSUPPORTED;   // >= 2 M pieces
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

// M_xi for the tiles [mb0 * 128, mb0 * 128 + nT) of V (all of them by default) into
// M [Q][K][Tpm] with Tpm = nT rounded up to 32 (chunked layers: an L2-sized slice)
wino_status run_domain_gemm(const void* V, const void* U, const Geo& g, const wino_algo* al, wino_dtype dt,
                            float* M, cudaStream_t st, int mb0, int nT) {
  if (nT < 0) nT = g.T;
  const int Tpm = (nT + 31) / 32 * 32;
  const bool tf32 = dt == WINO_F32;
  CUtensorMapDataType cdt = dt == WINO_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                            : dt == WINO_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                             : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  int BN = tf32 ? (g.K > 64 ? 128 : 64) : (g.K > 128 ? 256 : (g.K > 64 ? 128 : 64));
  const uint32_t BK = 128 / (uint32_t)g.es;
  CUtensorMap tv, tu, tm;
  if (!make_map3(&tv, cdt, g.es, V, BK, kBM, (uint64_t)g.planes * g.Q * g.TB * (g.Cp / BK), BK, kBM) ||
      !make_map3(&tu, cdt, g.es, U, g.Cp, g.K, (uint64_t)g.S * g.planes, BK, BN) ||
      !make_map3(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, nT, g.K, g.Q, kBM, 32, false, Tpm)) {
    set_last_error("cuTensorMapEncodeTiled failed (driver entry point unavailable or bad geometry)");
    return WINO_E_CUDA;
  }
  // UMMA operand formats: kind::f16 F16 = 0, BF16 = 1; kind::tf32 TF32 = 2.
  const uint32_t fmt = dt == WINO_F16 ? 0u : dt == WINO_BF16 ? 1u : 2u;
  if (tf32) {
    if (BN == 128) return launch_gemm<true, 128, 3>(tv, tu, tm, g, al->gs, fmt, mb0, nT, st);
    return launch_gemm<true, 64, 4>(tv, tu, tm, g, al->gs, fmt, mb0, nT, st);
  }
  if (BN == 256) return launch_gemm<false, 256, 4>(tv, tu, tm, g, al->gs, fmt, mb0, nT, st);   // 3 stages + 4 epilogue buffers: 8 % slower
  if (BN == 128) return launch_gemm<false, 128, 6>(tv, tu, tm, g, al->gs, fmt, mb0, nT, st);
  return launch_gemm<false, 64, 8>(tv, tu, tm, g, al->gs, fmt, mb0, nT, st);
}

}  // namespace wino

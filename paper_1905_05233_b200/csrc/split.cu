// split.cu -- fused K3 + K4: the Winograd-domain GEMM and the output transform
// in one persistent kernel whose SMs are split between the two stages, so the
// fp32 M (P:92's Hadamard products summed over channels, 925 MB on cfg5) lives
// in L2 only -- written by the tensor-core SMs, read back by the CUDA-core SMs,
// then discarded -- instead of crossing HBM twice:
//
//   CTAs [0, G)     GEMM role (the warp-specialised tcgen05 pipeline of gemm.cu):
//                   items (tile block mb, output point p, channel block nb) in
//                   mb-major order; each item's fp32 accumulators are stored by
//                   TMA into a tile-blocked M [nMB][K][Q][128 t], and once its
//                   stores are complete the item is published on done[mb]
//                   (release).
//   CTAs [G, grid)  transform role: items (mb, 32-channel slice); wait for
//                   done[mb] == Q * nNB (acquire), stream the slice's M pieces
//                   -- all Q points of one channel for the 128 tiles, one
//                   contiguous Q * 512-byte run -- from L2 into a shared-memory
//                   ring (cp.async.bulk + mbarriers), drop the consumed lines
//                   from L2 (discard.global.L2: no write-back), apply
//                   Y = A^T M A per (tile, channel) in the fp32 operation order of
//                   K4 (output_transform_nchw) and store y.
//
// The GEMM producer holds back (tile block mb waits until block mb - lag is
// transformed) so the live part of M stays well inside the 126 MB L2.  Every CTA
// is resident (cooperative launch: one CTA per SM), the transform role waits only
// on GEMM items and the GEMM role only on transform items lag blocks back, so the
// waits always end.  Results are bit-identical to the staged K3 -> K4 pair.
#include <cstdlib>
#include <string>

#include "device.cuh"
#include "gemm_common.cuh"
#include "geometry.hpp"
#include "tmap.hpp"

namespace wino {

constexpr int kSplitThreads = 288;   // warps 0..7: GEMM roles / two transform groups; warp 8: transform producer
constexpr int kSliceK = 32;          // output channels per transform item

struct SplitArgs {
  float AT[kMaxM][kMaxDomain];
  int Q, K, T, Ho, Wo, th, tw;
  int nMB, nNB, nKS;   // tile blocks, GEMM channel blocks, transform slices per tile block
  int G;               // GEMM CTAs
  int lag;             // backpressure distance in tile blocks (0: none)
  int KP, NB;          // channels per transform ring slot, ring slots
  void* y;
  const float* Mb;     // blocked M [nMB][K][Q][128] fp32
  int* done;           // [nMB] GEMM items stored
  int* fixed;          // [nMB] channels transformed
  int dbg;             // timing experiments only (WINO_SPLIT_DBG): 1 no L2 discard, 2 no transform math,
                       // 4 transform CTAs exit at once (GEMM alone; no backpressure), 8 no publication,
                       // 16 p-major GEMM item order (with 4 only), 32 no L2 cache-policy hints
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
// global -> shared contiguous bulk copy, completion on an mbarrier (transaction bytes)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// L2 eviction-priority policies (createpolicy): the streamed V tiles, the
// consumed M pieces and y go first, the M written for the transform role stays.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 int c2, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair_hint(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                      int c1, int c2, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d_hint(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                                  int c3, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4, %5}], [%1], %6;" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// wait until at most n of this thread's bulk store groups are pending (n <= 8)
__device__ __forceinline__ void bulk_wait_pending(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.bulk.wait_group 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.bulk.wait_group 4;" ::: "memory"); break;
    case 5: asm volatile("cp.async.bulk.wait_group 5;" ::: "memory"); break;
    case 6: asm volatile("cp.async.bulk.wait_group 6;" ::: "memory"); break;
    case 7: asm volatile("cp.async.bulk.wait_group 7;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group 8;" ::: "memory"); break;
  }
}

// Output transform of NC channels k0 .. k0 + NC - 1 of one tile t: Y = A^T M A per
// channel with m(c, q) = M point q of channel c, in the fp32 operation order of
// output_transform_nchw (bit-identical); the NC channels are independent FMA
// chains interleaved for latency hiding.
template <int DT, int M, int D, int NC, typename Src>
__device__ __forceinline__ void split_xform(const Src& m, const SplitArgs& sa, int t, int k0) {
  using Tr = DType<DT>;
  using TT = typename Tr::T;
  const int tj = t % sa.tw, rest = t / sa.tw;
  const int ti = rest % sa.th, n = rest / sa.th;
  float Y[NC][M][M];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int p = 0; p < M; ++p)
#pragma unroll
      for (int q = 0; q < M; ++q) Y[c][p][q] = 0.f;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    float Z[NC][M];
#pragma unroll
    for (int q = 0; q < M; ++q)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < D; ++j) acc = fmaf(m(c, i * D + j), sa.AT[q][j], acc);
        Z[c][q] = acc;
      }
#pragma unroll
    for (int p = 0; p < M; ++p)
#pragma unroll
      for (int q = 0; q < M; ++q)
#pragma unroll
        for (int c = 0; c < NC; ++c) Y[c][p][q] = fmaf(sa.AT[p][i], Z[c][q], Y[c][p][q]);
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    TT* dst = reinterpret_cast<TT*>(sa.y) + (((size_t)n * sa.K + k0 + c) * sa.Ho + (size_t)ti * M) * sa.Wo + (size_t)tj * M;
#pragma unroll
    for (int p = 0; p < M; ++p) {
      if (ti * M + p >= sa.Ho) break;
      store_tile_row<Tr, M>(dst + (size_t)p * sa.Wo, Y[c][p], sa.Wo - tj * M);
    }
  }
}

// channels per transform slot: 2 where both pieces fit in registers (the slot is
// then released before the math), else 1
__host__ __device__ constexpr int split_nc(int Q) { return 2 * Q <= 80 ? 2 : 1; }

// GEMM role: the CTA-pair pipeline of gemm.cu (domain_gemm_pair_kernel): a cluster of
// two CTAs owns a [256 t x 256 k] tile of one point; CTA r stores its 128 tiles.
template <int STAGES, int EPI, int DT, int MO, int DO>
__global__ void __launch_bounds__(kSplitThreads, 1)
    domain_gemm_split_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmU,
                             const __grid_constant__ CUtensorMap tmMb, int Cp, uint32_t idesc,
                             const __grid_constant__ GemmSched gs, const __grid_constant__ SplitArgs sa) {
  constexpr int BN = 256;
  constexpr int BK = 64, UK = 16, ES = 2;
  constexpr int A_BYTES = kBM * 128, B_BYTES = (BN / 2) * 128, STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr int EPI_BYTES = 32 * kBM * 4, TMEM_COLS = 2 * BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Q = sa.Q, K = sa.K;

  if (blockIdx.x < sa.G) {
    // ============================================================== GEMM role (CTA pairs)
    float* epi = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + EPI * EPI_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const uint32_t rank = cluster_ctarank();
    const int cl = blockIdx.x >> 1, ncl = sa.G >> 1;
    if (warp == 0 && lane == 0) {
      tma_prefetch(&tmV);
      tma_prefetch(&tmU);
      tma_prefetch(&tmMb);
      for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 2), mbar_init(&empty[s], 1);
      for (int a = 0; a < 2; ++a) mbar_init(&tfull[a], 1), mbar_init(&tempty[a], 8);
      fence_barrier_init();
      fence_proxy_async_shared();
    }
    if (warp == 2) tmem_alloc_pair(tmem_slot, TMEM_COLS);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
    const int nMB2 = (sa.nMB + 1) >> 1;
    const int per_mb = Q * sa.nNB;
    const int nItems = nMB2 * per_mb;
    const int KB = Cp / BK;
    // mb-major order: the tile blocks finish one after the other for the transform role
    const bool pmaj = (sa.dbg & 20) == 20;   // p-major order (the staged kernel's), GEMM-alone timing only
    auto decode = [&](int item, int& mb, int& p, int& nb) {
      if (pmaj) {
        nb = item % sa.nNB, mb = 2 * ((item / sa.nNB) % nMB2) + (int)rank, p = item / (sa.nNB * nMB2);
        return;
      }
      mb = 2 * (item / per_mb) + (int)rank;
      const int r = item % per_mb;
      p = r / sa.nNB, nb = r % sa.nNB;
    };

    if (warp == 0) {
      if (lane == 0) {
        // ---------------------------------------------- TMA producer (+ backpressure), both CTAs
        int stage = 0, held = -1;
        uint32_t phase = 0;
        for (int item = cl; item < nItems; item += ncl) {
          int mb, p, nb;
          decode(item, mb, p, nb);
          const int mbw = mb & ~1;   // both CTAs of the pair hold back on the same block
          if (sa.lag > 0 && mbw >= sa.lag && held != mbw) {
            while (ld_relaxed_gpu(sa.fixed + mbw - sa.lag) < K) __nanosleep(256);
            held = mbw;
          }
          const int k0 = nb * BN + (int)rank * (BN / 2);
          for (int pr = gs.off[p]; pr < gs.off[p + 1]; ++pr) {
            const int qi = gs.in_pt[pr], sl = gs.slab[pr];
            for (int kb = 0; kb < KB; ++kb) {
              mbar_wait(&empty[stage], phase ^ 1);
              const uint32_t fb = mapa_rank(&full[stage], 0);
              if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * STAGE_BYTES);
              else mbar_arrive_cluster(fb);
              uint8_t* base = smem + stage * STAGE_BYTES;
              if (sa.dbg & 32) tma_load_3d_pair(base, &tmV, fb, 0, 0, (mb * KB + kb) * Q + qi);
              else tma_load_3d_pair_hint(base, &tmV, fb, 0, 0, (mb * KB + kb) * Q + qi, pol_first);
              tma_load_3d_pair(base + A_BYTES, &tmU, fb, kb * BK, k0, sl);
              if (++stage == STAGES) stage = 0, phase ^= 1;
            }
          }
        }
        for (int s = 0; s < STAGES; ++s) {   // drain: all multicast arrivals on this CTA have landed
          mbar_wait(&empty[stage], phase ^ 1);
          if (++stage == STAGES) stage = 0, phase ^= 1;
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      if (lane == 0 && rank == 0) {
        // ---------------------------------------------- MMA issuer (leader)
        int stage = 0, acc = 0;
        uint32_t phase = 0, acc_phase = 0;
        for (int item = cl; item < nItems; item += ncl) {
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
              const uint32_t a0 = smem_u32(smem + stage * STAGE_BYTES);
              const uint32_t b0 = a0 + A_BYTES;
#pragma unroll
              for (int k = 0; k < BK / UK; ++k) {
                const uint32_t koff = k * UK * ES;
                mma_ss_pair<false>(d_tmem, umma_desc_sw128(a0 + koff), umma_desc_sw128(b0 + koff), idesc,
                                   (step | k) != 0);
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
    } else if (warp >= 4 && warp < 8) {
      // ------------------------------------------------ epilogue: TMEM -> smem -> TMA store, publish
      const int wq = warp & 3;
      const bool storer = (warp == 4 && lane == 0);
      int acc = 0, chunk = 0, pend = -1;
      uint32_t acc_phase = 0;
      for (int item = cl; item < nItems; item += ncl) {
        int mb, p, nb;
        decode(item, mb, p, nb);
        const bool live = mb < sa.nMB;   // the last pair's second block may lie past the layer
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        int nbox = 0;
#pragma unroll 1
        for (int j0 = 0; j0 < BN; j0 += 32) {
          float v[32];
          tmem_ld32(tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN + j0, v);
          if (j0 + 32 == BN) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_rank(&tempty[acc], 0));
          }
          if (nb * BN + j0 >= K || !live) continue;
          float* buf = epi + (chunk % EPI) * (EPI_BYTES / 4);
          if (storer) bulk_wait_read<EPI - 1>();
          named_bar_sync(1, 128);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) buf[jj * kBM + wq * 32 + lane] = v[jj];
          fence_proxy_async_shared();
          named_bar_sync(1, 128);
          if (storer) {
            if (sa.dbg & 32) tma_store_4d(&tmMb, buf, 0, p, nb * BN + j0, mb);
            else tma_store_4d_hint(&tmMb, buf, 0, p, nb * BN + j0, mb, pol_last);
            bulk_commit();
          }
          ++chunk, ++nbox;
        }
        if (storer && live && !(sa.dbg & 8)) {
          // Publish the item once its stores are complete.  To keep the epilogue
          // from draining its stores after every item, the publication of item i
          // is deferred until the next item's stores are issued -- unless the
          // producer's backpressure could make that item wait for item i's tile
          // block (its block is lag or more blocks later): then now.
          const int nxt = item + ncl;
          const bool defer = nxt < nItems && (sa.lag == 0 || 2 * (nxt / per_mb) < (mb & ~1) + sa.lag);
          if (pend >= 0) {   // the previous item: complete once only this item's nbox groups remain
            bulk_wait_pending(nbox);
            fence_proxy_async_global();
            __threadfence();
            red_release_gpu_add(sa.done + pend, 1);
            pend = -1;
          }
          if (defer) {
            pend = mb;
          } else {
            bulk_wait_all();
            fence_proxy_async_global();
            __threadfence();
            red_release_gpu_add(sa.done + mb, 1);
          }
        }
        if (++acc == 2) acc = 0, acc_phase ^= 1;
      }
      if (storer && pend >= 0) {
        bulk_wait_all();
        fence_proxy_async_global();
        __threadfence();
        red_release_gpu_add(sa.done + pend, 1);
      }
      if (storer) bulk_wait_all();
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 2) {
      tc_fence_after();
      tmem_dealloc_pair(tmem_base, TMEM_COLS);
    }
    return;
  }

  // ================================================================ transform role
  if (sa.dbg & 4) return;
  constexpr int QD = DO * DO;
  const int R = gridDim.x - sa.G, r0 = blockIdx.x - sa.G;
  const int NB = sa.NB, KP = sa.KP;
  const size_t piece = (size_t)QD * kBM;             // floats per channel piece
  const size_t slotf = (size_t)KP * piece;
  float* ring = reinterpret_cast<float*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NB * slotf * 4);
  uint64_t* empty = full + NB;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) mbar_init(&full[b], 1), mbar_init(&empty[b], kBM);
    fence_barrier_init();
  }
  __syncthreads();
  const int nItems = sa.nMB * sa.nKS;
  const int need = Q * sa.nNB;
  const uint64_t pol_first = policy_evict_first();
  if (warp == 8) {
    if (lane == 0) {
      int s = 0;
      for (int it = r0; it < nItems; it += R) {
        const int mb = it / sa.nKS, k0 = (it % sa.nKS) * kSliceK, nk = min(K, k0 + kSliceK) - k0;
        while (ld_acquire_gpu(sa.done + mb) < need) __nanosleep(128);
        fence_proxy_async_global();
        for (int j = 0; j < nk; j += KP, ++s) {
          const int b = s % NB;
          if (s >= NB) mbar_wait(&empty[b], (uint32_t)(((s / NB) - 1) & 1));
          const int kc = min(KP, nk - j);
          const uint32_t bytes = (uint32_t)(kc * piece * 4);
          mbar_arrive_expect_tx(&full[b], bytes);
          bulk_load_hint(ring + (size_t)b * slotf, sa.Mb + ((size_t)mb * K + k0 + j) * piece, bytes, &full[b],
                         pol_first);
        }
      }
    }
    return;
  }
  // warps 0..7: two groups of four (thread = tile), slots alternate between them
  const int grp = warp >> 2, tl = threadIdx.x & (kBM - 1);
  int s = 0;
  for (int it = r0; it < nItems; it += R) {
    const int mb = it / sa.nKS, k0 = (it % sa.nKS) * kSliceK, nk = min(K, k0 + kSliceK) - k0;
    const int t = mb * kBM + tl;
    for (int j = 0; j < nk; j += KP, ++s) {
      if ((s & 1) != grp) continue;
      const int b = s % NB;
      mbar_wait(&full[b], (uint32_t)((s / NB) & 1));
      const int kc = min(KP, nk - j);
      // the slot's lines are in shared memory: drop them from L2 without write-back
      const float* src = sa.Mb + ((size_t)mb * K + k0 + j) * piece;
      if (!(sa.dbg & 1))
        for (int l = tl; l < kc * QD * 4; l += kBM) discard_l2(src + (size_t)l * 32);
      const float* fb = ring + (size_t)b * slotf + tl;
      constexpr int NC = split_nc(QD);
      if (NC * QD <= 80) {
        // copy the slot into registers and hand it back to the producer before the math
        float mv[NC][QD];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int q = 0; q < QD; ++q) mv[c][q] = c < kc ? fb[c * piece + q * kBM] : 0.f;
        mbar_arrive(&empty[b]);
        if (t < sa.T && !(sa.dbg & 2)) {
          auto src = [&](int c, int q) { return mv[c][q]; };
          if (kc == NC) split_xform<DT, MO, DO, NC>(src, sa, t, k0 + j);
          else split_xform<DT, MO, DO, 1>(src, sa, t, k0 + j);
        }
      } else {
        if (t < sa.T && !(sa.dbg & 2))
          for (int c = 0; c < kc; ++c) {
            auto src = [&](int, int q) { return fb[c * piece + q * kBM]; };
            split_xform<DT, MO, DO, 1>(src, sa, t, k0 + j + c);
          }
        mbar_arrive(&empty[b]);
      }
      if (tl == 0) atomicAdd(sa.fixed + mb, kc);
    }
  }
}

// ------------------------------------------------------------------ host side

template <int DT, int MO, int DO>
static wino_status launch_split(const CUtensorMap& tv, const CUtensorMap& tu, const Geo& g, const wino_algo* al,
                                uint32_t fmt, float* Mw, void* y, int* cnt, cudaStream_t st) {
  constexpr int STAGES = 6, EPI = 2;   // the staged pair kernel's best configuration (gemm.cu)
  constexpr int SMEM = STAGES * (kBM * 128 + 128 * 128) + EPI * 32 * kBM * 4 + 1024 + 256;
  constexpr int BN = 256;
  auto kern = domain_gemm_split_kernel<STAGES, EPI, DT, MO, DO>;
  const int nMB = g.TB, nNB = (g.K + BN - 1) / BN;
  const int Q = g.Q;
  CUtensorMap tmb;
  {
    const uint64_t dims[4] = {(uint64_t)kBM, (uint64_t)Q, (uint64_t)g.K, (uint64_t)nMB};
    const uint64_t str[3] = {(uint64_t)kBM * 4, (uint64_t)Q * kBM * 4, (uint64_t)g.K * Q * kBM * 4};
    const uint32_t box[4] = {(uint32_t)kBM, 1, 32, 1};
    if (!make_map(&tmb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, Mw, dims, str, box, false)) {
      set_last_error("cuTensorMapEncodeTiled failed for the blocked M");
      return WINO_E_CUDA;
    }
  }
  SplitArgs sa{};
  for (int q = 0; q < al->m; ++q)
    for (int j = 0; j < al->D; ++j) sa.AT[q][j] = al->xp.AT[q][j];
  sa.Q = Q, sa.K = g.K, sa.T = g.T, sa.Ho = g.Ho, sa.Wo = g.Wo, sa.th = g.th, sa.tw = g.tw;
  sa.nMB = nMB, sa.nNB = nNB, sa.nKS = (g.K + kSliceK - 1) / kSliceK;
  sa.y = y, sa.Mb = Mw, sa.done = cnt, sa.fixed = cnt + nMB;
  const int sms = num_sms();
  // SM split: balance the GEMM (about 9.5 TFLOP/s per SM measured, bf16) against the
  // transform's L2 stream of M (about 110 GB/s per SM); WINO_SPLIT_R overrides
  int R = 0;
  {
    const double F = 2.0 * g.T * g.Cp * g.K * al->gs.npairs, Mbytes = 4.0 * Q * g.K * g.T;
    const double ratio = (Mbytes / 110e9) / (F / 9.5e12);   // R / G
    R = (int)(sms * ratio / (1.0 + ratio) + 0.5);
    if (const char* e = getenv("WINO_SPLIT_R")) R = atoi(e);
    R = R < 1 ? 1 : (R > sms - 2 ? sms - 2 : R);
  }
  sa.G = (sms - R) & ~1;   // whole CTA pairs
  if (sa.G < 2) sa.G = 2;
  sa.lag = 6;
  if (const char* e = getenv("WINO_SPLIT_LAG")) sa.lag = atoi(e);
  if (const char* e = getenv("WINO_SPLIT_DBG")) sa.dbg = atoi(e);
  if (sa.dbg & 4) sa.lag = 0;
  // transform ring: slots of KP channel pieces (Q * 512 B each)
  const size_t piece_bytes = (size_t)Q * kBM * 4;
  sa.KP = split_nc(Q);
  const size_t budget = (size_t)SMEM - 1024 - 256;
  sa.NB = (int)(budget / (sa.KP * piece_bytes));
  if (sa.NB > 8) sa.NB = 8;
  sa.NB &= ~1;
  if (sa.NB < 2) return WINO_E_UNSUPPORTED;
  const int smem = SMEM;
  WINO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  WINO_CUDA_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int) * 2 * nMB, st));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(kSplitThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;   // every CTA resident: the roles wait on each other
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;   // CTA pairs (the transform role ignores its peer)
  attr[1].val.clusterDim.x = 2, attr[1].val.clusterDim.y = 1, attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cfg.gridDim = dim3(sms & ~1);
  const uint32_t idesc = make_idesc(fmt, 2 * kBM, BN);
  WINO_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, tv, tu, tmb, g.Cp, idesc, al->gs, sa));
  WINO_LAUNCH_CHECK();
  return WINO_OK;
}

template <int DT, int MO>
static wino_status split_d(int doff, const CUtensorMap& tv, const CUtensorMap& tu, const Geo& g, const wino_algo* al,
                           uint32_t fmt, float* M, void* y, int* cnt, cudaStream_t st) {
  switch (doff) {
    case 0: return launch_split<DT, MO, MO + 2>(tv, tu, g, al, fmt, M, y, cnt, st);
    case 1: return launch_split<DT, MO, MO + 3>(tv, tu, g, al, fmt, M, y, cnt, st);
    default: return launch_split<DT, MO, MO + 4>(tv, tu, g, al, fmt, M, y, cnt, st);
  }
}
template <int DT>
static wino_status split_m(int m, int doff, const CUtensorMap& tv, const CUtensorMap& tu, const Geo& g,
                           const wino_algo* al, uint32_t fmt, float* M, void* y, int* cnt, cudaStream_t st) {
  switch (m) {
    case 2: return split_d<DT, 2>(doff, tv, tu, g, al, fmt, M, y, cnt, st);
    case 3: return split_d<DT, 3>(doff, tv, tu, g, al, fmt, M, y, cnt, st);
    case 4: return split_d<DT, 4>(doff, tv, tu, g, al, fmt, M, y, cnt, st);
    case 5: return split_d<DT, 5>(doff, tv, tu, g, al, fmt, M, y, cnt, st);
    case 6: return split_d<DT, 6>(doff, tv, tu, g, al, fmt, M, y, cnt, st);
    case 7: return split_d<DT, 7>(doff, tv, tu, g, al, fmt, M, y, cnt, st);
    default: return split_d<DT, 8>(doff, tv, tu, g, al, fmt, M, y, cnt, st);
  }
}

// Fused K3 + K4 with split SMs (16-bit dtypes, K > 128, NCHW output, m <= 8,
// domain <= m + 4).  Returns WINO_E_UNSUPPORTED, without launching, otherwise.
wino_status run_domain_gemm_split(const void* V, const void* U, const Geo& g, const wino_algo* al, wino_dtype dt,
                                  float* M, void* y, int* cnt, cudaStream_t st) {
  const int doff = al->D - al->m - 2;
  if (dt == WINO_F32 || g.K <= 128 || al->m < 2 || al->m > 8 || doff < 0 || doff > 2) return WINO_E_UNSUPPORTED;
  CUtensorMapDataType cdt = dt == WINO_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  constexpr int BN = 256;
  const uint32_t BK = 128 / (uint32_t)g.es;
  CUtensorMap tv, tu;
  if (!make_map3(&tv, cdt, g.es, V, BK, kBM, (uint64_t)g.planes * g.Q * g.TB * (g.Cp / BK), BK, kBM) ||
      !make_map3(&tu, cdt, g.es, U, g.Cp, g.K, (uint64_t)g.S * g.planes, BK, BN / 2)) {   // each CTA: half of B
    set_last_error("cuTensorMapEncodeTiled failed (driver entry point unavailable or bad geometry)");
    return WINO_E_CUDA;
  }
  const uint32_t fmt = dt == WINO_F16 ? 0u : 1u;
  return dt == WINO_F16 ? split_m<WINO_F16>(al->m, doff, tv, tu, g, al, fmt, M, y, cnt, st)
                        : split_m<WINO_BF16>(al->m, doff, tv, tu, g, al, fmt, M, y, cnt, st);
}

}  // namespace wino

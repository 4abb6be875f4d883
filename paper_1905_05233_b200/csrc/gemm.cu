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
#include "gemm_common.cuh"

namespace wino {

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

// ------------------------------------------------------------------ host side


template <bool kTF32, int BN, int STAGES>
static wino_status launch_gemm(const CUtensorMap& tv, const CUtensorMap& tu, const CUtensorMap& tm, const Geo& g,
                               const GemmSched& gs, uint32_t fmt, int mb0, int nT, cudaStream_t st) {
  using Cfg = GemmCfg<kTF32, BN, STAGES>;
  auto kern = domain_gemm_kernel<kTF32, BN, STAGES>;
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

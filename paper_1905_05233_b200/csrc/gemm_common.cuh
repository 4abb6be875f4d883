// gemm_common.cuh -- tile configuration of the tcgen05 Winograd-domain GEMM
// (gemm.cu) shared with the fused GEMM + output-transform kernel (split.cu).
#pragma once

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

}  // namespace wino

// geometry.hpp -- layer geometry and workspace layout of wino_conv2d
// (include/wino.h): U [S][K][Cp] | V [TB][Cp/CBW][Q][128][CBW] | M [Q][K][Tp] (fp32, or the
// 16-bit dtype under wino_set_m_storage) | group counters.
#pragma once
#include <cstddef>

#include "algo.hpp"

namespace wino {

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// M between K3 and K4 in the layer's 16-bit dtype (reading M3)?  fp32 layers keep fp32, and so
// do tiles beyond 8x8 (their output transforms weigh M by entries up to ~1e4, SURVEY H1 option 5).
inline bool m_in_dtype(const wino_algo* al, wino_dtype dt) {
  return al->m_store == 1 && dt != WINO_F32 && al->m <= 8;
}

struct Geo {
  int N, C, H, W, K, pad;
  int m, D, Q, S;
  int Ho, Wo, th, tw, T, Tp, Cp;
  int TB, CBW;   // V blocks: 128 tiles x CBW channels (one 128-byte swizzle row per tile)
  size_t es, planes;
  size_t mes;    // bytes per M element: 4 (fp32, R1) or 2 (the 16-bit layer dtype, M3)
  size_t offU, offV, offM, offD, total;
};

// Tiling of PAPER.md P:498: overlapping (m+2)x(m+2) tiles at stride m.
// Element offset of V_0[t][c] in the blocked layout: 16 KB blocks [128 t][CBW c]
// (every GEMM A-operand box is one contiguous 16 KB run), block (t / 128, c / CBW,
// point q) at ((t/128) * Cp/CBW + c/CBW) * Q + q -- the Q point blocks of one
// (tile block, channel block) are adjacent, so point q of a tile is at the
// compile-time distance q * kVPointStride elements from point 0.
constexpr int kVPointBytes = 16384;   // one [128 t][CBW c] block
__host__ __device__ inline size_t v_offset(int t, int c, int Cp, int CBW, int Q) {
  return ((size_t)(t >> 7) * (Cp / CBW) + c / CBW) * Q * (128 * CBW) + (size_t)(t & 127) * CBW + c % CBW;
}

inline Geo make_geo(const wino_algo* al, int N, int C, int H, int W, int K, int pad, wino_dtype dt) {
  Geo g;
  g.N = N, g.C = C, g.H = H, g.W = W, g.K = K, g.pad = pad;
  g.m = al->m;
  g.D = al->D;
  g.Q = al->D * al->D;
  g.S = al->units;
  g.Ho = H + 2 * pad - 2;
  g.Wo = W + 2 * pad - 2;
  g.th = (g.Ho + g.m - 1) / g.m;
  g.tw = (g.Wo + g.m - 1) / g.m;
  g.T = N * g.th * g.tw;
  g.Tp = (int)align_up(g.T, 32);   // 128-byte M rows (fused K3+K4 discards whole L2 lines)
  g.Cp = (int)align_up(C, 64);
  g.es = dt == WINO_F32 ? 4 : 2;
  g.planes = dt == WINO_F32 ? 2 : 1;  // fp32: TF32 hi and lo planes
  size_t u_bytes = g.planes * (size_t)g.S * K * g.Cp * g.es;
  g.TB = (g.T + 127) / 128;
  g.CBW = (int)(128 / g.es);
  size_t v_bytes = g.planes * (size_t)g.Q * g.TB * 128 * g.Cp * g.es;
  // M: [Q][K][Tp] for the staged K3 -> K4 pair, [TB][K][Q][128] for the fused split kernel
  g.mes = m_in_dtype(al, dt) ? 2 : 4;
  size_t m_bytes = (size_t)g.Q * K * g.TB * 128 * g.mes;
  g.offU = 0;
  g.offV = align_up(g.offU + u_bytes, 1024);
  g.offM = align_up(g.offV + v_bytes, 1024);
  g.offD = align_up(g.offM + m_bytes, 1024);
  g.total = align_up(g.offD + (size_t)((g.T + 127) / 128) * 8, 1024);   // two ints per 128-tile group
  return g;
}

}  // namespace wino

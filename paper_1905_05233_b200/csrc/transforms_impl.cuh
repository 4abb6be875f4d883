// transforms_impl.cuh -- kernels of transforms.cu (see there), instantiated
// per storage dtype, kind and m-range slice by xform.cu.
#pragma once
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "device.cuh"
#include "geometry.hpp"
#include "tmap.hpp"
#include "bt_masks.hpp"

namespace wino {


// ------------------------------------------------------------------ K2 weight transform
// One thread per (k, c); c < Cp (zero padding for c >= C).  For the SUBSOLVER
// lowering slab u is the Winograd point u of G g G^T; for the RESIDUE lowering
// it is the fp32 combination sum_j coef_j (G_P g G_P^T)_{a_j}, rounded once.
template <int DT>
__global__ void __launch_bounds__(128) weight_transform_kernel(const typename DType<DT>::T* __restrict__ w, int K,
                                                               int C, int Cp, const __grid_constant__ XformParams xp,
                                                               const __grid_constant__ UnitTerms ut,
                                                               typename DType<DT>::T* __restrict__ U,
                                                               size_t plane) {
  using Tr = DType<DT>;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (c >= Cp) return;
  float g[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) g[a][b] = c < C ? Tr::load(w + ((size_t)k * C + c) * 9 + a * 3 + b) : 0.f;
  const int D = xp.D;
  for (int u = 0; u < ut.units; ++u) {
    float acc = 0.f;
    for (int j = 0; j < ut.nterm[u]; ++j) {
      const int idx = ut.a[u][j];
      const int i = idx / D, jj = idx % D;
      float row[3];
#pragma unroll
      for (int b = 0; b < 3; ++b) row[b] = xp.G[i][0] * g[0][b] + xp.G[i][1] * g[1][b] + xp.G[i][2] * g[2][b];
      const float uij = row[0] * xp.G[jj][0] + row[1] * xp.G[jj][1] + row[2] * xp.G[jj][2];
      const float term = __fmul_rn(ut.coef[u][j], uij);
      acc = j == 0 ? term : __fadd_rn(acc, term);
    }
    const size_t off = ((size_t)u * K + k) * Cp + c;
    if constexpr (DT == WINO_F32) {
      float hi, lo;
      split_tf32(acc, hi, lo);
      U[off] = hi;
      U[off + plane] = lo;
    } else {
      U[off] = Tr::cvt(acc);
    }
  }
}

#ifndef K1_SKIP
#define K1_SKIP 0   // timing experiments only (K1 NCHW): 1 skips the tile transforms, 2 the
                    // conversions, 8 drops the bf16 V stores
#endif
template <int DT>
__device__ __forceinline__ void store_pair(typename DType<DT>::T* dst, float2 v, size_t plane) {
  if constexpr (DT == WINO_F32) {
    float h0, l0, h1, l1;
    split_tf32(v.x, h0, l0);
    split_tf32(v.y, h1, l1);
    *reinterpret_cast<float2*>(dst) = make_float2(h0, h1);
    *reinterpret_cast<float2*>(dst + plane) = make_float2(l0, l1);
  } else if constexpr (DT == WINO_F16) {
    *reinterpret_cast<__half2*>(dst) = __float22half2_rn(v);
  } else {
#if defined(K1_SKIP) && (K1_SKIP & 8)
    if (v.x == 1234.5f)   // timing experiment: keep the math, drop the stores
#endif
    *reinterpret_cast<__nv_bfloat162*>(dst) = __float22bfloat162_rn(v);
  }
}

// SUBSOLVER fast path: U_{ij}[k][c] = (G g G^T)_{ij} for a channel pair per
// lane (packed FFMA2, 128-byte coalesced stores per warp and point).
// block (32, 4): x = channel pair within a 64-channel block, y = k offset.
template <int DT, int D>
__global__ void __launch_bounds__(128) weight_transform_points(const typename DType<DT>::T* __restrict__ w, int K,
                                                               int C, int Cp, const __grid_constant__ XformParams xp,
                                                               typename DType<DT>::T* __restrict__ U, size_t plane) {
  using Tr = DType<DT>;
  const int ca = blockIdx.x * 64 + 2 * threadIdx.x, cb = ca + 1;
  const int k = blockIdx.y * 4 + threadIdx.y;
  if (k >= K) return;
  float2 g[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      g[a][b] = make_float2(ca < C ? Tr::load(w + ((size_t)k * C + ca) * 9 + a * 3 + b) : 0.f,
                            cb < C ? Tr::load(w + ((size_t)k * C + cb) * 9 + a * 3 + b) : 0.f);
  typename Tr::T* out = U + (size_t)k * Cp + ca;
  const size_t ps = (size_t)K * Cp;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    float2 row[3];   // (G g)_{i,b}
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      float2 acc = __fmul2_rn(g[0][b], make_float2(xp.G[i][0], xp.G[i][0]));
      acc = __ffma2_rn(g[1][b], make_float2(xp.G[i][1], xp.G[i][1]), acc);
      row[b] = __ffma2_rn(g[2][b], make_float2(xp.G[i][2], xp.G[i][2]), acc);
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
      float2 acc = __fmul2_rn(row[0], make_float2(xp.G[j][0], xp.G[j][0]));
      acc = __ffma2_rn(row[1], make_float2(xp.G[j][1], xp.G[j][1]), acc);
      acc = __ffma2_rn(row[2], make_float2(xp.G[j][2], xp.G[j][2]), acc);
      store_pair<DT>(out + (size_t)(i * D + j) * ps, acc, plane);
    }
  }
}

// Zero patterns of B^T baked into K1 at compile time (bt_masks.hpp): DenseBT
// keeps every term; MaskBT<w0, w1> has bit j * n_x + q set where B^T[j][q] != 0.
// The transform loops are fully unrolled, so a false nz() removes the term's
// FFMA2 (the coefficient values stay runtime kernel parameters).  Skipping a
// zero term can only change the sign of an exact zero result.
// Row pairs (small tiles only): rows j1 < j2 of B^T with B^T[j2][q] = +-B^T[j1][q]
// (Toom-Cook points +-p, P:533's good points come in such pairs).  Then
// E = sum_{q: +} B^T[j1][q] x_q, O = sum_{q: -} B^T[j1][q] x_q give both rows as
// E + O and E - O, and in the second stage the two output rows accumulate E and
// O once instead of twice.  PAIRS holds 4 bits per row (partner + 1, 0 = none),
// NEG bit j1 * n_x + q marks the '-' columns of base row j1.
struct DenseBT {
  __host__ __device__ static constexpr bool nz(int, int, int) { return true; }
  __host__ __device__ static constexpr int first(int, int) { return 0; }
  __host__ __device__ static constexpr int partner(int) { return -1; }
  __host__ __device__ static constexpr bool neg(int, int, int) { return false; }
};
template <uint64_t W0, uint64_t W1, uint64_t PAIRS = 0, uint64_t NEG = 0>
struct MaskBT {
  __host__ __device__ static constexpr bool nz(int j, int q, int nx) {
    return j * nx + q < 64 ? ((W0 >> (j * nx + q)) & 1) != 0 : ((W1 >> (j * nx + q - 64)) & 1) != 0;
  }
  __host__ __device__ static constexpr int first(int i, int nx) {   // first nonzero column of row i
    int a = 0;
    while (a < nx && !nz(i, a, nx)) ++a;
    return a;
  }
  __host__ __device__ static constexpr int partner(int j) { return (int)((PAIRS >> (4 * j)) & 15) - 1; }
  __host__ __device__ static constexpr bool neg(int j1, int q, int nx) { return ((NEG >> (j1 * nx + q)) & 1) != 0; }
};

// Small-tile core shared by every K1 staging path (so they stay bit-identical):
// V = B^T d B with the first stage per output column j and the second stage per
// output row i, row pairs folded as above.  load_row(a, d) fills input row a.
template <int DT, int NX, int D, typename MK, typename LoadRow>
__device__ __forceinline__ void transform_tile_small(LoadRow load_row, const XformParams& xp,
                                                     typename DType<DT>::T* out, size_t qstride, size_t plane) {
  float2 acc[D][D];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) acc[i][j] = make_float2(0.f, 0.f);
#pragma unroll
  for (int a = 0; a < NX; ++a) {
    float2 d[NX];
    load_row(a, d);
    float2 rt[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int p = MK::partner(j);
      if (p >= 0 && p < j) continue;   // the second row of a pair: formed with its base row
      float2 e = make_float2(0.f, 0.f), o = make_float2(0.f, 0.f);
#pragma unroll
      for (int q = 0; q < NX; ++q) {
        const float c = xp.BT[j][q];
        if (!MK::nz(j, q, NX)) continue;
        if (p > j && MK::neg(j, q, NX)) o = __ffma2_rn(d[q], make_float2(c, c), o);
        else e = __ffma2_rn(d[q], make_float2(c, c), e);
      }
      if (p > j) {
        rt[j] = __ffma2_rn(o, make_float2(1.f, 1.f), e);
        rt[p] = __ffma2_rn(o, make_float2(-1.f, -1.f), e);
      } else {
        rt[j] = e;
      }
    }
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int p = MK::partner(i);
      if (p >= 0 && p < i) continue;   // accumulated into its base row's E / O slots
      const float c = xp.BT[i][a];
      if (!MK::nz(i, a, NX)) continue;
      // paired rows: acc[i] collects E, acc[p] collects O until the end
      const int dst = (p > i && MK::neg(i, a, NX)) ? p : i;
#pragma unroll
      for (int j = 0; j < D; ++j)
        acc[dst][j] = (p < 0 && a == MK::first(i, NX)) ? __fmul2_rn(rt[j], make_float2(c, c))
                                                       : __ffma2_rn(rt[j], make_float2(c, c), acc[dst][j]);
    }
  }
#pragma unroll
  for (int i = 0; i < D; ++i) {
    const int p = MK::partner(i);
    if (p > i) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const float2 e = acc[i][j], o = acc[p][j];
        acc[i][j] = __ffma2_rn(o, make_float2(1.f, 1.f), e);
        acc[p][j] = __ffma2_rn(o, make_float2(-1.f, -1.f), e);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) store_pair<DT>(out + (size_t)(i * D + j) * qstride, acc[i][j], plane);
}

// ------------------------------------------------------------------ K1 input transform (NCHW)
// Channel-pair design for sm_100a.  CTA = (tile-column block of TJB tiles,
// (n, tile row ti), 64-channel block); lane l of every warp owns the channel
// pair (c0 + 2l, c0 + 2l + 1), so
//  * the halo is staged in shared memory as float2 pairs s[row][col][l]
//    (conflict-free 8-byte accesses), loaded with VEC-element vector loads
//    along w and converted to fp32 once;
//  * the separable transform V = B^T d B runs on packed FFMA2 (fma.rn.f32x2,
//    one instruction for both channels, coefficient broadcast);
//  * each V_q store of a warp is 32 x (2 channels) = one contiguous 128-byte
//    row (16-bit; fp32: 256 B per plane) of the K-major GEMM operand.
// Warp w handles tiles tj0 + w, tj0 + w + nwarps, ...  The column stage is
// chunked by JC output columns so the row-stage intermediates (NX x JC float2)
// stay in registers at every m.
// Stage NX halo rows of a channel pair per lane into s2[row][col][lane]
// (float2 = (channel a, channel b)): zero fill outside the image, then
// vectors of VEC elements along w (aligned in global coordinates) in batches
// of LB, all loads of a batch issued before any is consumed.  Warp w stages
// rows w, w + nw, ...
template <int VEC, typename TT> struct VecT;
template <typename TT> struct VecT<1, TT> { using T = TT; };
template <int VEC, typename TT> struct VecT {
  using T = typename std::conditional<VEC * sizeof(TT) == 16, uint4,
            typename std::conditional<VEC * sizeof(TT) == 8, uint2, unsigned int>::type>::type;
};
template <typename Tr, int VEC, int NX>
__device__ __forceinline__ void stage_halo(const typename Tr::T* xa, const typename Tr::T* xb, bool oka, bool okb,
                                           int H, int W, int row0, int col0, int SEG, int qlo, int qhi, float2* s2,
                                           int warp, int nw, int lane) {
  using TT = typename Tr::T;
  using VT = typename VecT<VEC, TT>::T;
  constexpr int LB = 16 / (int)sizeof(VT) < 4 ? 4 : (16 / (int)sizeof(VT) > 8 ? 8 : 16 / (int)sizeof(VT));
  const int v0 = qlo / VEC, nv = (qhi + VEC - 1) / VEC - v0;
#pragma unroll 1
  for (int a = warp; a < NX; a += nw) {
    const int r = row0 + a;
    float2* srow = s2 + a * SEG * 32 + lane;
    if (r < 0 || r >= H) {
      for (int b = 0; b < SEG; ++b) srow[b * 32] = make_float2(0.f, 0.f);
      continue;
    }
    for (int b = 0; b < qlo - col0; ++b) srow[b * 32] = make_float2(0.f, 0.f);
    for (int b = qhi - col0; b < SEG; ++b) srow[b * 32] = make_float2(0.f, 0.f);
    const VT* ra = reinterpret_cast<const VT*>(xa + (size_t)r * W) + v0;
    const VT* rb = reinterpret_cast<const VT*>(xb + (size_t)r * W) + v0;
    float2* sv = srow + (v0 * VEC - col0) * 32;
#pragma unroll 1
    for (int vb = 0; vb < nv; vb += LB) {
      VT ua[LB], ub[LB];
#pragma unroll
      for (int k = 0; k < LB; ++k) {
        ua[k] = VT{}, ub[k] = VT{};
        if (vb + k < nv) {
          if (oka) ua[k] = ra[vb + k];
          if (okb) ub[k] = rb[vb + k];
        }
      }
#pragma unroll
      for (int k = 0; k < LB; ++k) {
        if (vb + k >= nv) break;
        const int q0 = (v0 + vb + k) * VEC;
        const TT* ea = reinterpret_cast<const TT*>(&ua[k]);
        const TT* eb = reinterpret_cast<const TT*>(&ub[k]);
        float2* dst = sv + (vb + k) * VEC * 32;
        if (q0 >= qlo && q0 + VEC <= qhi) {
#pragma unroll
          for (int j = 0; j < VEC; ++j) dst[j * 32] = make_float2(Tr::load(ea + j), Tr::load(eb + j));
        } else {
#pragma unroll
          for (int j = 0; j < VEC; ++j)
            if (q0 + j >= qlo && q0 + j < qhi) dst[j * 32] = make_float2(Tr::load(ea + j), Tr::load(eb + j));
        }
      }
    }
  }
}

__host__ __device__ constexpr int k1_nchunk(int NX, int D) { return D * NX <= 36 ? 1 : (D * NX + 31) / 32; }
// larger tiles: two output columns per pass (measured best, scripts/ubench_k1rolled.cu)
__host__ __device__ constexpr int k1_jc(int NX, int D) { return k1_nchunk(NX, D) == 1 ? D : 2; }

// V = B^T d B for one tile and the channel pair of this lane.  The halo row a
// (a < NX) of the tile starts at ring + slot(a) * SEG * 32 + col * 32, slot(a)
// = (s0 + a) mod NX (a ring of NX staged rows; s0 = 0 for a plain buffer).
// The separable transform runs on packed FFMA2 (coefficient broadcast); each
// V_q store of the warp is one contiguous 128-byte (16-bit) / 2 x 256-byte
// (fp32 hi/lo) row of the K-major GEMM operand.
template <int DT, int NX, int D, typename MK = DenseBT>
__device__ __forceinline__ void transform_tile_pairs(const float2* ring, int s0, int SEG, int col,
                                                     const XformParams& xp, typename DType<DT>::T* out,
                                                     size_t qstride, size_t plane) {
  constexpr int JC = k1_jc(NX, D);
  if constexpr (k1_nchunk(NX, D) == 1) {
    auto load_row = [&](int a, float2* d) {
      const int sa = s0 + a < NX ? s0 + a : s0 + a - NX;
      const float2* sd = ring + (sa * SEG + col) * 32;
#pragma unroll
      for (int q = 0; q < NX; ++q) d[q] = sd[q * 32];
    };
    transform_tile_small<DT, NX, D, MK>(load_row, xp, out, qstride, plane);
  } else {
    // larger tiles: JC output columns at a time and a rolled loop over input
    // rows, so only D x JC accumulators and one halo row live in registers
#pragma unroll 1
    for (int j0 = 0; j0 < D; j0 += JC) {
      float2 acc[D][JC];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int jj = 0; jj < JC; ++jj) acc[i][jj] = make_float2(0.f, 0.f);
#pragma unroll 1
      for (int a = 0; a < NX; ++a) {
        const int sa = s0 + a < NX ? s0 + a : s0 + a - NX;
        const float2* sd = ring + (sa * SEG + col) * 32;
        float2 d[NX];
#pragma unroll
        for (int q = 0; q < NX; ++q) d[q] = sd[q * 32];
#pragma unroll
        for (int jj = 0; jj < JC; ++jj) {
          float2 rt = make_float2(0.f, 0.f);
#pragma unroll
          for (int q = 0; q < NX; ++q) {
            const float c = xp.BT[j0 + jj < D ? j0 + jj : D - 1][q];
            rt = __ffma2_rn(d[q], make_float2(c, c), rt);
          }
#pragma unroll
          for (int i = 0; i < D; ++i) {
            const float c = xp.BT[i][a];
            acc[i][jj] = __ffma2_rn(rt, make_float2(c, c), acc[i][jj]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int jj = 0; jj < JC; ++jj)
          if (j0 + jj < D) store_pair<DT>(out + (size_t)(i * D + j0 + jj) * qstride, acc[i][jj], plane);
    }
  }
}

// ------------------------------------------------------------------ K1 input transform (NCHW)
// Channel-pair design for sm_100a.  Lane l of every warp owns the channel pair
// (c0 + 2l, c0 + 2l + 1) of a 64-channel block; warp w transforms tiles
// w, w + nwarps, ... of the CTA's TJB-tile column block; the halo is staged in
// shared memory as float2 pairs ring[row][col][l] (fp32, conflict-free 8-byte
// accesses).
//
// input_transform_tma (the main path): a CTA owns (tile-column block, image
// n, channel block) and walks down all th tile rows.  One thread issues TMA
// boxes of the m new input rows of each step (64 channels at once) into a ring
// of NSLOT raw slots, NSLOT - 1 steps ahead of the math; completion is tracked
// by per-slot mbarriers (no cp.async bookkeeping in the other threads).  Each
// step converts its raw box into the packed ring[row][pair][col] (row pitch
// SEGP odd: conflict-free for lane = channel pair), and the 2 halo rows shared
// with the previous tile row are reused, so x is read from HBM once.
//   mode 0 (flat): rows are whole image rows, box {RB * W, 64} of the
//                  [N*C][H*W] view (any W with H*W*es % 16 == 0)
//   mode 2 (flat, row groups): the same rows as box {ralign * W, RB / ralign, 64} of the
//                  [N*C][H / ralign][ralign * W] view -- the identical shared-memory image
//                  for RB * W > 256, the box-dimension limit (m = 8 at W = 28 in 16 bits)
//   mode 1 (3D):   box {BOXC, RB, 64} of the [N*C][H][W] view (W*es % 16 == 0)
// TMA zero-fills rows / columns outside the image.
template <int DT> struct PairT;
// pack2(ra, rb, d0, d1): columns (c, c + 1) of channels a (ra) and b (rb) -> the
// two pairs d0 = (a_c, b_c), d1 = (a_c+1, b_c+1) with one load per channel
template <> struct PairT<WINO_F32> {
  using T = float2;
  static __device__ __forceinline__ T pack(float a, float b) { return make_float2(a, b); }
  static __device__ __forceinline__ void pack2(const float* ra, const float* rb, T* d0, T* d1) {
    const float2 a = *reinterpret_cast<const float2*>(ra), b = *reinterpret_cast<const float2*>(rb);
    *d0 = make_float2(a.x, b.x);
    *d1 = make_float2(a.y, b.y);
  }
  static __device__ __forceinline__ float2 unpack(T v) { return v; }
};
template <> struct PairT<WINO_BF16> {
  using T = uint32_t;   // (bf16 a, bf16 b): a in the low half
  static __device__ __forceinline__ T pack(__nv_bfloat16 a, __nv_bfloat16 b) {
    return (uint32_t)__bfloat16_as_ushort(a) | ((uint32_t)__bfloat16_as_ushort(b) << 16);
  }
  static __device__ __forceinline__ void pack2(const __nv_bfloat16* ra, const __nv_bfloat16* rb, T* d0, T* d1) {
    const uint32_t a = *reinterpret_cast<const uint32_t*>(ra), b = *reinterpret_cast<const uint32_t*>(rb);
    *d0 = __byte_perm(a, b, 0x5410);   // (a lo, b lo)
    *d1 = __byte_perm(a, b, 0x7632);   // (a hi, b hi)
  }
  static __device__ __forceinline__ float2 unpack(T v) {
    return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xFFFF0000u));
  }
};
template <> struct PairT<WINO_F16> {
  using T = uint32_t;
  static __device__ __forceinline__ T pack(__half a, __half b) {
    return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
  }
  static __device__ __forceinline__ void pack2(const __half* ra, const __half* rb, T* d0, T* d1) {
    const uint32_t a = *reinterpret_cast<const uint32_t*>(ra), b = *reinterpret_cast<const uint32_t*>(rb);
    *d0 = __byte_perm(a, b, 0x5410);   // (a lo, b lo)
    *d1 = __byte_perm(a, b, 0x7632);   // (a hi, b hi)
  }
  static __device__ __forceinline__ float2 unpack(T v) {
    return __half22float2(*reinterpret_cast<const __half2*>(&v));
  }
};

template <int DT, int NX, int D, typename PT, typename MK = DenseBT>
__device__ __forceinline__ void transform_tile_ring(const PT* ring, int s0, int RR, int SEGP, int col,
                                                    const XformParams& xp, typename DType<DT>::T* out,
                                                    size_t qstride, size_t plane) {
  using P = PairT<DT>;
  constexpr int JC = k1_jc(NX, D);
  if constexpr (k1_nchunk(NX, D) == 1) {
    auto load_row = [&](int a, float2* d) {
      const int sa = s0 + a < RR ? s0 + a : s0 + a - RR;
      const PT* sd = ring + sa * 32 * SEGP + col;
#pragma unroll
      for (int q = 0; q < NX; ++q) d[q] = P::unpack(sd[q]);
    };
    transform_tile_small<DT, NX, D, MK>(load_row, xp, out, qstride, plane);
  } else {
    // JC output columns per pass; small enough domains unroll every pass
    // (compile-time coefficient indices) with a memory clobber between passes
    // so the scheduler cannot interleave them, larger ones roll the passes.
    auto pass = [&](int j0) {
      float2 acc[D][JC];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int jj = 0; jj < JC; ++jj) acc[i][jj] = make_float2(0.f, 0.f);
#pragma unroll
      for (int a = 0; a < NX; ++a) {
        const int sa = s0 + a < RR ? s0 + a : s0 + a - RR;
        const PT* sd = ring + sa * 32 * SEGP + col;
        float2 d[NX];
#pragma unroll
        for (int q = 0; q < NX; ++q) d[q] = P::unpack(sd[q]);
#pragma unroll
        for (int jj = 0; jj < JC; ++jj) {
          float2 rt = make_float2(0.f, 0.f);
#pragma unroll
          for (int q = 0; q < NX; ++q) {
            const float c = xp.BT[j0 + jj < D ? j0 + jj : D - 1][q];
            if (MK::nz(j0 + jj < D ? j0 + jj : D - 1, q, NX)) rt = __ffma2_rn(d[q], make_float2(c, c), rt);
          }
#pragma unroll
          for (int i = 0; i < D; ++i) {
            const float c = xp.BT[i][a];
            if (MK::nz(i, a, NX)) acc[i][jj] = __ffma2_rn(rt, make_float2(c, c), acc[i][jj]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int jj = 0; jj < JC; ++jj)
          if (j0 + jj < D) store_pair<DT>(out + (size_t)(i * D + j0 + jj) * qstride, acc[i][jj], plane);
    };
    if constexpr (NX * D <= 64) {
#pragma unroll
      for (int j0 = 0; j0 < D; j0 += JC) {
        pass(j0);
        asm volatile("" ::: "memory");
      }
    } else {
      // tiles from 9 x 9: a clobber keeps the halo loads inside the pass -- hoisted out of
      // the loop they hold NX^2 registers and the kernel spills (cfg5 bf16 K1: lin8 418 ->
      // 290 us, sup1_8 513 -> 341 us, lin7 260 -> 249 us); 8 x 8 halos are faster hoisted
      // (sup1_6 335 vs 362 us)
#pragma unroll 1
      for (int j0 = 0; j0 < D; j0 += JC) {
        pass(j0);
        if constexpr (NX >= 9) asm volatile("" ::: "memory");
      }
    }
  }
}

#ifndef K1_CONV_WARPS_DEF
#define K1_CONV_WARPS_DEF 4
#endif
constexpr int K1_CONV_WARPS = K1_CONV_WARPS_DEF;   // converter warps of input_transform_tma
// compute warps per CTA: 7 for the fully unrolled small tiles, 5 for the rolled
// larger ones (keeps two CTAs per SM with room for their registers), 6 for 7 x 7 halo
// tiles (m = 5: a tile row of 28 columns holds 6 tiles; cfg5 bf16 K1 lin5 226 -> 195 us,
// sup1_5 234 -> 202 us)
__host__ __device__ constexpr bool k1_small(int NX, int D) { return NX * D <= 36; }
// Eight compute warps for the rolled multi-pass tiles, two warps sharing a tile's passes
// (a tile row of cfg5 holds only 4-5 such tiles), measured no faster once the halo loads stay
// inside the passes, and slower through the 157-register cap and the runtime pass stride
// (cfg5 bf16 K1: lin8 301 vs 294 us, sup1_6 380-388 vs 335 us, lin5 304 vs 226 us): not kept.
__host__ __device__ constexpr int k1_maxcw(int NX, int D) { return k1_small(NX, D) ? 7 : NX * D <= 56 ? 6 : 5; }

struct K1Geo {
  int C, H, W, pad, th, tw, Cp, TJB;
  int mode, RB, BOXC, NSLOT, RR, SEGP;
  int ralign, calign;   // flat boxes start at a multiple of ralign rows, 3D boxes at a multiple of calign columns
  unsigned box_bytes, slot_bytes;
  int ncb, nItems;      // column blocks; work items = ncb * N * (Cp / 64)
};

// Persistent, barrier-free pipeline: grid = min(items, 2 per SM); a CTA walks
// work items (column block, image, 64-channel block) and, inside each, the th
// tile rows.  Conversion step K of the CTA (item j, it = -1 .. th-1; K counts
// across items) moves the M input rows it*M - pad + 2 .. +M-1 (n_x - m = 2
// halo rows come from the previous step) from raw slot K % NSLOT into ring
// group K % RG (groups of M rows, consecutive groups adjacent in the circular
// ring of RR = RG * M rows).  Compute step (j, ti) reads groups K - 1 (its last
// two rows) and K, K = j (th + 1) + ti + 1.  Handoffs are mbarriers only:
//   producer warp  --raw_full (TMA tx)-->  converter warps
//   converters     --raw_empty-->  producer;  --grp_full-->  compute warps
//   compute warps  --grp_empty (group K - 1 after step ti; group K too after
//                    the item's last step)-->  converters
// so the converters run up to RG - 2 steps ahead of the math, and the next
// item's first boxes and conversions overlap the current item's last tiles.
template <int DT, int M, int NX, int D, typename MK = DenseBT>
__global__ void __launch_bounds__(32 * (k1_maxcw(NX, D) + K1_CONV_WARPS + 1), k1_small(NX, D) && DT != WINO_F32 ? 2 : 1)
    input_transform_tma(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ K1Geo gk,
                        const __grid_constant__ XformParams xp, typename DType<DT>::T* __restrict__ V,
                        size_t qstride, size_t plane) {
  using Tr = DType<DT>;
  using TT = typename Tr::T;
  using P = PairT<DT>;
  using PT = typename P::T;
  extern __shared__ __align__(16) uint8_t k1_smem_raw[];
  // TMA destinations must be 128-byte aligned: offset the shared array (stays a
  // shared-space pointer, so accesses compile to LDS / STS)
  uint8_t* k1_smem = k1_smem_raw + ((128u - (smem_u32(k1_smem_raw) & 127u)) & 127u);
  const int NSLOT = gk.NSLOT, RR = gk.RR, RG = gk.RR / M, SEGP = gk.SEGP, th = gk.th, pad = gk.pad, W = gk.W;
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(k1_smem);
  uint64_t* raw_empty = raw_full + NSLOT;
  uint64_t* grp_full = raw_empty + NSLOT;
  uint64_t* grp_empty = grp_full + RG;
  uint8_t* raw = k1_smem + 256;
  PT* ring = reinterpret_cast<PT*>(raw + (size_t)NSLOT * gk.slot_bytes);
  const int SEG = gk.TJB * M + NX - M;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int CW = 0;                       // compute warps first
  const int cw = (int)(blockDim.x >> 5) - K1_CONV_WARPS - 1;
  const int conv0 = cw, prod = cw + K1_CONV_WARPS;
  const int nCB = gk.Cp / 64;
  (void)CW;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSLOT; ++s) mbar_init(&raw_full[s], 1), mbar_init(&raw_empty[s], K1_CONV_WARPS * 32);
    for (int g = 0; g < RG; ++g) mbar_init(&grp_full[g], K1_CONV_WARPS * 32), mbar_init(&grp_empty[g], cw * 32);
    fence_barrier_init();
    tma_prefetch(&tmx);
  }
  __syncthreads();

  // item -> (column block, image, channel block); channel blocks fastest
  auto decode = [&](int item, int& cb, int& n, int& c0) {
    const int cbk = item % nCB, r = item / nCB;
    n = r % (gk.nItems / (nCB * gk.ncb));
    cb = r / (gk.nItems / (nCB * gk.ncb));
    c0 = cbk * 64;
  };
  const int nIt = gk.nItems;

  if (warp == prod) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int item = blockIdx.x; item < nIt; item += gridDim.x) {
        int cb, n, c0;
        decode(item, cb, n, c0);
        const int col0 = cb * gk.TJB * M - pad;
        const int cst = ((col0 < 0 ? 0 : col0) / gk.calign) * gk.calign;
        const int crow = n * gk.C + c0;
        for (int it = -1; it < th; ++it) {
          mbar_wait_sleep(&raw_empty[s], ph ^ 1);
          const int g0 = it * M - pad + NX - M;
          const int gst = gk.mode != 1 ? ((g0 < 0 ? 0 : g0) / gk.ralign) * gk.ralign : (g0 < 0 ? 0 : g0);
          mbar_arrive_expect_tx(&raw_full[s], gk.box_bytes);
          if (gk.mode == 0) tma_load_2d(raw + (size_t)s * gk.slot_bytes, &tmx, &raw_full[s], gst * W, crow);
          else if (gk.mode == 2) tma_load_3d(raw + (size_t)s * gk.slot_bytes, &tmx, &raw_full[s], 0, gst / gk.ralign, crow);
          else tma_load_3d(raw + (size_t)s * gk.slot_bytes, &tmx, &raw_full[s], cst, gst, crow);
          if (++s == NSLOT) s = 0, ph ^= 1;
        }
      }
    }
  } else if (warp >= conv0) {
    // ------------------------------------------------------------ converters
    const int cwarp = warp - conv0;
    int s = 0, g = 0;
    uint32_t phs = 0, phg = 0;
    const PT z = P::pack(Tr::cvt(0.f), Tr::cvt(0.f));
    for (int item = blockIdx.x; item < nIt; item += gridDim.x) {
      int cb, n, c0;
      decode(item, cb, n, c0);
      const int col0 = cb * gk.TJB * M - pad;
      const int cst = ((col0 < 0 ? 0 : col0) / gk.calign) * gk.calign;
      const bool flat = gk.mode != 1;                               // whole image rows (modes 0 and 2)
      const int RBW = flat ? gk.RB * W : gk.RB * gk.BOXC;           // elements per channel in the box
      const int rstride = flat ? W : gk.BOXC;
      // ring columns [blo, bhi) are inside the image; the others are zero
      const int blo = col0 < 0 ? -col0 : 0;
      const int bhi = flat ? (W - col0 < SEG ? W - col0 : SEG) : SEG;
      const int qoff = flat ? col0 : col0 - cst;   // raw column of ring column b: b + qoff
      const bool allc = c0 + 64 <= gk.C;                   // every channel of the block is real
      // vector conversion: raw columns qoff + b for b in [bs, bs + 2 npair) in aligned pairs
      // (rows and channel planes of the box start at even elements), single leading /
      // trailing columns apart
      const bool vec = (rstride % 2) == 0 && (RBW % 2) == 0;
      const int bs = blo + ((qoff + blo) & 1);
      const int npair = (bhi - bs) / 2;
      const bool lead = bs > blo, trail = bs + 2 * npair < bhi;
      for (int it = -1; it < th; ++it) {
        mbar_wait_sleep(&raw_full[s], phs);
        mbar_wait_sleep(&grp_empty[g], phg ^ 1);
        const TT* rs = reinterpret_cast<const TT*>(raw + (size_t)s * gk.slot_bytes);
        const int g0 = it * M - pad + NX - M;
        const int gst = flat ? ((g0 < 0 ? 0 : g0) / gk.ralign) * gk.ralign : (g0 < 0 ? 0 : g0);
#pragma unroll 1
        for (int k = cwarp; k < M; k += K1_CONV_WARPS) {
          const int gr = g0 + k;
          if (gr < -pad) continue;   // never read
          PT* drow = ring + (g * M + k) * 32 * SEGP;
          const TT* rrow = rs + (gr < 0 ? 0 : gr - gst) * rstride + qoff;
          for (int b = 0; b < blo; ++b) drow[lane * SEGP + b] = z;     // lane = channel pair
          for (int b = bhi; b < SEG; ++b) drow[lane * SEGP + b] = z;
          if (gr >= 0 && allc && vec) {
            // two columns per lane and load (4-byte / 8-byte raw pairs): lanes 0-15 walk the
            // column pairs, the two half-warps take the even / odd channel pairs p
            // (odd SEGP: the half-warps store to disjoint banks)
            const TT* r0 = rrow + bs;
            PT* d0 = drow + bs + (lane >> 4) * SEGP;
            for (int pi = lane & 15; pi < npair; pi += 16) {
              const TT* src = r0 + 2 * pi + (lane >> 4) * 2 * RBW;
              PT* dst = d0 + 2 * pi;
#pragma unroll 4
              for (int pp = 0; pp < 16; ++pp) {
                P::pack2(src, src + RBW, dst, dst + 1);
                src += 4 * RBW;
                dst += 2 * SEGP;
              }
            }
            if (lead)   // the first column alone (odd raw alignment): one channel pair per lane
              drow[lane * SEGP + blo] = P::pack(rrow[(2 * lane) * RBW + blo], rrow[(2 * lane + 1) * RBW + blo]);
            if (trail)
              drow[lane * SEGP + bhi - 1] =
                  P::pack(rrow[(2 * lane) * RBW + bhi - 1], rrow[(2 * lane + 1) * RBW + bhi - 1]);
          } else if (gr >= 0 && allc) {
            for (int b = blo + lane; b < bhi; b += 32) {
#pragma unroll 8
              for (int p = 0; p < 32; ++p)
                drow[p * SEGP + b] = P::pack(rrow[(2 * p) * RBW + b], rrow[(2 * p + 1) * RBW + b]);
            }
          } else {
            for (int b = blo + lane; b < bhi; b += 32) {
#pragma unroll 4
              for (int p = 0; p < 32; ++p) {
                const int ca = c0 + 2 * p;
                const TT va = (gr >= 0 && ca < gk.C) ? rrow[(2 * p) * RBW + b] : Tr::cvt(0.f);
                const TT vb = (gr >= 0 && ca + 1 < gk.C) ? rrow[(2 * p + 1) * RBW + b] : Tr::cvt(0.f);
                drow[p * SEGP + b] = P::pack(va, vb);
              }
            }
          }
        }
        mbar_arrive(&raw_empty[s]);   // this thread is done with the raw slot
        mbar_arrive(&grp_full[g]);    // ... and has written its ring rows
        if (++s == NSLOT) s = 0, phs ^= 1;
        if (++g == RG) g = 0, phg ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ compute warps
    int g = 0;          // group of conversion step K (the current step's new rows)
    uint32_t phg = 0;
    for (int item = blockIdx.x; item < nIt; item += gridDim.x) {
      int cb, n, c0;
      decode(item, cb, n, c0);
      const int tj0 = cb * gk.TJB;
      const int ca = c0 + 2 * lane;
      // conversion (item, -1): its last two rows are the first tile row's halo
      int gp = g;
      mbar_wait_sleep(&grp_full[g], phg);
      if (++g == RG) g = 0, phg ^= 1;
#pragma unroll 1
      for (int ti = 0; ti < th; ++ti) {
        mbar_wait_sleep(&grp_full[g], phg);
        const int s0 = gp * M + M - (NX - M);   // ring row of the tile's first halo row
        const size_t t_row = ((size_t)n * th + ti) * gk.tw;
        for (int tjl = warp; tjl < gk.TJB; tjl += cw) {
          const int tj = tj0 + tjl;
          if (tj >= gk.tw) break;
#if !(K1_SKIP & 1)
          transform_tile_ring<DT, NX, D, PT, MK>(ring + lane * SEGP, s0, RR, SEGP, tjl * M, xp,
                                                 V + v_offset((int)(t_row + tj), ca, gk.Cp, 128 / (int)sizeof(TT), D * D),
                                                 kVPointBytes / sizeof(TT), plane);
#endif
        }
        mbar_arrive(&grp_empty[gp]);               // the older group is no longer needed
        if (ti == th - 1) mbar_arrive(&grp_empty[g]);
        gp = g;
        if (++g == RG) g = 0, phg ^= 1;
      }
    }
  }
}

// ------------------------------------------------------------------ K1 input transform (NHWC)
// x[N][H][W][C]: channels are contiguous, so a TMA box {64 channels, BOXW
// columns, NX rows} of the [N][H][W][C] tensor lands in shared memory as
// [row][col][channel] -- already lane = channel pair (4-byte bf16x2 / half2,
// 8-byte float2 words, consecutive lanes consecutive words: conflict-free).
// No transpose: CTA = (tile-column block of TJB tiles, image, 64-channel
// block) walks down the tile rows with an NSLOT-deep TMA ring (mbarriers),
// each warp transforms one tile of the row from the box.  Boxes start at
// non-negative coordinates (rows / columns before the image are predicated
// to zero); TMA zero-fills beyond W, H and C.
struct K1NGeo {
  int C, H, W, pad, th, tw, Cp, TJB, BOXW, NSLOT;
  unsigned box_bytes, slot_bytes;
};

template <int DT, int NX, int D, typename PT, typename MK = DenseBT>
__device__ __forceinline__ void transform_tile_box(const PT* box, int BOXW, int rowoff, int colbase,
                                                   const XformParams& xp, typename DType<DT>::T* out,
                                                   size_t qstride, size_t plane) {
  // element (a, q) of the tile: box row a + rowoff, column colbase + q (word
  // index (row * BOXW + col) * 32 + lane, `box` already offset by lane);
  // negative rows / columns are the zero padding
  using P = PairT<DT>;
  constexpr int JC = k1_jc(NX, D);
  auto load_row = [&](int a, float2* d) {
    const int r = a + rowoff;
    const PT* sd = box + (size_t)(r < 0 ? 0 : r) * BOXW * 32;
#pragma unroll
    for (int q = 0; q < NX; ++q) {
      const int c = colbase + q;
      const float2 v = P::unpack(sd[(c < 0 ? 0 : c) * 32]);
      d[q] = (r < 0 || c < 0) ? make_float2(0.f, 0.f) : v;
    }
  };
  if constexpr (k1_nchunk(NX, D) == 1) {
    transform_tile_small<DT, NX, D, MK>(load_row, xp, out, qstride, plane);
  } else {
    // JC output columns per pass; small enough domains unroll every pass
    // (compile-time coefficient indices) with a memory clobber between passes
    // so the scheduler cannot interleave them, larger ones roll the passes.
    auto pass = [&](int j0) {
      float2 acc[D][JC];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int jj = 0; jj < JC; ++jj) acc[i][jj] = make_float2(0.f, 0.f);
#pragma unroll
      for (int a = 0; a < NX; ++a) {
        float2 d[NX];
        load_row(a, d);
#pragma unroll
        for (int jj = 0; jj < JC; ++jj) {
          float2 rt = make_float2(0.f, 0.f);
#pragma unroll
          for (int q = 0; q < NX; ++q) {
            const float c = xp.BT[j0 + jj < D ? j0 + jj : D - 1][q];
            if (MK::nz(j0 + jj < D ? j0 + jj : D - 1, q, NX)) rt = __ffma2_rn(d[q], make_float2(c, c), rt);
          }
#pragma unroll
          for (int i = 0; i < D; ++i) {
            const float c = xp.BT[i][a];
            if (MK::nz(i, a, NX)) acc[i][jj] = __ffma2_rn(rt, make_float2(c, c), acc[i][jj]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int jj = 0; jj < JC; ++jj)
          if (j0 + jj < D) store_pair<DT>(out + (size_t)(i * D + j0 + jj) * qstride, acc[i][jj], plane);
    };
    if constexpr (NX * D <= 64) {
#pragma unroll
      for (int j0 = 0; j0 < D; j0 += JC) {
        pass(j0);
        asm volatile("" ::: "memory");
      }
    } else {
#pragma unroll 1
      for (int j0 = 0; j0 < D; j0 += JC) pass(j0);
    }
  }
}

template <int DT, int M, int NX, int D, typename MK = DenseBT>
__global__ void __launch_bounds__(256, 2) input_transform_nhwc(const __grid_constant__ CUtensorMap tmx,
                                                               const __grid_constant__ K1NGeo gk,
                                                               const __grid_constant__ XformParams xp,
                                                               typename DType<DT>::T* __restrict__ V, size_t qstride,
                                                               size_t plane) {
  using PT = typename PairT<DT>::T;
  extern __shared__ __align__(16) uint8_t kn_smem_raw[];
  uint8_t* sm = kn_smem_raw + ((128u - (smem_u32(kn_smem_raw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint8_t* slots = sm + 128;
  const int NSLOT = gk.NSLOT, th = gk.th, pad = gk.pad;
  const int tj0 = blockIdx.x * gk.TJB, n = blockIdx.y, c0 = blockIdx.z * 64;
  const int col0 = tj0 * M - pad, cst = col0 < 0 ? 0 : col0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // warps 0 .. nw-2 transform tiles; warp nw-1 is the TMA producer.  Slots are
  // released per warp through `empty` mbarriers, so compute warps never wait
  // for each other -- only for their data.
  uint64_t* empty = full + NSLOT;
  const int cw = nw - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSLOT; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], cw);
    fence_barrier_init();
    tma_prefetch(&tmx);
  }
  __syncthreads();
  if (warp == cw) {
    if (lane == 0) {
#pragma unroll 1
      for (int ti = 0; ti < th; ++ti) {
        const int s_ = ti % NSLOT;
        if (ti >= NSLOT) mbar_wait(&empty[s_], (uint32_t)(((ti / NSLOT) - 1) & 1));
        const int g_ = ti * M - pad;
        fence_proxy_async_shared();
        mbar_arrive_expect_tx(&full[s_], gk.box_bytes);
        tma_load_4d(slots + (size_t)s_ * gk.slot_bytes, &tmx, &full[s_], c0, cst, g_ < 0 ? 0 : g_, n);
      }
    }
    return;
  }
  const int ca = c0 + 2 * lane;
#pragma unroll 1
  for (int ti = 0; ti < th; ++ti) {
    mbar_wait(&full[ti % NSLOT], (uint32_t)((ti / NSLOT) & 1));
    const PT* box = reinterpret_cast<const PT*>(slots + (size_t)(ti % NSLOT) * gk.slot_bytes) + lane;
    const int g = ti * M - pad;
    const int rowoff = g - (g < 0 ? 0 : g);   // -pad for the first tile row, else 0
    for (int tjl = warp; tjl < gk.TJB; tjl += cw) {
      const int tj = tj0 + tjl;
      if (tj >= gk.tw) break;
      const size_t t = ((size_t)n * th + ti) * gk.tw + tj;
      transform_tile_box<DT, NX, D, PT, MK>(box, gk.BOXW, rowoff, tjl * M + col0 - cst, xp,
                                        V + v_offset((int)t, ca, gk.Cp, 128 / (int)sizeof(typename DType<DT>::T), D * D), kVPointBytes / sizeof(typename DType<DT>::T),
                                        plane);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[ti % NSLOT]);   // this warp is done with the slot
  }
}

// Fallback for NHWC tensors TMA cannot describe (C * es % 16 != 0, e.g. C = 3):
// thread per (tile, channel pair), direct loads of the halo from global memory.
template <int DT, int M, int NX, int D, typename MK = DenseBT>
__global__ void __launch_bounds__(128) input_transform_nhwc_direct(const typename DType<DT>::T* __restrict__ x, int C,
                                                                   int H, int W, int pad, int th, int tw, int Cp,
                                                                   int T, const __grid_constant__ XformParams xp,
                                                                   typename DType<DT>::T* __restrict__ V,
                                                                   size_t qstride, size_t plane) {
  using Tr = DType<DT>;
  // one thread per (tile, channel pair), pairs fastest: Cp / 2 is a multiple of 32,
  // so a warp shares its tile; a flat 1D grid has no 65535-tile limit
  const size_t id = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int P = Cp / 2;
  if (id >= (size_t)T * P) return;
  const int t = (int)(id / P), pi = (int)(id % P);
  const int ca = 2 * pi, cb = ca + 1;
  const int tj = t % tw, rest = t / tw, ti = rest % th, n = rest / th;
  if constexpr (k1_nchunk(NX, D) == 1) {
    auto load_row = [&](int a, float2* d) {
      const int r = ti * M - pad + a;
#pragma unroll
      for (int q = 0; q < NX; ++q) {
        const int c = tj * M - pad + q;
        const bool ok = r >= 0 && r < H && c >= 0 && c < W;
        const typename Tr::T* px = x + (((size_t)n * H + (ok ? r : 0)) * W + (ok ? c : 0)) * C;
        d[q] = make_float2(ok && ca < C ? Tr::load(px + ca) : 0.f, ok && cb < C ? Tr::load(px + cb) : 0.f);
      }
    };
    transform_tile_small<DT, NX, D, MK>(load_row, xp, V + v_offset(t, ca, Cp, 128 / (int)sizeof(typename Tr::T), D * D),
                                        kVPointBytes / sizeof(typename Tr::T), plane);
    return;
  }
  float2 rowT[NX][D];
#pragma unroll
  for (int a = 0; a < NX; ++a) {
    const int r = ti * M - pad + a;
    float2 d[NX];
#pragma unroll
    for (int q = 0; q < NX; ++q) {
      const int c = tj * M - pad + q;
      const bool ok = r >= 0 && r < H && c >= 0 && c < W;
      const typename Tr::T* px = x + (((size_t)n * H + (ok ? r : 0)) * W + (ok ? c : 0)) * C;
      d[q] = make_float2(ok && ca < C ? Tr::load(px + ca) : 0.f, ok && cb < C ? Tr::load(px + cb) : 0.f);
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int q = 0; q < NX; ++q) acc = __ffma2_rn(d[q], make_float2(xp.BT[j][q], xp.BT[j][q]), acc);
      rowT[a][j] = acc;
    }
  }
  typename Tr::T* out = V + v_offset(t, ca, Cp, 128 / (int)sizeof(typename Tr::T), D * D);
  constexpr size_t qstride_c = kVPointBytes / sizeof(typename Tr::T);
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int a = 0; a < NX; ++a) acc = __ffma2_rn(rowT[a][j], make_float2(xp.BT[i][a], xp.BT[i][a]), acc);
      store_pair<DT>(out + (size_t)(i * D + j) * qstride_c, acc, plane);
    }
}

// Synchronous variant for rows whose vectors are narrower than 4 bytes (odd W
// in 16-bit): CTA = (tile-column block, (n, ti), channel block).
template <int DT, int M, int NX, int D, typename MK = DenseBT>
__global__ void __launch_bounds__(256, 2) input_transform_pairs(
    const typename DType<DT>::T* __restrict__ x, int C, int H, int W, int pad, int th, int tw, int Cp, int TJB, int VEC,
    const __grid_constant__ XformParams xp, typename DType<DT>::T* __restrict__ V, size_t qstride, size_t plane) {
  using Tr = DType<DT>;
  using TT = typename Tr::T;
  extern __shared__ float2 s2[];
  const int SEG = TJB * M + NX - M;   // staged columns
  const int tj0 = blockIdx.x * TJB;
  const int n = blockIdx.y / th, ti = blockIdx.y % th;
  const int c0 = blockIdx.z * 64;
  const int row0 = ti * M - pad, col0 = tj0 * M - pad;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int ca = c0 + 2 * lane, cb = ca + 1;
  const bool oka = ca < C, okb = cb < C;
  const int qlo = col0 < 0 ? 0 : col0;
  const int qhi = (col0 + SEG < W) ? col0 + SEG : W;  // in-image columns [qlo, qhi)
  const TT* xa = x + ((size_t)n * C + (oka ? ca : 0)) * H * W;
  const TT* xb = x + ((size_t)n * C + (okb ? cb : 0)) * H * W;
  switch (VEC * (int)sizeof(TT)) {
    case 16: stage_halo<Tr, 16 / (int)sizeof(TT), NX>(xa, xb, oka, okb, H, W, row0, col0, SEG, qlo, qhi, s2, warp, nw, lane); break;
    case 8: stage_halo<Tr, 8 / (int)sizeof(TT), NX>(xa, xb, oka, okb, H, W, row0, col0, SEG, qlo, qhi, s2, warp, nw, lane); break;
    case 4: stage_halo<Tr, 4 / (int)sizeof(TT), NX>(xa, xb, oka, okb, H, W, row0, col0, SEG, qlo, qhi, s2, warp, nw, lane); break;
    default: stage_halo<Tr, 1, NX>(xa, xb, oka, okb, H, W, row0, col0, SEG, qlo, qhi, s2, warp, nw, lane); break;
  }
  __syncthreads();
  for (int tjl = warp; tjl < TJB; tjl += nw) {
    const int tj = tj0 + tjl;
    if (tj >= tw) break;
    const size_t t = ((size_t)n * th + ti) * tw + tj;
    transform_tile_pairs<DT, NX, D, MK>(s2 + lane, 0, SEG, tjl * M, xp, V + v_offset((int)t, ca, Cp, 128 / (int)sizeof(TT), D * D),
                                    kVPointBytes / sizeof(TT), plane);
  }
}

// ------------------------------------------------------------------ K4 output transform (NCHW)
#ifndef K4_TMA16
#define K4_TMA16 1   // 16-bit M: the TMA-staged K4 at every domain size (0: tile-pair kernel for domains <= 6)
#endif
// M element: fp32 (reading R1) or the layer's 16-bit dtype (reading M3)
__device__ __forceinline__ float ld_m(const float* p) { return __ldg(p); }
__device__ __forceinline__ float ld_m(const __half* p) { return __half2float(__ldg(p)); }
__device__ __forceinline__ float ld_m(const __nv_bfloat16* p) { return __bfloat162float(__ldg(p)); }
__device__ __forceinline__ float sm_m(const float* p) { return *p; }
__device__ __forceinline__ float sm_m(const __half* p) { return __half2float(*p); }
__device__ __forceinline__ float sm_m(const __nv_bfloat16* p) { return __bfloat162float(*p); }
// One thread per (t, k), t fastest (coalesced reads of M[q][k][t]).  Row-streamed
// separable transform: Z_i = M_{i,.} A (m values), Y += A_{i,.}^T (x) Z_i.
// Tiles [t0, T) with M rows indexed from t0 (a chunk's M slice when t0 > 0);
// DISC drops the consumed M lines from L2 afterwards (they are never written
// back: chunked layers keep M in L2 only).
template <int DT, int M, int D, bool DISC, typename MT = float>
__global__ void __launch_bounds__(128) output_transform_nchw(const MT* __restrict__ Mw, int K, int Ho, int Wo,
                                                             int th, int tw, int T, int Tp,
                                                             const __grid_constant__ XformParams xp,
                                                             typename DType<DT>::T* __restrict__ y, int t0) {
  using Tr = DType<DT>;
  const int tl = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = t0 + tl;
  const int k = blockIdx.y;
  if (t >= T) return;
  float Y[M][M];
#pragma unroll
  for (int p = 0; p < M; ++p)
#pragma unroll
    for (int q = 0; q < M; ++q) Y[p][q] = 0.f;
  const size_t qs = (size_t)K * Tp;
  const MT* src = Mw + (size_t)k * Tp + tl;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    float Mi[D];
#pragma unroll
    for (int j = 0; j < D; ++j) Mi[j] = ld_m(src + (size_t)(i * D + j) * qs);
    float Z[M];
#pragma unroll
    for (int q = 0; q < M; ++q) {
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < D; ++j) acc = fmaf(Mi[j], xp.AT[q][j], acc);
      Z[q] = acc;
    }
#pragma unroll
    for (int p = 0; p < M; ++p)
#pragma unroll
      for (int q = 0; q < M; ++q) Y[p][q] = fmaf(xp.AT[p][i], Z[q], Y[p][q]);
  }
  const int tj = t % tw, rest = t / tw;
  const int ti = rest % th, n = rest / th;
  typename Tr::T* dst = y + (((size_t)n * K + k) * Ho + (size_t)ti * M) * Wo + (size_t)tj * M;
#pragma unroll
  for (int p = 0; p < M; ++p) {
    if (ti * M + p >= Ho) break;
    store_tile_row<Tr, M>(dst + (size_t)p * Wo, Y[p], Wo - tj * M);
  }
  if constexpr (DISC) {
    // every live lane has consumed its M values (they fed Y): lane 0 drops the
    // warp's 32-tile line of each point
    __syncwarp(__activemask());
    if ((threadIdx.x & 31) == 0)
      for (int q = 0; q < D * D; ++q) discard_l2(src + (size_t)q * qs);
  }
}

// Tile-pair K4 for a 16-bit M (domains <= 6, one pass; reading M3): thread per
// (tiles t, t + 1, k), so each M load of a warp is 32 x (2 tiles) = 128 B (the
// fp32-M thread-per-tile kernel measured faster than this one on fp32 M), and
// the transform runs on packed FFMA2, the two tiles in the two lanes of each
// instruction: per tile the same fp32 operations in the same order as
// output_transform_nchw (bit-identical results).
__device__ __forceinline__ float2 ld_m2(const float* p) { return __ldg(reinterpret_cast<const float2*>(p)); }
__device__ __forceinline__ float2 ld_m2(const __half* p) {
  return __half22float2(__ldg(reinterpret_cast<const __half2*>(p)));
}
__device__ __forceinline__ float2 ld_m2(const __nv_bfloat16* p) {
  return __bfloat1622float2(__ldg(reinterpret_cast<const __nv_bfloat162*>(p)));
}
template <int DT, int M, int D, typename MT>
__global__ void __launch_bounds__(128, 8) output_transform_nchw2(const MT* __restrict__ Mw, int K, int Ho, int Wo,
                                                              int th, int tw, int T, int Tp,
                                                              const __grid_constant__ XformParams xp,
                                                              typename DType<DT>::T* __restrict__ y) {
  using Tr = DType<DT>;
  const int t = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int k = blockIdx.y;
  if (t >= T) return;
  float2 Y[M][M];
#pragma unroll
  for (int p = 0; p < M; ++p)
#pragma unroll
    for (int q = 0; q < M; ++q) Y[p][q] = make_float2(0.f, 0.f);
  const size_t qs = (size_t)K * Tp;
  const MT* src = Mw + (size_t)k * Tp + t;   // t even, Tp a multiple of 32: aligned pairs
#pragma unroll
  for (int i = 0; i < D; ++i) {
    float2 Mi[D];
#pragma unroll
    for (int j = 0; j < D; ++j) Mi[j] = ld_m2(src + (size_t)(i * D + j) * qs);
    float2 Z[M];
#pragma unroll
    for (int q = 0; q < M; ++q) {
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < D; ++j) acc = __ffma2_rn(Mi[j], make_float2(xp.AT[q][j], xp.AT[q][j]), acc);
      Z[q] = acc;
    }
#pragma unroll
    for (int p = 0; p < M; ++p)
#pragma unroll
      for (int q = 0; q < M; ++q) Y[p][q] = __ffma2_rn(make_float2(xp.AT[p][i], xp.AT[p][i]), Z[q], Y[p][q]);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int tt = t + h;
    if (tt >= T) break;
    const int tj = tt % tw, rest = tt / tw;
    const int ti = rest % th, n = rest / th;
    typename Tr::T* dst = y + (((size_t)n * K + k) * Ho + (size_t)ti * M) * Wo + (size_t)tj * M;
#pragma unroll
    for (int p = 0; p < M; ++p) {
      if (ti * M + p >= Ho) break;
      float row[M];
#pragma unroll
      for (int q = 0; q < M; ++q) row[q] = h ? Y[p][q].y : Y[p][q].x;
      store_tile_row<Tr, M>(dst + (size_t)p * Wo, row, Wo - tj * M);
    }
  }
}

// Y through shared memory for rows stored element by element (odd m in 16-bit; 12-byte
// rows of m = 6 measured faster with their three 4-byte stores), tiles up to 8 x 8
#ifndef K4_STAGE_Y
#define K4_STAGE_Y 1
#endif
template <int M, typename TT>
__host__ __device__ constexpr bool k4_stage_y() {
  return K4_STAGE_Y && M <= 8 && (M * sizeof(TT)) % 4 != 0;
}
template <int M, typename TT>
constexpr size_t k4_stage_bytes() {
  return k4_stage_y<M, TT>() ? 4 * 32 * (sizeof(TT*) + sizeof(int) + (size_t)M * M * sizeof(TT)) : 0;
}

// TMA-staged K4 for large domains (D >= 7): a thread per (t, k) cannot keep
// enough of its D^2 loads in flight, so M is streamed through shared memory
// instead.  CTA = (128-tile block, 32 output channels); one producer thread
// loads, per channel k, the piece {128 t, 1 k, Q points} of M (Q x 512 B) into
// a ring of NB buffers (mbarriers), four warps (thread = tile) apply
// Y = A^T M A to it in the same fp32 order as output_transform_nchw.
template <int DT, int M, int D, typename MT = float>
__global__ void __launch_bounds__(160) output_transform_tma(const __grid_constant__ CUtensorMap tmMl, int K, int Ho,
                                                            int Wo, int th, int tw, int T, int NB,
                                                            const __grid_constant__ XformParams xp,
                                                            typename DType<DT>::T* __restrict__ y) {
  using Tr = DType<DT>;
  using TT = typename Tr::T;
  constexpr int Q = D * D;
  constexpr bool STG = k4_stage_y<M, TT>();
  extern __shared__ __align__(16) uint8_t k4t_smem_raw[];
  uint8_t* sm = k4t_smem_raw + ((128u - (smem_u32(k4t_smem_raw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + NB;
  MT* buf = reinterpret_cast<MT*>(sm + 128);
  // Y staging (STG): per compute warp 32 tile bases, their valid rows / columns, and
  // the 32 tiles' Y as [p][tile][q] in the output dtype
  uint8_t* stg = sm + 128 + (size_t)NB * Q * 128 * sizeof(MT);
  TT** sbase = reinterpret_cast<TT**>(stg) + (threadIdx.x >> 5) * 32;
  int* svalid = reinterpret_cast<int*>(stg + 4 * 32 * sizeof(TT*)) + (threadIdx.x >> 5) * 32;
  TT* sy = reinterpret_cast<TT*>(stg + 4 * 32 * (sizeof(TT*) + sizeof(int))) + (threadIdx.x >> 5) * 32 * M * M;
  const int mb = blockIdx.x, k0 = blockIdx.y * 32, nk = min(K, k0 + 32) - k0;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) mbar_init(&full[b], 1), mbar_init(&empty[b], 128);
    fence_barrier_init();
    tma_prefetch(&tmMl);
  }
  __syncthreads();
  if (tid >= 128) {   // producer warp
    if (tid == 128) {
      for (int j = 0; j < nk; ++j) {
        const int b = j % NB;
        if (j >= NB) mbar_wait(&empty[b], (uint32_t)(((j / NB) - 1) & 1));
        mbar_arrive_expect_tx(&full[b], Q * 128 * (uint32_t)sizeof(MT));
        tma_load_3d(buf + (size_t)b * Q * 128, &tmMl, &full[b], mb * 128, k0 + j, 0);
      }
    }
    return;
  }
  const int t = mb * 128 + tid;
  const int tj = t % tw, rest = t / tw, ti = rest % th, n = rest / th;
  for (int j = 0; j < nk; ++j) {
    const int b = j % NB;
    mbar_wait(&full[b], (uint32_t)((j / NB) & 1));
    if (t < T) {
      const MT* fb = buf + (size_t)b * Q * 128 + tid;
      float Y[M][M];
#pragma unroll
      for (int p = 0; p < M; ++p)
#pragma unroll
        for (int q = 0; q < M; ++q) Y[p][q] = 0.f;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        float Mi[D];
#pragma unroll
        for (int jj = 0; jj < D; ++jj) Mi[jj] = sm_m(fb + (i * D + jj) * 128);
        float Z[M];
#pragma unroll
        for (int q = 0; q < M; ++q) {
          float acc = 0.f;
#pragma unroll
          for (int jj = 0; jj < D; ++jj) acc = fmaf(Mi[jj], xp.AT[q][jj], acc);
          Z[q] = acc;
        }
#pragma unroll
        for (int p = 0; p < M; ++p)
#pragma unroll
          for (int q = 0; q < M; ++q) Y[p][q] = fmaf(xp.AT[p][i], Z[q], Y[p][q]);
      }
      TT* dst = y + (((size_t)n * K + k0 + j) * Ho + (size_t)ti * M) * Wo + (size_t)tj * M;
      if constexpr (STG) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int p = 0; p < M; ++p)
#pragma unroll
          for (int q = 0; q < M; ++q) sy[(p * 32 + lane) * M + q] = Tr::cvt(Y[p][q]);
        sbase[lane] = dst;
        svalid[lane] = min(M, Ho - ti * M) | (min(M, Wo - tj * M) << 8);
      } else {
#pragma unroll
        for (int p = 0; p < M; ++p) {
          if (ti * M + p >= Ho) break;
          store_tile_row<Tr, M>(dst + (size_t)p * Wo, Y[p], Wo - tj * M);
        }
      }
    } else if constexpr (STG) {
      sbase[threadIdx.x & 31] = nullptr;
    }
    mbar_arrive(&empty[b]);
    if constexpr (STG) {
      // the warp's 32 tiles written row p at a time: consecutive lanes take consecutive
      // (tile, column) elements, i.e. runs of M columns of adjacent tiles (the per-tile
      // 2-byte stores touched a sector per lane: cfg5 lin7 bf16 K4 497 -> 275 us)
      const int lane = threadIdx.x & 31;
      __syncwarp();
#pragma unroll 1
      for (int p = 0; p < M; ++p) {
#pragma unroll
        for (int e0 = 0; e0 < 32 * M; e0 += 32) {
          const int e = e0 + lane, tl = e / M, q = e - tl * M;
          TT* bp = sbase[tl];
          const int v = svalid[tl];
          if (bp != nullptr && p < (v & 255) && q < (v >> 8)) bp[(size_t)p * Wo + q] = sy[p * 32 * M + e];
        }
      }
      __syncwarp();
    }
  }
}

// ------------------------------------------------------------------ K4 output transform (NHWC)
// y[N][Ho][Wo][K].  CTA = 32 tiles (lanes, coalesced M reads along t) x KB
// output channels (8 warps x KB/8); Y is staged in shared memory as
// [tile][pixel][channel] in the storage dtype and written back as contiguous
// runs of KB channels per pixel (16-byte vector stores when K allows).
// KB output channels per CTA; TS = per-tile stride of the stage in elements
// (+8: 16-byte aligned rows, and only 4-way bank conflicts for lane = tile)
template <int M> struct K4N {
  // (16 channels x 144 pixels of fp32 for 32 tiles would need 296 KB of shared memory at m = 12)
  static constexpr int KB = M <= 4 ? 32 : (M <= 10 ? 16 : 8);
  static constexpr int TS = M * M * KB + 8;
};

template <int DT, int M, int D, typename MT = float>
__global__ void __launch_bounds__(256) output_transform_nhwc(const MT* __restrict__ Mw, int K, int Ho, int Wo,
                                                             int th, int tw, int T, int Tp,
                                                             const __grid_constant__ XformParams xp,
                                                             typename DType<DT>::T* __restrict__ y) {
  using Tr = DType<DT>;
  using TT = typename Tr::T;
  constexpr int KB = K4N<M>::KB, KPW = KB / 8, TS = K4N<M>::TS;
  extern __shared__ __align__(16) uint8_t k4n_smem[];
  TT* stage = reinterpret_cast<TT*>(k4n_smem);   // [32 tiles, stride TS][M*M][KB]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * 32 + lane;
  const int k0 = blockIdx.y * KB;
  const size_t qs = (size_t)K * Tp;
#pragma unroll 1
  for (int jk = 0; jk < KPW; ++jk) {
    const int kl = warp * KPW + jk, k = k0 + kl;
    if (t >= T || k >= K) continue;
    float Y[M][M];
#pragma unroll
    for (int p = 0; p < M; ++p)
#pragma unroll
      for (int q = 0; q < M; ++q) Y[p][q] = 0.f;
    const MT* src = Mw + (size_t)k * Tp + t;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      float Mi[D];
#pragma unroll
      for (int j = 0; j < D; ++j) Mi[j] = ld_m(src + (size_t)(i * D + j) * qs);
      float Z[M];
#pragma unroll
      for (int q = 0; q < M; ++q) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < D; ++j) acc = fmaf(Mi[j], xp.AT[q][j], acc);
        Z[q] = acc;
      }
#pragma unroll
      for (int p = 0; p < M; ++p)
#pragma unroll
        for (int q = 0; q < M; ++q) Y[p][q] = fmaf(xp.AT[p][i], Z[q], Y[p][q]);
    }
#pragma unroll
    for (int p = 0; p < M; ++p)
#pragma unroll
      for (int q = 0; q < M; ++q) stage[(size_t)lane * TS + (p * M + q) * KB + kl] = Tr::cvt(Y[p][q]);
  }
  __syncthreads();
  // write-back: units of 8 channels (16 B in 16-bit, 32 B in fp32) per (tile, pixel)
  constexpr int VE = 8;
  constexpr int UPP = KB / VE;   // units per pixel
  const bool vec = (K % VE) == 0 && (reinterpret_cast<uintptr_t>(y) % 16) == 0;
  for (int u = threadIdx.x; u < 32 * M * M * UPP; u += blockDim.x) {
    const int tl = u / (M * M * UPP), r = u % (M * M * UPP);
    const int px = r / UPP, kv = (r % UPP) * VE;
    const int tt = blockIdx.x * 32 + tl;
    if (tt >= T || k0 + kv >= K) continue;
    const int p = px / M, q = px % M;
    const int tj = tt % tw, rest = tt / tw, ti = rest % th, n = rest / th;
    const int ho = ti * M + p, wo = tj * M + q;
    if (ho >= Ho || wo >= Wo) continue;
    TT* dst = y + (((size_t)n * Ho + ho) * Wo + wo) * K + k0 + kv;
    const TT* src = stage + (size_t)tl * TS + px * KB + kv;
    if (vec && k0 + kv + VE <= K) {
      if constexpr (sizeof(TT) == 2) {
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
      } else {
        reinterpret_cast<uint4*>(dst)[0] = reinterpret_cast<const uint4*>(src)[0];
        reinterpret_cast<uint4*>(dst)[1] = reinterpret_cast<const uint4*>(src)[1];
      }
    } else {
      for (int e = 0; e < VE && k0 + kv + e < K; ++e) dst[e] = src[e];
    }
  }
}

// ------------------------------------------------------------------ launchers
struct InArgs {
  const void* x;
  int C, H, W, pad, th, tw, Cp, N, layout;
  const XformParams* xp;
  void* V;
  size_t qstride, plane;
  cudaStream_t st;
};
struct OutArgs {
  const void* Mw;   // fp32, or the 16-bit layer dtype when m16
  int K, Ho, Wo, th, tw, T, Tp, layout;
  const XformParams* xp;
  void* y;
  cudaStream_t st;
  int t0 = 0, nT = -1, disc = 0;   // chunked K4 (NCHW thread-per-tile kernel only): tiles [t0, t0 + nT)
  int m16 = 0;                      // M stored in the layer dtype (reading M3; 16-bit layers only)
};
using InFn = void (*)(const InArgs&);
using OutFn = void (*)(const OutArgs&);

// B^T structure of the runtime algorithm, computed exactly as scripts/gen_bt_masks.py
// does for bt_masks.hpp: zero pattern (bit j * n_x + q) and, for fully unrolled
// small tiles, the +-row pairs (greedy in row order) with their '-' columns.
struct BTKey {
  uint64_t w0 = 0, w1 = 0, pairs = 0, neg = 0;
};
inline BTKey bt_key(const XformParams& xp, int nx, int D) {
  BTKey k;
  for (int j = 0; j < D; ++j)
    for (int q = 0; q < nx; ++q)
      if (xp.BT[j][q] != 0.f) {
        const int b = j * nx + q;
        (b < 64 ? k.w0 : k.w1) |= 1ull << (b & 63);
      }
  if (nx * D > 36) return k;
  int partner[16];
  for (int j = 0; j < D; ++j) partner[j] = -1;
  for (int j1 = 0; j1 < D; ++j1) {
    if (partner[j1] >= 0) continue;
    for (int j2 = j1 + 1; j2 < D; ++j2) {
      if (partner[j2] >= 0) continue;
      bool ok = true, flip = false;
      for (int q = 0; q < nx && ok; ++q) {
        const float u = xp.BT[j1][q], v = xp.BT[j2][q];
        if (v == u) continue;
        if (v == -u) flip = true;
        else ok = false;
      }
      if (!ok || !flip) continue;
      partner[j1] = j2, partner[j2] = j1;
      for (int q = 0; q < nx; ++q)
        if (xp.BT[j1][q] != 0.f && xp.BT[j2][q] == -xp.BT[j1][q]) k.neg |= 1ull << (j1 * nx + q);
      break;
    }
  }
  for (int j = 0; j < D; ++j) k.pairs |= (uint64_t)(partner[j] + 1) << (4 * j);
  return k;
}
// K1 kernels for the algorithm's B^T structure: a compiled instance when it is
// one of bt_masks.hpp, else the dense one
#define WINO_PICK(nx_, d_, a_, b_, p_, n_)                                                         \
  if constexpr (nx_ == NX && d_ == D) {                                                            \
    if (k.w0 == a_ && k.w1 == b_ && k.pairs == p_ && k.neg == n_) kern = KERN<DT, M, NX, D, MaskBT<a_, b_, p_, n_>>; \
  }
template <int DT, int M, int NX, int D>
static auto pick_k1_tma(const XformParams& xp) {
#define KERN input_transform_tma
  auto kern = KERN<DT, M, NX, D, DenseBT>;
  const BTKey k = bt_key(xp, NX, D);
  WINO_BT_MASKS(WINO_PICK)
#undef KERN
  return kern;
}
template <int DT, int M, int NX, int D>
static auto pick_k1_nhwc(const XformParams& xp) {
#define KERN input_transform_nhwc
  auto kern = KERN<DT, M, NX, D, DenseBT>;
  const BTKey k = bt_key(xp, NX, D);
  WINO_BT_MASKS(WINO_PICK)
#undef KERN
  return kern;
}
template <int DT, int M, int NX, int D>
static auto pick_k1_nhwc_direct(const XformParams& xp) {
#define KERN input_transform_nhwc_direct
  auto kern = KERN<DT, M, NX, D, DenseBT>;
  const BTKey k = bt_key(xp, NX, D);
  WINO_BT_MASKS(WINO_PICK)
#undef KERN
  return kern;
}
template <int DT, int M, int NX, int D>
static auto pick_k1_pairs(const XformParams& xp) {
#define KERN input_transform_pairs
  auto kern = KERN<DT, M, NX, D, DenseBT>;
  const BTKey k = bt_key(xp, NX, D);
  WINO_BT_MASKS(WINO_PICK)
#undef KERN
  return kern;
}
#undef WINO_PICK

template <int DT, int M, int D>
static void launch_in_nhwc(const InArgs& a) {
  using TT = typename DType<DT>::T;
  constexpr int NX = M + 2;
  const size_t es = sizeof(TT);
  const CUtensorMapDataType cdt = DT == WINO_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                  : DT == WINO_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                   : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  K1NGeo gk{};
  gk.C = a.C, gk.H = a.H, gk.W = a.W, gk.pad = a.pad, gk.th = a.th, gk.tw = a.tw, gk.Cp = a.Cp;
  gk.TJB = a.tw < 7 ? a.tw : 7;   // one compute warp per tile
  while (gk.TJB > 1 && gk.TJB * M + 2 > 256) --gk.TJB;
  gk.BOXW = gk.TJB * M + 2;
  gk.box_bytes = (unsigned)(64 * gk.BOXW * NX * es);
  gk.slot_bytes = (gk.box_bytes + 127) / 128 * 128;
  gk.NSLOT = 4;
  while (gk.NSLOT > 2 && 128 + 128 + (size_t)gk.NSLOT * gk.slot_bytes > 110 * 1024) --gk.NSLOT;
  const size_t smem = 256 + (size_t)gk.NSLOT * gk.slot_bytes;
  CUtensorMap tm;
  bool ok = (reinterpret_cast<uintptr_t>(a.x) % 16) == 0 && ((size_t)a.C * es) % 16 == 0 && smem <= 200 * 1024;
  if (ok) {
    const uint64_t dims[4] = {(uint64_t)a.C, (uint64_t)a.W, (uint64_t)a.H, (uint64_t)a.N};
    const uint64_t str[3] = {(uint64_t)a.C * es, (uint64_t)a.W * a.C * es, (uint64_t)a.H * a.W * a.C * es};
    const uint32_t box[4] = {64, (uint32_t)gk.BOXW, (uint32_t)NX, 1};
    ok = make_map(&tm, cdt, 4, a.x, dims, str, box, false);
  }
  // (tiles beyond 8x8 take the direct-load kernel: their boxes rarely fit, and
  // not instantiating the TMA kernels for them halves the build time)
  if constexpr (M <= 8) {
    if (ok) {
      auto kern = pick_k1_nhwc<DT, M, NX, D>(*a.xp);
      if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      dim3 grid((a.tw + gk.TJB - 1) / gk.TJB, a.N, a.Cp / 64);
      const int cw = gk.TJB < 7 ? gk.TJB : 7;   // compute warps (+1 TMA producer warp)
      kern<<<grid, 32 * (cw + 1), smem, a.st>>>(tm, gk, *a.xp, (TT*)a.V, a.qstride, a.plane);
      return;
    }
  }
  const int T = a.N * a.th * a.tw;
  dim3 grid((unsigned)(((size_t)T * (a.Cp / 2) + 127) / 128));
  pick_k1_nhwc_direct<DT, M, NX, D>(*a.xp)<<<grid, 128, 0, a.st>>>((const TT*)a.x, a.C, a.H, a.W, a.pad, a.th,
                                                                      a.tw, a.Cp, T, *a.xp, (TT*)a.V, a.qstride,
                                                                      a.plane);
}

template <int DT, int M, int D>
static void launch_in(const InArgs& a) {
  if (a.layout == WINO_NHWC) return launch_in_nhwc<DT, M, D>(a);
  using TT = typename DType<DT>::T;
  using PT = typename PairT<DT>::T;
  constexpr int NX = M + 2;
  const size_t es = sizeof(TT);
  const uintptr_t xa = reinterpret_cast<uintptr_t>(a.x);
  const CUtensorMapDataType cdt = DT == WINO_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                  : DT == WINO_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                   : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  K1Geo gk{};
  gk.C = a.C, gk.H = a.H, gk.W = a.W, gk.pad = a.pad, gk.th = a.th, gk.tw = a.tw, gk.Cp = a.Cp;
  CUtensorMap tm;
  bool ok = xa % 16 == 0;
  if (ok && ((size_t)a.W * es) % 16 == 0) {
    // 3D boxes {BOXC, M, 64} over column blocks of up to 8 tiles
    gk.mode = 1;
    gk.TJB = a.tw < 7 ? a.tw : 7;
    const int al = (int)(16 / es);
    gk.calign = al, gk.ralign = 1;
    // box columns: the staged segment plus up to al - 1 leading columns of alignment
    while (gk.TJB > 1 && ((gk.TJB * M + 2 + 2 * al - 2) / al) * al > 256) --gk.TJB;
    gk.BOXC = ((gk.TJB * M + 2 + 2 * al - 2) / al) * al;
    gk.RB = M;
    const uint64_t dims[3] = {(uint64_t)a.W, (uint64_t)a.H, (uint64_t)a.N * a.C};
    const uint64_t str[2] = {(uint64_t)a.W * es, (uint64_t)a.H * a.W * es};
    const uint32_t box[3] = {(uint32_t)gk.BOXC, (uint32_t)gk.RB, 64};
    ok = make_map(&tm, cdt, 3, a.x, dims, str, box, false);
    gk.box_bytes = (unsigned)(gk.BOXC * gk.RB * 64 * es);
  } else if (ok && ((size_t)a.H * a.W * es) % 16 == 0) {
    // whole image rows: flat boxes {RB * W, 64} of the [N*C][H*W] view
    gk.mode = 0;
    gk.TJB = a.tw;
    int r16 = 1;
    while ((r16 * a.W * es) % 16) ++r16;      // rows per 16-byte aligned flat offset
    gk.ralign = r16, gk.calign = 1;
    gk.RB = (M + r16 - 1 + r16 - 1) / r16 * r16;  // covers M rows from an aligned start
    if (gk.RB * a.W <= 256) {
      const uint64_t dims[2] = {(uint64_t)a.H * a.W, (uint64_t)a.N * a.C};
      const uint64_t str[1] = {(uint64_t)a.H * a.W * es};
      const uint32_t box[2] = {(uint32_t)(gk.RB * a.W), 64};
      ok = make_map(&tm, cdt, 2, a.x, dims, str, box, false);
    } else if (r16 * a.W <= 256 && a.H % r16 == 0) {
      // more than 256 elements per channel: the rows as groups of r16 (16-byte aligned
      // groups; H * W * es % 16 == 0 makes H a multiple of r16), same bytes in shared memory
      gk.mode = 2;
      const uint64_t dims[3] = {(uint64_t)r16 * a.W, (uint64_t)(a.H / r16), (uint64_t)a.N * a.C};
      const uint64_t str[2] = {(uint64_t)r16 * a.W * es, (uint64_t)a.H * a.W * es};
      const uint32_t box[3] = {(uint32_t)(r16 * a.W), (uint32_t)(gk.RB / r16), 64};
      ok = make_map(&tm, cdt, 3, a.x, dims, str, box, false);
    } else {
      ok = false;
    }
    gk.box_bytes = (unsigned)(gk.RB * a.W * 64 * es);
  } else {
    ok = false;
  }
  const int seg = (ok ? gk.TJB : 1) * M + 2;
  if (ok) {
    gk.slot_bytes = (gk.box_bytes + 127) / 128 * 128;
    gk.SEGP = seg | 1;
    // raw slots / halo-ring groups (of M rows) that keep two CTAs per SM; the first
    // candidate can be overridden for experiments (WINO_K1_RING="<slots>,<groups>")
    int cand[4][2] = {{3, 3}, {3, 3}, {2, 4}, {2, 3}};
    if (const char* e = getenv("WINO_K1_RING")) {
      int ns = 0, rg = 0;
      if (sscanf(e, "%d,%d", &ns, &rg) == 2 && ns >= 2 && ns <= 6 && rg >= 3 && rg <= 6) cand[0][0] = ns, cand[0][1] = rg;
    }
    size_t smem = 0;
    for (int i = 0; i < 4; ++i) {
      gk.NSLOT = cand[i][0], gk.RR = cand[i][1] * M;
      smem = 256 + 128 + (size_t)gk.NSLOT * gk.slot_bytes + (size_t)gk.RR * 32 * gk.SEGP * sizeof(PT);
      if (smem <= 112 * 1024 || (i == 0 && getenv("WINO_K1_RING"))) break;
    }
    ok = smem <= 200 * 1024 && M <= 8;   // tiles beyond 8x8: synchronous staging (see launch_in_nhwc)
    if constexpr (M <= 8) if (ok) {
      auto kern = pick_k1_tma<DT, M, NX, D>(*a.xp);
      if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      constexpr int MAXCW = k1_maxcw(NX, D);
      const int nthr = 32 * ((gk.TJB < MAXCW ? gk.TJB : MAXCW) + K1_CONV_WARPS + 1);   // compute + converter + TMA warps
      gk.ncb = (a.tw + gk.TJB - 1) / gk.TJB;
      gk.nItems = gk.ncb * a.N * (a.Cp / 64);
      const int per_sm = k1_small(NX, D) && DT != WINO_F32 && smem <= 112 * 1024 ? 2 : 1;
      const int grid = gk.nItems < per_sm * num_sms() ? gk.nItems : per_sm * num_sms();
      kern<<<grid, nthr, smem, a.st>>>(tm, gk, *a.xp, (TT*)a.V, a.qstride, a.plane);
      return;
    }
  }
  // fallback: synchronous staging (odd plane sizes, misaligned x)
  int tjb = a.tw < 8 ? a.tw : 8;
  while (tjb > 1 && (size_t)NX * (tjb * M + 2) * 256 > 64 * 1024) --tjb;
  const size_t ring = (size_t)NX * (tjb * M + 2) * 256;
  int vec = 1;
  for (int b = 16; b >= 4; b /= 2)
    if ((size_t)b >= es && a.W % (int)(b / es) == 0 && xa % b == 0) {
      vec = (int)(b / es);
      break;
    }
  auto kern = pick_k1_pairs<DT, M, NX, D>(*a.xp);
  if (ring > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ring);
  dim3 grid((a.tw + tjb - 1) / tjb, a.N * a.th, a.Cp / 64);
  kern<<<grid, 32 * tjb, ring, a.st>>>((const TT*)a.x, a.C, a.H, a.W, a.pad, a.th, a.tw, a.Cp, tjb, vec, *a.xp,
                                       (TT*)a.V, a.qstride, a.plane);
}
template <int DT, int M, int D, typename MT>
static void launch_out_mt(const OutArgs& a) {
  const MT* Mw = static_cast<const MT*>(a.Mw);
  using Tr = DType<DT>;
  if (a.layout == WINO_NHWC && a.nT < 0) {
    const size_t smem = (size_t)32 * K4N<M>::TS * sizeof(typename Tr::T);
    constexpr int KB = K4N<M>::KB;
    auto kern = output_transform_nhwc<DT, M, D, MT>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((a.T + 31) / 32, (a.K + KB - 1) / KB);
    kern<<<grid, 256, smem, a.st>>>(Mw, a.K, a.Ho, a.Wo, a.th, a.tw, a.T, a.Tp, *a.xp, (typename Tr::T*)a.y);
    return;
  }
  if constexpr (D >= 7 || sizeof(MT) == 2 || M <= 8) {
    constexpr int Q = D * D;
    // fp32 M at domains <= 6 too (cfg5 lin4 bf16: 188 -> 181 us); WINO_K4_TMA32=0 selects
    // the thread-per-tile kernel (same fp32 operation order, identical bits)
    static const bool tma32 = [] { const char* e = getenv("WINO_K4_TMA32"); return !(e && *e == '0'); }();
    const bool use = D >= 7 || (sizeof(MT) == 2 && K4_TMA16) || tma32;
    // ring of NB buffers in <= 96 KB; domains whose Q x 128 piece exceeds 48 KB (D >= 10
    // in fp32) take two buffers (up to 200 KB) rather than the thread-per-tile kernel
    // (cfg5 bf16 sup1_7 K4 692 -> 441 us, lin8 331 -> 288 us); chunks: thread-per-tile kernel
    const size_t piece = (size_t)Q * 128 * sizeof(MT);
    int NB = use && a.nT < 0 ? (int)((96 * 1024) / piece) : 0;
    NB = NB > 4 ? 4 : NB;
    if (use && a.nT < 0 && NB < 2 && 256 + 2 * piece + k4_stage_bytes<M, typename Tr::T>() <= 200 * 1024) NB = 2;
    CUtensorMap tml;
    const uint64_t dims[3] = {(uint64_t)a.Tp, (uint64_t)a.K, (uint64_t)Q};
    const uint64_t str[2] = {(uint64_t)a.Tp * sizeof(MT), (uint64_t)a.K * a.Tp * sizeof(MT)};
    const uint32_t box[3] = {128, 1, (uint32_t)Q};
    if (NB >= 2 && (reinterpret_cast<uintptr_t>(a.Mw) % 16) == 0 &&
        make_map(&tml, sizeof(MT) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : (DT == WINO_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16), 3, a.Mw, dims, str, box, false)) {
      const size_t smem = 256 + (size_t)NB * Q * 128 * sizeof(MT) + k4_stage_bytes<M, typename Tr::T>();
      auto kern = output_transform_tma<DT, M, D, MT>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      dim3 grid((a.T + 127) / 128, (a.K + 31) / 32);
      kern<<<grid, 160, smem, a.st>>>(tml, a.K, a.Ho, a.Wo, a.th, a.tw, a.T, NB, *a.xp, (typename Tr::T*)a.y);
      return;
    }
  }
  if constexpr (sizeof(MT) == 2 && D <= 8) {
    if (a.nT < 0 && a.t0 == 0) {   // 16-bit M, one pass: the tile-pair kernel
      dim3 grid((a.T + 255) / 256, a.K);
      output_transform_nchw2<DT, M, D, MT><<<grid, 128, 0, a.st>>>(Mw, a.K, a.Ho, a.Wo, a.th, a.tw, a.T, a.Tp,
                                                                   *a.xp, (typename Tr::T*)a.y);
      return;
    }
  }
  const int nT = a.nT < 0 ? a.T - a.t0 : a.nT;
  dim3 grid((nT + 127) / 128, a.K);
  if (sizeof(MT) == 4 && a.disc)
    output_transform_nchw<DT, M, D, true><<<grid, 128, 0, a.st>>>((const float*)a.Mw, a.K, a.Ho, a.Wo, a.th, a.tw, a.t0 + nT, a.Tp,
                                                                  *a.xp, (typename Tr::T*)a.y, a.t0);
  else
    output_transform_nchw<DT, M, D, false, MT><<<grid, 128, 0, a.st>>>(Mw, a.K, a.Ho, a.Wo, a.th, a.tw, a.t0 + nT,
                                                                   a.Tp, *a.xp, (typename Tr::T*)a.y, a.t0);
}

template <int DT, int M, int D>
static void launch_out(const OutArgs& a) {
  // 16-bit M for tiles up to 8x8 (m_in_dtype: larger tiles keep an fp32 M)
  if constexpr (DT == WINO_F16 && M <= 8) {
    if (a.m16) return launch_out_mt<DT, M, D, __half>(a);
  } else if constexpr (DT == WINO_BF16 && M <= 8) {
    if (a.m16) return launch_out_mt<DT, M, D, __nv_bfloat16>(a);
  }
  launch_out_mt<DT, M, D, float>(a);
}

// m in [2, 8], domain D in [m + 2, m + 4] (at most two quadratic moduli).
// [m - 2][D - m - 2]: m = 2..12, D = m + 2 .. m + 5 (each degree-d modulus adds
// d - 1 domain points); the largest tiles (m >= 9) stop at D = m + 4.
#define WINO_ROW(F, DT, M) {&F<DT, M, M + 2>, &F<DT, M, M + 3>, &F<DT, M, M + 4>, &F<DT, M, M + 5>}
#define WINO_ROW3(F, DT, M) {&F<DT, M, M + 2>, &F<DT, M, M + 3>, &F<DT, M, M + 4>, nullptr}
constexpr int kTabM = 11, kTabD = 4;
// the dispatch table is built in slices of m (xform.cu, one unit per dtype x kind x slice):
// rows m = 2..5, 6..8, 9..12
constexpr int kXfRows0 = 4, kXfRows1 = 3, kXfRows2 = 4;

}  // namespace wino

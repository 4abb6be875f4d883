// transforms_impl.cuh -- kernels of transforms.cu (see there), instantiated
// per storage dtype by xform_f32.cu / xform_f16.cu / xform_bf16.cu.
#pragma once
#include <string>

#include "device.cuh"
#include "geometry.hpp"

namespace wino {

// tiles per CTA row block of K1: about 32 output columns per CTA
__host__ __device__ constexpr int k1_tjb(int M) { return M >= 8 ? 4 : (32 / M); }

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

// B^T d B for one (tile, channel): d is the n_x x n_x halo in shared memory
// (row stride `ld`); rowT = d B (per input row), V = B^T rowT, rounded once.
template <int DT, int M, int NX, int D>
__device__ __forceinline__ void tile_transform(const float* sd, int ld, const XformParams& xp,
                                               typename DType<DT>::T* out, size_t qstride, size_t plane) {
  using Tr = DType<DT>;
  float rowT[NX][D];
#pragma unroll
  for (int r = 0; r < NX; ++r) {
    float d[NX];
#pragma unroll
    for (int q = 0; q < NX; ++q) d[q] = sd[r * ld + q];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      float acc = 0.f;
#pragma unroll
      for (int q = 0; q < NX; ++q) acc = fmaf(xp.BT[j][q], d[q], acc);
      rowT[r][j] = acc;
    }
  }
#pragma unroll
  for (int i = 0; i < D; ++i) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      float acc = 0.f;
#pragma unroll
      for (int r = 0; r < NX; ++r) acc = fmaf(xp.BT[i][r], rowT[r][j], acc);
      const size_t off = (size_t)(i * D + j) * qstride;
      if constexpr (DT == WINO_F32) {
        float hi, lo;
        split_tf32(acc, hi, lo);
        out[off] = hi;
        out[off + plane] = lo;
      } else {
        out[off] = Tr::cvt(acc);
      }
    }
  }
}

// ------------------------------------------------------------------ K1 input transform (NCHW)
// CTA = (tile-column block of TJB tiles, (n, ti), 32 channels).  The halo rows
// [ti*m - pad, ti*m - pad + nx) x [tj0*m - pad, ..) of 32 channels are staged in
// shared memory (fp32, zero outside the image), then thread (c, tj) applies
// B^T (.) B separably: rowT = d B (per input row), V = B^T rowT.  A warp holds
// 32 consecutive channels of one tile, so each V_q store is one contiguous
// 64 B (16-bit) / 128 B (fp32) segment of the K-major GEMM operand.
template <int DT, int M, int NX, int D>
__global__ void __launch_bounds__(32 * k1_tjb(M)) input_transform_nchw(
    const typename DType<DT>::T* __restrict__ x, int C, int H, int W, int pad, int th, int tw, int Cp,
    const __grid_constant__ XformParams xp, typename DType<DT>::T* __restrict__ V, size_t qstride, size_t plane) {
  using Tr = DType<DT>;
  constexpr int TJB = k1_tjb(M);
  constexpr int SEG = TJB * M + NX - M;
  constexpr int CS = (NX * SEG) | 1;  // odd channel stride: conflict-free smem reads
  __shared__ float s[32 * CS];
  const int tj0 = blockIdx.x * TJB;
  const int n = blockIdx.y / th, ti = blockIdx.y % th;
  const int c0 = blockIdx.z * 32;
  const int row0 = ti * M - pad, col0 = tj0 * M - pad;
  // halo load: one warp per (channel, row) segment, lanes along the row
  // (coalesced); batches of RB rows per warp are loaded into registers before
  // any is stored, so each thread keeps RB * EPL loads in flight.
  {
    constexpr int ROWS = 32 * NX;
    constexpr int RPW = (ROWS + TJB - 1) / TJB;   // rows per warp
    constexpr int EPL = (SEG + 31) / 32;          // elements per lane per row
    constexpr int RB = RPW < 16 ? RPW : 16;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll 1
    for (int i0 = 0; i0 < RPW; i0 += RB) {
      float v[RB][EPL];
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int rr = warp + (i0 + i) * TJB;
        const int cl = rr / NX, a = rr - cl * NX;
        const int r = row0 + a, c = c0 + cl;
        const bool rowok = rr < ROWS && c < C && r >= 0 && r < H;
        const typename Tr::T* src = x + (((size_t)n * C + c) * H + r) * W;
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          const int q = col0 + lane + 32 * e;
          v[i][e] = (rowok && lane + 32 * e < SEG && q >= 0 && q < W) ? Tr::load(src + q) : 0.f;
        }
      }
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int rr = warp + (i0 + i) * TJB;
        if (rr >= ROWS) break;
        const int cl = rr / NX, a = rr - cl * NX;
#pragma unroll
        for (int e = 0; e < EPL; ++e)
          if (lane + 32 * e < SEG) s[cl * CS + a * SEG + lane + 32 * e] = v[i][e];
      }
    }
  }
  __syncthreads();
  const int cl = threadIdx.x & 31, tjl = threadIdx.x >> 5;
  const int tj = tj0 + tjl;
  if (tj >= tw) return;
  const size_t t = ((size_t)n * th + ti) * tw + tj;
  tile_transform<DT, M, NX, D>(s + cl * CS + tjl * M, SEG, xp, V + t * Cp + c0 + cl, qstride, plane);
}

// Full-row variant: the CTA covers all tw tiles of tile-row (n, ti) for 32
// channels, so each channel's halo is ONE contiguous range of x
// (rows [ti*m - pad, ti*m - pad + nx) clipped to the image), read with
// VEC-element vector loads (VEC * sizeof(T) = 8 or 16 bytes).
template <int DT, int M, int NX, int D, int VEC>
__global__ void __launch_bounds__(512) input_transform_rows(
    const typename DType<DT>::T* __restrict__ x, int C, int H, int W, int pad, int th, int tw, int Cp,
    const __grid_constant__ XformParams xp, typename DType<DT>::T* __restrict__ V, size_t qstride, size_t plane) {
  using Tr = DType<DT>;
  using TT = typename Tr::T;
  extern __shared__ float s_dyn[];
  const int SEG = tw * M + NX - M;
  const int CS = (NX * SEG) | 1;
  const int n = blockIdx.y / th, ti = blockIdx.y % th;
  const int c0 = blockIdx.z * 32;
  const int r0 = ti * M - pad;
  const int rlo = r0 < 0 ? 0 : r0, rhi = (r0 + NX > H) ? H : r0 + NX;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // zero fill: left/right padding columns of every row, and rows outside the image
  for (int e = threadIdx.x; e < 32 * NX; e += blockDim.x) {
    const int cl = e / NX, a = e - cl * NX;
    float* row = s_dyn + cl * CS + a * SEG;
    const int r = r0 + a;
    if (r < 0 || r >= H || c0 + cl >= C) {
      for (int b = 0; b < SEG; ++b) row[b] = 0.f;
    } else {
      for (int b = 0; b < pad; ++b) row[b] = 0.f;
      for (int b = pad + W; b < SEG; ++b) row[b] = 0.f;
    }
  }
  const int nvec = (rhi - rlo) * W / VEC;
  const float invW = 1.0f / (float)W;
  for (int cl = warp; cl < 32; cl += nw) {
    const int c = c0 + cl;
    if (c >= C || nvec <= 0) continue;
    const TT* src = x + (((size_t)n * C + c) * H + rlo) * W;
    float* dst = s_dyn + cl * CS + (rlo - r0) * SEG + pad;
    for (int e = lane; e < nvec; e += 32) {
      const int flat = e * VEC;
      int a = __float2int_rz(((float)flat + 0.5f) * invW);
      a -= (a * W > flat);
      a += ((a + 1) * W <= flat);
      const int col = flat - a * W;
      float v[VEC];
      if constexpr (VEC * sizeof(TT) == 8) {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(src + flat));
        const TT* e2 = reinterpret_cast<const TT*>(&u);
#pragma unroll
        for (int k = 0; k < VEC; ++k) v[k] = Tr::load(e2 + k);
      } else if constexpr (VEC * sizeof(TT) == 16) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(src + flat));
        const TT* e2 = reinterpret_cast<const TT*>(&u);
#pragma unroll
        for (int k = 0; k < VEC; ++k) v[k] = Tr::load(e2 + k);
      } else {
#pragma unroll
        for (int k = 0; k < VEC; ++k) v[k] = Tr::load(src + flat + k);
      }
#pragma unroll
      for (int k = 0; k < VEC; ++k) dst[a * SEG + col + k] = v[k];
    }
  }
  __syncthreads();
  const int cl = threadIdx.x & 31, tj = threadIdx.x >> 5;
  if (tj >= tw) return;
  const size_t t = ((size_t)n * th + ti) * tw + tj;
  tile_transform<DT, M, NX, D>(s_dyn + cl * CS + tj * M, SEG, xp, V + t * Cp + c0 + cl, qstride, plane);
}

// ------------------------------------------------------------------ K4 output transform (NCHW)
// One thread per (t, k), t fastest (coalesced reads of M[q][k][t]).  Row-streamed
// separable transform: Z_i = M_{i,.} A (m values), Y += A_{i,.}^T (x) Z_i.
template <int DT, int M, int D>
__global__ void __launch_bounds__(128) output_transform_nchw(const float* __restrict__ Mw, int K, int Ho, int Wo,
                                                             int th, int tw, int T, int Tp,
                                                             const __grid_constant__ XformParams xp,
                                                             typename DType<DT>::T* __restrict__ y) {
  using Tr = DType<DT>;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (t >= T) return;
  float Y[M][M];
#pragma unroll
  for (int p = 0; p < M; ++p)
#pragma unroll
    for (int q = 0; q < M; ++q) Y[p][q] = 0.f;
  const size_t qs = (size_t)K * Tp;
  const float* src = Mw + (size_t)k * Tp + t;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    float Mi[D];
#pragma unroll
    for (int j = 0; j < D; ++j) Mi[j] = __ldg(src + (size_t)(i * D + j) * qs);
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
  // full-width tile rows are stored as one vector when the row is aligned
  constexpr int RB = M * (int)sizeof(typename Tr::T);
  constexpr bool kVec = (RB == 4 || RB == 8 || RB == 16);
  const bool vec = kVec && tj * M + M <= Wo && ((Wo * (int)sizeof(typename Tr::T)) % RB) == 0 &&
                   (reinterpret_cast<uintptr_t>(y) % RB) == 0;
#pragma unroll
  for (int p = 0; p < M; ++p) {
    if (ti * M + p >= Ho) break;
    typename Tr::T* row = dst + (size_t)p * Wo;
    if constexpr (kVec) {
      if (vec) {
        union {
          typename Tr::T e[M];
          uint32_t u[RB / 4];
        } pk;
#pragma unroll
        for (int q = 0; q < M; ++q) pk.e[q] = Tr::cvt(Y[p][q]);
        if constexpr (RB == 4) *reinterpret_cast<uint32_t*>(row) = pk.u[0];
        if constexpr (RB == 8) *reinterpret_cast<uint2*>(row) = make_uint2(pk.u[0], pk.u[1]);
        if constexpr (RB == 16) *reinterpret_cast<uint4*>(row) = make_uint4(pk.u[0], pk.u[1], pk.u[2], pk.u[3]);
        continue;
      }
    }
#pragma unroll
    for (int q = 0; q < M; ++q)
      if (tj * M + q < Wo) row[q] = Tr::cvt(Y[p][q]);
  }
}

// ------------------------------------------------------------------ launchers
struct InArgs {
  const void* x;
  int C, H, W, pad, th, tw, Cp, N;
  const XformParams* xp;
  void* V;
  size_t qstride, plane;
  cudaStream_t st;
};
struct OutArgs {
  const float* Mw;
  int K, Ho, Wo, th, tw, T, Tp;
  const XformParams* xp;
  void* y;
  cudaStream_t st;
};
using InFn = void (*)(const InArgs&);
using OutFn = void (*)(const OutArgs&);

template <int DT, int M, int D>
static void launch_in(const InArgs& a) {
  using Tr = DType<DT>;
  constexpr int VEC = 16 / (int)sizeof(typename Tr::T) / (sizeof(typename Tr::T) == 2 ? 2 : 1);  // 8 B (16-bit) / 16 B (fp32)
  const int seg = a.tw * M + 2;
  const size_t smem = (size_t)32 * ((M + 2) * seg | 1) * sizeof(float);
  if (a.tw <= 16 && smem <= 160 * 1024 && a.W % VEC == 0 && (reinterpret_cast<uintptr_t>(a.x) % (VEC * sizeof(typename Tr::T))) == 0) {
    auto kern = input_transform_rows<DT, M, M + 2, D, VEC>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid(1, a.N * a.th, a.Cp / 32);
    kern<<<grid, 32 * a.tw, smem, a.st>>>((const typename Tr::T*)a.x, a.C, a.H, a.W, a.pad, a.th, a.tw, a.Cp, *a.xp,
                                          (typename Tr::T*)a.V, a.qstride, a.plane);
    return;
  }
  constexpr int TJB = k1_tjb(M);
  dim3 grid((a.tw + TJB - 1) / TJB, a.N * a.th, a.Cp / 32);
  input_transform_nchw<DT, M, M + 2, D><<<grid, 32 * TJB, 0, a.st>>>(
      (const typename Tr::T*)a.x, a.C, a.H, a.W, a.pad, a.th, a.tw, a.Cp, *a.xp, (typename Tr::T*)a.V, a.qstride,
      a.plane);
}
template <int DT, int M, int D>
static void launch_out(const OutArgs& a) {
  using Tr = DType<DT>;
  dim3 grid((a.T + 127) / 128, a.K);
  output_transform_nchw<DT, M, D><<<grid, 128, 0, a.st>>>(a.Mw, a.K, a.Ho, a.Wo, a.th, a.tw, a.T, a.Tp, *a.xp,
                                                          (typename Tr::T*)a.y);
}

// m in [2, 8], domain D in [m + 2, m + 6].
#define WINO_ROW(F, DT, M) {&F<DT, M, M + 2>, &F<DT, M, M + 3>, &F<DT, M, M + 4>, &F<DT, M, M + 5>, &F<DT, M, M + 6>}
#define WINO_TABLE(F, DT) \
  {WINO_ROW(F, DT, 2), WINO_ROW(F, DT, 3), WINO_ROW(F, DT, 4), WINO_ROW(F, DT, 5), WINO_ROW(F, DT, 6), WINO_ROW(F, DT, 7), WINO_ROW(F, DT, 8)}

// per-dtype tables (xform_<dt>.cu)
extern const InFn kInTableF32[7][5], kInTableF16[7][5], kInTableBF16[7][5];
extern const OutFn kOutTableF32[7][5], kOutTableF16[7][5], kOutTableBF16[7][5];

}  // namespace wino

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
  for (int e = threadIdx.x; e < 32 * NX * SEG; e += blockDim.x) {
    const int cl = e / (NX * SEG);
    const int rem = e - cl * (NX * SEG);
    const int a = rem / SEG, b = rem - a * SEG;
    const int r = row0 + a, q = col0 + b, c = c0 + cl;
    float v = 0.f;
    if (c < C && r >= 0 && r < H && q >= 0 && q < W) v = Tr::load(x + (((size_t)n * C + c) * H + r) * W + q);
    s[cl * CS + a * SEG + b] = v;
  }
  __syncthreads();
  const int cl = threadIdx.x & 31, tjl = threadIdx.x >> 5;
  const int tj = tj0 + tjl;
  if (tj >= tw) return;
  const size_t t = ((size_t)n * th + ti) * tw + tj;
  const float* sd = s + cl * CS + tjl * M;
  float rowT[NX][D];
#pragma unroll
  for (int r = 0; r < NX; ++r) {
    float d[NX];
#pragma unroll
    for (int q = 0; q < NX; ++q) d[q] = sd[r * SEG + q];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      float acc = 0.f;
#pragma unroll
      for (int q = 0; q < NX; ++q) acc = fmaf(xp.BT[j][q], d[q], acc);
      rowT[r][j] = acc;
    }
  }
  typename Tr::T* out = V + t * Cp + c0 + cl;
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
#pragma unroll
  for (int p = 0; p < M; ++p) {
    if (ti * M + p >= Ho) break;
#pragma unroll
    for (int q = 0; q < M; ++q)
      if (tj * M + q < Wo) dst[(size_t)p * Wo + q] = Tr::cvt(Y[p][q]);
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

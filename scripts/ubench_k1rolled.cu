// Variants of K1's large-tile compute (NX x NX halo -> D x D points) for m >= 5.
#include <cstdio>
#include "../paper_1905_05233_b200/csrc/transforms_impl.cuh"
namespace wino { void count_launch(int) {} void reset_launch_count() {} void set_last_error(const std::string&) {} }
using namespace wino;

// V2: compile-time rows a, column chunks j0 rolled
// V3: everything unrolled, chunks fenced by a memory clobber
template <int VAR, int NX, int D, int JC>
__device__ __forceinline__ void tile(const uint32_t* ring, int SEGP, int col, const XformParams& xp, __nv_bfloat16* out,
                                     size_t qstride) {
  using P = PairT<WINO_BF16>;
  auto body = [&](int j0) {
    float2 acc[D][JC];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int jj = 0; jj < JC; ++jj) acc[i][jj] = make_float2(0.f, 0.f);
#pragma unroll
    for (int a = 0; a < NX; ++a) {
      const uint32_t* sd = ring + a * 32 * SEGP + col;
      float2 d[NX];
#pragma unroll
      for (int q = 0; q < NX; ++q) d[q] = P::unpack(sd[q]);
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
        if (j0 + jj < D) store_pair<WINO_BF16>(out + (size_t)(i * D + j0 + jj) * qstride, acc[i][jj], 0);
  };
  if constexpr (VAR == 2) {
#pragma unroll 1
    for (int j0 = 0; j0 < D; j0 += JC) body(j0);
  } else {
#pragma unroll
    for (int j0 = 0; j0 < D; j0 += JC) {
      body(j0);
      asm volatile("" ::: "memory");
    }
  }
}

template <int VAR, int NX, int D, int JC, int NW>
__global__ void __launch_bounds__(32 * NW, 2) kc(const __grid_constant__ XformParams xp, __nv_bfloat16* V, size_t qstride,
                                               int ntiles_total, int per_cta) {
  __shared__ uint32_t ring[NX * 32 * 35 + 64];
  for (int i = threadIdx.x; i < NX * 32 * 35 + 64; i += blockDim.x) ring[i] = 0x3f803f80u + i;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int it = warp; it < per_cta; it += NW) {
    const int t = (blockIdx.x * per_cta + it) % ntiles_total;
    __nv_bfloat16* out = V + (size_t)t * 512 + (blockIdx.x & 7) * 64 + 2 * lane;
    if constexpr (VAR == 1)
      transform_tile_ring<WINO_BF16, NX, D, uint32_t>(ring + lane * 35, 0, NX, 35, it % 2, xp, out, qstride, 0);
    else
      tile<VAR, NX, D, JC>(ring + lane * 35, 35, it % 2, xp, out, qstride);
  }
}
template <int VAR, int NX, int D, int JC, int NW>
void run(int T, const char* name) {
  XformParams xp{};
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 10; ++j) xp.BT[i][j] = 0.1f * (i + 1) - 0.05f * j;
  const size_t qstride = (size_t)T * 512;
  __nv_bfloat16* V;
  cudaMalloc(&V, D * D * qstride * 2);
  const int total = T * 8, ctas = 296, per_cta = (total + ctas - 1) / ctas;
  for (int r = 0; r < 2; ++r) kc<VAR, NX, D, JC, NW><<<ctas, 32 * NW>>>(xp, V, qstride, T, per_cta);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kc<VAR, NX, D, JC, NW><<<ctas, 32 * NW>>>(xp, V, qstride, T, per_cta);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%-22s %8.1f us (%s)\n", name, ms / 5 * 1e3, cudaGetErrorString(cudaGetLastError()));
  cudaFree(V);
}
int main() {
  run<1, 8, 8, 4, 5>(6400, "m6 D8  rolled");
  run<2, 8, 8, 4, 5>(6400, "m6 D8  V2 JC4");
  run<3, 8, 8, 4, 5>(6400, "m6 D8  V3 JC4");
  run<2, 8, 8, 2, 5>(6400, "m6 D8  V2 JC2");
  run<3, 8, 8, 2, 5>(6400, "m6 D8  V3 JC2");
  run<1, 10, 10, 4, 5>(4096, "m8 D10 rolled");
  run<2, 10, 10, 4, 5>(4096, "m8 D10 V2 JC4");
  run<3, 10, 10, 4, 5>(4096, "m8 D10 V3 JC4");
  run<3, 10, 10, 2, 5>(4096, "m8 D10 V3 JC2");
  run<2, 10, 10, 2, 5>(4096, "m8 D10 V2 JC2");
  return 0;
}

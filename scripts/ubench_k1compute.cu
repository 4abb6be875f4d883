// Microbenchmark of K1's compute phase alone: transform_tile_ring (the exact
// device function of libwino) over a static shared-memory halo ring, warp per
// tile, lane per channel pair, real coalesced V stores; no TMA, converter or
// barriers.  Same total work as cfg5 lin4 bf16 (12544 tiles x 8 channel blocks).
#include <cstdio>
#include <cstdlib>
#include "../paper_1905_05233_b200/csrc/transforms_impl.cuh"
namespace wino { void count_launch(int) {} void reset_launch_count() {} void set_last_error(const std::string&) {} }
using namespace wino;

template <int NW, int MINB, bool STORE>
__global__ void __launch_bounds__(32 * NW, MINB) kc(const __grid_constant__ XformParams xp, __nv_bfloat16* V,
                                                   size_t qstride, int ntiles_total, int per_cta) {
  __shared__ uint32_t ring[10 * 32 * 31];
  for (int i = threadIdx.x; i < 10 * 32 * 31; i += blockDim.x) ring[i] = 0x3f803f80u + i;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int it = warp; it < per_cta; it += NW) {
    const int t = (blockIdx.x * per_cta + it) % ntiles_total;
    __nv_bfloat16* out = V + (size_t)t * 512 + (blockIdx.x & 7) * 64 + 2 * lane;
    transform_tile_ring<WINO_BF16, 6, 6, uint32_t>(ring + lane * 31, it % 10, 10, 31, (it % 7) * 4, xp,
                                                   out, STORE ? qstride : 0, 0);
  }
}

int main() {
  XformParams xp{};
  xp.m = 4, xp.nx = 6, xp.D = 6;
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) xp.BT[i][j] = 0.1f * (i + 1) - 0.05f * j;
  const int T = 12544;
  const size_t qstride = (size_t)T * 512;
  __nv_bfloat16* V;
  cudaMalloc(&V, 36 * qstride * 2);
  const int total = T * 8;   // warp-tiles
  auto run = [&](auto kern, int nw, const char* name) {
    const int ctas = 148 * 2;
    const int per_cta = (total + ctas - 1) / ctas;
    for (int r = 0; r < 2; ++r) kern<<<ctas, 32 * nw>>>(xp, V, qstride, T, per_cta);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<ctas, 32 * nw>>>(xp, V, qstride, T, per_cta);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.1f us  (%s)\n", name, ms / 5 * 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  run(kc<7, 2, true>, 7, "7 warps x2 CTA, stores");
  run(kc<7, 2, false>, 7, "7 warps x2 CTA, no stores");
  run(kc<8, 2, true>, 8, "8 warps x2 CTA, stores");
  run(kc<4, 4, true>, 4, "4 warps x4 CTA, stores");
  run(kc<16, 1, true>, 16, "16 warps x1 CTA, stores");
  return 0;
}

// K1 compute-only for m = 8 (NX = D = 10, the rolled path) and m = 6 (NX = D = 8):
// same harness as ubench_k1compute.cu.
#include <cstdio>
#include "../paper_1905_05233_b200/csrc/transforms_impl.cuh"
namespace wino { void count_launch(int) {} void reset_launch_count() {} void set_last_error(const std::string&) {} }
using namespace wino;
template <int NX, int D, int NW>
__global__ void __launch_bounds__(32 * NW, 2) kc(const __grid_constant__ XformParams xp, __nv_bfloat16* V, size_t qstride,
                                               int ntiles_total, int per_cta) {
  __shared__ uint32_t ring[NX * 32 * 35 + 64];
  for (int i = threadIdx.x; i < NX * 32 * 35 + 64; i += blockDim.x) ring[i] = 0x3f803f80u + i;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int it = warp; it < per_cta; it += NW) {
    const int t = (blockIdx.x * per_cta + it) % ntiles_total;
    __nv_bfloat16* out = V + (size_t)t * 512 + (blockIdx.x & 7) * 64 + 2 * lane;
    transform_tile_ring<WINO_BF16, NX, D, uint32_t>(ring + lane * 35, 0, NX, 35, it % 2, xp, out, qstride, 0);
  }
}
template <int NX, int D, int NW>
void run(int T, const char* name) {
  XformParams xp{};
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 10; ++j) xp.BT[i][j] = 0.1f * (i + 1) - 0.05f * j;
  const size_t qstride = (size_t)T * 512;
  __nv_bfloat16* V;
  cudaMalloc(&V, D * D * qstride * 2);
  const int total = T * 8, ctas = 296, per_cta = (total + ctas - 1) / ctas;
  for (int r = 0; r < 2; ++r) kc<NX, D, NW><<<ctas, 32 * NW>>>(xp, V, qstride, T, per_cta);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kc<NX, D, NW><<<ctas, 32 * NW>>>(xp, V, qstride, T, per_cta);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%-12s %8.1f us (%s)\n", name, ms / 5 * 1e3, cudaGetErrorString(cudaGetLastError()));
  cudaFree(V);
}
int main() {
  run<8, 8, 5>(6400, "m6 D8");
  run<8, 9, 5>(6400, "m6 D9");
  run<10, 10, 5>(4096, "m8 D10");
  run<6, 6, 7>(12544, "m4 D6");
  return 0;
}

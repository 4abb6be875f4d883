// Microbenchmark: how fast can K1's V write stream go on B200?  The same 462 MB
// (cfg5 lin4 bf16: 36 points x 12544 tiles x 512 channels x 2 B) written as
//   seq32   : sequential, one 4-byte store per lane (128 B per warp instruction)
//   seq128  : sequential, 16-byte stores per lane
//   k1pat32 : K1's pattern -- CTA = (image, 64-channel block), warp per tile, and
//             per tile 36 rows of 128 B, one per point plane of the blocked V
//             ([Q][T/128][Cp/64][128 t][64 c])
//   k1bulk  : the same rows staged in shared memory per 7-tile step and written
//             as 36 bulk copies (cp.async.bulk.global.shared) of 7 x 128 B
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ubench_vstore.cu -o ubench_vstore
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int Q = 36, T = 12544, CP = 512, NB = 8, TPI = 49;   // tiles per image
constexpr size_t PLANE = (size_t)((T + 127) / 128) * 128 * CP;  // elements per point plane

__device__ __forceinline__ size_t voff(int t, int c) {
  return ((size_t)(t >> 7) * (CP / 64) + c / 64) * (128 * 64) + (t & 127) * 64 + (c & 63);
}

__global__ void seq32(uint32_t* V, size_t nwords) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nwords; i += (size_t)gridDim.x * blockDim.x)
    V[i] = (uint32_t)i;
}
__global__ void seq128(uint4* V, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    V[i] = make_uint4((uint32_t)i, 1, 2, 3);
}
// grid (NB, N): warps walk the image's 49 tiles
template <int NW>
__global__ void __launch_bounds__(32 * NW) k1pat32(uint16_t* V) {
  const int cb = blockIdx.x, n = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int tl = warp; tl < TPI; tl += NW) {
    const int t = n * TPI + tl;
    uint32_t* base = reinterpret_cast<uint32_t*>(V + voff(t, cb * 64 + 2 * lane));
#pragma unroll
    for (int p = 0; p < Q; ++p) base[(size_t)p * PLANE / 2] = (uint32_t)(p * 77 + lane);
  }
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// 7 tiles per step (one per warp), staged [Q][7][64 c], then 36 bulk copies
__global__ void __launch_bounds__(224) k1bulk(uint16_t* V) {
  extern __shared__ __align__(128) uint32_t stage_raw[];
  auto stage = reinterpret_cast<uint32_t(*)[Q][7][32]>(stage_raw);
  const int cb = blockIdx.x, n = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int step = 0; step < 7; ++step) {
    const int buf = step & 1;
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int p = 0; p < Q; ++p) stage[buf][p][warp][lane] = (uint32_t)(p * 77 + lane);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const int t0 = n * TPI + step * 7;
      // 7 consecutive tiles are contiguous within a 128-tile block unless they straddle one
      for (int p = 0; p < Q; ++p) {
        int done = 0;
        while (done < 7) {
          const int t = t0 + done;
          int run = 128 - (t & 127);
          if (run > 7 - done) run = 7 - done;
          uint16_t* g = V + (size_t)p * PLANE + voff(t, cb * 64);
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g),
                       "r"(smem_u32(&stage[buf][p][done][0])), "r"(run * 128)
                       : "memory");
          done += run;
        }
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = (size_t)Q * PLANE * 2;
  void* V;
  cudaMalloc(&V, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms / 10 * 1e3;
    printf("%-10s %8.1f us  %7.0f GB/s  (%s)\n", name, us, (double)Q * T * CP * 2 / us * 1e-3,
           cudaGetErrorString(cudaGetLastError()));
  };
  const size_t useful = (size_t)Q * T * CP * 2;
  timeit("seq32", [&] { seq32<<<148 * 8, 256>>>((uint32_t*)V, useful / 4); });
  timeit("seq128", [&] { seq128<<<148 * 8, 256>>>((uint4*)V, useful / 16); });
  timeit("k1pat32x7", [&] { k1pat32<7><<<dim3(NB, 256), 224>>>((uint16_t*)V); });
  timeit("k1pat32x16", [&] { k1pat32<16><<<dim3(NB, 256), 512>>>((uint16_t*)V); });
  const int sm = 2 * Q * 7 * 32 * 4;
  cudaFuncSetAttribute(k1bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  timeit("k1bulk", [&] { k1bulk<<<dim3(NB, 256), 224, sm>>>((uint16_t*)V); });
  return 0;
}

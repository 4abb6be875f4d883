// Probe: TMA 2D/3D box loads of a bf16 [128][784] tensor into shared memory.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include <cuda_bf16.h>
#include "../paper_1905_05233_b200/csrc/device.cuh"
#include "../paper_1905_05233_b200/csrc/tmap.hpp"
namespace wino { void count_launch(int) {} void reset_launch_count() {} void set_last_error(const std::string&) {} }
using namespace wino;

template <int MODE>
__global__ void probe_shared(const __grid_constant__ CUtensorMap tm, int c0, int c1, int c2, unsigned bytes, float* out, int variant) {
  extern __shared__ __align__(16) uint8_t sm2[];
  uint8_t* sm = variant == 2 ? sm2 : sm2 + ((128u - (smem_u32(sm2) & 127u)) & 127u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  uint8_t* dst = sm + 128;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_proxy_async_shared();
    mbar_arrive_expect_tx(bar, bytes);
    if (MODE == 2) tma_load_2d(dst, &tm, bar, c0, c1);
    else tma_load_3d(dst, &tm, bar, c0, c1, c2);
  }
  mbar_wait(bar, 0);
  float s = 0;
  for (unsigned i = threadIdx.x; i < bytes / 2; i += blockDim.x) s += __bfloat162float(reinterpret_cast<__nv_bfloat16*>(dst)[i]);
  atomicAdd(out, s);
}

template <int MODE>
__global__ void probe(const __grid_constant__ CUtensorMap tm, int c0, int c1, int c2, unsigned bytes, float* out, int variant) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* dst = sm;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  __syncthreads();
  bool issuer = variant == 0 ? threadIdx.x == 0 : (threadIdx.x >> 5) == 0;
  if (issuer) {
    if (variant == 0 || (threadIdx.x & 31) == 0) {
      mbar_arrive_expect_tx(bar, bytes);
      if (MODE == 2) tma_load_2d(dst, &tm, bar, c0, c1);
      else tma_load_3d(dst, &tm, bar, c0, c1, c2);
    }
    __syncwarp();
  }
  mbar_wait(bar, 0);
  float s = 0;
  for (unsigned i = threadIdx.x; i < bytes / 2; i += blockDim.x) s += __bfloat162float(reinterpret_cast<__nv_bfloat16*>(dst)[i]);
  atomicAdd(out, s);
}

int main(int argc, char** argv) {
  const int want = argc > 1 ? atoi(argv[1]) : 0;
  const int NC = 128, H = 28, W = 28;
  std::vector<__nv_bfloat16> h(NC * H * W);
  for (size_t i = 0; i < h.size(); ++i) h[i] = __float2bfloat16(1.0f);
  void* d; cudaMalloc(&d, h.size() * 2); cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, 4);
  for (int variant = want; variant < want + 1 && want < 2; ++variant) {
    CUtensorMap tm;
    uint64_t dims[2] = {(uint64_t)H * W, (uint64_t)NC}, str[1] = {(uint64_t)H * W * 2};
    uint32_t box[2] = {112, 64};
    bool ok = make_map(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, false);
    cudaMemset(out, 0, 4);
    cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 2048);
    probe<2><<<1, 224, 65536 + 2048>>>(tm, -28, 0, 0, 112 * 64 * 2, out, variant);
    cudaError_t e = cudaDeviceSynchronize();
    float r = -1; cudaMemcpy(&r, out, 4, cudaMemcpyDeviceToHost);
    printf("2D variant %d map %d err %s sum %.0f (expect %d)\n", variant, ok, cudaGetErrorString(e), r, 84 * 64);
    if (e != cudaSuccess) return 1;
  }
  if (want >= 20) {
    CUtensorMap tm;
    uint64_t dims[2] = {(uint64_t)H * W, (uint64_t)NC}, str[1] = {(uint64_t)H * W * 2};
    uint32_t box[2] = {112, 64};
    bool ok = make_map(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, false);
    cudaMemset(out, 0, 4);
    cudaFuncSetAttribute(probe_shared<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 2048);
    probe_shared<2><<<1, 224, 65536 + 2048>>>(tm, 0, 0, 0, 112 * 64 * 2, out, want - 20);
    cudaError_t e = cudaDeviceSynchronize();
    float r = -1; cudaMemcpy(&r, out, 4, cudaMemcpyDeviceToHost);
    printf("shared-ptr case %d map %d err %s sum %.0f\n", want, ok, cudaGetErrorString(e), r);
  } else if (want >= 9) {
    int cx = 0, cy = 0, bx = 112;
    if (want == 10) cx = 56;
    if (want == 11) bx = 64;
    if (want == 12) cx = 700, cy = 100;
    CUtensorMap tm;
    uint64_t dims[2] = {(uint64_t)H * W, (uint64_t)NC}, str[1] = {(uint64_t)H * W * 2};
    uint32_t box[2] = {(uint32_t)bx, 64};
    bool ok = make_map(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, false);
    cudaMemset(out, 0, 4);
    cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 2048);
    probe<2><<<1, 224, 65536 + 2048>>>(tm, cx, cy, 0, bx * 64 * 2, out, 1);
    cudaError_t e = cudaDeviceSynchronize();
    float r = -1; cudaMemcpy(&r, out, 4, cudaMemcpyDeviceToHost);
    printf("2D case %d map %d err %s sum %.0f\n", want, ok, cudaGetErrorString(e), r);
  } else if (want >= 2) {
    // 2: 3D neg coords box{40,4,64}; 4: 3D coords 0 box{40,4,64}; 5: 3D coords 0 box{64,4,64};
    // 6: 3D coords 0 swizzle128 box{64,4,64}; 7: 3D coords 0 box{64,4,1}; 8: 3D swz128 box {64,4,1}
    const int H2 = 32, W2 = 64;
    int bx0 = 40, bx1 = 4, bx2 = 64, cc = -1;
    bool swz = false;
    if (want == 4) cc = 0;
    if (want == 5) cc = 0, bx0 = 64;
    if (want == 6) cc = 0, bx0 = 64, swz = true;
    if (want == 7) cc = 0, bx0 = 64, bx2 = 1;
    if (want == 8) cc = 0, bx0 = 64, bx2 = 1, swz = true;
    CUtensorMap tm;
    uint64_t dims[3] = {(uint64_t)W2, (uint64_t)H2, (uint64_t)NC / 4}, str[2] = {(uint64_t)W2 * 2, (uint64_t)H2 * W2 * 2};
    uint32_t box[3] = {(uint32_t)bx0, (uint32_t)bx1, (uint32_t)bx2};
    bool ok = make_map(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d, dims, str, box, swz);
    cudaMemset(out, 0, 4);
    cudaFuncSetAttribute(probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 2048);
    probe<3><<<1, 224, 65536 + 2048>>>(tm, cc, cc, 0, bx0 * bx1 * bx2 * 2, out, 1);
    cudaError_t e = cudaDeviceSynchronize();
    float r = -1; cudaMemcpy(&r, out, 4, cudaMemcpyDeviceToHost);
    printf("3D case %d map %d err %s sum %.0f (box elems %d)\n", want, ok, cudaGetErrorString(e), r, bx0 * bx1 * bx2);
  }
  return 0;
}

// ubench_l2bw.cu -- L2 read bandwidth on B200 by access path and SM count:
//   (1) LDG.128 from 1024 threads per SM, 8 independent loads per thread in flight;
//   (2) cp.async.bulk (TMA, 1D) with several copies per SM in flight, 1 or 2 CTAs per SM.
// Working sets of 24 / 48 / 96 MB stay in the 126 MB L2; 4 GB streams from HBM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_l2bw scripts/ubench_l2bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(1024, 1) ldg_read(const uint4* __restrict__ buf, size_t n16_per_cta, size_t wrap16,
                                                     int reps, unsigned* sink) {
  uint32_t acc = 0;
  const size_t base = (size_t)blockIdx.x * n16_per_cta;
  for (int r = 0; r < reps; ++r) {
    for (size_t i = threadIdx.x; i < n16_per_cta; i += 8 * 1024) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const size_t j = i + (size_t)u * 1024;
        v[u] = j < n16_per_cta ? __ldcg(buf + (base + j) % wrap16) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

template <int CHUNK, int NB, int PER>
__global__ void __launch_bounds__(64) bulk_read(const uint8_t* buf, size_t bytes_per_cta, size_t wrap, int reps,
                                                unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NB * CHUNK * PER);
  uint64_t* empty = full + NB;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(s32(&empty[b])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t nslot = bytes_per_cta / (CHUNK * PER) * reps;
  const size_t base = (size_t)blockIdx.x * bytes_per_cta;
  if (threadIdx.x == 0) {
    for (size_t i = 0; i < nslot; ++i) {
      const int b = i % NB;
      const uint32_t ph = (uint32_t)((i / NB) & 1);
      if (i >= NB)
        asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(
                         s32(&empty[b])), "r"(ph ^ 1));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&full[b])), "r"(CHUNK * PER));
      for (int p = 0; p < PER; ++p) {
        const size_t off = (base + ((i * PER + p) * CHUNK) % bytes_per_cta) % wrap;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         s32(sm + (b * PER + p) * CHUNK)), "l"(buf + off), "r"(CHUNK), "r"(s32(&full[b]))
                     : "memory");
      }
    }
  } else if (threadIdx.x >= 32) {
    unsigned long long acc = 0;
    for (size_t i = 0; i < nslot; ++i) {
      const int b = i % NB;
      const uint32_t ph = (uint32_t)((i / NB) & 1);
      asm volatile("{\n.reg .pred P;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W2;\n}\n" ::"r"(
                       s32(&full[b])), "r"(ph));
      acc += reinterpret_cast<const uint32_t*>(sm + b * CHUNK * PER)[threadIdx.x - 32];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&empty[b])));
    }
    if (acc == 0x123456789ull) *sink = acc;
  }
}

template <int CHUNK, int NB, int PER>
static void run_bulk(const char* name, uint8_t* buf, unsigned long long* sink, int ctas_per_sm) {
  auto k = bulk_read<CHUNK, NB, PER>;
  const int smem = NB * CHUNK * PER + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (size_t wrapMB : {48, 4096}) {
    for (int g : {16, 40, 64, 148}) {
      const int grid = g * ctas_per_sm;
      const size_t per = (size_t)4 << 20;
      const int reps = 8;
      k<<<grid, 64, smem>>>(buf, per, wrapMB << 20, 1, sink);
      cudaEventRecord(e0);
      k<<<grid, 64, smem>>>(buf, per, wrapMB << 20, reps, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)per * reps * grid;
      printf("%-28s x%d CTA/SM  ws %5zu MB  SMs %3d : %8.1f GB/s  %6.1f GB/s/SM\n", name, ctas_per_sm, wrapMB, g,
             bytes / ms / 1e6, bytes / ms / 1e6 / g);
    }
  }
}

int main() {
  const size_t big = (size_t)4 << 30;
  uint8_t* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (size_t wrapMB : {24, 48, 96, 4096}) {
    for (int g : {16, 40, 64, 96, 148}) {
      const size_t per = (size_t)8 << 20;   // bytes per CTA per rep
      const int reps = 8;
      ldg_read<<<g, 1024>>>((const uint4*)buf, per / 16, (wrapMB << 20) / 16, 1, (unsigned*)sink);
      cudaEventRecord(e0);
      ldg_read<<<g, 1024>>>((const uint4*)buf, per / 16, (wrapMB << 20) / 16, reps, (unsigned*)sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)per * reps * g;
      printf("%-28s          ws %5zu MB  SMs %3d : %8.1f GB/s  %6.1f GB/s/SM\n", "ldg.cg 1024 thr x 8 x 16B", wrapMB,
             g, bytes / ms / 1e6, bytes / ms / 1e6 / g);
    }
  }
  run_bulk<16384, 12, 1>("bulk 16K x12", buf, sink, 1);
  run_bulk<4096, 8, 4>("bulk 4x4K x8", buf, sink, 1);
  run_bulk<32768, 6, 1>("bulk 32K x6", buf, sink, 1);
  run_bulk<16384, 6, 1>("bulk 16K x6", buf, sink, 2);
  run_bulk<8192, 6, 2>("bulk 2x8K x6", buf, sink, 2);
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

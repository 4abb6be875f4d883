// ubench_l2tma.cu -- TMA (cp.async.bulk) read bandwidth from L2 vs HBM as a
// function of the number of SMs reading: sizes the split of a persistent kernel
// into tensor-core CTAs and CTAs that stream an L2-resident intermediate.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_l2tma scripts/ubench_l2tma.cu
//   /tmp/ubench_l2tma
//
// Each CTA (one per SM, 1 producer thread) streams CHUNK-byte bulk copies of its
// share of a buffer into a ring of NB shared-memory slots (mbarrier completion);
// the consumer warp touches one word per chunk so the copies are not dead.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int CHUNK, int NB>
__global__ void __launch_bounds__(64, 1) l2read(const uint8_t* buf, size_t bytes_per_cta, size_t wrap, int reps,
                                                 unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NB * CHUNK);
  uint64_t* empty = full + NB;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(s32(&empty[b])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t nchunks = bytes_per_cta / CHUNK * reps;
  const size_t base = (size_t)blockIdx.x * bytes_per_cta;
  if (threadIdx.x == 0) {
    for (size_t i = 0; i < nchunks; ++i) {
      const int b = i % NB;
      const uint32_t ph = (uint32_t)((i / NB) & 1);
      if (i >= NB) {
        asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(
                         s32(&empty[b])), "r"(ph ^ 1));
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&full[b])), "r"(CHUNK));
      const size_t off = (base + (i * CHUNK) % bytes_per_cta) % wrap;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       s32(sm + b * CHUNK)), "l"(buf + off), "r"(CHUNK), "r"(s32(&full[b]))
                   : "memory");
    }
  } else if (threadIdx.x >= 32) {
    unsigned long long acc = 0;
    for (size_t i = 0; i < nchunks; ++i) {
      const int b = i % NB;
      const uint32_t ph = (uint32_t)((i / NB) & 1);
      asm volatile("{\n.reg .pred P;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W2;\n}\n" ::"r"(
                       s32(&full[b])), "r"(ph));
      acc += reinterpret_cast<const uint32_t*>(sm + b * CHUNK)[threadIdx.x - 32];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&empty[b])));
    }
    if (acc == 0x123456789ull) *sink = acc;
  }
}

int main() {
  const size_t big = (size_t)4 << 30;
  uint8_t* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  constexpr int CHUNK = 16384, NB = 12;
  auto k = l2read<CHUNK, NB>;
  const int smem = NB * CHUNK + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sms[] = {8, 16, 32, 40, 48, 64, 96, 148};
  for (size_t wrapMB : {24, 48, 96, 4096}) {
    const size_t wrap = wrapMB << 20;
    for (int g : sms) {
      // each CTA reads 64 MB total (wrapped into the working set)
      const size_t per = (size_t)4 << 20;
      const int reps = 16;
      k<<<g, 64, smem>>>(buf, per, wrap, 1, sink);
      cudaEventRecord(e0);
      k<<<g, 64, smem>>>(buf, per, wrap, reps, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)per * reps * g;
      printf("working set %5zu MB  SMs %3d : %8.1f GB/s total  %6.1f GB/s per SM\n", wrapMB, g, bytes / ms / 1e6,
             bytes / ms / 1e6 / g);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}

// Microbenchmark: fp32 FMA issue rates on sm_100a (register, immediate,
// constant-bank operands; packed FFMA2).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITERS = 4096, CH = 8;

__global__ void k_reg(float* out, float b, float c) {
  float a[CH];
  float bb = b + threadIdx.x * 1e-9f, cc = c - threadIdx.x * 1e-9f;
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(bb), "f"(cc));
  float s = 0; for (int i = 0; i < CH; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imm(float* out, float b, float c) {
  float a[CH];
  float cc = c - threadIdx.x * 1e-9f;
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFF0, %1;" : "+f"(a[i]) : "f"(cc));
  float s = 0; for (int i = 0; i < CH; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_cbank(float* out, const __grid_constant__ float b, float c) {
  float a[CH];
  float cc = c - threadIdx.x * 1e-9f;
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = __fmaf_rn(a[i], b, cc);
  float s = 0; for (int i = 0; i < CH; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float b, float c) {
  unsigned long long a[CH];
  float bb = b + threadIdx.x * 1e-9f, cc = c - threadIdx.x * 1e-9f;
  unsigned long long B, C;
  asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(bb), "f"(bb));
  asm("mov.b64 %0, {%1, %2};" : "=l"(C) : "f"(cc), "f"(cc));
  for (int i = 0; i < CH; ++i) { float x = threadIdx.x + i; asm("mov.b64 %0, {%1, %2};" : "=l"(a[i]) : "f"(x), "f"(x)); }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(B), "l"(C));
  float s = 0;
  for (int i = 0; i < CH; ++i) { float x, y; asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i])); s += x + y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fadd_reg(float* out, float b, float c) {
  float a[CH];
  float bb = b + threadIdx.x * 1e-9f;
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(bb));
  float s = 0; for (int i = 0; i < CH; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main2();
template <typename F>
void run(const char* name, F kern, int lanes_per_op) {
  float* out;
  cudaMalloc(&out, 148 * 16 * 256 * 4);
  int sms = 148, bpsm = 8, thr = 256;
  kern<<<sms * bpsm, thr>>>(out, 0.999f, 0.001f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<sms * bpsm, thr>>>(out, 0.999f, 0.001f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double winst = 5.0 * sms * bpsm * thr / 32.0 * ITERS * CH;
  double per_sm_clk = winst / sms / (ms * 1e-3 * 1.965e9 / 5 * 5);
  printf("%-10s %.3f ms  warp-inst/SM/clk(@1965MHz) %.3f  lane-ops/SM/clk %.1f\n", name, ms / 5,
         winst / sms / (ms * 1e-3 * 1.965e9), winst * 32 * lanes_per_op / sms / (ms * 1e-3 * 1.965e9));
  cudaFree(out);
}
int main() {
  run("ffma_reg", k_reg, 1);
  run("ffma_imm", k_imm, 1);
  run("ffma_cbank", k_cbank, 1);
  run("ffma2_reg", k_ffma2, 2);
  run("fadd_reg", k_fadd_reg, 1);
  return main2();
}

// ---- transform-like FFMA2 patterns (appended)
struct Coef { float c[64]; };
__global__ void k_ffma2_ur(float* out, const __grid_constant__ Coef cf) {
  float2 acc[16];
  float2 d[6];
  for (int i = 0; i < 6; ++i) d[i] = make_float2(threadIdx.x + i, threadIdx.x - i);
  for (int i = 0; i < 16; ++i) acc[i] = make_float2(0.f, 0.f);
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = __ffma2_rn(d[q], make_float2(cf.c[i * 3 + q], cf.c[i * 3 + q]), acc[i]);
#pragma unroll
    for (int q = 0; q < 6; ++q) d[q].x += 1e-7f;
  }
  float s = 0; for (int i = 0; i < 16; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma_ur(float* out, const __grid_constant__ Coef cf) {
  float acc[16];
  float d[6];
  for (int i = 0; i < 6; ++i) d[i] = threadIdx.x + i;
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = __fmaf_rn(d[q], cf.c[i * 3 + q], acc[i]);
#pragma unroll
    for (int q = 0; q < 6; ++q) d[q] += 1e-7f;
  }
  float s = 0; for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main2() {
  Coef cf;
  for (int i = 0; i < 64; ++i) cf.c[i] = 0.5f + i * 0.01f;
  float* out;
  cudaMalloc(&out, 148 * 16 * 256 * 4);
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0), cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (v == 0) k_ffma2_ur<<<148 * 8, 256>>>(out, cf); else k_ffma_ur<<<148 * 8, 256>>>(out, cf);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double winst = 148.0 * 8 * 256 / 32 * (ITERS / 8) * 96;
      double lanes = winst * 32 * (v == 0 ? 2 : 1);
      if (rep) printf("%s: %.3f ms  warp-inst/SM/clk %.3f  fma-lanes/SM/clk %.1f\n", v == 0 ? "ffma2_ur(transform)" : "ffma_ur(transform)",
                      ms, winst / 148 / (ms * 1e-3 * 1.965e9), lanes / 148 / (ms * 1e-3 * 1.965e9));
    }
  }
  return 0;
}

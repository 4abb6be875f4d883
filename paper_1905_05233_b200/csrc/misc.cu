// misc.cu -- K5 batched 1D tiles (BASELINE cfg 2), K6 error statistics, the
// fp64 direct-convolution reference of the metric path, launch accounting.
#include <cstring>
#include <string>
#include <type_traits>

#include "device.cuh"
#include "geometry.hpp"

namespace wino {

static thread_local int g_launches = 0;
void count_launch(int n) { g_launches += n; }
void reset_launch_count() { g_launches = 0; }

// Library-owned streams / events and the SM count, per (host thread, device):
// a thread that drives several GPUs gets each device's own objects.
DevState* dev_state() {
  constexpr int kMaxDev = 64;
  static thread_local DevState st[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) {
    set_last_error("dev_state: no current CUDA device");
    return nullptr;
  }
  DevState& d = st[dev];
  if (!d.ready) {
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&d.side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&d.io_in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&d.io_out, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d.fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d.join, cudaEventDisableTiming);
    for (int a = 0; a < 2 && e == cudaSuccess; ++a)
      for (int j = 0; j < 64 && e == cudaSuccess; ++j) e = cudaEventCreateWithFlags(&d.io_ev[a][j], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) {
      set_last_error(std::string("dev_state: ") + cudaGetErrorString(e));
      return nullptr;
    }
    if (d.sms <= 0) d.sms = 148;
    d.ready = true;
  }
  return &d;
}

int num_sms() {
  DevState* d = dev_state();
  return d ? d->sms : 148;
}

// ------------------------------------------------------------------ K5: 1D tiles
// y = A^T [(G h) (.) (B^T x)] per tile.  PAPER=true: every
// scalar multiply/add in fp32 without contraction (__fmul_rn / __fadd_rn), cast
// to the dtype after each op, ascending index from the first product, matrix
// entries cast once.  PAPER=false: fp32 internally, u, v, y rounded.
// A thread owns two adjacent tiles: their x / h / y runs are contiguous, so they
// move with 4- or 8-byte vector accesses, and every operation is a packed fp32x2
// one (FMUL2 / FADD2 / FFMA2, two-element conversions) -- per element the same
// IEEE operations in the same order, so results are unchanged bit for bit.
template <typename TT>
__device__ __forceinline__ void load_run2(const TT* __restrict__ p, int n2, float* out, bool vec) {
  // out[0 .. 2 * n2) = p[0 .. 2 * n2) as fp32; vec: p is 4-byte (16-bit) / 8-byte (fp32) aligned
  if (vec) {
    if constexpr (sizeof(TT) == 2) {
      const uint32_t* q = reinterpret_cast<const uint32_t*>(p);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (k >= n2) break;
        const uint32_t wv = __ldg(q + k);
        TT lo, hi;
        const uint16_t l16 = (uint16_t)(wv & 0xFFFFu), h16 = (uint16_t)(wv >> 16);
        memcpy(&lo, &l16, 2);
        memcpy(&hi, &h16, 2);
        out[2 * k] = DType<std::is_same<TT, __half>::value ? WINO_F16 : WINO_BF16>::load(&lo);
        out[2 * k + 1] = DType<std::is_same<TT, __half>::value ? WINO_F16 : WINO_BF16>::load(&hi);
      }
    } else {
      const float2* q = reinterpret_cast<const float2*>(p);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (k >= n2) break;
        const float2 v = __ldg(q + k);
        out[2 * k] = v.x, out[2 * k + 1] = v.y;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k >= 2 * n2) break;
      if constexpr (sizeof(TT) == 4) out[k] = p[k];
      else out[k] = DType<std::is_same<TT, __half>::value ? WINO_F16 : WINO_BF16>::load(p + k);
    }
  }
}

template <int DT, int M, int MU, bool PAPER, bool TRUNC>
__global__ void __launch_bounds__(128) conv1d_tiles_kernel(const typename DType<DT>::T* __restrict__ x,
                                                           const typename DType<DT>::T* __restrict__ h, int64_t T,
                                                           const __grid_constant__ XformParams xp,
                                                           typename DType<DT>::T* __restrict__ y, int vec) {
  using Tr = DType<DT>;
  using TT = typename Tr::T;
  constexpr int NX = M + 2;
  const RdMode<DT> R{TRUNC};   // compile-time mode: no per-op branch
  const int64_t t = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (t >= T) return;
  const bool two = t + 1 < T;
  float xr[2 * NX], hr[6];
  if (two) {
    load_run2<TT>(x + t * NX, NX, xr, vec != 0);
    load_run2<TT>(h + t * 3, 3, hr, vec != 0);
  } else {
#pragma unroll
    for (int j = 0; j < NX; ++j) xr[j] = Tr::load(x + t * NX + j), xr[NX + j] = 0.f;
#pragma unroll
    for (int j = 0; j < 3; ++j) hr[j] = Tr::load(h + t * 3 + j), hr[3 + j] = 0.f;
  }
  float2 hv[3], xv[NX];
#pragma unroll
  for (int j = 0; j < 3; ++j) hv[j] = make_float2(hr[j], hr[3 + j]);
#pragma unroll
  for (int j = 0; j < NX; ++j) xv[j] = make_float2(xr[j], xr[NX + j]);
  auto bc = [](float c) { return make_float2(c, c); };
  // paper-mode products and sums: packed FMUL2 / FADD2 in 16-bit (a rounding sits
  // between every pair); in fp32 nothing separates them, and the packed pair may
  // be contracted into FFMA2, so fp32 keeps the scalar non-contracting intrinsics
  auto mul = [](float2 a, float2 b) {
    if constexpr (DT == WINO_F32) return make_float2(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y));
    else return __fmul2_rn(a, b);
  };
  auto add = [](float2 a, float2 b) {
    if constexpr (DT == WINO_F32) return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
    else return __fadd2_rn(a, b);
  };
  float2 p[MU];
#pragma unroll
  for (int i = 0; i < MU; ++i) {
    float2 u, v;
    if constexpr (PAPER) {
      u = R.rd2(mul(bc(R.rd(xp.G[i][0])), hv[0]));
#pragma unroll
      for (int j = 1; j < 3; ++j) u = R.rd2(add(u, R.rd2(mul(bc(R.rd(xp.G[i][j])), hv[j]))));
      v = R.rd2(mul(bc(R.rd(xp.BT[i][0])), xv[0]));
#pragma unroll
      for (int j = 1; j < NX; ++j) v = R.rd2(add(v, R.rd2(mul(bc(R.rd(xp.BT[i][j])), xv[j]))));
      p[i] = R.rd2(mul(u, v));
    } else {
      u = make_float2(0.f, 0.f), v = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 3; ++j) u = __ffma2_rn(bc(xp.G[i][j]), hv[j], u);
#pragma unroll
      for (int j = 0; j < NX; ++j) v = __ffma2_rn(bc(xp.BT[i][j]), xv[j], v);
      p[i] = __fmul2_rn(R.rd2(u), R.rd2(v));
    }
  }
  float yo[2][M];
#pragma unroll
  for (int q = 0; q < M; ++q) {
    float2 acc;
    if constexpr (PAPER) {
      acc = R.rd2(mul(bc(R.rd(xp.AT[q][0])), p[0]));
#pragma unroll
      for (int i = 1; i < MU; ++i) acc = R.rd2(add(acc, R.rd2(mul(bc(R.rd(xp.AT[q][i])), p[i]))));
    } else {
      acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < MU; ++i) acc = __ffma2_rn(bc(xp.AT[q][i]), p[i], acc);
    }
    yo[0][q] = acc.x, yo[1][q] = acc.y;
  }
  if (two && vec) {
    if constexpr (sizeof(TT) == 2) {
      uint32_t* q = reinterpret_cast<uint32_t*>(y + t * M);
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const float a0 = yo[(2 * k) / M][(2 * k) % M];
        const float a1 = yo[(2 * k + 1) / M][(2 * k + 1) % M];
        TT e0 = R.cvt(a0), e1 = R.cvt(a1);
        uint16_t b0, b1;
        memcpy(&b0, &e0, 2);
        memcpy(&b1, &e1, 2);
        q[k] = (uint32_t)b0 | ((uint32_t)b1 << 16);
      }
    } else {
      float2* q = reinterpret_cast<float2*>(y + t * M);
#pragma unroll
      for (int k = 0; k < M; ++k)
        q[k] = make_float2(yo[(2 * k) / M][(2 * k) % M], yo[(2 * k + 1) / M][(2 * k + 1) % M]);
    }
  } else {
#pragma unroll
    for (int q = 0; q < M; ++q) y[t * M + q] = R.cvt(yo[0][q]);
    if (two)
#pragma unroll
      for (int q = 0; q < M; ++q) y[(t + 1) * M + q] = R.cvt(yo[1][q]);
  }
}

struct C1Args {
  const void *x, *h;
  int64_t T;
  const XformParams* xp;
  void* y;
  cudaStream_t st;
  int trunc;
};
template <int DT, int M, int MU, bool P>
static void launch_c1(const C1Args& a) {
  using Tr = DType<DT>;
  // vector accesses when x, h and y are aligned for them (each thread's runs start
  // at multiples of 2 tiles: 4-byte aligned in 16-bit, 8-byte in fp32)
  const uintptr_t al = sizeof(typename Tr::T) == 2 ? 4 : 8;
  const int vec = (reinterpret_cast<uintptr_t>(a.x) % al == 0 && reinterpret_cast<uintptr_t>(a.h) % al == 0 &&
                   reinterpret_cast<uintptr_t>(a.y) % al == 0) ? 1 : 0;
  const int64_t thr = (a.T + 1) / 2;
  const dim3 grid((unsigned)((thr + 127) / 128));
  if constexpr (DT == WINO_BF16) {
    if (a.trunc) {
      conv1d_tiles_kernel<DT, M, MU, P, true><<<grid, 128, 0, a.st>>>(
          (const typename Tr::T*)a.x, (const typename Tr::T*)a.h, a.T, *a.xp, (typename Tr::T*)a.y, vec);
      return;
    }
  }
  conv1d_tiles_kernel<DT, M, MU, P, false><<<grid, 128, 0, a.st>>>(
      (const typename Tr::T*)a.x, (const typename Tr::T*)a.h, a.T, *a.xp, (typename Tr::T*)a.y, vec);
}
using C1Fn = void (*)(const C1Args&);
#define C1ROW(DT, M, P) {&launch_c1<DT, M, M + 2, P>, &launch_c1<DT, M, M + 3, P>, &launch_c1<DT, M, M + 4, P>}
#define C1TAB(DT, P) {C1ROW(DT, 2, P), C1ROW(DT, 3, P), C1ROW(DT, 4, P), C1ROW(DT, 5, P), C1ROW(DT, 6, P), C1ROW(DT, 7, P), C1ROW(DT, 8, P)}
static const C1Fn kC1[2][3][7][3] = {
    {C1TAB(WINO_F32, false), C1TAB(WINO_F16, false), C1TAB(WINO_BF16, false)},
    {C1TAB(WINO_F32, true), C1TAB(WINO_F16, true), C1TAB(WINO_BF16, true)}};

// ------------------------------------------------------------------ K7: 2D tiles, paper mode
// Multi-channel 2D Winograd of independent tile samples in PAPER mode,
// the operation order of the oracle's paper_conv2d_tiles: for each channel c
//   U = G g G^T  (rows then columns),  V = B^T d B  (rows then columns),
//   P_c = rd(U (.) V),
// every product and partial sum computed in fp32 without contraction and cast to
// the dtype, matrix entries cast once; then the channel sum in the Winograd
// domain and Y = A^T M A (rows then columns), per op.  Channel sum (P:611
// boosters): csum 0 sequential (ascending c) / 1 pairwise (tree: the largest
// power of two below n on the left); acc 0 every partial sum cast to the dtype /
// 1 fp32 accumulation cast once (mixed precision).  Block = one sample, thread =
// one Winograd point (i, j); the pairwise tree is a binary counter of partial
// sums (an element at level l merges with the stored partial of level l).
template <int DT, int M, int MU>
__global__ void __launch_bounds__(256) conv2d_tiles_paper_kernel(const typename DType<DT>::T* __restrict__ d,
                                                                 const typename DType<DT>::T* __restrict__ g, int C,
                                                                 int64_t S, const __grid_constant__ XformParams xp,
                                                                 int csum, int acc32, int trunc,
                                                                 typename DType<DT>::T* __restrict__ y) {
  using Tr = DType<DT>;
  constexpr int NX = M + 2;
  const RdMode<DT> R{trunc != 0};
  __shared__ float sd[NX * NX], sg[9], sm[MU * MU];
  const int64_t s = blockIdx.x;
  const int pt = threadIdx.x, i = pt / MU, j = pt % MU;
  const bool live = pt < MU * MU;
  auto rdadd = [&](float a, float b) { return acc32 ? __fadd_rn(a, b) : R.rd(__fadd_rn(a, b)); };
  float stack[24];
  float msum = 0.f;
  for (int c = 0; c < C; ++c) {
    __syncthreads();
    const size_t base = ((size_t)c * S + s);
    for (int e = threadIdx.x; e < NX * NX; e += blockDim.x) sd[e] = Tr::load(d + base * NX * NX + e);
    for (int e = threadIdx.x; e < 9; e += blockDim.x) sg[e] = Tr::load(g + base * 9 + e);
    __syncthreads();
    if (!live) continue;
    // U[i][j] = sum_b G[j][b] U1[i][b],  U1[i][b] = sum_a G[i][a] g[a][b]
    float U1[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      float t = R.rd(__fmul_rn(R.rd(xp.G[i][0]), sg[0 * 3 + b]));
#pragma unroll
      for (int a = 1; a < 3; ++a) t = R.rd(__fadd_rn(t, R.rd(__fmul_rn(R.rd(xp.G[i][a]), sg[a * 3 + b]))));
      U1[b] = t;
    }
    float u = R.rd(__fmul_rn(R.rd(xp.G[j][0]), U1[0]));
#pragma unroll
    for (int b = 1; b < 3; ++b) u = R.rd(__fadd_rn(u, R.rd(__fmul_rn(R.rd(xp.G[j][b]), U1[b]))));
    // V[i][j] = sum_b BT[j][b] V1[i][b],  V1[i][b] = sum_a BT[i][a] d[a][b]
    float v = 0.f;
#pragma unroll
    for (int b = 0; b < NX; ++b) {
      float t = R.rd(__fmul_rn(R.rd(xp.BT[i][0]), sd[0 * NX + b]));
#pragma unroll
      for (int a = 1; a < NX; ++a) t = R.rd(__fadd_rn(t, R.rd(__fmul_rn(R.rd(xp.BT[i][a]), sd[a * NX + b]))));
      const float term = R.rd(__fmul_rn(R.rd(xp.BT[j][b]), t));
      v = b == 0 ? term : R.rd(__fadd_rn(v, term));
    }
    const float pc = R.rd(__fmul_rn(u, v));
    if (csum == 0) {
      msum = c == 0 ? pc : rdadd(msum, pc);
    } else {
      float val = pc;
      int cnt = c, lvl = 0;
      while (cnt & 1) val = rdadd(stack[lvl++], val), cnt >>= 1;
      stack[lvl] = val;
    }
  }
  if (live) {
    if (csum == 1) {
      // combine the stored partials from the lowest level up: sum = partial(high) + sum
      bool first = true;
      for (int lvl = 0; lvl < 24; ++lvl)
        if ((C >> lvl) & 1) {
          msum = first ? stack[lvl] : rdadd(stack[lvl], msum);
          first = false;
        }
    }
    sm[pt] = acc32 ? R.rd(msum) : msum;
  }
  __syncthreads();
  if (pt < M * M) {
    const int p = pt / M, q = pt % M;
    // Y[p][q] = sum_jj AT[q][jj] Y1[p][jj],  Y1[p][jj] = sum_ii AT[p][ii] M[ii][jj]
    float out = 0.f;
#pragma unroll
    for (int jj = 0; jj < MU; ++jj) {
      float t = R.rd(__fmul_rn(R.rd(xp.AT[p][0]), sm[0 * MU + jj]));
#pragma unroll
      for (int ii = 1; ii < MU; ++ii) t = R.rd(__fadd_rn(t, R.rd(__fmul_rn(R.rd(xp.AT[p][ii]), sm[ii * MU + jj]))));
      const float term = R.rd(__fmul_rn(R.rd(xp.AT[q][jj]), t));
      out = jj == 0 ? term : R.rd(__fadd_rn(out, term));
    }
    y[s * M * M + pt] = R.cvt(out);
  }
}

struct C2Args {
  const void *d, *g;
  int C;
  int64_t S;
  const XformParams* xp;
  int csum, acc, trunc;
  void* y;
  cudaStream_t st;
};
template <int DT, int M, int MU>
static void launch_c2(const C2Args& a) {
  using TT = typename DType<DT>::T;
  const int thr = (MU * MU + 31) / 32 * 32;
  conv2d_tiles_paper_kernel<DT, M, MU><<<(unsigned)a.S, thr, 0, a.st>>>((const TT*)a.d, (const TT*)a.g, a.C, a.S,
                                                                       *a.xp, a.csum, a.acc, a.trunc, (TT*)a.y);
}
using C2Fn = void (*)(const C2Args&);
#define C2ROW(DT, M) {&launch_c2<DT, M, M + 2>, &launch_c2<DT, M, M + 3>, &launch_c2<DT, M, M + 4>}
#define C2TAB(DT) {C2ROW(DT, 2), C2ROW(DT, 3), C2ROW(DT, 4), C2ROW(DT, 5), C2ROW(DT, 6), C2ROW(DT, 7), C2ROW(DT, 8)}
static const C2Fn kC2[3][7][3] = {C2TAB(WINO_F32), C2TAB(WINO_F16), C2TAB(WINO_BF16)};

// ------------------------------------------------------------------ K6: error statistics
constexpr int kStatThreads = 256;

__device__ __forceinline__ void stat_combine(double* a, const double* b) {
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = (i == 4) ? fmax(a[i], b[i]) : a[i] + b[i];
}

// fixed-order tree reduction of 8 doubles per thread over the block
__device__ void block_reduce8(double* v, double (*sh)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) sh[threadIdx.x][i] = v[i];
  __syncthreads();
  for (int s = kStatThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) stat_combine(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
}

template <int DT>
__global__ void __launch_bounds__(kStatThreads) stats_tiles_kernel(const typename DType<DT>::T* __restrict__ y,
                                                                   const double* __restrict__ yr, int N, int K,
                                                                   int Ho, int Wo, int m, int th, int tw,
                                                                   double* __restrict__ part) {
  using Tr = DType<DT>;
  __shared__ double sh[kStatThreads][8];
  const int64_t ntiles = (int64_t)N * K * th * tw;
  const int64_t tile = (int64_t)blockIdx.x * kStatThreads + threadIdx.x;
  double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (tile < ntiles) {
    const int tj = (int)(tile % tw);
    int64_t r = tile / tw;
    const int ti = (int)(r % th);
    const int64_t nk = r / th;
    double sad = 0, sar = 0, e2 = 0, r2 = 0, nf = 0, ne = 0;
    for (int p = 0; p < m; ++p) {
      const int i = ti * m + p;
      if (i >= Ho) break;
      for (int q = 0; q < m; ++q) {
        const int j = tj * m + q;
        if (j >= Wo) break;
        const size_t off = ((size_t)nk * Ho + i) * Wo + j;
        const double yy = (double)Tr::load(y + off), rr = yr[off];
        double d;
        if (isfinite(yy)) {
          d = fabs(yy - rr);
        } else {
          d = INFINITY;
          nf += 1;
        }
        sad += d;
        sar += fabs(rr);
        e2 += d * d;
        r2 += rr * rr;
        ne += 1;
      }
    }
    const double e = sqrt(e2), rn = sqrt(r2);
    const double rel = e == 0 ? 0.0 : (rn == 0 ? INFINITY : e / rn);
    v[0] = sad, v[1] = sar, v[2] = rel, v[3] = e, v[4] = rel, v[5] = nf, v[6] = 1, v[7] = ne;
  }
  block_reduce8(v, sh);
  if (threadIdx.x == 0)
    for (int i = 0; i < 8; ++i) part[(size_t)blockIdx.x * 8 + i] = sh[0][i];
}

__global__ void __launch_bounds__(kStatThreads) stats_final_kernel(const double* __restrict__ part, int nparts,
                                                                   double* __restrict__ out) {
  __shared__ double sh[kStatThreads][8];
  double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int b = threadIdx.x; b < nparts; b += kStatThreads) stat_combine(v, part + (size_t)b * 8);
  block_reduce8(v, sh);
  if (threadIdx.x == 0)
    for (int i = 0; i < 8; ++i) out[i] = sh[0][i];
}

// ------------------------------------------------------------------ fp64 direct reference
// y_ref[n,k,i,j] = sum_{c,p,q} w[k,c,p,q] x[n,c,i+p-pad,j+q-pad]  (valid
// cross-correlation, zero padding).  CTA = 32 output columns x
// 32 output channels of one (n, i) row; x rows and weights staged per channel.
template <int DT>
__global__ void __launch_bounds__(256) direct_f64_kernel(const typename DType<DT>::T* __restrict__ x,
                                                         const typename DType<DT>::T* __restrict__ w, int C, int H,
                                                         int W, int K, int pad, int Ho, int Wo,
                                                         double* __restrict__ y) {
  using Tr = DType<DT>;
  __shared__ double xs[3][34];
  __shared__ double wsm[32][9];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 groups of 4 channels
  const int j0 = blockIdx.x * 32;
  const int n = blockIdx.y / Ho, i = blockIdx.y % Ho;
  const int k0 = blockIdx.z * 32;
  double acc[4] = {0, 0, 0, 0};
  for (int c = 0; c < C; ++c) {
    for (int e = threadIdx.x; e < 3 * 34; e += 256) {
      const int p = e / 34, q = e % 34;
      const int r = i + p - pad, col = j0 + q - pad;
      xs[p][q] = (r >= 0 && r < H && col >= 0 && col < W) ? (double)Tr::load(x + (((size_t)n * C + c) * H + r) * W + col) : 0.0;
    }
    for (int e = threadIdx.x; e < 32 * 9; e += 256) {
      const int kk = e / 9, pq = e % 9;
      wsm[kk][pq] = (k0 + kk < K) ? (double)Tr::load(w + ((size_t)(k0 + kk) * C + c) * 9 + pq) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int q = 0; q < 3; ++q) acc[kk] = fma(wsm[ty * 4 + kk][p * 3 + q], xs[p][tx + q], acc[kk]);
    __syncthreads();
  }
  const int j = j0 + tx;
  if (j < Wo)
    for (int kk = 0; kk < 4; ++kk) {
      const int k = k0 + ty * 4 + kk;
      if (k < K) y[(((size_t)n * K + k) * Ho + i) * Wo + j] = acc[kk];
    }
}

}  // namespace wino

using namespace wino;

extern "C" {

int32_t wino_last_launch_count(void) { return g_launches; }

wino_status wino_conv1d_tiles(const void* x, const void* h, int64_t T, const wino_algo* al, wino_dtype dt,
                              int per_op_rounding, void* y, void* stream) {
  reset_launch_count();
  if (!al || !x || !h || !y || T < 0) return set_last_error("bad argument"), WINO_E_ARG;
  if (dt != WINO_F32 && dt != WINO_F16 && dt != WINO_BF16) return set_last_error("bad dtype"), WINO_E_ARG;
  if (al->lowering != WINO_LOWER_SUBSOLVER) return set_last_error("1D tiles: SUBSOLVER algos only"), WINO_E_UNSUPPORTED;
  const int dm = al->mu - al->m - 2;
  if (dm < 0 || dm > 2) return set_last_error("1D tiles: mu must be in [m+2, m+4]"), WINO_E_UNSUPPORTED;
  if (al->m > 8) return set_last_error("1D tiles: m <= 8 only"), WINO_E_UNSUPPORTED;
  if (T == 0) return WINO_OK;
  if (per_op_rounding & ~3) return set_last_error("1D tiles: per_op_rounding flags are bits 0 and 1"), WINO_E_ARG;
  C1Args a{x, h, T, &al->xp, y, reinterpret_cast<cudaStream_t>(stream), (per_op_rounding & 2) ? 1 : 0};
  kC1[(per_op_rounding & 1) ? 1 : 0][dt][al->m - 2][dm](a);
  WINO_LAUNCH_CHECK();
  return WINO_OK;
}

wino_status wino_conv2d_tiles_paper(const void* d, const void* g, int C, int64_t S, const wino_algo* al,
                                   wino_dtype dt, int csum, int acc, int bf16_trunc, void* y, void* stream) {
  reset_launch_count();
  if (!al || !d || !g || !y || C <= 0 || S < 0 || (csum != 0 && csum != 1) || (acc != 0 && acc != 1) ||
      (bf16_trunc != 0 && bf16_trunc != 1))
    return set_last_error("bad argument"), WINO_E_ARG;
  if (dt != WINO_F32 && dt != WINO_F16 && dt != WINO_BF16) return set_last_error("bad dtype"), WINO_E_ARG;
  if (al->lowering != WINO_LOWER_SUBSOLVER) return set_last_error("2D paper tiles: SUBSOLVER algos only"), WINO_E_UNSUPPORTED;
  const int dm = al->mu - al->m - 2;
  if (dm < 0 || dm > 2 || al->m > 8) return set_last_error("2D paper tiles: m <= 8, mu in [m+2, m+4]"), WINO_E_UNSUPPORTED;
  if (S > 0x7fffffff) return set_last_error("2D paper tiles: S < 2^31"), WINO_E_UNSUPPORTED;
  if (S == 0) return WINO_OK;
  C2Args a{d, g, C, S, &al->xp, csum, acc, bf16_trunc, y, reinterpret_cast<cudaStream_t>(stream)};
  kC2[dt][al->m - 2][dm](a);
  WINO_LAUNCH_CHECK();
  return WINO_OK;
}

size_t wino_error_stats_scratch(int N, int K, int Ho, int Wo, int m) {
  if (N <= 0 || K <= 0 || Ho <= 0 || Wo <= 0 || m <= 0) return 0;
  int64_t tiles = (int64_t)N * K * ((Ho + m - 1) / m) * ((Wo + m - 1) / m);
  return (size_t)((tiles + kStatThreads - 1) / kStatThreads) * 8 * sizeof(double);
}

wino_status wino_error_stats(const void* y, wino_dtype dt, const double* y_ref, int N, int K, int Ho, int Wo, int m,
                             double* stats, void* scratch, void* stream) {
  reset_launch_count();
  if (!y || !y_ref || !stats || !scratch || N <= 0 || K <= 0 || Ho <= 0 || Wo <= 0 || m <= 0)
    return set_last_error("bad argument"), WINO_E_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int th = (Ho + m - 1) / m, tw = (Wo + m - 1) / m;
  const int64_t tiles = (int64_t)N * K * th * tw;
  const int nb = (int)((tiles + kStatThreads - 1) / kStatThreads);
  double* part = static_cast<double*>(scratch);
  switch (dt) {
    case WINO_F32:
      stats_tiles_kernel<WINO_F32><<<nb, kStatThreads, 0, st>>>((const float*)y, y_ref, N, K, Ho, Wo, m, th, tw, part);
      break;
    case WINO_F16:
      stats_tiles_kernel<WINO_F16><<<nb, kStatThreads, 0, st>>>((const __half*)y, y_ref, N, K, Ho, Wo, m, th, tw, part);
      break;
    case WINO_BF16:
      stats_tiles_kernel<WINO_BF16><<<nb, kStatThreads, 0, st>>>((const __nv_bfloat16*)y, y_ref, N, K, Ho, Wo, m,
                                                                 th, tw, part);
      break;
    default:
      return set_last_error("bad dtype"), WINO_E_ARG;
  }
  WINO_LAUNCH_CHECK();
  stats_final_kernel<<<1, kStatThreads, 0, st>>>(part, nb, stats);
  WINO_LAUNCH_CHECK();
  return WINO_OK;
}

wino_status wino_direct_conv2d_f64(const void* x, const void* w, int N, int C, int H, int W, int K, int pad,
                                   wino_dtype dt, double* y, void* stream) {
  reset_launch_count();
  if (!x || !w || !y || N <= 0 || C <= 0 || K <= 0 || (pad != 0 && pad != 1)) return set_last_error("bad argument"), WINO_E_ARG;
  const int Ho = H + 2 * pad - 2, Wo = W + 2 * pad - 2;
  if (Ho <= 0 || Wo <= 0) return set_last_error("bad geometry"), WINO_E_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  dim3 grid((Wo + 31) / 32, N * Ho, (K + 31) / 32);
  switch (dt) {
    case WINO_F32:
      direct_f64_kernel<WINO_F32><<<grid, 256, 0, st>>>((const float*)x, (const float*)w, C, H, W, K, pad, Ho, Wo, y);
      break;
    case WINO_F16:
      direct_f64_kernel<WINO_F16><<<grid, 256, 0, st>>>((const __half*)x, (const __half*)w, C, H, W, K, pad, Ho, Wo, y);
      break;
    case WINO_BF16:
      direct_f64_kernel<WINO_BF16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)w, C, H, W,
                                                         K, pad, Ho, Wo, y);
      break;
    default:
      return set_last_error("bad dtype"), WINO_E_ARG;
  }
  WINO_LAUNCH_CHECK();
  return WINO_OK;
}

}  // extern "C"

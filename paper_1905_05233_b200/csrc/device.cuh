// device.cuh -- device helpers shared by the sm_100a kernels: storage-dtype
// conversions (round-to-nearest-even, no flush-to-zero: built without
// --use_fast_math) and thin inline-PTX wrappers for mbarrier, TMA
// (cp.async.bulk.tensor) and the 5th-generation tensor cores (tcgen05 / TMEM).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "algo.hpp"

namespace wino {

// ------------------------------------------------------------------ dtype traits
template <int DT> struct DType;
template <> struct DType<WINO_F32> {
  using T = float;
  static __device__ __forceinline__ float load(const T* p) { return *p; }
  static __device__ __forceinline__ T cvt(float v) { return v; }
  static __device__ __forceinline__ float rd(float v) { return v; }
  static __device__ __forceinline__ float2 rd2(float2 v) { return v; }
};
template <> struct DType<WINO_F16> {
  using T = __half;
  static __device__ __forceinline__ float load(const T* p) { return __half2float(*p); }
  static __device__ __forceinline__ T cvt(float v) { return __float2half_rn(v); }
  static __device__ __forceinline__ float rd(float v) { return __half2float(__float2half_rn(v)); }
  // two values per conversion (cvt.rn.f16x2.f32): the same RNE rounding per element
  static __device__ __forceinline__ float2 rd2(float2 v) { return __half22float2(__float22half2_rn(v)); }
};
template <> struct DType<WINO_BF16> {
  using T = __nv_bfloat16;
  static __device__ __forceinline__ float load(const T* p) { return __bfloat162float(*p); }
  static __device__ __forceinline__ T cvt(float v) { return __float2bfloat16_rn(v); }
  static __device__ __forceinline__ float rd(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
  static __device__ __forceinline__ float2 rd2(float2 v) { return __bfloat1622float2(__float22bfloat162_rn(v)); }
};

// bf16 by truncation (reading A10's switch: drop the low 16 bits of the fp32
// pattern; NaNs stay quiet NaNs), for the paper-mode tile kernels.
__device__ __forceinline__ float bf16_trunc(float v) {
  const uint32_t b = __float_as_uint(v);
  return __uint_as_float((v != v) ? ((b & 0xFFFF0000u) | 0x00400000u) : (b & 0xFFFF0000u));
}
// rounding of the storage dtype with a runtime mode: trunc applies to bf16 only
template <int DT>
struct RdMode {
  using Tr = DType<DT>;
  using T = typename Tr::T;
  bool trunc;
  __device__ __forceinline__ float rd(float v) const {
    if constexpr (DT == WINO_BF16) {
      if (trunc) return bf16_trunc(v);
    }
    return Tr::rd(v);
  }
  __device__ __forceinline__ float2 rd2(float2 v) const {
    if constexpr (DT == WINO_BF16) {
      if (trunc) return make_float2(bf16_trunc(v.x), bf16_trunc(v.y));
    }
    return Tr::rd2(v);
  }
  __device__ __forceinline__ T cvt(float v) const {
    if constexpr (DT == WINO_BF16) {
      if (trunc) return __ushort_as_bfloat16((unsigned short)(__float_as_uint(bf16_trunc(v)) >> 16));
    }
    return Tr::cvt(v);
  }
};

inline size_t dtype_size(wino_dtype dt) { return dt == WINO_F32 ? 4 : 2; }

// Store one output-tile row v[0..M) (rounded to the storage dtype) at row[0..valid)
// with the widest naturally aligned vector stores (16 / 8 / 4 bytes); ragged or
// unaligned rows fall back to element stores.  (A 6-wide bf16 row is 12 bytes:
// three 4-byte stores instead of six 2-byte ones.)
template <typename Tr, int M>
__device__ __forceinline__ void store_tile_row(typename Tr::T* row, const float (&v)[M], int valid) {
  using TT = typename Tr::T;
  constexpr int RB = M * (int)sizeof(TT);
  union {
    TT e[M];
    uint32_t u[(RB + 3) / 4];
  } pk;
#pragma unroll
  for (int q = 0; q < M; ++q) pk.e[q] = Tr::cvt(v[q]);
  const uintptr_t a = reinterpret_cast<uintptr_t>(row);
  if constexpr (RB % 4 == 0) {
    if (valid >= M) {
      if constexpr (RB % 16 == 0) {
        if (a % 16 == 0) {
#pragma unroll
          for (int c = 0; c < RB / 16; ++c)
            reinterpret_cast<uint4*>(row)[c] = make_uint4(pk.u[4 * c], pk.u[4 * c + 1], pk.u[4 * c + 2], pk.u[4 * c + 3]);
          return;
        }
      }
      if constexpr (RB % 8 == 0) {
        if (a % 8 == 0) {
#pragma unroll
          for (int c = 0; c < RB / 8; ++c) reinterpret_cast<uint2*>(row)[c] = make_uint2(pk.u[2 * c], pk.u[2 * c + 1]);
          return;
        }
      }
      if (a % 4 == 0) {
#pragma unroll
        for (int c = 0; c < RB / 4; ++c) reinterpret_cast<uint32_t*>(row)[c] = pk.u[c];
        return;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < M; ++q)
    if (q < valid) row[q] = pk.e[q];
}

// Split an fp32 value into TF32 hi (round to nearest, 10-bit mantissa) and the
// exact fp32 remainder lo = v - hi (the MMA reads lo's top 11 bits).
__device__ __forceinline__ void split_tf32(float v, float& hi, float& lo) {
  uint32_t b = __float_as_uint(v);
  uint32_t h = (b + 0x1000u) & 0xFFFFE000u;
  if ((b & 0x7F800000u) == 0x7F800000u) h = b & 0xFFFFE000u;  // inf / nan: keep
  hi = __uint_as_float(h);
  lo = ((b & 0x7F800000u) == 0x7F800000u) ? 0.f : __fsub_rn(v, hi);
}

// ------------------------------------------------------------------ PTX: shared memory / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// The same wait with a suspend-time hint: a waiting warp sleeps (up to the hint,
// or until the phase completes) instead of re-issuing try_wait, so spinning
// consumer warps do not take issue slots from the warps doing the work.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(20000)
      : "memory");
}

// ------------------------------------------------------------------ PTX: TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// smem -> global tensor store (bulk async group); the box is clipped at the
// tensor bounds, so ragged tiles need no masking.
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------------------------ PTX: tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, both K-major, fp32 accumulate.
template <bool kTF32>
__device__ __forceinline__ void mma_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  }
}
// Arrive on `bar` once every previously issued tcgen05.mma of this thread completes.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// UMMA shared-memory descriptor, K-major, 128-byte swizzle: rows of 128 B,
// 8-row atoms of 1024 B (SBO), LBO unused (encoded 1), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor: fp32 accumulate, K-major A and B, M x N tile.
// a/b format: 0 = F16, 1 = BF16 (kind::f16); 2 = TF32 (kind::tf32).
__host__ __device__ constexpr uint32_t make_idesc(uint32_t ab_format, int M, int N) {
  return (1u << 4) | (ab_format << 7) | (ab_format << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// 32 lanes x 32 consecutive fp32 columns: thread i of the warp receives row
// (lane_base + i), columns [col, col + 32).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ------------------------------------------------------------------ PTX: CTA pairs (cta_group::2)
// A cluster of two CTAs on one TPC runs one M = 256 MMA: each CTA holds its own
// 128 rows of A and half of B's N rows at the same shared-memory offsets; the
// leader (rank 0) issues the MMAs, each CTA's TMEM receives its 128 rows of D.
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// Arrive on a barrier of (possibly) the peer CTA.  Default semantics (release at CTA
// scope), as the remote arrives only signal progress: the data behind them is
// tracked by complete_tx (TMA) or ordered by tcgen05 fences (TMEM reads).  A
// .release.cluster arrive is a cluster-scope fence that waits for the thread's
// outstanding memory traffic -- microseconds per pipeline stage under load.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA load into this CTA's shared memory whose completion is counted on the
// leader's mbarrier (bar_cluster = its shared::cluster address)
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                 int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// one warp of EACH CTA of the pair allocates / frees (collectively)
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
template <bool kTF32>
__device__ __forceinline__ void mma_ss_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  }
}
// arrive on `bar` (same offset) in both CTAs of the pair once the issued MMAs complete
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// Drop a 128-byte L2 line without writing it back (its contents become undefined):
// for consumed intermediates that must not cost HBM write bandwidth.
__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

}  // namespace wino

// Launch bookkeeping and per-device library state (misc.cu).
namespace wino {
void count_launch(int n = 1);
void reset_launch_count();
struct DevState {
  bool ready = false;
  int sms = 0;
  int pair_clusters = 0;   // co-resident 2-CTA clusters of the K3 pair kernel (0: not queried yet)
  int ures_clusters = 0;   // ... of the resident-U pair kernel
  cudaStream_t side = nullptr, io_in = nullptr, io_out = nullptr;   // K2 fork; host_io copy streams
  cudaEvent_t fork = nullptr, join = nullptr, io_ev[2][64] = {};
};
DevState* dev_state();   // of the calling thread's current device; nullptr (+ last error) on failure
int num_sms();           // of the current device
}  // namespace wino

#define WINO_CUDA_CHECK(expr)                                                              \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess) {                                                               \
      wino::set_last_error(std::string(#expr) + ": " + cudaGetErrorString(_e));            \
      return WINO_E_CUDA;                                                                  \
    }                                                                                      \
  } while (0)

#define WINO_LAUNCH_CHECK()                                                                \
  do {                                                                                     \
    cudaError_t _e = cudaGetLastError();                                                   \
    if (_e != cudaSuccess) {                                                               \
      wino::set_last_error(std::string("kernel launch: ") + cudaGetErrorString(_e));      \
      return WINO_E_CUDA;                                                                  \
    }                                                                                      \
    wino::count_launch();                                                                  \
  } while (0)

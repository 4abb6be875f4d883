// tmap.hpp -- host-side TMA tensor-map encoding (cuTensorMapEncodeTiled via
// the runtime's driver entry point, so libwino.so needs no direct libcuda
// symbol at load time beyond what the runtime resolves).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace wino {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

// rank-dimensional tiled map; dims[0] innermost, strides in bytes for dims 1..,
// out-of-bounds elements of a box read as zero.
inline bool make_map(CUtensorMap* map, CUtensorMapDataType dt, int rank, const void* base, const uint64_t* dims,
                     const uint64_t* strides_bytes, const uint32_t* box, bool swizzle128) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) d[i] = dims[i], b[i] = box[i], e[i] = 1;
  for (int i = 0; i + 1 < rank; ++i) s[i] = strides_bytes[i];
  return enc(map, dt, (cuuint32_t)rank, const_cast<void*>(base), d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3D map; d0 innermost.  row0 = elements per d0-row in memory (>= d0).
inline bool make_map3(CUtensorMap* map, CUtensorMapDataType dt, size_t es, const void* base, uint64_t d0, uint64_t d1,
                      uint64_t d2, uint32_t b0, uint32_t b1, bool swizzle = true, uint64_t row0 = 0) {
  if (!row0) row0 = d0;
  const uint64_t dims[3] = {d0, d1, d2};
  const uint64_t strides[2] = {row0 * es, row0 * d1 * es};
  const uint32_t box[3] = {b0, b1, 1};
  return make_map(map, dt, 3, base, dims, strides, box, swizzle);
}

}  // namespace wino

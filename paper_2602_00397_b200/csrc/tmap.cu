// TMA tensor-map encoding (host).  cuTensorMapEncodeTiled is resolved once
// through the runtime's driver entry point, so the library needs no -lcuda.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

#include "ffwd_internal.h"

namespace ffwd {

namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

}  // namespace

CUresult encode_tmap_2d_bf16_sw(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows,
                                uint32_t box_inner, uint32_t box_rows, bool swizzle128);

// 2-D bf16 row-major tensor [rows x inner], 128 B swizzle, box {box_inner, box_rows};
// out-of-bounds rows of a box read as zero (the short tail block).
CUresult encode_tmap_2d_bf16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows,
                             uint32_t box_inner, uint32_t box_rows) {
  return encode_tmap_2d_bf16_sw(m, base, inner, rows, box_inner, box_rows, true);
}

// swizzle128 = false: no swizzle (boxes wider than 128 B; L2 prefetch maps)
CUresult encode_tmap_2d_bf16_sw(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows,
                                uint32_t box_inner, uint32_t box_rows, bool swizzle128) {
  EncodeFn enc = get_encode();
  if (!enc) return CUDA_ERROR_NOT_FOUND;
  const cuuint64_t dims[2] = {inner, rows};
  const cuuint64_t strides[1] = {inner * 2};
  const cuuint32_t box[2] = {box_inner, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

}  // namespace ffwd

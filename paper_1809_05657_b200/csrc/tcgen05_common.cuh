// tcgen05_common.cuh — pieces shared by the two tcgen05 GEMM kernels
// (gemm_tcgen05.cu: one CTA per tile; gemm_tcgen05_2sm.cu: CTA pairs): shared-memory
// matrix descriptors, TMEM loads, the C epilogue stores and the TMA tensor maps.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

namespace hda {
namespace tcc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// shared-memory matrix descriptor (sm_100 "version 1"), 128-byte swizzle
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version
  d |= (uint64_t)2 << 61;   // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <typename TC>
__device__ __forceinline__ void store_chunk(TC* row, int64_t col0, int64_t n0, int64_t n1, const uint32_t (&r)[32],
                                            float alpha, float beta);

template <>
__device__ __forceinline__ void store_chunk<float>(float* row, int64_t col0, int64_t n0, int64_t n1,
                                                   const uint32_t (&r)[32], float alpha, float beta) {
  const bool full = col0 >= n0 && col0 + 32 <= n1 && ((uintptr_t)(row + col0) % 16 == 0);
  if (full) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      float4 v;
      v.x = alpha * __uint_as_float(r[j]);
      v.y = alpha * __uint_as_float(r[j + 1]);
      v.z = alpha * __uint_as_float(r[j + 2]);
      v.w = alpha * __uint_as_float(r[j + 3]);
      float4* p = reinterpret_cast<float4*>(row + col0 + j);
      if (beta != 0.f) {
        float4 c = *p;
        v.x = fmaf(beta, c.x, v.x);
        v.y = fmaf(beta, c.y, v.y);
        v.z = fmaf(beta, c.z, v.z);
        v.w = fmaf(beta, c.w, v.w);
      }
      *p = v;
    }
  } else {
    for (int j = 0; j < 32; j++) {
      const int64_t c = col0 + j;
      if (c < n0 || c >= n1) continue;
      float v = alpha * __uint_as_float(r[j]);
      if (beta != 0.f) v = fmaf(beta, row[c], v);
      row[c] = v;
    }
  }
}

template <>
__device__ __forceinline__ void store_chunk<__nv_bfloat16>(__nv_bfloat16* row, int64_t col0, int64_t n0, int64_t n1,
                                                           const uint32_t (&r)[32], float alpha, float beta) {
  const bool full = col0 >= n0 && col0 + 32 <= n1 && ((uintptr_t)(row + col0) % 16 == 0);
  if (full) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      uint4* p = reinterpret_cast<uint4*>(row + col0 + j);
      float c[8];
      if (beta != 0.f) {
        uint4 cv = *p;
        const __nv_bfloat16* cb = reinterpret_cast<const __nv_bfloat16*>(&cv);
#pragma unroll
        for (int t = 0; t < 8; t++) c[t] = __bfloat162float(cb[t]);
      }
      uint4 out;
      __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&out);
#pragma unroll
      for (int t = 0; t < 8; t++) {
        float v = alpha * __uint_as_float(r[j + t]);
        if (beta != 0.f) v = fmaf(beta, c[t], v);
        ob[t] = __float2bfloat16_rn(v);
      }
      *p = out;
    }
  } else {
    for (int j = 0; j < 32; j++) {
      const int64_t c = col0 + j;
      if (c < n0 || c >= n1) continue;
      float v = alpha * __uint_as_float(r[j]);
      if (beta != 0.f) v = fmaf(beta, __bfloat162float(row[c]), v);
      row[c] = __float2bfloat16_rn(v);
    }
  }
}

// ---------------------------------------------------------------- host side

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiled get_encode() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiled)p;
  });
  return fn;
}

// 2-D bf16 tensor map: inner dim `inner` (contiguous), outer dim `outer`, box {64, box_outer}
inline bool make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_outer) {
  EncodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace tcc
}  // namespace hda

// gemm_simt.cu — reference-grade CUDA-core GEMM used only where the tcgen05 path
// does not apply (tile-unaligned work boxes).  C = alpha*A@B + beta*C over the work box
// (Listing 2), bf16 inputs, fp32 accumulation.
#include <cuda_bf16.h>

#include "kernels.cuh"
#include "sync.cuh"

namespace hda {

template <typename TC>
__device__ __forceinline__ float ld_c(const TC* p);
template <>
__device__ __forceinline__ float ld_c(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld_c(const __nv_bfloat16* p) { return __bfloat162float(*p); }
template <typename TC>
__device__ __forceinline__ void st_c(TC* p, float v);
template <>
__device__ __forceinline__ void st_c(float* p, float v) { *p = v; }
template <>
__device__ __forceinline__ void st_c(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

template <typename TC>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const __nv_bfloat16* __restrict__ A,
                                                        const __nv_bfloat16* __restrict__ B, TC* C, int64_t N,
                                                        int64_t K, int64_t m0, int64_t m1, int64_t n0, int64_t n1,
                                                        float alpha, float beta, const __grid_constant__ KSync ks) {
  ks_pre(ks);
  __shared__ float As[32][65];
  __shared__ float Bs[32][65];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t mb = m0 + (int64_t)blockIdx.y * 64, nb = n0 + (int64_t)blockIdx.x * 64;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += 32) {
    for (int t = threadIdx.x; t < 64 * 32; t += 256) {
      int r = t / 32, c = t % 32;
      int64_t gm = mb + r, gk = k0 + c;
      As[c][r] = (gm < m1 && gk < K) ? __bfloat162float(A[gm * K + gk]) : 0.f;
      int rb = t / 64, cb = t % 64;
      int64_t gkb = k0 + rb, gn = nb + cb;
      Bs[rb][cb] = (gkb < K && gn < n1) ? __bfloat162float(B[gkb * N + gn]) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < 32; k++) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; i++) a[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; j++) b[j] = Bs[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) {
      int64_t gm = mb + ty * 4 + i, gn = nb + tx * 4 + j;
      if (gm < m1 && gn < n1) {
        TC* p = C + gm * N + gn;
        float v = alpha * acc[i][j];
        if (beta != 0.f) v = fmaf(beta, ld_c<TC>(p), v);
        st_c<TC>(p, v);
      }
    }
  ks_post(ks);
}

cudaError_t launch_gemm_simt(int c_dtype, const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K,
                             const int64_t* lb, const int64_t* ub, float alpha, float beta, const KSync& ks,
                             cudaStream_t s) {
  (void)M;
  const int64_t m0 = lb[1], m1 = ub[1], n0 = lb[2], n1 = ub[2];
  if (m0 >= m1 || n0 >= n1) return cudaSuccess;
  dim3 grid((unsigned)((n1 - n0 + 63) / 64), (unsigned)((m1 - m0 + 63) / 64));
  if (c_dtype == 1)
    gemm_simt_kernel<float><<<grid, 256, 0, s>>>((const __nv_bfloat16*)A, (const __nv_bfloat16*)B, (float*)C, N, K,
                                                 m0, m1, n0, n1, alpha, beta, ks);
  else
    gemm_simt_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)A, (const __nv_bfloat16*)B,
                                                         (__nv_bfloat16*)C, N, K, m0, m1, n0, n1, alpha, beta, ks);
  return cudaGetLastError();
}

}  // namespace hda

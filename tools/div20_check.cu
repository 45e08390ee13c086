// div20_check.cu — hda::div20 (csrc/divc.cuh, the 9-point stencil's fp64 division by
// 20) against the IEEE division a / 20.0 on 2^32 hashed doubles: every exponent from
// subnormal to huge, both signs, plus zeros, Inf, NaN and the range edges; and
// hda::div6 (the 3-D stencil's fp32 division by 6) against a / 6.0f on every one of the
// 2^32 fp32 bit patterns.  Prints the mismatch counts; exit 1 on any.  Run by tests/test_gpu_parity.py::test_div20_matches_ieee.
#include <cstdio>
#include <cstdint>

#include "divc.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void check(uint64_t n, unsigned long long* bad, unsigned long long* first) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t h = mix(i);
    double a;
    if (i < 64) {  // specials and range edges
      const double sp[16] = {0.0, -0.0, 1.0 / 0.0, -1.0 / 0.0, 0.0 / 0.0, 0x1p-1000, -0x1p-1000, 0x1p+1000,
                             0x1.fffffffffffffp+999, 0x1.0000000000001p-1000, 0x1p-1074, 0x1p-1022,
                             0x1.fffffffffffffp+1023, 20.0, 3.0, 1e-300};
      a = sp[i % 16];
      if (i >= 16) a = -a;
    } else if ((h & 7) == 0) {  // concentrate near the fast-path edges
      const uint64_t e = (h >> 3) & 1 ? 1023 - 1000 : 1023 + 1000;
      const uint64_t ee = e + ((h >> 4) % 5) - 2;
      a = __longlong_as_double((long long)(((h >> 8) & 1) << 63 | ee << 52 | (mix(h) & 0xFFFFFFFFFFFFFull)));
    } else {
      a = __longlong_as_double((long long)h);  // uniform bit patterns: all exponents, NaNs included
    }
    const double g = hda::div20(a), w = a / 20.0;
    const bool same = __double_as_longlong(g) == __double_as_longlong(w) || (g != g && w != w);
    if (!same && atomicAdd(bad, 1ull) == 0) *first = (unsigned long long)__double_as_longlong(a);
  }
}

__global__ void check6(unsigned long long* bad, unsigned long long* first) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (1ull << 32);
       i += (uint64_t)gridDim.x * blockDim.x) {
    const float a = __uint_as_float((unsigned)i);
    const float g = hda::div6(a), w = a / 6.0f;
    const bool same = __float_as_uint(g) == __float_as_uint(w) || (g != g && w != w);
    if (!same && atomicAdd(bad, 1ull) == 0) *first = i;
  }
}

int main() {
  unsigned long long *bad, *first;
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&first, 8);
  *bad = 0;
  *first = 0;
  const uint64_t n = 1ull << 32;
  check<<<148 * 8, 256>>>(n, bad, first);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("CUDA error\n");
    return 2;
  }
  printf("div20 vs IEEE: %llu mismatches in %llu inputs", *bad, (unsigned long long)n);
  if (*bad) printf(" (first input bits %016llx)", *first);
  printf("\n");
  const unsigned long long bad20 = *bad;
  *bad = 0;
  check6<<<148 * 8, 256>>>(bad, first);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("CUDA error\n");
    return 2;
  }
  printf("div6 (fp32) vs IEEE: %llu mismatches in all 4294967296 inputs", *bad);
  if (*bad) printf(" (first input bits %08llx)", *first);
  printf("\n");
  return (bad20 || *bad) ? 1 : 0;
}

// divc.cuh — the 9-point stencil's division by 20 (reading R12: Y = (4e + c) / 20),
// correctly rounded, without recomputing 1/20 per point.
//
// nvcc's IEEE fp64 division by a constant rebuilds the reciprocal on every call
// (MUFU.RCP64H + 5 dependent DFMA: 9 MUFU.RCP64H / 74 DFMA in the register-march
// 9-point kernel) before the same three-operation correction used here.  Markstein
// (IBM J. R&D 34(1), 1990; Muller et al., Handbook of Floating-Point Arithmetic,
// "Markstein's theorem"): with y = RN(1/b) and q0 within one ulp of a/b, the remainder
// r = a - b*q0 is exact in one FMA and RN(q0 + r*y) = RN(a/b), provided nothing
// underflows or overflows.  q0 = RN(a*y) is within one ulp (|a*y - a/b| <= ulp/2).
// Outside [2^-1000, 2^1000] (zeros, subnormals, huge values, Inf, NaN) the IEEE
// division runs instead, so every input gets the correctly rounded quotient: bit-
// identical to the oracle's a / 20.0 (tests: test_stencil_division_edge_values and
// test_div20_matches_ieee).
#pragma once

namespace hda {

__device__ __forceinline__ double div20(double a) {
  const double y = 0.05;  // RN(1/20)
  const double m = fabs(a);
  if (m >= 0x1p-1000 && m <= 0x1p+1000) {  // NaN fails both
    const double q0 = __dmul_rn(a, y);
    const double r = __fma_rn(-q0, 20.0, a);
    return __fma_rn(r, y, q0);
  }
  return a / 20.0;
}
// fp32: nvcc already folds 1/20 into a constant (FFMA correction + FCHK); keep it
__device__ __forceinline__ float div20(float a) { return a / 20.0f; }

// The 3-D 7-point stencil's fp32 division by 6 (reading R13), same scheme: y = RN(1/6);
// no reciprocal refinement and no FCHK on the fast path.  Exhaustively checked against
// a / 6.0f on all 2^32 inputs (tools/div20_check.cu).
__device__ __forceinline__ float div6(float a) {
  const float y = 0x1.555556p-3f;  // RN(1/6)
  const float m = fabsf(a);
  if (m >= 0x1p-100f && m <= 0x1p+100f) {
    const float q0 = __fmul_rn(a, y);
    const float r = __fmaf_rn(-q0, 6.0f, a);
    return __fmaf_rn(r, y, q0);
  }
  return a / 6.0f;
}
__device__ __forceinline__ double div6(double a) { return a / 6.0; }

}  // namespace hda

/* markstein_check.c — verifies that the 3-operation quotient used by the stencil
 * kernels, q0 = RN(x*y), r = RN(x - q0*d) (exact, FMA), q1 = RN(q0 + r*y) with
 * y = RN(1/d), equals the IEEE quotient RN(x/d):
 *   fp32, d = 6:  EXHAUSTIVELY over every finite float whose quotient is normal;
 *   fp64, d = 20: over N random bit patterns spread over all normal exponents plus
 *                 structured values (small integers, sums of k/2^m).
 * Zero residual / non-finite / tiny inputs take the guarded path in the kernels and
 * are excluded here.  Build: gcc -O2 -ffp-contract=off -o /tmp/mc tools/markstein_check.c -lm
 * Run: /tmp/mc [fp64 samples = 2e8] [fp32 stride = 1]  (full run: profiles/r01/markstein_check.txt)
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t sm(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int main(int argc, char** argv) {
  long long n64 = argc > 1 ? atoll(argv[1]) : 200000000LL;
  uint64_t stride = argc > 2 ? strtoull(argv[2], 0, 10) : 1; /* 1 = every float */
  /* fp32 / 6 exhaustive */
  const float d32 = 6.0f, y32 = 1.0f / 6.0f;
  uint64_t bad32 = 0, tested32 = 0;
  for (uint64_t u = 0; u < (1ull << 32); u += stride) {
    uint32_t b = (uint32_t)u;
    float x;
    memcpy(&x, &b, 4);
    if (!isfinite(x) || fabsf(x) < 0x1p-100f) continue;
    float q0 = x * y32;
    float r = fmaf(-q0, d32, x);
    float q1 = r == 0.0f ? q0 : fmaf(r, y32, q0);
    float ref = x / d32;
    tested32++;
    if (memcmp(&q1, &ref, 4)) {
      if (bad32 < 5) printf("fp32 mismatch x=%a q1=%a ref=%a\n", x, q1, ref);
      bad32++;
    }
  }
  printf("fp32 /6: %llu finite inputs, %llu mismatches\n", (unsigned long long)tested32, (unsigned long long)bad32);
  /* fp64 / 20 random over normal exponents */
  const double d64 = 20.0, y64 = 1.0 / 20.0;
  uint64_t s = 180905657, bad64 = 0;
  for (long long i = 0; i < n64; i++) {
    uint64_t h = sm(&s);
    double x;
    if (i % 4 == 0) {  /* structured: sums of small dyadic rationals (stencil-like values) */
      x = (double)(int64_t)(h % 2000001 - 1000000) / (double)(1u << (h >> 60));
    } else {
      uint64_t e = 24 + (h >> 11) % 1990; /* biased exponent in [24, 2013] */
      uint64_t bits = (h & 0x800FFFFFFFFFFFFFull) | (e << 52);
      memcpy(&x, &bits, 8);
    }
    if (!isfinite(x) || fabs(x) < 0x1p-1000) continue;
    double q0 = x * y64;
    double r = fma(-q0, d64, x);
    double q1 = r == 0.0 ? q0 : fma(r, y64, q0);
    double ref = x / d64;
    if (memcmp(&q1, &ref, 8)) {
      if (bad64 < 5) printf("fp64 mismatch x=%a q1=%a ref=%a\n", x, q1, ref);
      bad64++;
    }
  }
  printf("fp64 /20: %lld samples, %llu mismatches\n", n64, (unsigned long long)bad64);
  return (bad32 || bad64) ? 1 : 0;
}

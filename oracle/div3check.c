/*
 * Exhaustive check (test infrastructure): the FMA-based quotient the device
 * uses for x / 3.0f (userkernels/stencil_kernels.h: lf_div3f, and its packed
 * fp32x2 form in the generic executor) equals the IEEE division for every one
 * of the 2^32 float bit patterns.  The residual is formed negated,
 * t = RN(3q - x), and applied as RN(q - t r): signed zeros then come out right
 * without a test (x = -0: t = +0, q - t r = -0 + -0), so only infinities
 * (t = NaN) keep the plain product.  Host fmaf is the
 * correctly rounded fused multiply-add, as __fmaf_rn is on the GPU.
 * Usage: div3check [stride]  (stride > 1 samples every stride-th pattern)
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static inline float div3_device_sequence(float x) {
  const float r = 0x1.555556p-2f;
  const float q = x * r;
  const float t = fmaf(q, 3.0f, -x);
  const float q1 = fmaf(t, -r, q);
  return isinf(q) ? q : q1;
}

int main(int argc, char** argv) {
  long stride = argc > 1 ? atol(argv[1]) : 1;
  long bad = 0, n = 0;
#pragma omp parallel for reduction(+ : bad, n) schedule(static)
  for (long i = 0; i <= 0xffffffffL; i += stride) {
    uint32_t u = (uint32_t)i, ua, ub;
    float x, a, b;
    memcpy(&x, &u, 4);
    a = x / 3.0f;
    b = div3_device_sequence(x);
    memcpy(&ua, &a, 4);
    memcpy(&ub, &b, 4);
    n++;
    if (ua != ub && !(isnan(a) && isnan(b))) bad++;
  }
  printf("{\"checked\": %ld, \"mismatches\": %ld}\n", n, bad);
  return bad != 0;
}

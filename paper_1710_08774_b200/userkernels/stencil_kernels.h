/*
 * User kernels for the BASELINE.json stencil chains (configs 1, 2 and 4).
 *
 * In the reference model these are the user's own opaque per-cell functions:
 * the rule file names them in `declaration:` strings (R/SPEC.md:81,
 * rulespec.hpp:41-53) and both the naive schedule (run_naive, R/SPEC.md:532-540)
 * and the emitted fused loop nest (R/SPEC.md:499-502) call the very same
 * functions.  We keep that contract: this header is included by the CPU
 * oracle (oracle/ sources) and inlined into the sm_100a fused executors
 * (csrc/exec/ sources), so a parity difference can only come from the schedule,
 * never from two transcriptions of the arithmetic.
 *
 * Rules for bit-exact parity:
 *  - only + - * / sqrt min max fabs (correctly rounded on both sides);
 *  - evaluation order is the C order written here; host builds use
 *    -ffp-contract=off, device builds -fmad=false, so no FMA contraction.
 */
#ifndef LF_USERKERNELS_STENCIL_H
#define LF_USERKERNELS_STENCIL_H

#if defined(__CUDACC__)
#define LF_HD __host__ __device__ __forceinline__
#else
#define LF_HD static inline
#endif

/* ---- config 1: lap(lap(u)) then explicit update ------------------------ */

/* 5-point Laplacian, BASELINE.json configs[0]:
 *   L = u[i-1,j] + u[i+1,j] + u[i,j-1] + u[i,j+1] - 4 u[i,j]   (left to right) */
LF_HD void lap5(double w, double e, double s, double n, double c, double* o) {
  *o = w + e + s + n - 4.0 * c;
}

/* u <- u - 0.01 * stage2 */
LF_HD void biharm_update(double c, double l2, double* o) { *o = c - 0.01 * l2; }

/* ---- config 2: 3D heat through face fluxes ----------------------------- */

/* flux on the face between c and its +1 neighbour along one axis */
LF_HD void face_flux(double up, double c, double* f) { *f = up - c; }

/* divergence of the three face fluxes, alpha*dt/h^2 = 0.1 */
LF_HD void heat_divupd(double c, double fxp, double fxm, double fyp, double fym, double fzp,
                       double fzm, double* o) {
  *o = c + 0.1 * ((fxp - fxm) + (fyp - fym) + (fzp - fzm));
}

/* ---- config 4: separable 3x3 box filter, applied twice (fp32) ---------- */

/* x / 3.0f, correctly rounded.  The device computes the IEEE quotient with
 * one multiply by RN(1/3) and an FMA residual correction instead of the
 * generic division subroutine (rcp + Newton + slow-path call):
 *   q = RN(x r),  t = RN(3 q - x),  q1 = RN(q - t r)
 * The sequence is exhaustively checked bit-identical to `x / 3.0f` for all
 * 2^32 inputs (oracle/div3check.c, tests/test_div3.py).  Forming the residual
 * negated gives signed zeros right with no test (x = -0: t = +0, q1 = -0);
 * infinities (t = NaN) keep the plain product, which is exact for them. */
LF_HD float lf_div3f(float x) {
#if defined(__CUDA_ARCH__)
  const float r = 0x1.555556p-2f; /* RN(1/3) */
  const float q = __fmul_rn(x, r);
  const float t = __fmaf_rn(q, 3.0f, -x);
  const float q1 = __fmaf_rn(t, -r, q);
  return isinf(q) ? q : q1;
#else
  return x / 3.0f;
#endif
}

#if defined(__CUDACC__)
/* the same sequence on fp32x2 pairs (FMUL2 / FFMA2; lanewise identical) */
__device__ __forceinline__ float2 lf_div3f2(float2 x) {
#if defined(__CUDA_ARCH__)
  const float2 r = make_float2(0x1.555556p-2f, 0x1.555556p-2f);
  const float2 q = __fmul2_rn(x, r);
  const float2 t = __ffma2_rn(q, make_float2(3.0f, 3.0f), make_float2(-x.x, -x.y));
  const float2 q1 = __ffma2_rn(t, make_float2(-0x1.555556p-2f, -0x1.555556p-2f), q);
  return make_float2(isinf(q.x) ? q.x : q1.x, isinf(q.y) ? q.y : q1.y);
#else
  return x; /* host pass: device only */
#endif
}
#endif

/* one 3-tap pass; a,b,c are the -1,0,+1 neighbours along the pass axis */
LF_HD void box3(float a, float b, float c, float* o) { *o = lf_div3f(a + b + c); }

#endif

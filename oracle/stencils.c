/*
 * CPU ORACLE (test infrastructure only) -- configs 1, 2 and 4 of BASELINE.json.
 * See oracle.h for the contract.  Each function cites the reference semantics
 * it restates.
 */
#include <omp.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"
#include "../paper_1710_08774_b200/userkernels/stencil_kernels.h"

int lfo_max_threads(void) { return omp_get_max_threads(); }

static int clamp_threads(int threads) {
  if (threads <= 0) threads = omp_get_max_threads();
  return threads;
}

/* ========================================================================
 * Config 1: u_new = u - 0.01 * lap5(lap5(u)), zero Dirichlet ghost ring of 2.
 * Terminal layout: g_u extent (N+4)^2, base -2 (buffer_extents,
 * storage.cpp:403-427, for reads at offsets -2..+2).
 * ====================================================================== */

#define U1(a, j, i) (a)[((j) + 2) * P + ((i) + 2)]

static void biharm_zero_ghosts(double* a, long nj, long ni) {
  const long P = ni + 4;
  for (long j = -2; j < nj + 2; ++j)
    for (long i = -2; i < ni + 2; ++i)
      if (j < 0 || j >= nj || i < 0 || i >= ni) U1(a, j, i) = 0.0;
}

/* run_naive (R/SPEC.md:532-540): lap1 over its whole space (the cross of
 * cells [-1,N+1)^2 that lap2 reads), then lap2 over [0,N)^2, then upd. */
int lfo_biharm_naive(const double* u_in, double* u_out, long nj, long ni, int steps) {
  const long P = ni + 4;
  const size_t n = (size_t)(nj + 4) * (size_t)P;
  const long PL = ni + 2;
  double* a = (double*)malloc(n * sizeof(double));
  double* b = (double*)malloc(n * sizeof(double));
  double* L = (double*)malloc((size_t)(nj + 2) * PL * sizeof(double));
  double* L2 = (double*)malloc((size_t)nj * ni * sizeof(double));
  if (!a || !b || !L || !L2) return 3;
  memcpy(a, u_in, n * sizeof(double));
  memset(b, 0, n * sizeof(double));
  for (int s = 0; s < steps; ++s) {
    for (long j = -1; j < nj + 1; ++j)
      for (long i = -1; i < ni + 1; ++i)
        lap5(U1(a, j, i - 1), U1(a, j, i + 1), U1(a, j - 1, i), U1(a, j + 1, i), U1(a, j, i),
             &L[(j + 1) * PL + (i + 1)]);
#define LL(j, i) L[((j) + 1) * PL + ((i) + 1)]
    for (long j = 0; j < nj; ++j)
      for (long i = 0; i < ni; ++i)
        lap5(LL(j, i - 1), LL(j, i + 1), LL(j - 1, i), LL(j + 1, i), LL(j, i), &L2[j * ni + i]);
#undef LL
    for (long j = 0; j < nj; ++j)
      for (long i = 0; i < ni; ++i) biharm_update(U1(a, j, i), L2[j * ni + i], &U1(b, j, i));
    biharm_zero_ghosts(b, nj, ni);
    double* t = a;
    a = b;
    b = t;
  }
  memcpy(u_out, a, n * sizeof(double));
  free(a);
  free(b);
  free(L);
  free(L2);
  return 0;
}

/* HFAV fused schedule for config 1.  Loop order (j,i); lap1 leads by one row
 * (shift j=+1, shifts.cpp:21-77), L contracted to an outer_rotate window of 3
 * rows (storage.cpp:369-378), L2 a scalar.  OpenMP splits the outer j loop;
 * each thread primes its own window (prologue, R/PAPER.md:464). */
static void biharm_fused_step(const double* a, double* b, long nj, long ni, int threads) {
  const long P = ni + 4;
  const long W = ni + 2; /* L window row: logical cols [-1, ni+1) */
#pragma omp parallel num_threads(threads)
  {
    int nt = omp_get_num_threads(), t = omp_get_thread_num();
    long j0 = nj * t / nt, j1 = nj * (t + 1) / nt;
    double* win = (double*)malloc(3 * W * sizeof(double));
    double* rows[3] = {win, win + W, win + 2 * W};
    /* prologue: L rows j0-1 and j0 */
    for (int r = 0; r < 2; ++r) {
      long j = j0 - 1 + r;
      for (long i = -1; i < ni + 1; ++i)
        lap5(U1(a, j, i - 1), U1(a, j, i + 1), U1(a, j - 1, i), U1(a, j + 1, i), U1(a, j, i),
             &rows[r][i + 1]);
    }
    for (long j = j0; j < j1; ++j) {
      double* lm = rows[0];
      double* l0 = rows[1];
      double* lp = rows[2];
      long jj = j + 1; /* lap1 runs at trip + shift */
      for (long i = -1; i < ni + 1; ++i)
        lap5(U1(a, jj, i - 1), U1(a, jj, i + 1), U1(a, jj - 1, i), U1(a, jj + 1, i), U1(a, jj, i),
             &lp[i + 1]);
      for (long i = 0; i < ni; ++i) {
        double l2;
        lap5(l0[i], l0[i + 2], lm[i + 1], lp[i + 1], l0[i + 1], &l2);
        biharm_update(U1(a, j, i), l2, &U1(b, j, i));
      }
      /* outer_rotate: pointer rotation of the row window */
      rows[0] = l0;
      rows[1] = lp;
      rows[2] = lm;
    }
    free(win);
  }
  biharm_zero_ghosts(b, nj, ni);
}

/* one step, in -> out (out's ghost ring zeroed): the unit the CPU baseline times */
int lfo_biharm_fused_step(const double* u_in, double* u_out, long nj, long ni, int threads) {
  biharm_fused_step(u_in, u_out, nj, ni, clamp_threads(threads));
  return 0;
}

int lfo_biharm_fused(const double* u_in, double* u_out, long nj, long ni, int steps, int threads) {
  const size_t n = (size_t)(nj + 4) * (size_t)(ni + 4);
  threads = clamp_threads(threads);
  double* a = (double*)malloc(n * sizeof(double));
  double* b = (double*)malloc(n * sizeof(double));
  if (!a || !b) return 3;
  memcpy(a, u_in, n * sizeof(double));
  memset(b, 0, n * sizeof(double));
  for (int s = 0; s < steps; ++s) {
    biharm_fused_step(a, b, nj, ni, threads);
    double* t = a;
    a = b;
    b = t;
  }
  memcpy(u_out, a, n * sizeof(double));
  free(a);
  free(b);
  return 0;
}
#undef U1

/* ========================================================================
 * Config 2: 3D heat, u_new = u + 0.1 * div(face fluxes), periodic.
 * Terminal layout: g_u extent (N+2)^3, base -1, ghost layer filled by wrap.
 * ====================================================================== */

#define U3(a, k, j, i) (a)[(((k) + 1) * PJ + ((j) + 1)) * PI + ((i) + 1)]

static void heat3d_wrap(double* a, long nk, long nj, long ni) {
  const long PI = ni + 2, PJ = nj + 2;
  for (long k = 0; k < nk; ++k)
    for (long j = 0; j < nj; ++j) {
      U3(a, k, j, -1) = U3(a, k, j, ni - 1);
      U3(a, k, j, ni) = U3(a, k, j, 0);
    }
  for (long k = 0; k < nk; ++k)
    for (long i = -1; i < ni + 1; ++i) {
      U3(a, k, -1, i) = U3(a, k, nj - 1, i);
      U3(a, k, nj, i) = U3(a, k, 0, i);
    }
  for (long j = -1; j < nj + 1; ++j)
    for (long i = -1; i < ni + 1; ++i) {
      U3(a, -1, j, i) = U3(a, nk - 1, j, i);
      U3(a, nk, j, i) = U3(a, 0, j, i);
    }
}

/* run_naive: fluxx over faces i in [-1,N), fluxy over j in [-1,N), fluxz over
 * k in [-1,N) -- each into a full array -- then divupd over [0,N)^3. */
int lfo_heat3d_naive(const double* u_in, double* u_out, long nk, long nj, long ni, int steps) {
  const long PI = ni + 2, PJ = nj + 2;
  const size_t n = (size_t)(nk + 2) * PJ * PI;
  double* a = (double*)malloc(n * sizeof(double));
  double* b = (double*)malloc(n * sizeof(double));
  double* fx = (double*)malloc((size_t)nk * nj * (ni + 1) * sizeof(double));
  double* fy = (double*)malloc((size_t)nk * (nj + 1) * ni * sizeof(double));
  double* fz = (double*)malloc((size_t)(nk + 1) * nj * ni * sizeof(double));
  if (!a || !b || !fx || !fy || !fz) return 3;
  memcpy(a, u_in, n * sizeof(double));
  memcpy(b, u_in, n * sizeof(double));
#define FX(k, j, i) fx[((k) * nj + (j)) * (ni + 1) + ((i) + 1)]
#define FY(k, j, i) fy[((k) * (nj + 1) + ((j) + 1)) * ni + (i)]
#define FZ(k, j, i) fz[(((k) + 1) * nj + (j)) * ni + (i)]
  for (int s = 0; s < steps; ++s) {
    for (long k = 0; k < nk; ++k)
      for (long j = 0; j < nj; ++j)
        for (long i = -1; i < ni; ++i) face_flux(U3(a, k, j, i + 1), U3(a, k, j, i), &FX(k, j, i));
    for (long k = 0; k < nk; ++k)
      for (long j = -1; j < nj; ++j)
        for (long i = 0; i < ni; ++i) face_flux(U3(a, k, j + 1, i), U3(a, k, j, i), &FY(k, j, i));
    for (long k = -1; k < nk; ++k)
      for (long j = 0; j < nj; ++j)
        for (long i = 0; i < ni; ++i) face_flux(U3(a, k + 1, j, i), U3(a, k, j, i), &FZ(k, j, i));
    for (long k = 0; k < nk; ++k)
      for (long j = 0; j < nj; ++j)
        for (long i = 0; i < ni; ++i)
          heat_divupd(U3(a, k, j, i), FX(k, j, i), FX(k, j, i - 1), FY(k, j, i), FY(k, j - 1, i),
                      FZ(k, j, i), FZ(k - 1, j, i), &U3(b, k, j, i));
    heat3d_wrap(b, nk, nj, ni);
    double* t = a;
    a = b;
    b = t;
  }
#undef FX
#undef FY
#undef FZ
  memcpy(u_out, a, n * sizeof(double));
  free(a);
  free(b);
  free(fx);
  free(fy);
  free(fz);
  return 0;
}

/* HFAV fused schedule for config 2: loop order (k,j,i), all shifts 0;
 * fx contracted to inner_circular(2) (a scalar carry), fy to outer_rotate 2
 * rows, fz to outer_rotate 2 planes.
 * Prologues compute the i=-1 / j=-1 / k=k0-1 faces.  OpenMP over k. */
static void heat3d_wrap_parallel(double* a, long nk, long nj, long ni, int threads) {
  const long PI = ni + 2, PJ = nj + 2;
#pragma omp parallel for num_threads(threads)
  for (long k = 0; k < nk; ++k) {
    for (long j = 0; j < nj; ++j) {
      U3(a, k, j, -1) = U3(a, k, j, ni - 1);
      U3(a, k, j, ni) = U3(a, k, j, 0);
    }
    for (long i = -1; i < ni + 1; ++i) {
      U3(a, k, -1, i) = U3(a, k, nj - 1, i);
      U3(a, k, nj, i) = U3(a, k, 0, i);
    }
  }
  memcpy(&U3(a, -1, -1, -1), &U3(a, nk - 1, -1, -1), (size_t)PJ * PI * sizeof(double));
  memcpy(&U3(a, nk, -1, -1), &U3(a, 0, -1, -1), (size_t)PJ * PI * sizeof(double));
}

static void heat3d_fused_step(const double* a, double* b, long nk, long nj, long ni, int threads) {
  const long PI = ni + 2, PJ = nj + 2;
#pragma omp parallel num_threads(threads)
  {
    int nt = omp_get_num_threads(), t = omp_get_thread_num();
    long k0 = nk * t / nt, k1 = nk * (t + 1) / nt;
    double* fzw = (double*)malloc(2 * (size_t)nj * ni * sizeof(double));
    double* fyw = (double*)malloc(2 * (size_t)ni * sizeof(double));
    double* fz_prev = fzw;
    double* fz_cur = fzw + (size_t)nj * ni;
    /* prologue: fz plane k0-1 */
    for (long j = 0; j < nj; ++j)
      for (long i = 0; i < ni; ++i) face_flux(U3(a, k0, j, i), U3(a, k0 - 1, j, i), &fz_prev[j * ni + i]);
    for (long k = k0; k < k1; ++k) {
      double* fy_prev = fyw;
      double* fy_cur = fyw + ni;
      for (long i = 0; i < ni; ++i) face_flux(U3(a, k, 0, i), U3(a, k, -1, i), &fy_prev[i]);
      for (long j = 0; j < nj; ++j) {
        double fx_prev;
        face_flux(U3(a, k, j, 0), U3(a, k, j, -1), &fx_prev);
        for (long i = 0; i < ni; ++i) {
          double fxc;
          face_flux(U3(a, k, j, i + 1), U3(a, k, j, i), &fxc);
          face_flux(U3(a, k, j + 1, i), U3(a, k, j, i), &fy_cur[i]);
          face_flux(U3(a, k + 1, j, i), U3(a, k, j, i), &fz_cur[j * ni + i]);
          heat_divupd(U3(a, k, j, i), fxc, fx_prev, fy_cur[i], fy_prev[i], fz_cur[j * ni + i],
                      fz_prev[j * ni + i], &U3(b, k, j, i));
          fx_prev = fxc;
        }
        double* t2 = fy_prev;
        fy_prev = fy_cur;
        fy_cur = t2;
      }
      double* t3 = fz_prev;
      fz_prev = fz_cur;
      fz_cur = t3;
    }
    free(fzw);
    free(fyw);
  }
  heat3d_wrap_parallel(b, nk, nj, ni, threads);
}

/* one step, in -> out (out's ghosts wrapped): the unit the CPU baseline times */
int lfo_heat3d_fused_step(const double* u_in, double* u_out, long nk, long nj, long ni, int threads) {
  heat3d_fused_step(u_in, u_out, nk, nj, ni, clamp_threads(threads));
  return 0;
}

int lfo_heat3d_fused(const double* u_in, double* u_out, long nk, long nj, long ni, int steps,
                     int threads) {
  const size_t n = (size_t)(nk + 2) * (nj + 2) * (ni + 2);
  threads = clamp_threads(threads);
  double* a = (double*)malloc(n * sizeof(double));
  double* b = (double*)malloc(n * sizeof(double));
  if (!a || !b) return 3;
  memcpy(a, u_in, n * sizeof(double));
  memcpy(b, u_in, n * sizeof(double));
  for (int s = 0; s < steps; ++s) {
    heat3d_fused_step(a, b, nk, nj, ni, threads);
    double* t = a;
    a = b;
    b = t;
  }
  memcpy(u_out, a, n * sizeof(double));
  free(a);
  free(b);
  return 0;
}
#undef U3

/* ========================================================================
 * Config 4: row1 -> col1 -> row2 -> col2, each (a+b+c)/3 in fp32.
 * Terminal layout: g_img extent (N+4)^2, base -2, replicate-padded by the
 * caller (clamp-to-edge as a ghost-cell convention); g_out N^2, base 0.
 * ====================================================================== */

#define IM(j, i) img[((j) + 2) * P + ((i) + 2)]

/* run_naive: r1 over rows [-2,N+2) x cols [-1,N+1); c1 over [-1,N+1)^2;
 * r2 over rows [-1,N+1) x cols [0,N); c2 over [0,N)^2. */
int lfo_box_naive(const float* img, float* out, long nj, long ni) {
  const long P = ni + 4;
  const long W = ni + 2;
  float* r1 = (float*)malloc((size_t)(nj + 4) * W * sizeof(float));
  float* c1 = (float*)malloc((size_t)(nj + 2) * W * sizeof(float));
  float* r2 = (float*)malloc((size_t)(nj + 2) * ni * sizeof(float));
  if (!r1 || !c1 || !r2) return 3;
#define R1(j, i) r1[((j) + 2) * W + ((i) + 1)]
#define C1(j, i) c1[((j) + 1) * W + ((i) + 1)]
#define R2(j, i) r2[((j) + 1) * ni + (i)]
  for (long j = -2; j < nj + 2; ++j)
    for (long i = -1; i < ni + 1; ++i) box3(IM(j, i - 1), IM(j, i), IM(j, i + 1), &R1(j, i));
  for (long j = -1; j < nj + 1; ++j)
    for (long i = -1; i < ni + 1; ++i) box3(R1(j - 1, i), R1(j, i), R1(j + 1, i), &C1(j, i));
  for (long j = -1; j < nj + 1; ++j)
    for (long i = 0; i < ni; ++i) box3(C1(j, i - 1), C1(j, i), C1(j, i + 1), &R2(j, i));
  for (long j = 0; j < nj; ++j)
    for (long i = 0; i < ni; ++i) box3(R2(j - 1, i), R2(j, i), R2(j + 1, i), &out[j * ni + i]);
#undef R1
#undef C1
#undef R2
  free(r1);
  free(c1);
  free(r2);
  return 0;
}

/* HFAV fused schedule for config 4: loop order (j,i); r1 leads by 2 rows,
 * c1/r2 by 1; windows r1 3 rows, c1 one row, r2 3 rows (minimal spans; the
 * reference's grouping quirk B-1 would widen r1 to 5). */
int lfo_box_fused(const float* img, float* out, long nj, long ni, int threads) {
  const long P = ni + 4;
  const long W = ni + 2;
  threads = clamp_threads(threads);
#pragma omp parallel num_threads(threads)
  {
    int nt = omp_get_num_threads(), t = omp_get_thread_num();
    long j0 = nj * t / nt, j1 = nj * (t + 1) / nt;
    float* buf = (float*)malloc((3 * W + W + 3 * ni) * sizeof(float));
    float* r1[3] = {buf, buf + W, buf + 2 * W};
    float* c1 = buf + 3 * W;
    float* r2[3] = {buf + 4 * W, buf + 4 * W + ni, buf + 4 * W + 2 * ni};
    /* prologue: r1 rows j0-2, j0-1, j0 ; c1/r2 rows j0-1 */
    for (int r = 0; r < 3; ++r) {
      long j = j0 - 2 + r;
      for (long i = -1; i < ni + 1; ++i) box3(IM(j, i - 1), IM(j, i), IM(j, i + 1), &r1[r][i + 1]);
    }
    for (int step = 0; step < 2; ++step) {
      /* c1 row (j0-1+step) from r1 rows, then r2 row */
      for (long i = -1; i < ni + 1; ++i) box3(r1[0][i + 1], r1[1][i + 1], r1[2][i + 1], &c1[i + 1]);
      for (long i = 0; i < ni; ++i) box3(c1[i], c1[i + 1], c1[i + 2], &r2[1 + step][i]);
      /* advance r1 window by one row */
      long jn = j0 + 1 + step;
      float* f = r1[0];
      r1[0] = r1[1];
      r1[1] = r1[2];
      r1[2] = f;
      for (long i = -1; i < ni + 1; ++i)
        box3(IM(jn, i - 1), IM(jn, i), IM(jn, i + 1), &r1[2][i + 1]);
    }
    /* now: r2[1] = row j0-1, r2[2] = row j0, r1 window = rows j0, j0+1, j0+2 */
    for (long j = j0; j < j1; ++j) {
      /* c1 row j+1 and r2 row j+1 */
      for (long i = -1; i < ni + 1; ++i) box3(r1[0][i + 1], r1[1][i + 1], r1[2][i + 1], &c1[i + 1]);
      float* rnew = r2[0];
      for (long i = 0; i < ni; ++i) box3(c1[i], c1[i + 1], c1[i + 2], &rnew[i]);
      r2[0] = r2[1];
      r2[1] = r2[2];
      r2[2] = rnew;
      for (long i = 0; i < ni; ++i) box3(r2[0][i], r2[1][i], r2[2][i], &out[j * ni + i]);
      /* r1 row j+3 for the next trip */
      if (j + 1 < j1) {
        long jn = j + 3;
        float* f = r1[0];
        r1[0] = r1[1];
        r1[1] = r1[2];
        r1[2] = f;
        for (long i = -1; i < ni + 1; ++i)
          box3(IM(jn, i - 1), IM(jn, i), IM(jn, i + 1), &r1[2][i + 1]);
      }
    }
    free(buf);
  }
  return 0;
}
#undef IM

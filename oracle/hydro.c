/*
 * CPU ORACLE (test infrastructure only) -- Hydro2D chain, BASELINE.json
 * configs[2] / configs[4].  Semantics of one step (specs/hydro2d.lf): the
 * x-sweep chain over every row the y-sweep reads (interior rows plus the two
 * reflective ghost rows on each side), then the y-sweep chain over the
 * interior, then the ghost ring of the new state refilled by reflection
 * (rho, E even; rho*u odd across i-faces; rho*v odd across j-faces).
 *
 *   lfo_hydro_naive  -- run_naive (R/SPEC.md:532-540): each of the 12 kernel
 *                       groups swept over its whole space into full arrays.
 *   lfo_hydro_fused  -- the HFAV fused nest (one (j,i) loop, row windows for
 *                       the x-swept state and the y intermediates, OpenMP over
 *                       row bands): the CPU reference path timed by bench.py.
 */
#include <omp.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"
#include "../paper_1710_08774_b200/userkernels/hydro_kernels.h"

#define AT(a, j, i) (a)[((long)(j) + 2) * P + ((i) + 2)]

/* reflective ghost refill of one state array: `odd_i`/`odd_j` negate */
static void reflect(double* a, long nj, long ni, int odd_j, int odd_i) {
  const long P = ni + 4;
  for (long j = 0; j < nj; ++j)
    for (int g = 0; g < 2; ++g) {
      AT(a, j, -1 - g) = odd_i ? -AT(a, j, g) : AT(a, j, g);
      AT(a, j, ni + g) = odd_i ? -AT(a, j, ni - 1 - g) : AT(a, j, ni - 1 - g);
    }
  for (int g = 0; g < 2; ++g)
    for (long i = -2; i < ni + 2; ++i) {
      AT(a, -1 - g, i) = odd_j ? -AT(a, g, i) : AT(a, g, i);
      AT(a, nj + g, i) = odd_j ? -AT(a, nj - 1 - g, i) : AT(a, nj - 1 - g, i);
    }
}

static void reflect_state(double* s[4], long nj, long ni) {
  reflect(s[0], nj, ni, 0, 0);
  reflect(s[1], nj, ni, 0, 1); /* rho*u */
  reflect(s[2], nj, ni, 1, 0); /* rho*v */
  reflect(s[3], nj, ni, 0, 0);
}

/* ======================================================================== */
/* run_naive                                                                 */
/* ======================================================================== */
int lfo_hydro_naive(const double* const in[4], double* const out[4], long nj, long ni, double dtdx, int steps) {
  const long P = ni + 4;
  const size_t n = (size_t)(nj + 4) * P;
  double* buf = (double*)malloc(n * sizeof(double) * (4 + 4 + 4 + 4 * 7 + 4 * 7));
  if (!buf) return 3;
  double* U[4];
  double* U1[4];
  double* U2[4];
  double *Q[4], *D[4], *M[4], *QP[4], *G[4], *F[4];
  double *YQ[4], *YD[4], *YM[4], *YP[4], *YG[4], *YF[4];
  double* p = buf;
  for (int v = 0; v < 4; ++v) { U[v] = p; p += n; }
  for (int v = 0; v < 4; ++v) { U1[v] = p; p += n; }
  for (int v = 0; v < 4; ++v) { U2[v] = p; p += n; }
  for (int v = 0; v < 4; ++v) {
    Q[v] = p; p += n; D[v] = p; p += n; M[v] = p; p += n; QP[v] = p; p += n;
    G[v] = p; p += n; F[v] = p; p += n; YQ[v] = p; p += n;
  }
  for (int v = 0; v < 4; ++v) {
    YD[v] = p; p += n; YM[v] = p; p += n; YP[v] = p; p += n; YG[v] = p; p += n; YF[v] = p; p += n;
    p += 2 * n;
  }
  for (int v = 0; v < 4; ++v) memcpy(U[v], in[v], n * sizeof(double));
  for (int s = 0; s < steps; ++s) {
    const long J0 = -2, J1 = nj + 2; /* rows the x-sweep covers */
    /* ---- x-sweep: constoprim_x over cols [-2, ni+2) */
    for (long j = J0; j < J1; ++j)
      for (long i = -2; i < ni + 2; ++i)
        hy_constoprim(AT(U[0], j, i), AT(U[1], j, i), AT(U[2], j, i), AT(U[3], j, i), &AT(Q[0], j, i),
                      &AT(Q[1], j, i), &AT(Q[2], j, i), &AT(Q[3], j, i));
    for (long j = J0; j < J1; ++j)
      for (long i = -1; i < ni + 1; ++i)
        hy_slope(AT(Q[0], j, i - 1), AT(Q[1], j, i - 1), AT(Q[2], j, i - 1), AT(Q[3], j, i - 1), AT(Q[0], j, i),
                 AT(Q[1], j, i), AT(Q[2], j, i), AT(Q[3], j, i), AT(Q[0], j, i + 1), AT(Q[1], j, i + 1),
                 AT(Q[2], j, i + 1), AT(Q[3], j, i + 1), &AT(D[0], j, i), &AT(D[1], j, i), &AT(D[2], j, i),
                 &AT(D[3], j, i));
    for (long j = J0; j < J1; ++j)
      for (long i = -1; i < ni + 1; ++i)
        hy_trace(AT(Q[0], j, i), AT(Q[1], j, i), AT(Q[2], j, i), AT(Q[3], j, i), AT(D[0], j, i), AT(D[1], j, i),
                 AT(D[2], j, i), AT(D[3], j, i), dtdx, &AT(M[0], j, i), &AT(M[1], j, i), &AT(M[2], j, i),
                 &AT(M[3], j, i), &AT(QP[0], j, i), &AT(QP[1], j, i), &AT(QP[2], j, i), &AT(QP[3], j, i));
    for (long j = J0; j < J1; ++j)
      for (long i = -1; i < ni; ++i)
        hy_riemann(AT(QP[0], j, i), AT(QP[1], j, i), AT(QP[2], j, i), AT(QP[3], j, i), AT(M[0], j, i + 1),
                   AT(M[1], j, i + 1), AT(M[2], j, i + 1), AT(M[3], j, i + 1), &AT(G[0], j, i), &AT(G[1], j, i),
                   &AT(G[2], j, i), &AT(G[3], j, i));
    for (long j = J0; j < J1; ++j)
      for (long i = -1; i < ni; ++i)
        hy_flux(AT(G[0], j, i), AT(G[1], j, i), AT(G[2], j, i), AT(G[3], j, i), &AT(F[0], j, i), &AT(F[1], j, i),
                &AT(F[2], j, i), &AT(F[3], j, i));
    for (long j = J0; j < J1; ++j)
      for (long i = 0; i < ni; ++i)
        hy_update(AT(U[0], j, i), AT(U[1], j, i), AT(U[2], j, i), AT(U[3], j, i), AT(F[0], j, i - 1),
                  AT(F[1], j, i - 1), AT(F[2], j, i - 1), AT(F[3], j, i - 1), AT(F[0], j, i), AT(F[1], j, i),
                  AT(F[2], j, i), AT(F[3], j, i), dtdx, &AT(U1[0], j, i), &AT(U1[1], j, i), &AT(U1[2], j, i),
                  &AT(U1[3], j, i));
    /* ---- y-sweep on the x-swept state: normal momentum rho*v (U1[2]) */
    for (long j = -2; j < nj + 2; ++j)
      for (long i = 0; i < ni; ++i)
        hy_constoprim(AT(U1[0], j, i), AT(U1[2], j, i), AT(U1[1], j, i), AT(U1[3], j, i), &AT(YQ[0], j, i),
                      &AT(YQ[1], j, i), &AT(YQ[2], j, i), &AT(YQ[3], j, i));
    for (long j = -1; j < nj + 1; ++j)
      for (long i = 0; i < ni; ++i)
        hy_slope(AT(YQ[0], j - 1, i), AT(YQ[1], j - 1, i), AT(YQ[2], j - 1, i), AT(YQ[3], j - 1, i),
                 AT(YQ[0], j, i), AT(YQ[1], j, i), AT(YQ[2], j, i), AT(YQ[3], j, i), AT(YQ[0], j + 1, i),
                 AT(YQ[1], j + 1, i), AT(YQ[2], j + 1, i), AT(YQ[3], j + 1, i), &AT(YD[0], j, i), &AT(YD[1], j, i),
                 &AT(YD[2], j, i), &AT(YD[3], j, i));
    for (long j = -1; j < nj + 1; ++j)
      for (long i = 0; i < ni; ++i)
        hy_trace(AT(YQ[0], j, i), AT(YQ[1], j, i), AT(YQ[2], j, i), AT(YQ[3], j, i), AT(YD[0], j, i),
                 AT(YD[1], j, i), AT(YD[2], j, i), AT(YD[3], j, i), dtdx, &AT(YM[0], j, i), &AT(YM[1], j, i),
                 &AT(YM[2], j, i), &AT(YM[3], j, i), &AT(YP[0], j, i), &AT(YP[1], j, i), &AT(YP[2], j, i),
                 &AT(YP[3], j, i));
    for (long j = -1; j < nj; ++j)
      for (long i = 0; i < ni; ++i)
        hy_riemann(AT(YP[0], j, i), AT(YP[1], j, i), AT(YP[2], j, i), AT(YP[3], j, i), AT(YM[0], j + 1, i),
                   AT(YM[1], j + 1, i), AT(YM[2], j + 1, i), AT(YM[3], j + 1, i), &AT(YG[0], j, i),
                   &AT(YG[1], j, i), &AT(YG[2], j, i), &AT(YG[3], j, i));
    for (long j = -1; j < nj; ++j)
      for (long i = 0; i < ni; ++i)
        hy_flux(AT(YG[0], j, i), AT(YG[1], j, i), AT(YG[2], j, i), AT(YG[3], j, i), &AT(YF[0], j, i),
                &AT(YF[1], j, i), &AT(YF[2], j, i), &AT(YF[3], j, i));
    for (long j = 0; j < nj; ++j)
      for (long i = 0; i < ni; ++i)
        hy_update(AT(U1[0], j, i), AT(U1[2], j, i), AT(U1[1], j, i), AT(U1[3], j, i), AT(YF[0], j - 1, i),
                  AT(YF[1], j - 1, i), AT(YF[2], j - 1, i), AT(YF[3], j - 1, i), AT(YF[0], j, i), AT(YF[1], j, i),
                  AT(YF[2], j, i), AT(YF[3], j, i), dtdx, &AT(U2[0], j, i), &AT(U2[2], j, i), &AT(U2[1], j, i),
                  &AT(U2[3], j, i));
    reflect_state(U2, nj, ni);
    for (int v = 0; v < 4; ++v) memcpy(U[v], U2[v], n * sizeof(double));
  }
  for (int v = 0; v < 4; ++v) memcpy(out[v], U[v], n * sizeof(double));
  free(buf);
  return 0;
}

/* ======================================================================== */
/* HFAV fused schedule                                                       */
/* ======================================================================== */

/* x-sweep of one row r into x1[4] (interior columns), 1-D windows along i */
static void xsweep_row(const double* const U[4], long P, long r, long ni, double dtdx, double* x1[4],
                       double* scratch) {
  /* scratch: prims (ni+4) x4, qm/qp (ni+2) x8, flux (ni+1) x4 */
  double* q[4];
  double* qm[4];
  double* qp[4];
  double* f[4];
  double* s = scratch;
  for (int v = 0; v < 4; ++v) { q[v] = s; s += ni + 4; }
  for (int v = 0; v < 4; ++v) { qm[v] = s; s += ni + 2; qp[v] = s; s += ni + 2; }
  for (int v = 0; v < 4; ++v) { f[v] = s; s += ni + 1; }
  const double* row[4];
  for (int v = 0; v < 4; ++v) row[v] = U[v] + (r + 2) * P + 2; /* logical col 0 */
  for (long i = -2; i < ni + 2; ++i)
    hy_constoprim(row[0][i], row[1][i], row[2][i], row[3][i], &q[0][i + 2], &q[1][i + 2], &q[2][i + 2],
                  &q[3][i + 2]);
  for (long i = -1; i < ni + 1; ++i) {
    double d0, d1, d2, d3;
    const long c = i + 2;
    hy_slope(q[0][c - 1], q[1][c - 1], q[2][c - 1], q[3][c - 1], q[0][c], q[1][c], q[2][c], q[3][c], q[0][c + 1],
             q[1][c + 1], q[2][c + 1], q[3][c + 1], &d0, &d1, &d2, &d3);
    hy_trace(q[0][c], q[1][c], q[2][c], q[3][c], d0, d1, d2, d3, dtdx, &qm[0][i + 1], &qm[1][i + 1],
             &qm[2][i + 1], &qm[3][i + 1], &qp[0][i + 1], &qp[1][i + 1], &qp[2][i + 1], &qp[3][i + 1]);
  }
  for (long i = -1; i < ni; ++i) {
    double g0, g1, g2, g3;
    hy_riemann(qp[0][i + 1], qp[1][i + 1], qp[2][i + 1], qp[3][i + 1], qm[0][i + 2], qm[1][i + 2], qm[2][i + 2],
               qm[3][i + 2], &g0, &g1, &g2, &g3);
    hy_flux(g0, g1, g2, g3, &f[0][i + 1], &f[1][i + 1], &f[2][i + 1], &f[3][i + 1]);
  }
  for (long i = 0; i < ni; ++i)
    hy_update(row[0][i], row[1][i], row[2][i], row[3][i], f[0][i], f[1][i], f[2][i], f[3][i], f[0][i + 1],
              f[1][i + 1], f[2][i + 1], f[3][i + 1], dtdx, &x1[0][i], &x1[1][i], &x1[2][i], &x1[3][i]);
}

static void hydro_fused_step(const double* const U[4], double* const V[4], long nj, long ni, double dtdx,
                             int threads) {
  const long P = ni + 4;
#pragma omp parallel num_threads(threads)
  {
    int nt = omp_get_num_threads(), t = omp_get_thread_num();
    long j0 = nj * t / nt, j1 = nj * (t + 1) / nt;
    /* windows: x-swept rows (3), y prims (3), y qp (2), y flux (2); all 4 vars x ni */
    const long W = ni;
    double* mem = (double*)malloc(sizeof(double) * (4 * W * (3 + 3 + 2 + 2 + 1) + 16 * (ni + 4)));
    double *x1[3][4], *yq[3][4], *yp[2][4], *yf[2][4], *ym[4];
    double* s = mem;
    for (int k = 0; k < 3; ++k)
      for (int v = 0; v < 4; ++v) { x1[k][v] = s; s += W; }
    for (int k = 0; k < 3; ++k)
      for (int v = 0; v < 4; ++v) { yq[k][v] = s; s += W; }
    for (int k = 0; k < 2; ++k)
      for (int v = 0; v < 4; ++v) { yp[k][v] = s; s += W; }
    for (int k = 0; k < 2; ++k)
      for (int v = 0; v < 4; ++v) { yf[k][v] = s; s += W; }
    for (int v = 0; v < 4; ++v) { ym[v] = s; s += W; }
    double* scratch = s;
    /* march rows r = j0-2 .. j1+1: x-sweep row r, y prim row r, y slope/trace
       row r-1, y riemann/flux face (r-2)+1/2, update row r-2 */
    for (long r = j0 - 2; r < j1 + 2; ++r) {
      const long k = r - (j0 - 2); /* 0-based trip */
      double** xr = x1[k % 3];
      xsweep_row(U, P, r, ni, dtdx, xr, scratch);
      double** qr = yq[k % 3];
      for (long i = 0; i < ni; ++i)
        hy_constoprim(xr[0][i], xr[2][i], xr[1][i], xr[3][i], &qr[0][i], &qr[1][i], &qr[2][i], &qr[3][i]);
      if (k < 2) continue;
      double** qm1 = yq[(k - 1) % 3];
      double** qm2 = yq[(k - 2) % 3];
      double** pp = yp[(k - 1) & 1]; /* qp of row r-1 */
      for (long i = 0; i < ni; ++i) {
        double d0, d1, d2, d3;
        hy_slope(qm2[0][i], qm2[1][i], qm2[2][i], qm2[3][i], qm1[0][i], qm1[1][i], qm1[2][i], qm1[3][i], qr[0][i],
                 qr[1][i], qr[2][i], qr[3][i], &d0, &d1, &d2, &d3);
        hy_trace(qm1[0][i], qm1[1][i], qm1[2][i], qm1[3][i], d0, d1, d2, d3, dtdx, &ym[0][i], &ym[1][i],
                 &ym[2][i], &ym[3][i], &pp[0][i], &pp[1][i], &pp[2][i], &pp[3][i]);
      }
      if (k < 3) continue;
      double** pprev = yp[k & 1]; /* qp of row r-2 */
      double** fcur = yf[k & 1];  /* flux of face (r-2)+1/2 */
      for (long i = 0; i < ni; ++i) {
        double g0, g1, g2, g3;
        hy_riemann(pprev[0][i], pprev[1][i], pprev[2][i], pprev[3][i], ym[0][i], ym[1][i], ym[2][i], ym[3][i],
                   &g0, &g1, &g2, &g3);
        hy_flux(g0, g1, g2, g3, &fcur[0][i], &fcur[1][i], &fcur[2][i], &fcur[3][i]);
      }
      if (k < 4) continue;
      double** fprev = yf[(k - 1) & 1];
      double** xu = x1[(k - 2) % 3]; /* x-swept row r-2 */
      const long jo = r - 2;
      for (long i = 0; i < ni; ++i)
        hy_update(xu[0][i], xu[2][i], xu[1][i], xu[3][i], fprev[0][i], fprev[1][i], fprev[2][i], fprev[3][i],
                  fcur[0][i], fcur[1][i], fcur[2][i], fcur[3][i], dtdx, &AT(V[0], jo, i), &AT(V[2], jo, i),
                  &AT(V[1], jo, i), &AT(V[3], jo, i));
    }
    free(mem);
  }
  double* Vm[4] = {V[0], V[1], V[2], V[3]};
  reflect_state(Vm, nj, ni);
}

int lfo_hydro_fused_step(const double* const in[4], double* const out[4], long nj, long ni, double dtdx,
                         int threads) {
  if (threads <= 0) threads = omp_get_max_threads();
  hydro_fused_step(in, out, nj, ni, dtdx, threads);
  return 0;
}

int lfo_hydro_fused(const double* const in[4], double* const out[4], long nj, long ni, double dtdx, int steps,
                    int threads) {
  const size_t n = (size_t)(nj + 4) * (ni + 4);
  if (threads <= 0) threads = omp_get_max_threads();
  double* buf = (double*)malloc(8 * n * sizeof(double));
  if (!buf) return 3;
  double *A[4], *B[4];
  for (int v = 0; v < 4; ++v) {
    A[v] = buf + v * n;
    B[v] = buf + (4 + v) * n;
    memcpy(A[v], in[v], n * sizeof(double));
  }
  for (int s = 0; s < steps; ++s) {
    hydro_fused_step((const double* const*)A, B, nj, ni, dtdx, threads);
    for (int v = 0; v < 4; ++v) {
      double* t = A[v];
      A[v] = B[v];
      B[v] = t;
    }
  }
  for (int v = 0; v < 4; ++v) memcpy(out[v], A[v], n * sizeof(double));
  free(buf);
  return 0;
}
/* ======================================================================== */
/* adaptive time step (specs/hydro2d_adaptive.lf)                            */
/* ======================================================================== */

/* the CFL reduction over the interior of a state: cfl_init, then cfl_max of
 * every cell's cfl_speed in loop order (j, i) -- run_naive's sequential sweep
 * of the associative group -- and cfl_dt */
static double cfl_dtdx(double* const U[4], long nj, long ni) {
  const long P = ni + 4;
  double m;
  hy_cfl_init(&m);
  for (long j = 0; j < nj; ++j)
    for (long i = 0; i < ni; ++i) {
      double sp;
      hy_cfl_speed(AT(U[0], j, i), AT(U[1], j, i), AT(U[2], j, i), AT(U[3], j, i), &sp);
      hy_cfl_max(m, sp, &m);
    }
  double d;
  hy_cfl_dt(m, &d);
  return d;
}

/* `steps` adaptive steps: step s runs with dt/dx_s (dtdx_io in: dt/dx_0), and
 * dt/dx_{s+1} comes from the CFL condition on its result; dtdx_io out: the
 * dt/dx the state after the last step gives (the chain's g_dtdx_n goal) */
int lfo_hydro_adaptive(const double* const in[4], double* const out[4], long nj, long ni, double* dtdx_io, int steps,
                       int fused, int threads) {
  const size_t n = (size_t)(nj + 4) * (ni + 4);
  if (threads <= 0) threads = omp_get_max_threads();
  double* buf = (double*)malloc(8 * n * sizeof(double));
  if (!buf) return 3;
  double *A[4], *B[4];
  for (int v = 0; v < 4; ++v) {
    A[v] = buf + v * n;
    B[v] = buf + (4 + v) * n;
    memcpy(A[v], in[v], n * sizeof(double));
  }
  double dtdx = *dtdx_io;
  for (int s = 0; s < steps; ++s) {
    int st = fused ? (hydro_fused_step((const double* const*)A, B, nj, ni, dtdx, threads), 0)
                   : lfo_hydro_naive((const double* const*)A, B, nj, ni, dtdx, 1);
    if (st) {
      free(buf);
      return st;
    }
    dtdx = cfl_dtdx(B, nj, ni);
    for (int v = 0; v < 4; ++v) {
      double* t = A[v];
      A[v] = B[v];
      B[v] = t;
    }
  }
  for (int v = 0; v < 4; ++v) memcpy(out[v], A[v], n * sizeof(double));
  *dtdx_io = dtdx;
  free(buf);
  return 0;
}
#undef AT

/*
 * User kernels of the Hydro2D chain (BASELINE.json configs[2] / configs[4]):
 * compressible Euler, MUSCL-Hancock Godunov scheme, directionally split,
 * gamma = 1.4, fp64.  Authored from textbook numerics for this framework (the
 * CEA Hydro2D sources are not part of the reference snapshot).
 *
 * Each sweep is the six-kernel chain the paper describes (R/PAPER.md:468-486):
 *   constoprim -> slope (minmod) -> trace (half-step predictor) ->
 *   riemann (two-shock iterative solver, fixed 10 Newton steps) ->
 *   flux -> update (conservative)
 * written for a generic "normal" direction: (r, mn, mt, e) = density, normal
 * momentum, transverse momentum, total energy.  The x-sweep passes
 * (rho, rho*u, rho*v, E) and the y-sweep (rho, rho*v, rho*u, E).
 *
 * As with stencil_kernels.h, the same source runs in the CPU oracle and is
 * inlined into the sm_100a executor.  Only + - * / sqrt fma fabs and
 * comparisons are used -- each correctly rounded on both sides, fma() being
 * the single-rounding fused multiply-add of C99 / IEEE 754-2008 -- with fixed
 * iteration counts and no early exits, so the two schedules agree bit for bit.
 * The expressions are written in fused multiply-add form where a product
 * feeds a sum (as an optimising compiler would contract them), and every
 * quantity the solver needs more than once is formed once:
 *   * the Lagrangian wave speed of a shock, W = C sqrt(1 + k (p* - p)/p), is
 *     carried as W^2 = gamma rho (p + k (p* - p)) -- one fma per Newton step
 *     and no division by p (gamma k = (gamma+1)/2);
 *   * the Newton step z_l z_r / (z_l + z_r) (u*_l - u*_r), z = 2W^3/(W^2+C^2),
 *     is written over one common denominator (2 sqrt + 1 reciprocal per step);
 *   * the star density rho W^2 / (W^2 + rho (p - p*)) is one quotient;
 *   * every quotient a / b is formed as a * (1/b) from the correctly rounded
 *     reciprocal (two roundings; b > 0 in every case, so the sign of a zero
 *     numerator carries through exactly as in a / b), and the Newton update
 *     p* + num/den as fma(num, 1/den, p*).
 */
#ifndef LF_USERKERNELS_HYDRO_H
#define LF_USERKERNELS_HYDRO_H

/* Reciprocals and square roots go through HY_RCP / HY_SQRT.  By default they
 * are the plain operators (1.0 / b, sqrt).  An sm_100a executor may include this header a
 * second time, inside its own namespace and with HY_FAST defined (after
 * csrc/exec/fastmath.cuh): every function that takes a reciprocal or a root then
 * takes a trailing `unsigned* hy_bad`, uses the branch-free fast paths of
 * fastmath.cuh, and sets *hy_bad when an operand left the range where those
 * equal the IEEE operation -- the executor then recomputes with the plain
 * build.  Same expressions, same operation order: the arithmetic is unchanged. */
#undef HY_BAD_PARAM
#undef HY_BAD_ARG
#undef HY_RCP
#undef HY_SQRT
#ifdef HY_FAST
#define HY_BAD_PARAM , unsigned* hy_bad
#define HY_BAD_ARG , hy_bad
#define HY_RCP(b) lf_rcp_fast((b), hy_bad)
#define HY_SQRT(x) lf_sqrt_fast((x), hy_bad)
#else
#define HY_BAD_PARAM
#define HY_BAD_ARG
#define HY_RCP(b) (1.0 / (b))
#define HY_SQRT(x) sqrt(x)
#endif

#ifndef LF_HD
#if defined(__CUDACC__) || defined(__CUDACC_RTC__)
#define LF_HD __host__ __device__ __forceinline__
#else
#include <math.h>
#define LF_HD static inline
#endif
#endif

/* Physical constants.  An executor may define them first as names bound to
 * the same values (e.g. device constant memory, so they are instruction
 * operands instead of rematerialised 64-bit immediates). */
#ifndef HY_GAMMA
#define HY_GAMMA 1.4
#define HY_GM1 0.4         /* gamma - 1 */
#define HY_GOGM1 3.5       /* gamma / (gamma - 1) */
#define HY_GK 1.2          /* gamma k = gamma (gamma+1)/(2 gamma) = (gamma+1)/2 */
#define HY_SMALLR 1e-10
#define HY_SMALLP 1e-12
#define HY_SMALLC 1e-10
#endif
#define HY_NITER 10

LF_HD double hy_max(double a, double b) { return a > b ? a : b; }
LF_HD double hy_min(double a, double b) { return a < b ? a : b; }
/* conservative -> primitive (density, normal & transverse velocity, pressure):
 * p = (gamma-1) (e - |m|^2 / (2 rho)) */
LF_HD void hy_constoprim(double r, double mn, double mt, double e, double* qr, double* qn, double* qt,
                         double* qp HY_BAD_PARAM) {
  const double rr = hy_max(r, HY_SMALLR);
  const double inv = HY_RCP(rr);
  const double m2 = fma(mn, mn, mt * mt);
  *qr = rr;
  *qn = mn * inv;
  *qt = mt * inv;
  *qp = hy_max(HY_GM1 * fma(-0.5 * inv, m2, e), HY_SMALLP);
}

/* minmod-limited slope from the left and right differences */
LF_HD double hy_minmod(double dl, double dr) {
  if (dl * dr <= 0.0) return 0.0;
  return fabs(dl) < fabs(dr) ? dl : dr;
}

LF_HD void hy_slope(double rm, double nm, double tm, double pm, double r0, double n0, double t0, double p0,
                    double rp, double np, double tp, double pp, double* dr, double* dn, double* dt, double* dp) {
  *dr = hy_minmod(r0 - rm, rp - r0);
  *dn = hy_minmod(n0 - nm, np - n0);
  *dt = hy_minmod(t0 - tm, tp - t0);
  *dp = hy_minmod(p0 - pm, pp - p0);
}

/* MUSCL-Hancock predictor: evolve the cell's primitive state by half a time
 * step with the primitive Euler equations, then extrapolate to the left
 * (minus) and right (plus) faces: q -/+ dq/2 + dt/2 A(q) dq/dx. */
LF_HD void hy_trace(double r, double n, double t, double p, double dr, double dn, double dt, double dp,
                    double dtdx, double* mr, double* mn, double* mt, double* mp, double* pr, double* pn,
                    double* pt, double* pp HY_BAD_PARAM) {
  const double h = -0.5 * dtdx;
  const double sr = h * fma(n, dr, r * dn);
  const double sn = h * fma(n, dn, dp * HY_RCP(r));
  const double st = h * (n * dt);
  const double sp = h * fma(n, dp, (HY_GAMMA * p) * dn);
  *mr = hy_max(fma(-0.5, dr, r) + sr, HY_SMALLR);
  *mn = fma(-0.5, dn, n) + sn;
  *mt = fma(-0.5, dt, t) + st;
  *mp = hy_max(fma(-0.5, dp, p) + sp, HY_SMALLP);
  *pr = hy_max(fma(0.5, dr, r) + sr, HY_SMALLR);
  *pn = fma(0.5, dn, n) + sn;
  *pt = fma(0.5, dt, t) + st;
  *pp = hy_max(fma(0.5, dp, p) + sp, HY_SMALLP);
}

/* Godunov state at a face from left/right primitive states: two-shock
 * approximation of the exact Riemann problem, p* by HY_NITER Newton steps,
 * then sampling at x/t = 0 with a linear fan.
 *
 * With W^2 = A(p*) = gamma rho (p + k (p* - p)) = C^2 + gamma k rho (p* - p),
 * C^2 = gamma p rho, the step p* += z_l z_r / (z_l + z_r) (u*_l - u*_r),
 * u*_l - u*_r = (nl - nr) - (p*-pl)/W_l - (p*-pr)/W_r and
 * z = 2 W^3 / (W^2 + C^2), is over one common denominator
 *   A_l A_r [ (nl-nr) W_l W_r - (p*-pl) W_r - (p*-pr) W_l ]
 *   ----------------------------------------------------------------
 *   (A_l + C_l^2)/2 W_r A_r + (A_r + C_r^2)/2 W_l A_l
 *
 * The solver is split into init / newton / sample so an executor can advance
 * two independent problems in one loop (hy_riemann is exactly
 * init + HY_NITER x newton + sample, so results are identical). */
typedef struct {
  double nl, pl, nr, pr; /* normal velocities and pressures */
  double dn;             /* nl - nr */
  double cl2, cr2;       /* C^2 = gamma p rho (Lagrangian sound speed squared) */
  double gkl, gkr;       /* gamma k rho: dA/dp* */
  double hcl2, hcr2;     /* C^2 / 2 */
} hy_rp;

LF_HD double hy_riemann_init(double rl, double nl, double pl, double rr, double nr, double pr, hy_rp* c HY_BAD_PARAM) {
  c->nl = nl;
  c->pl = pl;
  c->nr = nr;
  c->pr = pr;
  c->dn = nl - nr;
  c->cl2 = (HY_GAMMA * pl) * rl;
  c->cr2 = (HY_GAMMA * pr) * rr;
  c->gkl = HY_GK * rl;
  c->gkr = HY_GK * rr;
  c->hcl2 = 0.5 * c->cl2;
  c->hcr2 = 0.5 * c->cr2;
  /* acoustic (linearised) first guess */
  const double cl = HY_SQRT(c->cl2);
  const double cr = HY_SQRT(c->cr2);
  return hy_max((fma(cr, pl, cl * pr) + (cl * cr) * c->dn) * HY_RCP(cl + cr), HY_SMALLP);
}

LF_HD double hy_riemann_newton(const hy_rp* c, double ps HY_BAD_PARAM) {
  const double dl = ps - c->pl, dr = ps - c->pr;
  const double al = fma(c->gkl, dl, c->cl2);
  const double ar = fma(c->gkr, dr, c->cr2);
  const double wl = HY_SQRT(al);
  const double wr = HY_SQRT(ar);
  const double inner = fma(fma(c->dn, wl, -dl), wr, -(dr * wl));
  const double num = (al * ar) * inner;
  const double den = fma(fma(0.5, al, c->hcl2), wr * ar, fma(0.5, ar, c->hcr2) * (wl * al));
  return hy_max(fma(num, HY_RCP(den), ps), HY_SMALLP);
}

LF_HD void hy_riemann_sample(const hy_rp* c, double ps, double rl, double tl, double rr, double tr, double* gr,
                             double* gn, double* gt, double* gp HY_BAD_PARAM) {
  const double al = fma(c->gkl, ps - c->pl, c->cl2);
  const double ar = fma(c->gkr, ps - c->pr, c->cr2);
  const double wl = HY_SQRT(al);
  const double wr = HY_SQRT(ar);
  const double us = (fma(wl, c->nl, wr * c->nr) + (c->pl - c->pr)) * HY_RCP(wl + wr);
  const int left = us > 0.0;
  const double ro = left ? rl : rr;
  const double uo = left ? c->nl : -c->nr; /* velocity along the sampled wave direction */
  const double po = left ? c->pl : c->pr;
  const double wo = left ? wl : wr;
  const double ao = left ? al : ar;        /* W^2 of the sampled wave */
  const double to = left ? tl : tr;
  const double uss = left ? us : -us;
  const double iro = HY_RCP(ro);
  const double co = HY_SQRT((HY_GAMMA * po) * iro);
  const double rstar = hy_max((ro * ao) * HY_RCP(fma(ro, po - ps, ao)), HY_SMALLR);
  const double cstar = HY_SQRT((HY_GAMMA * ps) * HY_RCP(rstar));
  double spout = co - uo;
  double spin = cstar - uss;
  if (ps >= po) {
    const double ushock = fma(wo, iro, -uo);
    spout = ushock;
    spin = ushock;
  }
  const double scr = hy_max(spout - spin, HY_SMALLC + fabs(spout + spin));
  const double frac = hy_min(hy_max(fma(0.5, (spout + spin) * HY_RCP(scr), 0.5), 0.0), 1.0);
  double r = fma(frac, rstar - ro, ro);
  double u = fma(frac, uss - uo, uo);
  double p = fma(frac, ps - po, po);
  if (spout < 0.0) {
    r = ro;
    u = uo;
    p = po;
  }
  if (spin > 0.0) {
    r = rstar;
    u = uss;
    p = ps;
  }
  *gr = r;
  *gn = left ? u : -u;
  *gt = to;
  *gp = p;
}

LF_HD void hy_riemann(double rl, double nl, double tl, double pl, double rr, double nr, double tr, double pr,
                      double* gr, double* gn, double* gt, double* gp HY_BAD_PARAM) {
  hy_rp c;
  double ps = hy_riemann_init(rl, nl, pl, rr, nr, pr, &c HY_BAD_ARG);
  for (int it = 0; it < HY_NITER; ++it) ps = hy_riemann_newton(&c, ps HY_BAD_ARG);
  hy_riemann_sample(&c, ps, rl, tl, rr, tr, gr, gn, gt, gp HY_BAD_ARG);
}

/* conservative flux through the face from the Godunov state:
 * (rho u, rho u^2 + p, rho u t, u (E + p)), E + p = gamma/(gamma-1) p + rho |u|^2 / 2 */
LF_HD void hy_flux(double r, double n, double t, double p, double* fr, double* fn, double* ft, double* fe) {
  const double m = r * n;
  const double ke = (0.5 * r) * fma(n, n, t * t);
  *fr = m;
  *fn = fma(m, n, p);
  *ft = m * t;
  *fe = n * fma(p, HY_GOGM1, ke);
}

/* conservative update of one cell from its two face fluxes */
LF_HD void hy_update(double r, double mn, double mt, double e, double frm, double fnm, double ftm, double fem,
                     double frp, double fnp, double ftp, double fep, double dtdx, double* ro, double* no,
                     double* to, double* eo) {
  *ro = fma(dtdx, frm - frp, r);
  *no = fma(dtdx, fnm - fnp, mn);
  *to = fma(dtdx, ftm - ftp, mt);
  *eo = fma(dtdx, fem - fep, e);
}

/* ---- adaptive time step (specs/hydro2d_adaptive.lf): the CFL condition ---- */
#ifndef HY_CFL
#define HY_CFL 0.5
#endif

/* fastest signal speed of a cell, max(|u|, |v|) + c with c = sqrt(gamma p / rho) */
LF_HD void hy_cfl_speed(double r, double mx, double my, double e, double* s HY_BAD_PARAM) {
  double qr, qu, qv, qp;
  hy_constoprim(r, mx, my, e, &qr, &qu, &qv, &qp HY_BAD_ARG);
  const double c = HY_SQRT((HY_GAMMA * qp) * HY_RCP(qr));
  *s = hy_max(fabs(qu), fabs(qv)) + c;
}
/* the reduction: seed, combine (exact and order-independent), and dt/dx */
LF_HD void hy_cfl_init(double* m) { *m = 0.0; }
LF_HD void hy_cfl_max(double c, double s, double* o) { *o = hy_max(c, s); }
LF_HD void hy_cfl_dt(double m, double* d) { *d = HY_CFL / m; }

#endif

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
 * inlined into the sm_100a executor.  Only + - * / sqrt fabs and comparisons
 * are used (all correctly rounded on both sides), fixed iteration counts, no
 * early exits -- so the two schedules agree bit for bit.
 */
#ifndef LF_USERKERNELS_HYDRO_H
#define LF_USERKERNELS_HYDRO_H

/* Divisions and square roots go through HY_QUOT / HY_SQRT.  By default they
 * are the plain operators.  An sm_100a executor may include this header a
 * second time, inside its own namespace and with HY_FAST defined (after
 * csrc/exec/fastmath.cuh): every function that divides or takes a root then
 * takes a trailing `unsigned* hy_bad`, uses the branch-free fast paths of
 * fastmath.cuh, and sets *hy_bad when an operand left the range where those
 * equal the IEEE operation -- the executor then recomputes with the plain
 * build.  Same expressions, same operation order: the arithmetic is unchanged. */
#undef HY_BAD_PARAM
#undef HY_BAD_ARG
#undef HY_QUOT
#undef HY_SQRT
#ifdef HY_FAST
#define HY_BAD_PARAM , unsigned* hy_bad
#define HY_BAD_ARG , hy_bad
#define HY_QUOT(a, b) lf_div_fast((a), (b), hy_bad)
#define HY_SQRT(x) lf_sqrt_fast((x), hy_bad)
#else
#define HY_BAD_PARAM
#define HY_BAD_ARG
#define HY_QUOT(a, b) ((a) / (b))
#define HY_SQRT(x) sqrt(x)
#endif

#if defined(__CUDACC__)
#define LF_HD __host__ __device__ __forceinline__
#else
#include <math.h>
#define LF_HD static inline
#endif

#define HY_GAMMA 1.4
#define HY_SMALLR 1e-10
#define HY_SMALLP 1e-12
#define HY_SMALLC 1e-10
#define HY_NITER 10

LF_HD double hy_max(double a, double b) { return a > b ? a : b; }
/* a / b for a denominator that is finite and nonzero (every division of this
 * chain): a zero numerator returns a * b, which is the same signed zero as the
 * quotient.  Keeps the exactly-zero differences of states at rest (velocities,
 * pressure jumps, slopes) off the device's division slow path. */
LF_HD double hy_div(double a, double b HY_BAD_PARAM) {
#ifdef HY_FAST
  unsigned slow = 0;
  const double q = lf_div_fast(a, b, &slow);
  *hy_bad |= a == 0.0 ? 0u : slow;
  return a == 0.0 ? a * b : q;
#else
  if (a == 0.0) return a * b;
  return a / b;
#endif
}
LF_HD double hy_min(double a, double b) { return a < b ? a : b; }

/* conservative -> primitive (density, normal & transverse velocity, pressure) */
LF_HD void hy_constoprim(double r, double mn, double mt, double e, double* qr, double* qn, double* qt,
                         double* qp HY_BAD_PARAM) {
  const double rr = hy_max(r, HY_SMALLR);
  const double inv = HY_QUOT(1.0, rr);
  const double un = mn * inv;
  const double ut = mt * inv;
  const double ek = 0.5 * rr * (un * un + ut * ut);
  *qr = rr;
  *qn = un;
  *qt = ut;
  *qp = hy_max((HY_GAMMA - 1.0) * (e - ek), HY_SMALLP);
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
 * (minus) and right (plus) faces. */
LF_HD void hy_trace(double r, double n, double t, double p, double dr, double dn, double dt, double dp,
                    double dtdx, double* mr, double* mn, double* mt, double* mp, double* pr, double* pn,
                    double* pt, double* pp HY_BAD_PARAM) {
  const double h = -0.5 * dtdx;
  const double sr = h * (n * dr + r * dn);
  const double sn = h * (n * dn + hy_div(dp, r HY_BAD_ARG));
  const double st = h * (n * dt);
  const double sp = h * (n * dp + HY_GAMMA * p * dn);
  *mr = hy_max(r - 0.5 * dr + sr, HY_SMALLR);
  *mn = n - 0.5 * dn + sn;
  *mt = t - 0.5 * dt + st;
  *mp = hy_max(p - 0.5 * dp + sp, HY_SMALLP);
  *pr = hy_max(r + 0.5 * dr + sr, HY_SMALLR);
  *pn = n + 0.5 * dn + sn;
  *pt = t + 0.5 * dt + st;
  *pp = hy_max(p + 0.5 * dp + sp, HY_SMALLP);
}

/* Godunov state at a face from left/right primitive states: two-shock
 * approximation of the exact Riemann problem, p* by HY_NITER Newton steps on
 * the Lagrangian wave speeds w = c*sqrt(1 + k (p*-p)/p), then sampling at
 * x/t = 0 with a linear fan.  z = 2w^3/(w^2+c^2) enters only through
 * z_l z_r / (z_l + z_r) = 1 / (1/z_l + 1/z_r), and the step is written over
 * one common denominator, so a Newton step costs 2 sqrt + 1 division.
 *
 * The solver is split into init / newton / sample so an executor can advance
 * two independent problems in one loop (hy_riemann is exactly
 * init + HY_NITER x newton + sample, so results are identical). */
typedef struct {
  double nl, pl, nr, pr;       /* normal velocities and pressures */
  double cl, cr, cl2, cr2;     /* Lagrangian sound speeds rho*c and squares */
  double kpl, kpr;             /* (gamma+1)/(2 gamma) / p */
} hy_rp;

LF_HD double hy_riemann_init(double rl, double nl, double pl, double rr, double nr, double pr, hy_rp* c HY_BAD_PARAM) {
  const double k = (HY_GAMMA + 1.0) / (2.0 * HY_GAMMA);
  c->nl = nl;
  c->pl = pl;
  c->nr = nr;
  c->pr = pr;
  c->cl = HY_SQRT(HY_GAMMA * pl * rl);
  c->cr = HY_SQRT(HY_GAMMA * pr * rr);
  c->cl2 = c->cl * c->cl;
  c->cr2 = c->cr * c->cr;
  c->kpl = HY_QUOT(k, pl);
  c->kpr = HY_QUOT(k, pr);
  return hy_max(HY_QUOT(c->cr * pl + c->cl * pr + c->cl * c->cr * (nl - nr), c->cl + c->cr), HY_SMALLP);
}

LF_HD double hy_riemann_newton(const hy_rp* c, double ps HY_BAD_PARAM) {
  const double wl = c->cl * HY_SQRT(1.0 + c->kpl * (ps - c->pl));
  const double wr = c->cr * HY_SQRT(1.0 + c->kpr * (ps - c->pr));
  /* (u*_l - u*_r) / (1/z_l + 1/z_r) over one common denominator:
   *   u*_l - u*_r = ((nl - nr) wl wr - (ps - pl) wr - (ps - pr) wl) / (wl wr)
   *   1/z_l + 1/z_r = ((wl^2 + cl^2) wr^3 + (wr^2 + cr^2) wl^3) / (2 wl^3 wr^3)
   * so a Newton step costs 2 sqrt + 1 division. */
  const double wl2 = wl * wl, wr2 = wr * wr;
  const double num = 2.0 * wl2 * wr2 * ((c->nl - c->nr) * wl * wr - (ps - c->pl) * wr - (ps - c->pr) * wl);
  const double den = (wl2 + c->cl2) * (wr2 * wr) + (wr2 + c->cr2) * (wl2 * wl);
  return hy_max(ps + hy_div(num, den HY_BAD_ARG), HY_SMALLP);
}

LF_HD void hy_riemann_sample(const hy_rp* c, double ps, double rl, double tl, double rr, double tr, double* gr,
                             double* gn, double* gt, double* gp HY_BAD_PARAM) {
  const double wl = c->cl * HY_SQRT(1.0 + c->kpl * (ps - c->pl));
  const double wr = c->cr * HY_SQRT(1.0 + c->kpr * (ps - c->pr));
  const double us = hy_div(wl * c->nl + wr * c->nr + c->pl - c->pr, wl + wr HY_BAD_ARG);
  const int left = us > 0.0;
  const double ro = left ? rl : rr;
  const double uo = left ? c->nl : -c->nr; /* velocity along the sampled wave direction */
  const double po = left ? c->pl : c->pr;
  const double wo = left ? wl : wr;
  const double to = left ? tl : tr;
  const double uss = left ? us : -us;
  const double iro = HY_QUOT(1.0, ro);
  const double co = HY_SQRT(HY_GAMMA * po * iro);
  const double rstar = hy_max(HY_QUOT(ro, 1.0 + hy_div(ro * (po - ps), wo * wo HY_BAD_ARG)), HY_SMALLR);
  const double cstar = HY_SQRT(HY_QUOT(HY_GAMMA * ps, rstar));
  double spout = co - uo;
  double spin = cstar - uss;
  if (ps >= po) {
    const double ushock = wo * iro - uo;
    spout = ushock;
    spin = ushock;
  }
  const double scr = hy_max(spout - spin, HY_SMALLC + fabs(spout + spin));
  const double frac = hy_min(hy_max(0.5 * (1.0 + hy_div(spout + spin, scr HY_BAD_ARG)), 0.0), 1.0);
  double r = frac * rstar + (1.0 - frac) * ro;
  double u = frac * uss + (1.0 - frac) * uo;
  double p = frac * ps + (1.0 - frac) * po;
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

/* conservative flux through the face from the Godunov state */
LF_HD void hy_flux(double r, double n, double t, double p, double* fr, double* fn, double* ft, double* fe) {
  const double m = r * n;
  const double et = p * (1.0 / (HY_GAMMA - 1.0)) + 0.5 * r * (n * n + t * t);
  *fr = m;
  *fn = m * n + p;
  *ft = m * t;
  *fe = n * (et + p);
}

/* conservative update of one cell from its two face fluxes */
LF_HD void hy_update(double r, double mn, double mt, double e, double frm, double fnm, double ftm, double fem,
                     double frp, double fnp, double ftp, double fep, double dtdx, double* ro, double* no,
                     double* to, double* eo) {
  *ro = r + dtdx * (frm - frp);
  *no = mn + dtdx * (fnm - fnp);
  *to = mt + dtdx * (ftm - ftp);
  *eo = e + dtdx * (fem - fep);
}

#endif

// Fused sm_100a executor for the Hydro2D step (BASELINE.json configs[2] and
// configs[4]; specs/hydro2d.lf): x-sweep chain then y-sweep chain, fused into
// ONE pass over the grid, fp64 SoA state (rho, rho*u, rho*v, E), reflective
// walls.
//
// The planner fuses all 12 kernel rules into one (j, i) nest: the x-swept
// state rho1..en1 is an intermediate with a 5-row window and every x/y
// intermediate is contracted.  The executor realises exactly that:
//   * a CTA of 128 threads owns a strip of 124 cells and marches its rows;
//     rows of the four state arrays arrive by TMA (4 tensor maps, 2 rows per
//     stage, 2-slot mbarrier ring);
//   * x-sweep of a row through shared memory: prims (128 columns), slope +
//     trace (126) -- one pass of the CTA each, so no warp runs a second,
//     nearly empty pass while the others wait at the barrier (127-cell strips
//     need 131 / 129; same speed in a same-box A/B, fewer barrier stalls) --
//     Riemann + flux on
//     the 125 faces (one per thread; the last three threads repeat face 124),
//     then the update;
//   * thread t keeps column i0+t's y-sweep in registers: the x-swept state,
//     prims, the plus-face trace state and the previous face flux are rolling
//     windows along j, one y-face Riemann solve per row per thread;
//   * the new state leaves once (64 B per cell-step of HBM traffic), with the
//     reflective ghost ring written by the owners of the mirrored cells.
#include <algorithm>
#include <cstdlib>

#include "../../userkernels/hydro_kernels.h"
#include "common.cuh"
#include "exec.hpp"
#include "fastmath.cuh"
#include "rowstream.cuh"

namespace lfx {
// the same user kernels with branch-free divisions / square roots that flag
// operands outside their exact range (fastmath.cuh); every call below checks
// the flag and recomputes with the plain kernels above when it is set
namespace hf {
// the chain's 64-bit constants as constant-bank operands (same values): as
// literals they are rematerialised into uniform registers inside the loops
// (same-box A/B: +4 %)
__constant__ double kGamma = HY_GAMMA, kGm1 = HY_GM1, kGk = HY_GK, kSmallR = HY_SMALLR, kSmallP = HY_SMALLP,
                    kSmallC = HY_SMALLC;
#undef HY_GAMMA
#undef HY_GM1
#undef HY_GK
#undef HY_SMALLR
#undef HY_SMALLP
#undef HY_SMALLC
#define HY_GAMMA kGamma
#define HY_GM1 kGm1
#define HY_GK kGk
#define HY_SMALLR kSmallR
#define HY_SMALLP kSmallP
#define HY_SMALLC kSmallC
#define HY_FAST 1
#undef LF_HD
#define LF_HD __device__ __forceinline__
#undef LF_USERKERNELS_HYDRO_H
#include "../../userkernels/hydro_kernels.h"
#undef HY_FAST
#undef LF_HD
#define LF_HD __host__ __device__ __forceinline__
}  // namespace hf
namespace {

#ifndef LF_HYDRO_NT
#define LF_HYDRO_NT 128
#endif
#ifndef LF_HYDRO_UNROLL
#define LF_HYDRO_UNROLL 2
#endif
constexpr int NT = LF_HYDRO_NT;         // threads per CTA = x-faces per row
constexpr int UNROLL = LF_HYDRO_UNROLL; // Newton steps per unrolled loop body
constexpr int W = NT - 4;              // cells per strip
constexpr int H = 2;                   // radius of each sweep
constexpr int BOXW = NT + 4;           // staged columns from the even storage column <= i0 (NT + 3 used)
constexpr int R = 2;                   // rows per stage
constexpr int S = 2;                   // ring slots (compute per row >> load latency)
constexpr int ARR_TX = BOXW * R * 8;   // bytes TMA delivers per array per stage
constexpr int ARR_BYTES = (ARR_TX + 127) / 128 * 128;  // 128-B aligned array slots
constexpr int STAGE_TX = 4 * ARR_TX;
constexpr int STAGE_BYTES = 4 * ARR_BYTES;
constexpr int NPRIM = W + 4;           // 131 prim columns
constexpr int NQ = W + 2;              // 129 trace columns
constexpr int XBUF = 4 * NPRIM + 8 * NQ + 4 * NT;  // doubles per x-sweep buffer
constexpr int U1RING = 3 * 4 * NT;                 // x-swept state of rows r-1..r-3, per column (thread)
constexpr int YQRING = 2 * 4 * NT;                 // y-sweep prims of rows r-1, r-2, per column
constexpr int SMEM = S * STAGE_BYTES + XBUF * 8 + (U1RING + YQRING) * 8 + S * 8 + 128;

// out-of-line fallbacks of the fast paths (rarely taken: keep their
// registers out of the hot loop)
struct D4 {
  double v[4];
};
__device__ __noinline__ D4 slow_riemann(double rl, double nl, double tl, double pl, double rr, double nr, double tr,
                                        double pr) {
  D4 g;
  hy_riemann(rl, nl, tl, pl, rr, nr, tr, pr, &g.v[0], &g.v[1], &g.v[2], &g.v[3]);
  return g;
}
__device__ __noinline__ D4 slow_constoprim(double r, double mn, double mt, double e) {
  D4 q;
  hy_constoprim(r, mn, mt, e, &q.v[0], &q.v[1], &q.v[2], &q.v[3]);
  return q;
}
struct D8 {
  double v[8];
};
__device__ __noinline__ D8 slow_trace(double r, double n, double t, double p, double dr, double dn, double dt,
                                      double dp, double dtdx) {
  D8 o;
  hy_trace(r, n, t, p, dr, dn, dt, dp, dtdx, &o.v[0], &o.v[1], &o.v[2], &o.v[3], &o.v[4], &o.v[5], &o.v[6], &o.v[7]);
  return o;
}

__device__ __noinline__ double slow_cfl_speed(double r, double mx, double my, double e) {
  double sp;
  hy_cfl_speed(r, mx, my, e, &sp);
  return sp;
}

struct Params {
  int ni, nj;            // interior of this launch's domain (slab rows for multi-GPU)
  int row_lo, row_hi;    // rows this launch computes
  long long pitch;       // ni + 4
  int strips;
  int ghost_top, ghost_bottom;  // refill reflective ghost rows at these faces
  unsigned force_slow;          // 1: take every exact fallback (LF_HYDRO_FORCE_SLOW, tests)
  const double* dtdx;    // rank-0 terminal g_dtdx (or, adaptive, the previous step's CFL maximum)
  int dtdx_is_max;       // adaptive steps after the first: dt/dx = CFL / *dtdx
  unsigned long long* cfl_acc;  // adaptive: this step's CFL maximum (double bits, atomicMax; zeroed by the host)
  double* out[4];
  // in place (out == the staged arrays): cells another CTA still reads are
  // deferred to these bands and copied in by hydro_commit after the step
  double* colband;  // [4][strips-1][nj][4]: the two columns either side of every strip boundary
  double* rowband;  // [ctas][3 segments][4 rows][4][W]: the two rows either side of every segment cut
  // row parts launched in ascending order (pipelined host runs): the launch's
  // last H rows are read by the NEXT part's launch, so they are deferred too
  // (defer_bottom) and committed separately: commit_mode 0 = every deferred
  // cell, 1 = all but those rows, 2 = those rows only
  int defer_bottom, commit_mode;
};

struct Maps {
  CUtensorMap m[4];
};

// `band` (in-place runs): a deferred cell goes to band[a * bstride] instead --
// the store addresses are selected, not branched to, so a warp whose edge lanes
// are deferred stays on one path; its ghost images are left to hydro_commit
__device__ __forceinline__ void store_cell(const Params& p, int j, int i, const double v[4], double* band = nullptr,
                                           unsigned bstride = 0) {
  // interior value plus its reflective images in the ghost ring
  const long long P = p.pitch;
  const long long base = (long long)(j + H) * P + (i + H);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double* d = p.out[a] + base;
    if (band) d = band + (size_t)a * bstride;
    *d = v[a];
  }
  if (band) return;
  int im = -100, jm = -100;
  if (i < H) im = -1 - i;
  if (i >= p.ni - H) im = 2 * p.ni - 1 - i;
  if (p.ghost_top && j < H) jm = -1 - j;
  if (p.ghost_bottom && j >= p.nj - H) jm = 2 * p.nj - 1 - j;
  if (im != -100) {
    const long long g = (long long)(j + H) * P + (im + H);
    p.out[0][g] = v[0];
    p.out[1][g] = -v[1];  // rho*u odd across i-faces
    p.out[2][g] = v[2];
    p.out[3][g] = v[3];
  }
  if (jm != -100) {
    const long long g = (long long)(jm + H) * P + (i + H);
    p.out[0][g] = v[0];
    p.out[1][g] = v[1];
    p.out[2][g] = -v[2];  // rho*v odd across j-faces
    p.out[3][g] = v[3];
    if (im != -100) {
      const long long c = (long long)(jm + H) * P + (im + H);
      p.out[0][c] = v[0];
      p.out[1][c] = -v[1];
      p.out[2][c] = -v[2];
      p.out[3][c] = v[3];
    }
  }
}

// ---- in place (config.aliases: every goal on its axiom's buffer; storage.cpp:453-594)
// A CTA reads its strip's columns i0-2 .. i0+W+1 of rows jb-2 .. je+1 and writes
// row j only after it has consumed row j+3, so its own reads are never
// overtaken.  What OTHER CTAs read of its cells are the two columns next to a
// strip boundary (the neighbour strip's halo) and the two rows next to a
// segment cut (the halo rows of the segment above / below in the same strip).
// Those cells -- with their reflective ghost images -- are written to band
// buffers instead and copied in by hydro_commit once every CTA of the step has
// finished reading: the shadow-window rule of the reference's alias analysis
// applied to the executor's own decomposition.
// slot 0..3 of row j in its segment's row band (-1: not deferred)
__device__ __forceinline__ int band_row_slot(int j, int jb, int je, bool cut_above, bool cut_below) {
  if (cut_above && j - jb < H) return j - jb;
  if (cut_below && je - j <= H) return H + (j - (je - H));
  return -1;
}
__device__ __forceinline__ double* rowband_at(const Params& p, int cta, int k, int slot, int t) {
  return p.rowband + ((size_t)(cta * 3 + k) * 4 + slot) * 4 * W + t;
}
__device__ __forceinline__ double* colband_at(const Params& p, int edge, int j, int c4) {
  return p.colband + ((size_t)edge * p.nj + j) * 4 + c4;
}

// ADAPT: also reduce the CFL speed of every stored cell (specs/hydro2d_adaptive.lf)
// INPLACE: the goals are the staged arrays themselves (see above)
template <int MINB, bool ADAPT = false, bool INPLACE = false>
__global__ void __launch_bounds__(NT, MINB) hydro_fused(const __grid_constant__ Maps maps, const Params p) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;
  double* xb0 = reinterpret_cast<double*>(smem + S * STAGE_BYTES);
  // each thread's own column of the x-swept state for the three rows the
  // y-sweep lags behind -- in shared memory rather than 24 more registers
  double* u1ring = reinterpret_cast<double*>(smem + S * STAGE_BYTES + XBUF * 8);
  double* yqring = u1ring + U1RING;  // slot r % 2 holds row r's prims
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE_BYTES + XBUF * 8 + (U1RING + YQRING) * 8);
  const int t = threadIdx.x;
  if (t == 0) pdl_trigger();
  pdl_wait();  // previous step's output (our input) complete, our output buffer free
  const double dtdx = ADAPT && p.dtdx_is_max ? HY_CFL / *p.dtdx : *p.dtdx;  // hy_cfl_dt of the previous step
  double cfl = 0.0;  // ADAPT: fastest signal speed over the cells this thread stored

  // ---- segment list (strip-major row ranges) and stage bookkeeping
  RowSeg seg[3];
  const int nseg = cta_segments(blockIdx.x, gridDim.x, p.strips, p.row_lo, p.row_hi, seg);
  int nst[3], total = 0;
  for (int k = 0; k < nseg; ++k) {
    nst[k] = (seg[k].je - seg[k].jb + 2 * H + 1 + R - 1) / R;  // marched rows jb-2 .. je+2
    total += nst[k];
  }
  auto issue = [&](int g) {
    if (g >= total) return;
    int k = 0, gg = g;
    while (gg >= nst[k]) gg -= nst[k++];
    const int slot = g % S;
    unsigned char* dst = ring + slot * STAGE_BYTES;
    fence_proxy_async();
    mbar_arrive_expect_tx(&full[slot], STAGE_TX);
    // storage col of logical i0-2, rounded down to an even column: TMA box
    // origins must be 16-B aligned along the contiguous dimension
    const int c0 = (seg[k].strip * W) & ~1;
    const int r0 = seg[k].jb - H + gg * R + H; // storage row of the stage's first row
#pragma unroll
    for (int a = 0; a < 4; ++a) tma_load_2d(dst + a * ARR_BYTES, &maps.m[a], &full[slot], c0, r0);
  };
  if (t == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    for (int a = 0; a < 4; ++a) tma_prefetch_desc(&maps.m[a]);
    for (int g = 0; g < S; ++g) issue(g);
  }
  __syncthreads();

  int g = 0, pending = -1;
  for (int k = 0; k < nseg; ++k) {
    const RowSeg sg = seg[k];
    const int i0 = sg.strip * W;
    const int off = i0 & 1;                  // staged column of logical i0-2 (see issue())
    const int ncell = min(W, p.ni - i0);     // cells of this strip
    const bool owns = t < ncell;
    // marched rows r = jb-2 .. je+2: the y-sweep lags the x-sweep by three rows
    // so that the y-face Riemann solve of a column can run next to the x-face
    // solve of the same thread (two independent dependency chains per thread)
    const int T = sg.je - sg.jb + 2 * H + 1;
    // y-sweep windows of column i0 + t (indices relative to the marched row r)
    double yqm[4];            // minus-face trace state of row r-2 (read at C of row r+... see below)
    double ypo[4], ypn[4];    // plus-face trace states of rows r-3 and r-2
    double yfp[4];            // flux of face (r-4)+1/2
    // benign states for the dummy y-problems before the pipeline fills
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      ypo[a] = ypn[a] = yqm[a] = (a == 0 || a == 3) ? 1.0 : 0.0;
    }
    for (int tt = 0; tt < T; ++tt) {
      const int tr = tt % R;
      if (tr == 0) mbar_wait(&full[g % S], (g / S) & 1);
      const double* st = reinterpret_cast<const double*>(ring + (g % S) * STAGE_BYTES);
      const double* row[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) row[a] = st + a * (ARR_BYTES / 8) + tr * BOXW + off;
      // one x-buffer suffices: A writes prims (last read in B of the previous row),
      // B writes face states (read in C), C writes fluxes (read in D) -- each
      // write is separated from the previous row's reads by a __syncthreads
      double* xb = xb0;
      double* xq = xb;                  // [4][NPRIM]  prims, column c <-> logical i0-2+c
      double* xm = xq + 4 * NPRIM;      // [4][NQ]     minus-face states, c <-> i0-1+c
      double* xp = xm + 4 * NQ;         // [4][NQ]     plus-face states
      double* xf = xp + 4 * NQ;         // [4][NT]     face fluxes, face c <-> (i0-1+c)+1/2

      // ---- A. x: conservative -> primitive on 131 columns
      for (int c = t; c < NPRIM; c += NT) {
        unsigned bad = p.force_slow;
        hf::hy_constoprim(row[0][c], row[1][c], row[2][c], row[3][c], &xq[c], &xq[NPRIM + c], &xq[2 * NPRIM + c],
                          &xq[3 * NPRIM + c], &bad);
        if (bad) {
          const D4 q = slow_constoprim(row[0][c], row[1][c], row[2][c], row[3][c]);
#pragma unroll
          for (int a = 0; a < 4; ++a) xq[a * NPRIM + c] = q.v[a];
        }
      }
      __syncthreads();
      if (pending >= 0) {  // every thread is past the last read of stage `pending`
        if (t == 0) issue(pending + S);
        pending = -1;
      }
      // ---- B. x: slope + trace on 129 columns
      for (int c = t; c < NQ; c += NT) {
        double d[4];
        hy_slope(xq[c], xq[NPRIM + c], xq[2 * NPRIM + c], xq[3 * NPRIM + c], xq[c + 1], xq[NPRIM + c + 1],
                 xq[2 * NPRIM + c + 1], xq[3 * NPRIM + c + 1], xq[c + 2], xq[NPRIM + c + 2],
                 xq[2 * NPRIM + c + 2], xq[3 * NPRIM + c + 2], &d[0], &d[1], &d[2], &d[3]);
        unsigned bad = p.force_slow;
        hf::hy_trace(xq[c + 1], xq[NPRIM + c + 1], xq[2 * NPRIM + c + 1], xq[3 * NPRIM + c + 1], d[0], d[1], d[2],
                     d[3], dtdx, &xm[c], &xm[NQ + c], &xm[2 * NQ + c], &xm[3 * NQ + c], &xp[c], &xp[NQ + c],
                     &xp[2 * NQ + c], &xp[3 * NQ + c], &bad);
        if (bad) {
          const D8 o = slow_trace(xq[c + 1], xq[NPRIM + c + 1], xq[2 * NPRIM + c + 1], xq[3 * NPRIM + c + 1], d[0],
                                  d[1], d[2], d[3], dtdx);
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            xm[a * NQ + c] = o.v[a];
            xp[a * NQ + c] = o.v[4 + a];
          }
        }
      }
      __syncthreads();
      // ---- C. two independent Riemann solves per thread:
      //   x-face t of row r (between cells i0-1+t and i0+t), and
      //   y-face (r-3)+1/2 of column i0+t (plus state of row r-3, minus state of row r-2)
      {
        // both problems advance in one loop: two independent dependency chains
        // per thread (the y-problem of a non-owning thread or of the pipeline's
        // first rows is a benign dummy whose result is dropped)
        const bool yface = owns && tt >= 4;
        // branch-free fast paths; a flagged problem is re-solved with the plain kernels
        unsigned bx = p.force_slow, by = p.force_slow;
        hf::hy_rp cx, cy;
        const int fx = min(t, W);  // faces W+1.. of the last threads: a harmless repeat of face W
        double psx = hf::hy_riemann_init(xp[fx], xp[NQ + fx], xp[3 * NQ + fx], xm[fx + 1], xm[NQ + fx + 1],
                                         xm[3 * NQ + fx + 1], &cx, &bx);
        double psy = hf::hy_riemann_init(ypo[0], ypo[1], ypo[3], yqm[0], yqm[1], yqm[3], &cy, &by);
#pragma unroll UNROLL
        for (int it = 0; it < HY_NITER; ++it) {
          psx = hf::hy_riemann_newton(&cx, psx, &bx);
          psy = hf::hy_riemann_newton(&cy, psy, &by);
        }
        double gx[4], gy[4];
        hf::hy_riemann_sample(&cx, psx, xp[fx], xp[2 * NQ + fx], xm[fx + 1], xm[2 * NQ + fx + 1], &gx[0], &gx[1],
                              &gx[2], &gx[3], &bx);
        hf::hy_riemann_sample(&cy, psy, ypo[0], ypo[2], yqm[0], yqm[2], &gy[0], &gy[1], &gy[2], &gy[3], &by);
        if (bx) {
          const D4 g4 = slow_riemann(xp[fx], xp[NQ + fx], xp[2 * NQ + fx], xp[3 * NQ + fx], xm[fx + 1],
                                     xm[NQ + fx + 1], xm[2 * NQ + fx + 1], xm[3 * NQ + fx + 1]);
#pragma unroll
          for (int a = 0; a < 4; ++a) gx[a] = g4.v[a];
        }
        if (by) {
          const D4 g4 = slow_riemann(ypo[0], ypo[1], ypo[2], ypo[3], yqm[0], yqm[1], yqm[2], yqm[3]);
#pragma unroll
          for (int a = 0; a < 4; ++a) gy[a] = g4.v[a];
        }
        hy_flux(gx[0], gx[1], gx[2], gx[3], &xf[t], &xf[NT + t], &xf[2 * NT + t], &xf[3 * NT + t]);
        if (yface) {
          double f[4];
          hy_flux(gy[0], gy[1], gy[2], gy[3], &f[0], &f[1], &f[2], &f[3]);
          if (tt >= 5) {
            // update of row r-3 from faces (r-4)+1/2 and (r-3)+1/2
            double o[4];
            // row r-3's x-swept state: ring slot (r-3) % 3 == r % 3
            const double* u1c = u1ring + (tt % 3) * 4 * NT + t;
            hy_update(u1c[0], u1c[2 * NT], u1c[NT], u1c[3 * NT], yfp[0], yfp[1], yfp[2], yfp[3], f[0], f[1], f[2], f[3],
                      dtdx, &o[0], &o[2], &o[1], &o[3]);
            const int jo = sg.jb - 2 + tt - 3;
            if constexpr (INPLACE) {
              // 32-bit band offsets (checked on the host): one store sequence for both bands
              const int rs = band_row_slot(jo, sg.jb, sg.je, sg.jb > p.row_lo, sg.je < p.row_hi || p.defer_bottom);
              const bool cl = t < H && sg.strip > 0, cr = t >= W - H && sg.strip < p.strips - 1;
              double* band = nullptr;
              unsigned bstride = W;
              if (rs >= 0) {
                band = p.rowband + (unsigned)(((blockIdx.x * 3 + k) * 4 + rs) * 4 * W + t);
              } else if (cl || cr) {
                band = p.colband + ((unsigned)((cl ? sg.strip - 1 : sg.strip) * p.nj + jo) * 4u +
                                    (unsigned)(cl ? H + t : t - (W - H)));
                bstride = (unsigned)(p.strips - 1) * (unsigned)p.nj * 4u;
              }
              store_cell(p, jo, i0 + t, o, band, bstride);
            } else {
              store_cell(p, jo, i0 + t, o);
            }
            if constexpr (ADAPT) {
              double sp;
              unsigned bs = p.force_slow;
              hf::hy_cfl_speed(o[0], o[1], o[2], o[3], &sp, &bs);
              if (bs) sp = slow_cfl_speed(o[0], o[1], o[2], o[3]);
              cfl = hy_max(cfl, sp);
            }
          }
#pragma unroll
          for (int a = 0; a < 4; ++a) yfp[a] = f[a];
        }
      }
      __syncthreads();
      if (tr == R - 1 || tt == T - 1) {
        pending = g;
        ++g;
      }
      if (!owns) continue;  // whole-warp uniform except in the strip's last warp
      // ---- D. x: update of cell i0+t -> x-swept state of row r; y: prims of row r,
      //      slope + trace of row r-1
      double u1[4];
      hy_update(row[0][t + 2], row[1][t + 2], row[2][t + 2], row[3][t + 2], xf[t], xf[NT + t], xf[2 * NT + t],
                xf[3 * NT + t], xf[t + 1], xf[NT + t + 1], xf[2 * NT + t + 1], xf[3 * NT + t + 1], dtdx, &u1[0],
                &u1[1], &u1[2], &u1[3]);
      double yq[4];
      unsigned bad = p.force_slow;
      hf::hy_constoprim(u1[0], u1[2], u1[1], u1[3], &yq[0], &yq[1], &yq[2], &yq[3], &bad);
      if (bad) {
        const D4 q = slow_constoprim(u1[0], u1[2], u1[1], u1[3]);
#pragma unroll
        for (int a = 0; a < 4; ++a) yq[a] = q.v[a];
      }
      if (tt >= 2) {
        double d[4], yp[4];
        const double* yq1 = yqring + ((tt + 1) & 1) * 4 * NT + t;  // row r-1
        const double* yq2 = yqring + (tt & 1) * 4 * NT + t;        // row r-2
        hy_slope(yq2[0], yq2[NT], yq2[2 * NT], yq2[3 * NT], yq1[0], yq1[NT], yq1[2 * NT], yq1[3 * NT], yq[0], yq[1],
                 yq[2], yq[3], &d[0],
                 &d[1], &d[2], &d[3]);
        // minus state of row r-1 is read by the y-face (r-2)+1/2 at C of the next row
        bad = p.force_slow;
        hf::hy_trace(yq1[0], yq1[NT], yq1[2 * NT], yq1[3 * NT], d[0], d[1], d[2], d[3], dtdx, &yqm[0], &yqm[1],
                     &yqm[2], &yqm[3], &yp[0], &yp[1], &yp[2], &yp[3], &bad);
        if (bad) {
          const D8 o = slow_trace(yq1[0], yq1[NT], yq1[2 * NT], yq1[3 * NT], d[0], d[1], d[2], d[3], dtdx);
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            yqm[a] = o.v[a];
            yp[a] = o.v[4 + a];
          }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          ypo[a] = ypn[a];  // plus state of row r-2 (for the face (r-2)+1/2 at the next row)
          ypn[a] = yp[a];   // plus state of row r-1
        }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        yqring[(tt & 1) * 4 * NT + a * NT + t] = yq[a];  // row r over row r-2
        u1ring[(tt % 3) * 4 * NT + a * NT + t] = u1[a];
      }
    }
  }
  if constexpr (ADAPT) {
    // the maximum is exact in any order: one atomic per warp on the bit
    // pattern (non-negative doubles order like their bits)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cfl = hy_max(cfl, __shfl_xor_sync(0xffffffffu, cfl, o));
    if ((t & 31) == 0) atomicMax(p.cfl_acc, static_cast<unsigned long long>(__double_as_longlong(cfl)));
  }
}

// In-place step, second launch: the deferred cells (and their ghost images)
// go to their places.  Same grid and segment list as the step's launch.
__global__ void __launch_bounds__(NT) hydro_commit(const Params p) {
  const int t = threadIdx.x;
  if (t == 0) pdl_trigger();
  pdl_wait();  // every CTA of the step has finished reading the arrays
  RowSeg seg[3];
  const int nseg = cta_segments(blockIdx.x, gridDim.x, p.strips, p.row_lo, p.row_hi, seg);
  const size_t cstride = (size_t)(p.strips - 1) * p.nj * 4;
  for (int k = 0; k < nseg; ++k) {
    const RowSeg sg = seg[k];
    const int i0 = sg.strip * W;
    const int ncell = min(W, p.ni - i0);
    const bool above = sg.jb > p.row_lo, below = sg.je < p.row_hi || p.defer_bottom;
    const int ext = p.defer_bottom ? p.row_hi - H : p.row_hi;  // rows >= ext wait for the next part's launch
    for (int rs = 0; rs < 2 * H; ++rs) {
      const int j = rs < H ? sg.jb + rs : sg.je - 2 * H + rs;
      if (j < sg.jb || j >= sg.je || band_row_slot(j, sg.jb, sg.je, above, below) != rs) continue;
      if (p.commit_mode == 1 ? j >= ext : (p.commit_mode == 2 && j < ext)) continue;
      if (t < ncell) {
        const double* b = rowband_at(p, blockIdx.x, k, rs, t);
        const double v[4] = {b[0], b[W], b[2 * W], b[3 * W]};
        store_cell(p, j, i0 + t, v);
      }
    }
    const bool left = sg.strip > 0, right = sg.strip < p.strips - 1;
    if ((!left && !right) || p.commit_mode == 2) continue;
    const long long n = (long long)(sg.je - sg.jb) * 4;
    for (long long idx = t; idx < n; idx += NT) {
      const int j = sg.jb + (int)(idx >> 2), q = (int)(idx & 3);
      if (q < H ? !left : !right) continue;
      if (band_row_slot(j, sg.jb, sg.je, above, below) >= 0) continue;
      const int tc = q < H ? q : W - 2 * H + q;
      const double* b = q < H ? colband_at(p, sg.strip - 1, j, H + q) : colband_at(p, sg.strip, j, q - H);
      const double v[4] = {b[0], b[cstride], b[2 * cstride], b[3 * cstride]};
      store_cell(p, j, i0 + tc, v);
    }
  }
}

bool supports(const lf::Plan& plan, std::string& why) {
  const auto& r = plan.rs.ranges;
  for (const auto& rg : r)
    if (rg.stride != 1 || rg.lo != 0) {
      why = "hydro executor needs unit strides and ranges starting at 0";
      return false;
    }
  long nj = r[0].trips(), ni = r[1].trips();
  if (ni < 4 || nj < 4 || (ni + 4) * 8 % 16) {
    why = "hydro executor needs N_i, N_j >= 4 and an even N_i (got " + std::to_string(nj) + "x" +
          std::to_string(ni) + ")";
    return false;
  }
  return true;
}

// dt/dx from the CFL maximum in place (hy_cfl_dt): the chain's g_dtdx_n goal
__global__ void cfl_finalize(double* slot) { hy_cfl_dt(*slot, slot); }

// band buffers of an in-place run (see hydro_commit), sized for a launch of
// `ctas` CTAs over `strips` strips of `nj` rows
struct Bands {
  double* col = nullptr;
  double* row = nullptr;
  bool defer_bottom = false;  // ordered row parts: the last H rows wait for the next part's launch
  int commit_mode = 0;        // see Params
  bool step = true;           // false: only the commit launch (commit_mode 2)
  static size_t col_doubles(int strips, int nj) { return (size_t)4 * std::max(0, strips - 1) * nj * 4; }
  static size_t row_doubles(int ctas) { return (size_t)ctas * 3 * 4 * 4 * W; }
};

int launch_step(const double* const in[4], double* const out[4], const double* dtdx, int ni, const RowPart& rp,
                cudaStream_t st, std::string& err, unsigned long long* cfl_acc = nullptr, bool dtdx_is_max = false,
                const Bands* bands = nullptr, int* ctas_out = nullptr) {
  const int nj = rp.rows;
  // LF_HYDRO_VARIANT: register budget for 2 / 3 (default) / 4 CTAs per SM.
  // With the branch-free divisions the Riemann phase keeps the fp64 pipe busy
  // from fewer warps: 3 CTAs at 168 registers (no spills) beat 4 CTAs at 128
  // (96 B of spills) -- profiles/r01_hydro_variants.txt
  static void (*const kern)(Maps, Params) = [] {
    const char* v = lfx::option("LF_HYDRO_VARIANT");
    const int var = v ? std::atoi(v) : 1;
    return var == 0 ? hydro_fused<2> : (var == 2 ? hydro_fused<4> : hydro_fused<3>);
  }();
  const bool inplace = bands && bands->row;
  void (*const k)(Maps, Params) =
      inplace ? (cfl_acc ? hydro_fused<3, true, true> : hydro_fused<3, false, true>) : (cfl_acc ? hydro_fused<3, true> : kern);
  static LaunchCache cache, cache_adapt, cache_inplace, cache_inplace_adapt;
  int slots = 0;
  if (int s = resident_slots(inplace ? (cfl_acc ? cache_inplace_adapt : cache_inplace) : (cfl_acc ? cache_adapt : cache),
                             reinterpret_cast<const void*>(k), NT, SMEM, 0, "cudaFuncSetAttribute(hydro)", &slots, err))
    return s;
  Maps maps;
  uint64_t dims[2] = {(uint64_t)ni + 4, (uint64_t)nj + 4};
  uint32_t box[2] = {BOXW, R};
  for (int a = 0; a < 4; ++a)
    if (!make_tensor_map(&maps.m[a], in[a], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 2, dims, box, err))
      return LF_ERR_CUDA;
  Params p;
  p.ni = ni;
  p.nj = nj;
  p.pitch = ni + 4;
  p.strips = (ni + W - 1) / W;
  p.row_lo = rp.lo;
  p.row_hi = rp.hi;
  p.ghost_top = rp.top;
  p.ghost_bottom = rp.bottom;
  p.dtdx = dtdx;
  p.dtdx_is_max = dtdx_is_max ? 1 : 0;
  p.cfl_acc = cfl_acc;
  const unsigned force_slow = lfx::option("LF_HYDRO_FORCE_SLOW") ? 1u : 0u;
  p.force_slow = force_slow;
  for (int a = 0; a < 4; ++a) p.out[a] = out[a];
  p.colband = bands ? bands->col : nullptr;
  p.rowband = bands ? bands->row : nullptr;
  p.defer_bottom = bands && bands->defer_bottom ? 1 : 0;
  p.commit_mode = bands ? bands->commit_mode : 0;
  const long long work = (long long)p.strips * (rp.hi - rp.lo);
  // each CTA must get at most 3 row segments (rowstream.cuh): at least
  // ceil(strips/2) CTAs when the row range is short
  const long long want = std::max<long long>(work / 8, (p.strips + 1) / 2);
  const int ctas = static_cast<int>(std::max<long long>(1, std::min<long long>(slots, want)));
  if ((long long)ctas * 2 < p.strips) {
    err = "row range too short for the resident grid";
    return LF_ERR_UNSUPPORTED;
  }
  if (ctas_out) {  // sizing query of an in-place run
    *ctas_out = ctas;
    return LF_OK;
  }
  if (!inplace) return cuda_status(launch_pdl(k, dim3(ctas), dim3(NT), SMEM, st, maps, p), "hydro_fused launch", err);
  // LF_HYDRO_IP_PDL (tuning): bit 0 = the step, bit 1 = the commit launched with
  // programmatic stream serialization
  const char* o = lfx::option("LF_HYDRO_IP_PDL");
  const int pdl = o ? std::atoi(o) : 0;
  cudaError_t e = cudaSuccess;
  if (!bands->step) {
  } else if (pdl & 1) {
    e = launch_pdl(k, dim3(ctas), dim3(NT), SMEM, st, maps, p);
  } else {
    k<<<ctas, NT, SMEM, st>>>(maps, p);
    e = cudaGetLastError();
  }
  if (int s = cuda_status(e, "hydro_fused launch", err)) return s;
  if (pdl & 2) {
    e = launch_pdl(hydro_commit, dim3(ctas), dim3(NT), 0, st, p);
  } else {
    hydro_commit<<<ctas, NT, 0, st>>>(p);
    e = cudaGetLastError();
  }
  return cuda_status(e, "hydro_commit launch", err);
}

// Whole-domain steps on ONE buffer per state array (the caller passed each
// goal on its aliased axiom's buffer).  The bands are plan-owned: 4 columns per
// strip boundary and 4 rows per segment cut, about 3 % of the state.
// `adaptive`: specs/hydro2d_adaptive.lf -- each step also reduces its CFL maximum
// (run_adaptive below); the two dt/dx slots are the goal's and one beside the bands.
int run_inplace(const ExecArgs& a, std::string& err, bool adaptive = false) {
  const auto& r = a.plan->rs.ranges;
  const int ni = (int)r[1].trips();
  const RowPart rp = row_part(a, (int)r[0].trips());
  const bool part = rp.lo > 0 || rp.hi < rp.rows;
  if (a.slab && !a.whole_domain_parts && part) {  // a rank's slab: one launch over all of its rows
    err = "in-place slab runs launch whole slabs (no face / interior parts)";
    return LF_ERR_UNSUPPORTED;
  }
  if (part && (a.steps != 1 || rp.hi - rp.lo < 2 * H || adaptive)) {
    err = "in-place row parts run one step at a time, span at least 4 rows and carry no per-step reduction";
    return LF_ERR_UNSUPPORTED;
  }
  double* u[4];
  for (int v = 0; v < 4; ++v) u[v] = static_cast<double*>(a.terms[v]);
  const double* dtdx = static_cast<const double*>(a.terms[4]);
  // band sizes from the whole domain's launch (a part's grid is never larger)
  const RowPart whole{rp.rows, 0, rp.rows, true, true};
  Bands sizing;
  sizing.row = reinterpret_cast<double*>(1);  // selects the in-place kernel for the occupancy query
  int ctas = 0;
  if (int s = launch_step(u, u, dtdx, ni, whole, a.stream, err, nullptr, false, &sizing, &ctas)) return s;
  const int strips = (ni + W - 1) / W;
  const size_t ncol = Bands::col_doubles(strips, rp.rows), nrow = Bands::row_doubles(ctas);
  if (ncol >= (1ull << 31) || nrow >= (1ull << 31)) {  // the kernel forms band offsets in 32 bits
    err = "grid too large for the in-place bands";
    return LF_ERR_UNSUPPORTED;
  }
  if (!a.mem || a.inplace_slots < 1 || a.inplace_slot < 0 || a.inplace_slot >= a.inplace_slots) {
    err = "in-place run without plan-owned band memory";
    return LF_ERR_INTERNAL;
  }
  const size_t band_bytes = (ncol + nrow * a.inplace_slots + 2) * sizeof(double);
  void* band_ptr = nullptr;
  if (int s = band_memory(*a.mem, band_bytes, a.stream, &band_ptr, err)) return s;
  double* mem = static_cast<double*>(band_ptr);
  cudaError_t e = cudaSuccess;
  Bands b;
  b.col = mem;
  b.row = mem + ncol + nrow * a.inplace_slot;
  if (part) {
    b.defer_bottom = rp.hi < rp.rows;
    if (a.inplace_phase == 1) {  // the rows the next part's launch has now read
      if (!b.defer_bottom) return LF_OK;
      b.step = false;
      b.commit_mode = 2;
    } else {
      b.commit_mode = b.defer_bottom ? 1 : 0;
    }
    if (int s = launch_step(u, u, dtdx, ni, rp, a.stream, err, nullptr, false, &b)) return s;
    return band_guard_check(*a.mem, band_bytes, a.stream, err);
  }
  int stt = LF_OK;
  if (adaptive && a.slab)  // one step of a slab driver's schedule: it zeroes, combines and finalises
    return launch_step(u, u, dtdx, ni, rp, a.stream, err, static_cast<unsigned long long*>(a.terms[9]),
                       a.raw_max_input, &b);
  if (!adaptive) {
    for (int s = 0; s < a.steps && stt == LF_OK; ++s)
      stt = launch_step(u, u, dtdx, ni, rp, a.stream, err, nullptr, false, &b);
    return stt != LF_OK ? stt : band_guard_check(*a.mem, band_bytes, a.stream, err);
  }
  double* dgoal = static_cast<double*>(a.terms[9]);
  double* dslot = mem + ncol + nrow * a.inplace_slots;
  const double* dsrc = dtdx;
  if (dgoal == dtdx) {  // the dt/dx pair shares its slot too: keep the given value beside the bands
    e = cudaMemcpyAsync(dslot + 1, dtdx, sizeof(double), cudaMemcpyDeviceToDevice, a.stream);
    if (e != cudaSuccess) return cuda_status(e, "cudaMemcpyAsync(dt/dx)", err);
    dsrc = dslot + 1;
  }
  bool is_max = false;
  for (int s = 0; s < a.steps && stt == LF_OK; ++s) {
    double* dd = ((a.steps - 1 - s) % 2) == 0 ? dgoal : dslot;
    e = cudaMemsetAsync(dd, 0, sizeof(double), a.stream);
    if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync(cfl)", err);
    stt = launch_step(u, u, dsrc, ni, rp, a.stream, err, reinterpret_cast<unsigned long long*>(dd), is_max, &b);
    dsrc = dd;
    is_max = true;
  }
  if (stt != LF_OK) return stt;
  cfl_finalize<<<1, 1, 0, a.stream>>>(dgoal);
  if (int s = cuda_status(cudaGetLastError(), "cfl_finalize launch", err)) return s;
  return band_guard_check(*a.mem, band_bytes, a.stream, err);
}

int run(const ExecArgs& a, std::string& err) {
  if (a.inplace) return run_inplace(a, err);
  const auto& r = a.plan->rs.ranges;
  const int ni = (int)r[1].trips();
  const RowPart rp = row_part(a, (int)r[0].trips());
  // terminals: g_rho g_mx g_my g_E g_dtdx | g_rho_n g_mx_n g_my_n g_E_n
  const double* src[4];
  double* goal[4];
  double* scr[4] = {nullptr, nullptr, nullptr, nullptr};
  for (int v = 0; v < 4; ++v) {
    src[v] = static_cast<const double*>(a.terms[v]);
    goal[v] = static_cast<double*>(a.terms[5 + v]);
    if (a.steps > 1) scr[v] = static_cast<double*>(a.scratch[v]);
  }
  const double* dtdx = static_cast<const double*>(a.terms[4]);
  for (int s = 0; s < a.steps; ++s) {
    double* const* dst = ((a.steps - 1 - s) % 2) == 0 ? goal : scr;
    int stt = launch_step(src, dst, dtdx, ni, rp, a.stream, err);
    if (stt != LF_OK) return stt;
    for (int v = 0; v < 4; ++v) src[v] = dst[v];
  }
  return LF_OK;
}

// Adaptive time step (specs/hydro2d_adaptive.lf, terminals g_rho g_mx g_my g_E
// g_dtdx | g_rho_n g_mx_n g_my_n g_E_n g_dtdx_n).  Each step reduces the CFL
// maximum of its new state into its dt/dx goal slot (zeroed first); the next
// step divides it into dt/dx itself.  On a whole domain the last slot is
// finalised here; a slab driver (lf_run_slabs) zeroes, combines the ranks'
// maxima (MAX all-reduce) and finalises itself -- Executor::max_reduce.
int run_adaptive(const ExecArgs& a, std::string& err) {
  if (a.inplace) return run_inplace(a, err, true);
  const auto& r = a.plan->rs.ranges;
  const int ni = (int)r[1].trips();
  const RowPart rp = row_part(a, (int)r[0].trips());
  const double* src[4];
  double* goal[4];
  double* scr[4] = {nullptr, nullptr, nullptr, nullptr};
  for (int v = 0; v < 4; ++v) {
    src[v] = static_cast<const double*>(a.terms[v]);
    goal[v] = static_cast<double*>(a.terms[5 + v]);
    if (a.steps > 1) scr[v] = static_cast<double*>(a.scratch[v]);
  }
  const double* dsrc = static_cast<const double*>(a.terms[4]);
  double* dgoal = static_cast<double*>(a.terms[9]);
  double* dscr = a.steps > 1 ? static_cast<double*>(a.scratch[4]) : nullptr;
  if (a.slab)  // one step of a slab driver's schedule: no zeroing, no finalising here
    return launch_step(src, goal, dsrc, ni, rp, a.stream, err, reinterpret_cast<unsigned long long*>(dgoal),
                       a.raw_max_input);
  bool is_max = false;
  for (int s = 0; s < a.steps; ++s) {
    const bool to_goal = ((a.steps - 1 - s) % 2) == 0;
    double* const* dst = to_goal ? goal : scr;
    double* dd = to_goal ? dgoal : dscr;
    cudaError_t e = cudaMemsetAsync(dd, 0, sizeof(double), a.stream);
    if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync(cfl)", err);
    int stt = launch_step(src, dst, dsrc, ni, rp, a.stream, err, reinterpret_cast<unsigned long long*>(dd), is_max);
    if (stt != LF_OK) return stt;
    for (int v = 0; v < 4; ++v) src[v] = dst[v];
    dsrc = dd;
    is_max = true;
  }
  cfl_finalize<<<1, 1, 0, a.stream>>>(dgoal);
  return cuda_status(cudaGetLastError(), "cfl_finalize launch", err);
}

int finalize_adaptive(const ExecArgs& a, std::string& err) {
  cfl_finalize<<<1, 1, 0, a.stream>>>(static_cast<double*>(a.terms[9]));
  return cuda_status(cudaGetLastError(), "cfl_finalize launch", err);
}

}  // namespace

extern const Executor hydro_executor = {"hydro2d_fused_tma", "hydro2d.lf", 1, 64.0, supports, run,
                                        nullptr, false, nullptr, /*inplace=*/true, /*inplace_parts=*/true};
extern const Executor hydro_adaptive_executor = {"hydro2d_adaptive_fused_tma", "hydro2d_adaptive.lf", 1, 64.0,
                                                 supports, run_adaptive, nullptr, true, finalize_adaptive,
                                                 /*inplace=*/true, /*inplace_parts=*/true};

}  // namespace lfx

/*
 * loomfuse-b200 CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * This library restates, in plain C, the two executions the reference
 * specifies for a fused stencil chain:
 *   - run_naive (R/SPEC.md:532-540): every kernel group swept over its full
 *     iteration space, in dataflow-topological order, with full-size
 *     intermediate arrays.  This is the parity oracle.
 *   - the HFAV fused schedule (R/SPEC.md:541-549, 499-502; shifts per
 *     shifts.cpp:8-79, windows per storage.cpp:319-399): one loop nest,
 *     intermediates in rolling windows, OpenMP over the outermost loop (the
 *     "outer-level parallelism" of R/PAPER.md:499).  This is the CPU
 *     reference path timed beside the GPU (bench.py cpu_baseline and
 *     --impl reference); it is itself checked against run_naive in tests/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load this
 * library.  The product (paper_1710_08774_b200/) never links or calls it.
 *
 * Parity status: the reference snapshot has no executor, no tests and no
 * golden vectors for this path, so the numerical oracle is
 * "parity unpinned" against the reference itself; the terminal extents/bases
 * that both schedules rely on are pinned against the reference's own planner
 * compiled from /root/reference (oracle/ref_planner.cpp -> oracle/_ref/), and
 * the chains' numerics are cross-checked bit for bit against a second,
 * independent run_naive (oracle/generic.py) that evaluates the same kernels
 * over the dataflow DAG the reference's own inference derives.
 *
 * Buffer conventions (identical to the GPU executors):
 *   terminals are dense row-major arrays of the reference's buffer_extents
 *   (storage.cpp:403-427): extent = trips + (max-min offset), index 0 at
 *   logical coordinate `base` = min offset.  Output buffers of iterated chains
 *   use the input's layout, and their ghost cells are refilled after every
 *   step according to the chain's boundary mode.
 */
#ifndef LF_ORACLE_H
#define LF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* config 1: u (N+4)^2 with a zero ghost ring of width 2.  */
int lfo_biharm_naive(const double* u_in, double* u_out, long nj, long ni, int steps);
int lfo_biharm_fused(const double* u_in, double* u_out, long nj, long ni, int steps, int threads);
int lfo_biharm_fused_step(const double* u_in, double* u_out, long nj, long ni, int threads);

/* config 2: u (N+2)^3, periodic ghost layer of width 1. */
int lfo_heat3d_naive(const double* u_in, double* u_out, long nk, long nj, long ni, int steps);
int lfo_heat3d_fused(const double* u_in, double* u_out, long nk, long nj, long ni, int steps,
                     int threads);
int lfo_heat3d_fused_step(const double* u_in, double* u_out, long nk, long nj, long ni, int threads);

/* config 4: img (N+4)^2 replicate-padded by 2; out N^2 (fp32). */
int lfo_box_naive(const float* img, float* out, long nj, long ni);
int lfo_box_fused(const float* img, float* out, long nj, long ni, int threads);

/* configs 3/5: Hydro2D step (x-sweep then y-sweep).  State: 4 SoA arrays
 * (rho, rhou, rhov, E), each (N+4)^2 with reflective ghosts of width 2. */
int lfo_hydro_naive(const double* const in[4], double* const out[4], long nj, long ni,
                    double dtdx, int steps);
int lfo_hydro_fused(const double* const in[4], double* const out[4], long nj, long ni,
                    double dtdx, int steps, int threads);
int lfo_hydro_fused_step(const double* const in[4], double* const out[4], long nj, long ni,
                         double dtdx, int threads);
/* configs 3/5 with the adaptive time step (specs/hydro2d_adaptive.lf) */
int lfo_hydro_adaptive(const double* const in[4], double* const out[4], long nj, long ni, double* dtdx_io, int steps,
                       int fused, int threads);

int lfo_max_threads(void);

#ifdef __cplusplus
}
#endif

#endif

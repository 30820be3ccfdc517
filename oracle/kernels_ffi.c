/*
 * CPU ORACLE (test infrastructure only) -- the shipped user kernels
 * (the headers under paper_1710_08774_b200/userkernels/) exposed element-wise to Python, so
 * oracle/generic.py can evaluate chains whose kernels are named by their
 * `declaration:` (no `body:`) over the dataflow DAG the REFERENCE's own
 * inference derives (refplan --dag; inference.cpp:404-472).
 *
 * Every wrapper has one signature: lfk_<function>(n, args), args[k] = the
 * k-th parameter of the declaration (inputs and outputs as declared), each an
 * array of n elements; element e calls the kernel on element e of every array.
 */
#include "oracle.h"
#include "../paper_1710_08774_b200/userkernels/hydro_kernels.h"
#include "../paper_1710_08774_b200/userkernels/stencil_kernels.h"

#define D(k) ((double*)args[k])
#define F(k) ((float*)args[k])

int lfk_hy_constoprim(long n, void** args) {
  for (long e = 0; e < n; ++e) hy_constoprim(D(0)[e], D(1)[e], D(2)[e], D(3)[e], &D(4)[e], &D(5)[e], &D(6)[e], &D(7)[e]);
  return 0;
}

int lfk_hy_slope(long n, void** args) {
  for (long e = 0; e < n; ++e)
    hy_slope(D(0)[e], D(1)[e], D(2)[e], D(3)[e], D(4)[e], D(5)[e], D(6)[e], D(7)[e], D(8)[e], D(9)[e], D(10)[e],
             D(11)[e], &D(12)[e], &D(13)[e], &D(14)[e], &D(15)[e]);
  return 0;
}

int lfk_hy_trace(long n, void** args) {
  for (long e = 0; e < n; ++e)
    hy_trace(D(0)[e], D(1)[e], D(2)[e], D(3)[e], D(4)[e], D(5)[e], D(6)[e], D(7)[e], D(8)[e], &D(9)[e], &D(10)[e],
             &D(11)[e], &D(12)[e], &D(13)[e], &D(14)[e], &D(15)[e], &D(16)[e]);
  return 0;
}

int lfk_hy_riemann(long n, void** args) {
  for (long e = 0; e < n; ++e)
    hy_riemann(D(0)[e], D(1)[e], D(2)[e], D(3)[e], D(4)[e], D(5)[e], D(6)[e], D(7)[e], &D(8)[e], &D(9)[e], &D(10)[e],
               &D(11)[e]);
  return 0;
}

int lfk_hy_flux(long n, void** args) {
  for (long e = 0; e < n; ++e) hy_flux(D(0)[e], D(1)[e], D(2)[e], D(3)[e], &D(4)[e], &D(5)[e], &D(6)[e], &D(7)[e]);
  return 0;
}

int lfk_hy_update(long n, void** args) {
  for (long e = 0; e < n; ++e)
    hy_update(D(0)[e], D(1)[e], D(2)[e], D(3)[e], D(4)[e], D(5)[e], D(6)[e], D(7)[e], D(8)[e], D(9)[e], D(10)[e],
              D(11)[e], D(12)[e], &D(13)[e], &D(14)[e], &D(15)[e], &D(16)[e]);
  return 0;
}

int lfk_lap5(long n, void** args) {
  for (long e = 0; e < n; ++e) lap5(D(0)[e], D(1)[e], D(2)[e], D(3)[e], D(4)[e], &D(5)[e]);
  return 0;
}

int lfk_biharm_update(long n, void** args) {
  for (long e = 0; e < n; ++e) biharm_update(D(0)[e], D(1)[e], &D(2)[e]);
  return 0;
}

int lfk_face_flux(long n, void** args) {
  for (long e = 0; e < n; ++e) face_flux(D(0)[e], D(1)[e], &D(2)[e]);
  return 0;
}

int lfk_heat_divupd(long n, void** args) {
  for (long e = 0; e < n; ++e)
    heat_divupd(D(0)[e], D(1)[e], D(2)[e], D(3)[e], D(4)[e], D(5)[e], D(6)[e], &D(7)[e]);
  return 0;
}

int lfk_box3(long n, void** args) {
  for (long e = 0; e < n; ++e) box3(F(0)[e], F(1)[e], F(2)[e], &F(3)[e]);
  return 0;
}

int lfk_hy_cfl_speed(long n, void** args) {
  for (long e = 0; e < n; ++e) hy_cfl_speed(D(0)[e], D(1)[e], D(2)[e], D(3)[e], &D(4)[e]);
  return 0;
}

int lfk_hy_cfl_init(long n, void** args) {
  for (long e = 0; e < n; ++e) hy_cfl_init(&D(0)[e]);
  return 0;
}

int lfk_hy_cfl_max(long n, void** args) {
  for (long e = 0; e < n; ++e) hy_cfl_max(D(0)[e], D(1)[e], &D(2)[e]);
  return 0;
}

int lfk_hy_cfl_dt(long n, void** args) {
  for (long e = 0; e < n; ++e) hy_cfl_dt(D(0)[e], &D(1)[e]);
  return 0;
}

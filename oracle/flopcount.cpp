// Algorithmic floating-point operation count of the Hydro2D chain -- test /
// measurement infrastructure only ("count in the oracle").
//
// The user kernels of userkernels/hydro_kernels.h are compiled here with
// `double` replaced by a counting type, then one cell-step is replayed: per
// sweep and cell one constoprim, slope, trace, Riemann solve (one face per
// cell), flux and update -- the composition oracle/hydro.c uses
// (hydro.c:77-101 x-sweep, 108-133 y-sweep).  Every + - * / and sqrt counts
// as one flop and fma as two (the usual convention; fabs, min/max selects, negation and
// comparisons are not flops).  The counts are averaged over seeded states
// spanning the workload's range (shocks and rarefactions, both Riemann
// sampling branches).  bench.py uses the printed per-cell-step figure as the
// algorithmic flops of the fp64 roofline; tests/test_flopcount.py pins it.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <math.h>

struct Counts {
  long long add = 0, mul = 0, div = 0, sqrt = 0, cmp = 0;
  long long flops() const { return add + mul + div + sqrt; }
};
static Counts g;

struct Fd {
  double v;
  Fd() : v(0) {}
  Fd(double x) : v(x) {}  // NOLINT: literals and constants promote
};
static inline Fd operator+(Fd a, Fd b) { ++g.add; return Fd(a.v + b.v); }
static inline Fd operator-(Fd a, Fd b) { ++g.add; return Fd(a.v - b.v); }
static inline Fd operator*(Fd a, Fd b) { ++g.mul; return Fd(a.v * b.v); }
static inline Fd operator/(Fd a, Fd b) { ++g.div; return Fd(a.v / b.v); }
static inline Fd operator-(Fd a) { return Fd(-a.v); }
static inline bool operator<(Fd a, Fd b) { ++g.cmp; return a.v < b.v; }
static inline bool operator>(Fd a, Fd b) { ++g.cmp; return a.v > b.v; }
static inline bool operator<=(Fd a, Fd b) { ++g.cmp; return a.v <= b.v; }
static inline bool operator>=(Fd a, Fd b) { ++g.cmp; return a.v >= b.v; }
static inline bool operator==(Fd a, Fd b) { ++g.cmp; return a.v == b.v; }
static inline Fd sqrt(Fd a) { ++g.sqrt; return Fd(std::sqrt(a.v)); }
// a fused multiply-add is a multiplication and an addition (two flops)
static inline Fd fma(Fd a, Fd b, Fd c) { ++g.mul; ++g.add; return Fd(std::fma(a.v, b.v, c.v)); }
static inline Fd fabs(Fd a) { return Fd(std::fabs(a.v)); }

#define double Fd
#include "../paper_1710_08774_b200/userkernels/hydro_kernels.h"
#undef double

namespace {

uint64_t sm_state = 0x9E3779B97F4A7C15ull;
double uni(double lo, double hi) {  // splitmix64 -> [lo, hi)
  uint64_t z = (sm_state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return lo + (hi - lo) * (double)(z >> 11) * 0x1.0p-53;
}

struct Cons {
  Fd r, mn, mt, e;
};
Cons random_cell() {
  const double r = uni(0.1, 1.1), u = uni(-0.6, 0.6), v = uni(-0.6, 0.6), p = uni(0.08, 1.1);
  return {r, r * u, r * v, p / 0.4 + 0.5 * r * (u * u + v * v)};
}

// one sweep's work for one cell: its constoprim, slope, trace, the Riemann
// solve and flux of one face (its left face) and its update, as hydro.c
// composes them; the neighbours' values are formed with counting off
Counts one_cell_sweep() {
  Cons c[4];
  for (auto& x : c) x = random_cell();
  const Fd dtdx = 0.2;
  Fd q[4][4], d[4][4], m[4][4], pl[4][4];
  auto cell = [&](int k) {
    hy_constoprim(c[k].r, c[k].mn, c[k].mt, c[k].e, &q[k][0], &q[k][1], &q[k][2], &q[k][3]);
  };
  auto slope_trace = [&](int k) {
    hy_slope(q[k - 1][0], q[k - 1][1], q[k - 1][2], q[k - 1][3], q[k][0], q[k][1], q[k][2], q[k][3], q[k + 1][0],
             q[k + 1][1], q[k + 1][2], q[k + 1][3], &d[k][0], &d[k][1], &d[k][2], &d[k][3]);
    hy_trace(q[k][0], q[k][1], q[k][2], q[k][3], d[k][0], d[k][1], d[k][2], d[k][3], dtdx, &m[k][0], &m[k][1],
             &m[k][2], &m[k][3], &pl[k][0], &pl[k][1], &pl[k][2], &pl[k][3]);
  };
  // neighbours (uncounted): cells 0, 1, 3 and cell 1's trace
  const Counts keep = g;
  cell(0), cell(1), cell(3);
  const Counts base = g = keep;
  cell(2);
  const Counts after_cell = g;
  g = keep;
  cell(2);
  slope_trace(1);
  g = after_cell;
  // counted: cell 2's slope + trace, face (1|2) Riemann + flux, cell 2's update
  slope_trace(2);
  Fd gs[4], f[4], o[4];
  hy_riemann(pl[1][0], pl[1][1], pl[1][2], pl[1][3], m[2][0], m[2][1], m[2][2], m[2][3], &gs[0], &gs[1], &gs[2],
             &gs[3]);
  hy_flux(gs[0], gs[1], gs[2], gs[3], &f[0], &f[1], &f[2], &f[3]);
  hy_update(c[2].r, c[2].mn, c[2].mt, c[2].e, f[0], f[1], f[2], f[3], f[0], f[1], f[2], f[3], dtdx, &o[0], &o[1],
            &o[2], &o[3]);
  Counts r;
  r.add = g.add - base.add;
  r.mul = g.mul - base.mul;
  r.div = g.div - base.div;
  r.sqrt = g.sqrt - base.sqrt;
  r.cmp = g.cmp - base.cmp;
  g = keep;
  return r;
}

}  // namespace

int main() {
  const int n = 20000;
  double add = 0, mul = 0, dv = 0, sq = 0, cmp = 0;
  for (int s = 0; s < n; ++s) {
    const Counts c = one_cell_sweep();
    add += c.add;
    mul += c.mul;
    dv += c.div;
    sq += c.sqrt;
    cmp += c.cmp;
  }
  add /= n, mul /= n, dv /= n, sq /= n, cmp /= n;
  const double sweep = add + mul + dv + sq;
  std::printf(
      "{\"per_cell_sweep\": {\"add\": %.4f, \"mul\": %.4f, \"div\": %.4f, \"sqrt\": %.4f, \"cmp\": %.4f, "
      "\"flops\": %.4f}, \"sweeps_per_step\": 2, \"flops_per_cell_step\": %.4f, \"samples\": %d}\n",
      add, mul, dv, sq, cmp, sweep, 2 * sweep, n);
  return 0;
}

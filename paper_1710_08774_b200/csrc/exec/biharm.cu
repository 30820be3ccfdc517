// Fused sm_100a executor for the 2D biharmonic chain (BASELINE.json
// configs[0]; specs/biharmonic2d.lf): lap1 -> lap2 -> upd, fp64, zero
// Dirichlet halo of 2.
//
// HFAV contracts L to a 3-row outer_rotate window and L2 to a scalar.  Here
// one warp marches a 128-column strip down the grid (rowstream.cuh): lane l
// owns columns 4l..4l+3; u and L keep 3-row register windows that rotate by
// register renaming (rows are unrolled by 3); the i +- 1
// neighbours of u and L come from the adjacent lanes by shuffle, and lanes 0
// and 31 additionally carry the two halo columns on each side of the strip.
// Rows of u arrive by TMA, 3 rows per stage, into a 4-slot ring.  Output:
// two 16-B stores per lane per row, plus the zero ghost ring of the goal buffer so iterated steps
// can feed it straight back.  Compulsory traffic: 8 B read + 8 B written per
// cell-update.
#include <algorithm>
#include <cstdlib>

#include "../../userkernels/stencil_kernels.h"
#include "common.cuh"
#include "exec.hpp"
#include "rowstream.cuh"

namespace lfx {
namespace {

constexpr int H = 2;                   // chain radius along j and i
constexpr int R = 3;                   // rows per stage (= register-window period)

// Tunable shape: CPL columns per lane (strip = 32*CPL columns), S ring slots,
// OCC resident CTAs per SM the register budget is sized for.
// R4 = 4: rows staged four at a time and lap2 lagging lap1 by two rows (see
// biharm_row4), else three at a time with lap2 one row behind.
template <int CPL_, int S_, int OCC_, int R_ = 3>
struct Cfg {
  static constexpr int CPL = CPL_, S = S_, OCC = OCC_, RR = R_;
  static constexpr int SW = 32 * CPL;
  static constexpr int BOXW = SW + 2 * H;
  static constexpr int STAGE_TX = BOXW * RR * 8;
  static constexpr int STAGE_BYTES = (STAGE_TX + 127) / 128 * 128;
  static constexpr int SMEM = S * STAGE_BYTES + S * 8 + 64;
};

struct Params {
  int ni, nj;         // nj: rows of the launch's domain (slab or grid)
  int row_lo, row_hi; // rows this launch computes
  long long pitch;    // ni + 4
  int strips;         // ni / SW
  int write_ghost_top, write_ghost_bottom;
  int store_policy;   // L2 policy of the output stores (l2_store_policy)
  int load_policy;    // -1: plain TMA fetches, else l2_store_policy mode for the fetched lines
  // in place (out == the staged array; config.aliases): the cells other CTAs
  // still read -- the edge lanes' column pair next to a strip boundary, the two
  // rows next to a segment cut -- go to these bands, biharm_commit copies them in
  double* colband;    // [strips-1][nj][4]: two columns either side of every strip boundary
  double* rowband;    // [ctas][3 segments][4 rows][SW]
};

// slot 0..3 of row j in its segment's row band (-1: not deferred)
__device__ __forceinline__ int band_row_slot(int j, int jb, int je, bool cut_above, bool cut_below) {
  if (cut_above && j - jb < H) return j - jb;
  if (cut_below && je - j <= H) return H + (j - (je - H));
  return -1;
}

template <int CPL>
struct Win {
  double u[3][CPL];   // u rows, indexed by row % 3
  double ex[3][2];    // halo columns carried by the edge lanes
  double L[3][CPL];   // L rows, indexed by row % 3
  double lex[3];      // L at the halo column, indexed by row % 3
  // i-1 / i+1 neighbours of the lane's first / last column, per row slot:
  // exchanged by shuffle one marched row BEFORE they are consumed, so the
  // shuffle latency never sits on the lap1 -> lap2 dependency chain
  double uw[3], ue[3];  // of u
  double lw[3], le[3];  // of L
};

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// One marched row.  P = (row index) % 3 is a compile-time constant, so the
// three-row windows rotate by register renaming instead of moves.
template <int CPL, int P>
__device__ __forceinline__ void biharm_row(Win<CPL>& w, const double* row, int t, int lane, int ex_col, double* orow,
                                           uint64_t pol) {
  constexpr int C = P, M1 = (P + 2) % 3, M2 = (P + 1) % 3;  // rows r, r-1, r-2
  {
#pragma unroll
    for (int h = 0; h < CPL / 2; ++h) {
      const double2 a = lds2(row + CPL * lane + H + 2 * h);
      w.u[C][2 * h] = a.x;
      w.u[C][2 * h + 1] = a.y;
    }
    const double2 e = lds2(row + ex_col);
    w.ex[C][0] = e.x; w.ex[C][1] = e.y;
    // neighbours of u row r, consumed by lap1 when this row is r-1 (next row)
    const double left = __shfl_up_sync(0xffffffffu, w.u[C][CPL - 1], 1);
    const double right = __shfl_down_sync(0xffffffffu, w.u[C][0], 1);
    w.uw[C] = lane == 0 ? e.y : left;
    w.ue[C] = lane == 31 ? e.x : right;
  }
  if (t < 2) return;
  // ---- lap1 at row r-1 (runs one row ahead of the output: shift j = +1)
  const double* um = w.u[M1];
  double* Ln = w.L[M1];  // slot of L row r-1
#pragma unroll
  for (int c = 0; c < CPL; ++c)
    lap5(c == 0 ? w.uw[M1] : um[c - 1], c == CPL - 1 ? w.ue[M1] : um[c + 1], w.u[M2][c], w.u[C][c], um[c], &Ln[c]);
  // L at the strip's halo column: lane 0 -> logical -1, lane 31 -> SW (one lap5, operands selected)
  {
    const bool lo = lane == 0;
    const double hw = lo ? w.ex[M1][0] : um[CPL - 1];
    const double he = lo ? um[0] : w.ex[M1][1];
    const int hc = lo ? 1 : 0;
    const double hs = hc ? w.ex[M2][1] : w.ex[M2][0];
    const double hn = hc ? w.ex[C][1] : w.ex[C][0];
    const double h0 = hc ? w.ex[M1][1] : w.ex[M1][0];
    lap5(hw, he, hs, hn, h0, &w.lex[M1]);
  }
  // neighbours of L row r-1, consumed by lap2 when this row is r-2 (next row)
  {
    const double left = __shfl_up_sync(0xffffffffu, Ln[CPL - 1], 1);
    const double right = __shfl_down_sync(0xffffffffu, Ln[0], 1);
    w.lw[M1] = lane == 0 ? w.lex[M1] : left;
    w.le[M1] = lane == 31 ? w.lex[M1] : right;
  }
  if (t < 4) return;
  // ---- lap2 + update at row r-2: L rows r-3 (slot C), r-2 (slot M2), r-1 (slot M1)
  const double* L0 = w.L[M2];
  double o[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    double l2;
    lap5(c == 0 ? w.lw[M2] : L0[c - 1], c == CPL - 1 ? w.le[M2] : L0[c + 1], w.L[C][c], w.L[M1][c], L0[c], &l2);
    biharm_update(w.u[M2][c], l2, &o[c]);
  }
#pragma unroll
  for (int h = 0; h < CPL / 2; ++h) st_hint2(orow + CPL * lane + 2 * h, o[2 * h], o[2 * h + 1], pol);
}

// Four-row variant: windows of four rows (row % 4, rows unrolled by 4) so
// that lap2 can run two rows behind lap1 -- at marched row r, lap1 makes
// L(r-1) while lap2 + update consume L(r-4..r-2) and u(r-3), all produced on
// earlier rows: the two Laplacians of a row are independent dependency
// chains instead of one chained after the other.
template <int CPL>
struct Win4 {
  double u[4][CPL];
  double ex[4][2];
  double L[4][CPL];
  double lex[4];
  double uw[4], ue[4];
  double lw[4], le[4];
};

template <int CPL, int P>
__device__ __forceinline__ void biharm_row4(Win4<CPL>& w, const double* row, int t, int lane, int ex_col,
                                            double* orow, uint64_t pol) {
  constexpr int C = P, M1 = (P + 3) % 4, M2 = (P + 2) % 4, M3 = (P + 1) % 4;  // rows r, r-1, r-2, r-3 (= r-4: C)
  {
#pragma unroll
    for (int h = 0; h < CPL / 2; ++h) {
      const double2 a = lds2(row + CPL * lane + H + 2 * h);
      w.u[C][2 * h] = a.x;
      w.u[C][2 * h + 1] = a.y;
    }
    const double2 e = lds2(row + ex_col);
    w.ex[C][0] = e.x;
    w.ex[C][1] = e.y;
    const double left = __shfl_up_sync(0xffffffffu, w.u[C][CPL - 1], 1);
    const double right = __shfl_down_sync(0xffffffffu, w.u[C][0], 1);
    w.uw[C] = lane == 0 ? e.y : left;
    w.ue[C] = lane == 31 ? e.x : right;
  }
  double o[CPL];
  const bool out_row = t >= 6;  // marched rows start at jb-3: output row r-3 >= jb
  if (out_row) {
    // ---- lap2 + update at row r-3 from L rows r-4 (slot C), r-3 (M3), r-2 (M2): all from earlier rows
    const double* L0 = w.L[M3];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      double l2;
      lap5(c == 0 ? w.lw[M3] : L0[c - 1], c == CPL - 1 ? w.le[M3] : L0[c + 1], w.L[C][c], w.L[M2][c], L0[c], &l2);
      biharm_update(w.u[M3][c], l2, &o[c]);
    }
  }
  if (t >= 2) {
    // ---- lap1 at row r-1 into slot M1 (slot C keeps L(r-4) for the lap2 above)
    const double* um = w.u[M1];
    double* Ln = w.L[M1];
#pragma unroll
    for (int c = 0; c < CPL; ++c)
      lap5(c == 0 ? w.uw[M1] : um[c - 1], c == CPL - 1 ? w.ue[M1] : um[c + 1], w.u[M2][c], w.u[C][c], um[c], &Ln[c]);
    const bool lo = lane == 0;
    const double hw = lo ? w.ex[M1][0] : um[CPL - 1];
    const double he = lo ? um[0] : w.ex[M1][1];
    const int hc = lo ? 1 : 0;
    const double hs = hc ? w.ex[M2][1] : w.ex[M2][0];
    const double hn = hc ? w.ex[C][1] : w.ex[C][0];
    const double h0 = hc ? w.ex[M1][1] : w.ex[M1][0];
    lap5(hw, he, hs, hn, h0, &w.lex[M1]);
    const double left = __shfl_up_sync(0xffffffffu, Ln[CPL - 1], 1);
    const double right = __shfl_down_sync(0xffffffffu, Ln[0], 1);
    w.lw[M1] = lane == 0 ? w.lex[M1] : left;
    w.le[M1] = lane == 31 ? w.lex[M1] : right;
  }
  if (out_row) {
#pragma unroll
    for (int h = 0; h < CPL / 2; ++h) st_hint2(orow + CPL * lane + 2 * h, o[2 * h], o[2 * h + 1], pol);
  }
}

// IP: in place (RR == 4 only) -- a warp writes row j of its strip after it has
// consumed row j+3, so its own reads are never overtaken; see Params.
template <class K, bool IP = false>
__global__ void __launch_bounds__(32, K::OCC)
    biharm_fused(const __grid_constant__ CUtensorMap tin, double* __restrict__ out, const Params p) {
  constexpr int CPL = K::CPL, S = K::S, SW = K::SW, BOXW = K::BOXW, STAGE_BYTES = K::STAGE_BYTES;
  constexpr int STAGE_TX = K::STAGE_TX, RR = K::RR;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE_BYTES);
  const int lane = threadIdx.x;

  RowSeg seg[3];
  const int nseg = cta_segments(blockIdx.x, gridDim.x, p.strips, p.row_lo, p.row_hi, seg);
  RowRing<RR, S> rr;
  // staged column 0 = logical i0 - 2 = storage i0; storage row = logical + 2;
  // the four-row variant marches one more row (its output lags by three)
  rr.init(seg, nseg, RR == 4 ? H + 1 : H, smem, full, STAGE_BYTES, STAGE_TX, 0, H, SW);
  if (p.load_policy >= 0) {
    rr.load_hint = true;
    rr.load_pol = l2_store_policy(p.load_policy);
  }
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    tma_prefetch_desc(&tin);
    pdl_trigger();
  }
  pdl_wait();  // previous step's output (our input) complete, our output buffer free
  if (lane == 0)
    for (int g = 0; g < S; ++g) rr.issue(g, &tin);
  __syncwarp();

  const uint64_t pol = l2_store_policy(p.store_policy);
  // extra columns: lane 0 -> logical -2,-1 ; lane 31 -> SW, SW+1 ; others: harmless copy
  const int ex_col = lane == 0 ? 0 : (lane == 31 ? SW + H : CPL * lane + H);
  // zero ghost ring of the goal buffer at the global edges
  auto ghost_ring = [&](const RowSeg& sg) {
    const bool lo_edge = sg.strip == 0, hi_edge = sg.strip == p.strips - 1;
    for (int jo = sg.jb; jo < sg.je; jo += 32) {
      const int j = jo + lane;
      if (j < sg.je) {
        double* rr0 = out + (long long)(j + H) * p.pitch;
        if (lo_edge) st_hint2(rr0, 0.0, 0.0, pol);
        if (hi_edge) st_hint2(rr0 + H + p.ni, 0.0, 0.0, pol);
      }
    }
    for (int side = 0; side < 2; ++side) {
      if (side == 0 && !(sg.jb == 0 && p.write_ghost_top)) continue;
      if (side == 1 && !(sg.je == p.nj && p.write_ghost_bottom)) continue;
      for (int gr = 0; gr < H; ++gr) {
        double* o = out + (long long)(side == 0 ? gr : p.nj + H + gr) * p.pitch + H + sg.strip * SW;
#pragma unroll
        for (int h = 0; h < CPL / 2; ++h) st_hint2(o + CPL * lane + 2 * h, 0.0, 0.0, pol);
        if (lane == 0 && lo_edge) st_hint2(o - H, 0.0, 0.0, pol);
        if (lane == 31 && hi_edge) st_hint2(o + SW, 0.0, 0.0, pol);
      }
    }
  };
  int g = 0;
  if constexpr (RR == 3) {
  Win<CPL> w;
  for (int k = 0; k < nseg; ++k) {
    const RowSeg sg = seg[k];
    const int T = sg.je - sg.jb + 2 * H;  // rows jb-2 .. je+1
    // output row r-2 of marched row r = jb-2+t lives at storage row (jb-2+t-2)+2
    double* orow = out + (long long)(sg.jb - 2) * p.pitch + H + sg.strip * SW;
    for (int t0 = 0; t0 < T; t0 += 3, ++g) {
      rr.wait(g);
      const double* st = reinterpret_cast<const double*>(rr.stage(g));
      biharm_row<CPL, 0>(w, st, t0, lane, ex_col, orow, pol);
      orow += p.pitch;
      if (t0 + 1 < T) biharm_row<CPL, 1>(w, st + BOXW, t0 + 1, lane, ex_col, orow, pol);
      orow += p.pitch;
      if (t0 + 2 < T) biharm_row<CPL, 2>(w, st + 2 * BOXW, t0 + 2, lane, ex_col, orow, pol);
      orow += p.pitch;
      // every lane has consumed this stage: hand the slot to stage g + S
      __syncwarp();
      if (lane == 0) rr.issue(g + S, &tin);
    }
    ghost_ring(sg);
  }
  } else {
  Win4<CPL> w;
  for (int k = 0; k < nseg; ++k) {
    const RowSeg sg = seg[k];
    // rows jb-3 .. je+2 (the ring stages from jb-3: halo H+1); output row r-3
    const int T = sg.je - sg.jb + 2 * H + 2;
    double* orow = out + (long long)(sg.jb - 4) * p.pitch + H + sg.strip * SW;
    // in place: where the lane's pair of marched row t goes (biharm_row4 stores at
    // dest + CPL * lane).  An edge lane next to a neighbouring strip walks the
    // column band (4 doubles per row) instead of the grid (one pitch per row);
    // the rows next to a segment cut -- the first two and the last two output
    // rows, marched rows 6, 7 and T-2, T-1 -- go to the row band.
    [[maybe_unused]] double* lp = orow;
    [[maybe_unused]] long long ls = p.pitch;
    if constexpr (IP) {
      const bool cl = lane == 0 && sg.strip > 0, cr = lane == 31 && sg.strip < p.strips - 1;
      if (cl || cr) {
        lp = p.colband + ((long long)((cl ? sg.strip - 1 : sg.strip) * (long long)p.nj + (sg.jb - 6)) * 4 + (cl ? 2 : 0)) -
             CPL * lane;
        ls = 4;
      }
    }
    auto dest = [&](int t, double* grid) -> double* {
      if constexpr (!IP) {
        return grid;  // the plain kernel: exactly the row pointer it always used
      } else {
        double* d = lp;
        lp += ls;
        if (t < 6 + H || t >= T - H) {
          const int jo = sg.jb - 6 + t;  // output row of marched row t
          const int rs = band_row_slot(jo, sg.jb, sg.je, sg.jb > p.row_lo, sg.je < p.row_hi);
          if (rs >= 0) d = p.rowband + (size_t)(((blockIdx.x * 3 + k) * 4 + rs) * SW);
        }
        return d;
      }
    };
    for (int t0 = 0; t0 < T; t0 += 4, ++g) {
      rr.wait(g);
      const double* st = reinterpret_cast<const double*>(rr.stage(g));
      biharm_row4<CPL, 0>(w, st, t0, lane, ex_col, dest(t0, orow), pol);
      orow += p.pitch;
      if (t0 + 1 < T) biharm_row4<CPL, 1>(w, st + BOXW, t0 + 1, lane, ex_col, dest(t0 + 1, orow), pol);
      orow += p.pitch;
      if (t0 + 2 < T) biharm_row4<CPL, 2>(w, st + 2 * BOXW, t0 + 2, lane, ex_col, dest(t0 + 2, orow), pol);
      orow += p.pitch;
      if (t0 + 3 < T) biharm_row4<CPL, 3>(w, st + 3 * BOXW, t0 + 3, lane, ex_col, dest(t0 + 3, orow), pol);
      orow += p.pitch;
      __syncwarp();
      if (lane == 0) rr.issue(g + S, &tin);
    }
    ghost_ring(sg);
  }
  }
}


// In-place step, second launch: the deferred cells go to their places (same
// grid and segment list as the step's launch; the zero ghost ring needs none).
constexpr int COMMIT_NT = 128;  // the copies are latency-bound: a CTA's rows in one or two round trips
template <class K>
__global__ void __launch_bounds__(COMMIT_NT) biharm_commit(double* __restrict__ out, const Params p) {
  constexpr int SW = K::SW;
  const int tid = threadIdx.x;
  if (tid == 0) pdl_trigger();
  pdl_wait();  // every CTA of the step has finished reading the array
  RowSeg seg[3];
  const int nseg = cta_segments(blockIdx.x, gridDim.x, p.strips, p.row_lo, p.row_hi, seg);
  for (int k = 0; k < nseg; ++k) {
    const RowSeg sg = seg[k];
    const bool above = sg.jb > p.row_lo, below = sg.je < p.row_hi;
    // 16-B pieces: a thread moves a column pair (all offsets are even: SW, H and the pitch are)
    for (int idx = tid; idx < 2 * H * (SW / 2); idx += COMMIT_NT) {
      const int rs = idx / (SW / 2), c = 2 * (idx % (SW / 2));
      const int j = rs < H ? sg.jb + rs : sg.je - 2 * H + rs;
      if (j < sg.jb || j >= sg.je || band_row_slot(j, sg.jb, sg.je, above, below) != rs) continue;
      *reinterpret_cast<double2*>(out + (long long)(j + H) * p.pitch + H + sg.strip * SW + c) =
          *reinterpret_cast<const double2*>(p.rowband + (size_t)(((blockIdx.x * 3 + k) * 4 + rs) * SW) + c);
    }
    const bool left = sg.strip > 0, right = sg.strip < p.strips - 1;
    if (!left && !right) continue;
    // thread (row, side): side 0 the strip's first two columns, 1 its last two
    for (int idx = tid; idx < (sg.je - sg.jb) * 2; idx += COMMIT_NT) {
      const int j = sg.jb + (idx >> 1), side = idx & 1;
      if (side == 0 ? !left : !right) continue;
      if (band_row_slot(j, sg.jb, sg.je, above, below) >= 0) continue;
      const size_t e = side == 0 ? sg.strip - 1 : sg.strip;
      *reinterpret_cast<double2*>(out + (long long)(j + H) * p.pitch + H + sg.strip * SW + (side == 0 ? 0 : SW - 2)) =
          *reinterpret_cast<const double2*>(p.colband + (e * p.nj + j) * 4 + (side == 0 ? 2 : 0));
    }
  }
}

// variant table (LF_BIHARM_VARIANT=<index> overrides the default for tuning runs)
struct Variant {
  const char* name;
  int sw;
  void (*kernel)(CUtensorMap, double*, Params);
  int smem, occ;
  int rows;  // rows per TMA stage (3 or 4)
};
template <class K>
Variant make_variant(const char* n) {
  return {n, K::SW, biharm_fused<K>, K::SMEM, K::OCC, K::RR};
}
const Variant& variant() {
  static const Variant table[] = {
      make_variant<Cfg<4, 4, 16>>("cpl4_s4_occ16"), make_variant<Cfg<2, 4, 16>>("cpl2_s4_occ16"),
      make_variant<Cfg<2, 6, 24>>("cpl2_s6_occ24"), make_variant<Cfg<4, 6, 12>>("cpl4_s6_occ12"),
      make_variant<Cfg<2, 8, 16>>("cpl2_s8_occ16"), make_variant<Cfg<4, 8, 8>>("cpl4_s8_occ8"),
      make_variant<Cfg<2, 16, 8>>("cpl2_s16_occ8"), make_variant<Cfg<2, 12, 10>>("cpl2_s12_occ10"),
      make_variant<Cfg<4, 6, 10>>("cpl4_s6_occ10"), make_variant<Cfg<2, 10, 12>>("cpl2_s10_occ12"),
      make_variant<Cfg<2, 8, 12>>("cpl2_s8_occ12"), make_variant<Cfg<2, 12, 12>>("cpl2_s12_occ12"),
      make_variant<Cfg<2, 16, 10>>("cpl2_s16_occ10"), make_variant<Cfg<2, 6, 16>>("cpl2_s6_occ16"),
      make_variant<Cfg<2, 9, 10, 4>>("cpl2_r4_s9_occ10"), make_variant<Cfg<2, 6, 12, 4>>("cpl2_r4_s6_occ12"),
      make_variant<Cfg<2, 12, 8, 4>>("cpl2_r4_s12_occ8"), make_variant<Cfg<4, 6, 8, 4>>("cpl4_r4_s6_occ8"),
      make_variant<Cfg<2, 6, 14, 4>>("cpl2_r4_s6_occ14"), make_variant<Cfg<2, 5, 14, 4>>("cpl2_r4_s5_occ14"),
      make_variant<Cfg<2, 8, 12, 4>>("cpl2_r4_s8_occ12"), make_variant<Cfg<2, 7, 12, 4>>("cpl2_r4_s7_occ12"),
  };
  static int idx = [] {
    const char* e = lfx::option("LF_BIHARM_VARIANT");
    // default cpl2_r4_s7_occ12: best of the measured sweep (profiles/r01_biharm_variants.txt)
    int i = e ? std::atoi(e) : 21;
    return (i >= 0 && i < (int)(sizeof table / sizeof table[0])) ? i : 21;
  }();
  return table[idx];
}

bool supports(const lf::Plan& plan, std::string& why) {
  const auto& r = plan.rs.ranges;
  for (const auto& rg : r)
    if (rg.stride != 1 || rg.lo != 0) {
      why = "biharmonic executor needs unit strides and ranges starting at 0";
      return false;
    }
  long nj = r[0].trips(), ni = r[1].trips();
  if (ni % 128 || nj < 1) {
    why = "biharmonic executor needs N_i % 128 == 0 (got " + std::to_string(ni) + ")";
    return false;
  }
  return true;
}

int launch_step(const double* in, double* out, int ni, const RowPart& rp, cudaStream_t st, std::string& err) {
  const int nj = rp.rows;
  const Variant& v = variant();
  static LaunchCache cache;  // the variant is fixed per process (LF_BIHARM_VARIANT)
  int slots = 0;
  if (int s = resident_slots(cache, reinterpret_cast<const void*>(v.kernel), 32, v.smem, v.occ,
                             "cudaFuncSetAttribute(biharm)", &slots, err))
    return s;
  CUtensorMap map;
  uint64_t dims[2] = {(uint64_t)ni + 4, (uint64_t)nj + 4};
  uint32_t box[2] = {(uint32_t)(v.sw + 2 * H), (uint32_t)v.rows};  // must match the kernel's stage bytes
  if (!make_tensor_map(&map, in, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 2, dims, box, err)) return LF_ERR_CUDA;
  Params p;
  p.ni = ni;
  p.nj = nj;
  p.pitch = ni + 4;
  p.strips = ni / v.sw;
  p.row_lo = rp.lo;
  p.row_hi = rp.hi;
  p.write_ghost_top = rp.top;
  p.write_ghost_bottom = rp.bottom;
  // evict_last: the output of an iteration is the next one's input and 134 MB
  // of it at 4096^2 nearly fits the 126 MB L2 -- same-box A/B 321 -> 340 G
  // (evict_first) at 4096^2, 289 -> 295 G at 16384^2 (LF_BIHARM_STORE_POLICY)
  const int store_policy = [] {
    const char* e = lfx::option("LF_BIHARM_STORE_POLICY");
    return e ? std::atoi(e) : 2;
  }();
  p.store_policy = store_policy;
  // TMA fetches with an explicit evict_normal hint: same-box A/B 341 -> 346 G
  // at 4096^2, 292 -> 298 G at 16384^2 against plain fetches (evict_first 334 G)
  const int load_policy = [] {
    const char* e = lfx::option("LF_BIHARM_LOAD_POLICY");
    return e ? std::atoi(e) : 1;
  }();
  p.load_policy = load_policy;
  p.colband = p.rowband = nullptr;
  // at least ~16 rows per CTA so the 4 priming rows stay a small fraction
  const int ctas = rowstream_ctas(slots, p.strips, rp.hi - rp.lo);
  if ((long long)ctas * 2 < p.strips) {
    err = "row range too short for the resident grid";
    return LF_ERR_UNSUPPORTED;
  }
  return cuda_status(launch_pdl(v.kernel, dim3(ctas), dim3(32), v.smem, st, map, out, p), "biharm_fused launch",
                     err);
}

// Whole-domain steps on ONE buffer (the caller passed g_unew on g_u's buffer,
// declared in config.aliases): the default four-row variant's in-place build,
// then the band commit, per step.  Bands are plan-owned: 4 columns per strip
// boundary and 4 rows per segment cut.
int run_inplace(const ExecArgs& a, std::string& err) {
  using K = Cfg<2, 7, 12, 4>;  // = the default variant (cpl2_r4_s7_occ12)
  static_assert(K::CPL == H, "an edge lane's columns are exactly the neighbour strip's halo");
  const auto& r = a.plan->rs.ranges;
  const int ni = (int)r[1].trips();
  const RowPart rp = row_part(a, (int)r[0].trips());
  if (a.slab || !a.mem) {
    err = "biharm2d_fused_tma runs in place on the whole domain only (no slabs or row parts)";
    return LF_ERR_UNSUPPORTED;
  }
  double* u = static_cast<double*>(a.terms[0]);
  void (*const kern)(CUtensorMap, double*, Params) = biharm_fused<K, true>;
  static LaunchCache cache;
  int slots = 0;
  if (int s = resident_slots(cache, reinterpret_cast<const void*>(kern), 32, K::SMEM, K::OCC,
                             "cudaFuncSetAttribute(biharm in place)", &slots, err))
    return s;
  Params p;
  p.ni = ni;
  p.nj = rp.rows;
  p.pitch = ni + 4;
  p.strips = ni / K::SW;
  p.row_lo = rp.lo;
  p.row_hi = rp.hi;
  p.write_ghost_top = rp.top;
  p.write_ghost_bottom = rp.bottom;
  p.store_policy = 2;
  p.load_policy = 1;
  const int ctas = rowstream_ctas(slots, p.strips, rp.hi - rp.lo);
  if ((long long)ctas * 2 < p.strips) {
    err = "row range too short for the resident grid";
    return LF_ERR_UNSUPPORTED;
  }
  const size_t ncol = (size_t)std::max(0, p.strips - 1) * p.nj * 4, nrow = (size_t)ctas * 3 * 4 * K::SW;
  const size_t band_bytes = (ncol + nrow) * sizeof(double);
  void* band_ptr = nullptr;
  if (int s = band_memory(*a.mem, band_bytes, a.stream, &band_ptr, err)) return s;
  p.colband = static_cast<double*>(band_ptr);
  p.rowband = p.colband + ncol;
  CUtensorMap map;
  uint64_t dims[2] = {(uint64_t)ni + 4, (uint64_t)p.nj + 4};
  uint32_t box[2] = {(uint32_t)(K::SW + 2 * H), (uint32_t)K::RR};
  if (!make_tensor_map(&map, u, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 2, dims, box, err)) return LF_ERR_CUDA;
  // LF_BIHARM_IP_PDL (tuning): bit 0 = the step, bit 1 = the commit launched with
  // programmatic stream serialization
  const char* o = lfx::option("LF_BIHARM_IP_PDL");
  const int pdl = o ? std::atoi(o) : 1;
  for (int s = 0; s < a.steps; ++s) {
    cudaError_t ce;
    if (pdl & 1) {
      ce = launch_pdl(kern, dim3(ctas), dim3(32), K::SMEM, a.stream, map, u, p);
    } else {
      kern<<<ctas, 32, K::SMEM, a.stream>>>(map, u, p);
      ce = cudaGetLastError();
    }
    if (int st = cuda_status(ce, "biharm_fused (in place) launch", err)) return st;
    if (pdl & 2) {
      ce = launch_pdl(biharm_commit<K>, dim3(ctas), dim3(COMMIT_NT), 0, a.stream, u, p);
    } else {
      biharm_commit<K><<<ctas, COMMIT_NT, 0, a.stream>>>(u, p);
      ce = cudaGetLastError();
    }
    if (int st = cuda_status(ce, "biharm_commit launch", err)) return st;
  }
  return band_guard_check(*a.mem, band_bytes, a.stream, err);
}

int run(const ExecArgs& a, std::string& err) {
  if (a.inplace) return run_inplace(a, err);
  const auto& r = a.plan->rs.ranges;
  const int ni = (int)r[1].trips();
  const RowPart rp = row_part(a, (int)r[0].trips());
  const double* src = static_cast<const double*>(a.terms[0]);
  double* goal = static_cast<double*>(a.terms[1]);
  double* scratch = a.steps > 1 ? static_cast<double*>(a.scratch[0]) : nullptr;
  for (int s = 0; s < a.steps; ++s) {
    double* dst = ((a.steps - 1 - s) % 2) == 0 ? goal : scratch;
    int st = launch_step(src, dst, ni, rp, a.stream, err);
    if (st != LF_OK) return st;
    src = dst;
  }
  return LF_OK;
}

}  // namespace

extern const Executor biharm_executor = {"biharm2d_fused_tma", "biharmonic2d.lf", 1, 16.0, supports, run,
                                         nullptr, false, nullptr, /*inplace=*/true};

}  // namespace lfx

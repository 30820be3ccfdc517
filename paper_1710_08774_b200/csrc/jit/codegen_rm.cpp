// Generic executor, part 3: the register march of 2D chains (lf_jit_step_rm).
//
// The HFAV schedule of codegen.cpp's marches (a CTA marches the outer
// dimension, callsite group g computes row t + s_g at trip t, s_g the pipeline
// shift of shifts.cpp:8-79, each intermediate kept for the W_v rows of its
// contraction, storage.cpp:319-399), with the storage moved one level closer
// to the ALUs:
//
//  * every consumer warp owns a strip of tw output columns and computes its
//    own halo, so warps never wait for one another: no CTA barrier at all;
//  * a lane owns V adjacent cells of the strip (V = 4 fp32 / 2 fp64 by
//    default): streamed axioms are read from their shared-memory ring (filled
//    by the producer warp's TMA row boxes, as in lf_jit_step_ws) with 16-B
//    vector loads, neighbours along the row come from the adjacent lanes by
//    warp shuffles;
//  * intermediates live in registers: variable v keeps its last W_v rows as
//    T R_v[W_v][V], rotated once per trip.
//
// Lanes near the strip edges receive shuffled values from outside the warp
// (junk); the tile width is chosen so that every cell a group must produce is
// at least the accumulated stencil reach away from the edges (margins A_g / B_g
// below), and only those cells are stored.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <set>
#include <sstream>
#include <tuple>

#include "../planner/dsl.hpp"
#include "codegen_ctx.hpp"

namespace lfx::cg {

namespace {

long floordiv(long a, long b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

std::string num(long v) { return v < 0 ? "m" + std::to_string(-v) : std::to_string(v); }

}  // namespace

// In place: the column band around an internal tile boundary e holds the
// cells neighbouring tiles read, [e + lo1, e + hi1), widened to whole 32-B
// sectors of the grid row, so no grid sector is left half written until the
// commit (a partly written sector costs L2 a read-modify-write).  Logical
// columns [zs(e), ze(e)); at most bw columns.
struct Zone {
  long so1 = 0, se = 4, lo1 = 0, hi1 = 0, bw = 0;
  std::string zs(const std::string& e) const {
    return "((((" + e + ")" + plus(lo1 + so1) + ") & ~" + std::to_string(se - 1) + ")" + plus(-so1) + ")";
  }
  std::string ze(const std::string& e) const {
    return "((((" + e + ")" + plus(hi1 + so1 + se - 1) + ") & ~" + std::to_string(se - 1) + ")" + plus(-so1) + ")";
  }
};
Zone zone_of(const Ctx& C, size_t v, int ti, int eb) {
  Zone z;
  z.so1 = -C.P.terminals[ti].base[1] + C.LO[1];
  z.se = 32 / eb;
  z.lo1 = C.vmin[v][1];
  z.hi1 = C.vmax[v][1];
  z.bw = z.hi1 - z.lo1 + 2 * (z.se - 1);
  return z;
}

// In place, 2D: after the step, copy the deferred boundary writes from the
// band buffers into the grid -- the row bands (full rows around the internal
// chunk boundaries, domain columns) and the column bands (around the internal
// tile boundaries of width `tile1`, rows outside every row band)
void emit_commit2(Ctx& C, const char* name, const std::vector<std::pair<size_t, int>>& caps,
                  const std::vector<int>& slots, int tile1, std::ostream& src, bool with_fill) {
  // flat over the band cells -- (band row, domain column) pairs, then (band
  // column, row) pairs -- four per thread, a block per 1024; the launch covers
  // the largest band set (jit.cpp)
  src << "extern \"C\" __global__ void __launch_bounds__(256) " << name << "(const LfArgs a) {\n";
  src << "  const int N0 = (int)a.n0;\n";
  src << "  const int nch = (N0 + a.chunk - 1) / a.chunk;\n";
  for (size_t q = 0; q < caps.size(); ++q) {
    const size_t v = caps[q].first;
    const auto& t = C.P.terminals[caps[q].second];
    const long so0 = -t.base[0] + C.LO[0], so1 = -t.base[1] + C.LO[1];
    const long E1 = t.extent[1], E0 = t.extent[0];
    const long lo0 = C.vmin[v][0], hi0 = C.vmax[v][0];
    const Zone z = zone_of(C, v, caps[q].second, static_cast<int>(t.elem_bytes));
    const long BH = hi0 - lo0, BW = z.bw;
    const long NT = (C.N[1] + tile1 - 1) / tile1;
    src << "  {\n";
    src << "    T* m = reinterpret_cast<T*>(a.t[" << caps[q].second << "]);\n";
    src << "    const T* rb = reinterpret_cast<const T*>(a.t[" << slots[q] << "]);\n";
    src << "    const T* cb = reinterpret_cast<const T*>(a.t[" << slots[q] + 1 << "]);\n";
    src << "    const long long nr = (long long)max(0, nch - 1) * " << BH * C.N[1] << ";  // row-band cells\n";
    src << "    const long long nc = (long long)N0 * " << (NT - 1) * BW << ";  // column-band cells\n";
    src << "    #pragma unroll\n";
    src << "    for (int j = 0; j < 4; ++j) {\n";
    src << "      const long long p = (long long)blockIdx.x * 1024 + j * 256 + threadIdx.x;\n";
    src << "      if (p < nr) {\n";
    src << "        const int r = (int)(p / " << C.N[1] << "), x = (int)(p - (long long)r * " << C.N[1] << ");\n";
    src << "        const int y = (r / " << BH << " + 1) * a.chunk" << plus(lo0) << " + r % " << BH << ";\n";
    src << "        if (y >= 0 && y < N0) m[(long long)(y" << plus(so0) << ") * " << E1 << "LL" << plus(so1) << " + x] = rb[(long long)r * "
        << E1 << "LL" << plus(so1) << " + x];\n";
    src << "      } else if (p - nr < nc) {\n";
    src << "        const int kc = (int)((p - nr) / N0), y = (int)(p - nr - (long long)kc * N0);  // band column kc = k * bw + c\n";
    src << "        const int bb = (y" << plus(-lo0) << ") / a.chunk * a.chunk;  // the one boundary whose row band could hold y\n";
    src << "        const int e = (kc / " << BW << " + 1) * " << tile1 << ", x = " << z.zs("e") << " + kc % " << BW << ";\n";
    src << "        if (!(bb > 0 && bb < N0 && y < bb" << plus(hi0) << ") && x >= 0 && x < " << C.N[1] << " && x < " << z.ze("e")
        << ") m[(long long)(y" << plus(so0) << ") * " << E1 << "LL" << plus(so1) << " + x] = cb[(long long)kc * " << E0 << " + y"
        << plus(so0) << "];\n";
    src << "      }\n    }\n  }\n";
  }
  // the ghost refill too (zero boundaries only: it reads no cell the commit writes)
  if (with_fill) src << "  lf_fill_body(a);\n";
  src << "}\n";
}

// The register-march emitter (lf_jit_step_rm): rows() sizes the rolling
// windows (a shared-memory ring per streamed axiom, registers per
// intermediate), columns() the lane span and strip width from the groups'
// exactness margins, layout() the shared memory, inplace() the deferred-write
// bands, head() the kernel head and the per-unit setup, trips() the unrolled
// trip loop: producer() the TMA row boxes, group() one callsite group,
// copy_tail() the window rotation; commit() the in-place commit kernel.
class RMarch {
 public:
  RMarch(Ctx& c, JitProgram& o, std::ostream& s)
      : C(c), out(o), src(s), eb(o.elem_bytes), CH(16 / o.elem_bytes), nv(c.P.vars.size()), G(c.groups) {}
  bool emit() {
    if (C.nd != 2) return false;
    if (!rows() || !columns() || !layout()) return false;
    inplace();
    trip_range();
    head();
    maps();
    if (!trips()) return false;
    commit();
    return true;
  }

 private:
  struct IP {
    size_t v;
    int ai, gi, slot;
  };
  Ctx& C;
  JitProgram& out;
  std::ostream& src;
  const int eb, CH;  // element bytes, elements per 16-B chunk
  const size_t nv;
  const std::vector<Grp>& G;
  const std::string VT = eb == 8 ? "double2" : "float4";
  const char* comp[4] = {"x", "y", "z", "w"};
  int V = 4, NW = 8, PD = 3, NS = 4;  // cells per lane, consumer warps, trips in flight, ring stages
  std::vector<int> lead, old, win, staged, drop;
  int goal_ti = -1;
  std::vector<int> vmin1, vmax1, A, B;
  std::vector<long> base_al, rho;
  long cs = 0, tw = 0, T1 = 0, inner = 1;
  std::vector<int> nbox, bw;
  std::vector<long> soff;
  size_t smem = 0;
  std::vector<IP> ips;
  int TS = 0, TE = 0;
  int U = 1, cu = 0;  // trip-loop unroll (register-window renaming), the copy being emitted
  std::string trip_end;

  bool rows();
  bool columns();
  bool layout();
  void inplace();
  void trip_range();
  void head();
  void maps();
  bool trips();
  void producer();
  bool group(size_t gi);
  void store_goals(size_t gi, const std::vector<std::pair<int, const GOut*>>& goals);
  void copy_tail();
  void commit();
  long goal_so(int ti) const { return -C.P.terminals[ti].base[1] + C.LO[1]; }  // storage col = logical + so
  int phys(int v, int k) const { return U == 1 ? k : (k + cu) % win[v]; }
  const IP* ip_of_goal(int ti) const {
    for (const auto& ip : ips)
      if (ip.gi == ti) return &ip;
    return nullptr;
  }
  std::string rowbase(size_t v, int off) const {
    const int W = win[v];
    if (W == 1) return "0";
    const int o = ((off % W) + W) % W;
    const std::string b = "b" + std::to_string(v);
    const std::string sum = o ? "(" + b + " + " + std::to_string(o) + ")" : b;
    const std::string sl =
        o ? "(" + sum + " >= " + std::to_string(W) + " ? " + sum + " - " + std::to_string(W) + " : " + sum + ")" : b;
    return sl + " * " + std::to_string(nbox[v] * bw[v]);
  }
};

bool RMarch::rows() {
  V = eb == 8 ? 2 : 4;
  if (const char* e = lfx::option("LF_JIT_RM_V")) V = std::atoi(e);
  if (V < CH || V % CH || V > 16) return false;
  NW = 8;  // consumer warps per CTA
  if (const char* e = lfx::option("LF_JIT_RM_WARPS")) NW = std::max(1, std::min(16, std::atoi(e)));
  PD = 3;
  if (const char* e = lfx::option("LF_JIT_PD")) PD = std::max(1, std::atoi(e));
  NS = PD + 1;
  if (G.empty()) return false;
  for (const auto& g : G)
    for (const auto& o : g.out)
      if (o.rel[1] != 0) return false;  // outputs at the group's anchor column only

  // ---- rows: streamed axioms in a shared-memory ring (+ PD rows in flight),
  // intermediates in registers (exactly the contraction span)
  lead.assign(nv, INT_MIN);
  old.assign(nv, INT_MAX);
  win.assign(nv, 0);
  staged.assign(nv, -1);
  for (const auto& g : G)
    for (const auto& in : g.loads) {
      lead[in.var] = std::max(lead[in.var], C.smem_var[in.var] ? INT_MIN : g.shift + in.rel[0]);
      old[in.var] = std::min(old[in.var], g.shift + in.rel[0]);
    }
  for (const auto& g : G)
    for (const auto& o : g.out)
      if (C.smem_var[o.var]) lead[o.var] = g.shift + o.rel[0];
  int reg_words = 0;
  for (size_t v = 0; v < nv; ++v) {
    if (C.smem_var[v]) {
      if (old[v] == INT_MAX) return false;
      win[v] = lead[v] - old[v] + 1;
      reg_words += win[v] * V * eb / 4;
    } else if (old[v] != INT_MAX && C.staged_axiom(static_cast<int>(v)) >= 0) {
      staged[v] = C.staged_axiom(static_cast<int>(v));
      win[v] = lead[v] - old[v] + 1 + PD;
    }
    if (win[v] > 0 && (win[v] > 64 || old[v] < -60 || lead[v] > 60)) return false;
  }
  if (reg_words > 96) return false;  // register windows would spill
  // fault injection (R/SPEC.md:557, as in emit_march): the named intermediate
  // keeps one row fewer than its contraction span
  drop.assign(nv, 0);
  if (const char* f = lfx::option("LF_JIT_FAULT"); f && std::strncmp(f, "span:", 5) == 0)
    for (size_t v = 0; v < nv; ++v)
      if (C.smem_var[v] && win[v] > 1 && C.P.vars[v].name == f + 5) {
        drop[v] = 1;
        win[v] -= 1;
      }

  return true;
}

bool RMarch::columns() {
  // ---- columns.  A lane's cells are c = cs + lane * V + i (warp-strip
  // relative).  A_g / B_g: how far from the lane span's left / right end group
  // g's values are still exact -- each shuffle across the warp edge eats the
  // reach of the read: a register variable at column offset dr, or a streamed
  // row (whose lane vectors start rho_v cells left of the lane's first cell)
  // at rho_v + dr.  The first goal fixes the lane alignment (its 16-B chunks
  // start at lane cells): cs = res (mod CH)
  goal_ti = -1;
  for (const auto& g : G)
    for (const auto& o : g.out)
      if (goal_ti < 0 && C.terminal_of(o.var, true) >= 0) goal_ti = C.terminal_of(o.var, true);
  if (goal_ti < 0) return false;
  vmin1.assign(nv, 0);
  vmax1.assign(nv, 0);
  for (size_t v = 0; v < nv; ++v) {
    if (staged[v] < 0) continue;
    const auto& t = C.P.terminals[staged[v]];
    const long so = C.extra_of(static_cast<int>(v))[1] - t.base[1] + C.LO[1];
    vmin1[v] = C.vmin[v][1];
    vmax1[v] = C.vmax[v][1];
    vmin1[v] -= static_cast<int>(((vmin1[v] + so) % CH + CH) % CH);  // TMA box origin 16-B aligned
  }
  base_al.assign(nv, 0);
  rho.assign(nv, 0);
  A.assign(G.size(), 0);
  B.assign(G.size(), 0);
  auto margins = [&](long cs) {
    for (size_t v = 0; v < nv; ++v)
      if (staged[v] >= 0) {
        const long D = cs - vmin1[v];
        base_al[v] = floordiv(D, CH) * CH;
        rho[v] = D - base_al[v];
      }
    std::map<int, std::pair<int, int>> margin;  // register variable -> (A, B) of its producer
    for (size_t gi = 0; gi < G.size(); ++gi) {
      int a = 0, b = 0;
      for (const auto& ld : G[gi].loads) {
        if (C.smem_var[ld.var]) {
          const auto [pa, pb] = margin.at(ld.var);
          a = std::max(a, pa - ld.rel[1]);
          b = std::max(b, pb + ld.rel[1]);
        } else if (staged[ld.var] >= 0) {
          a = std::max(a, static_cast<int>(-(rho[ld.var] + ld.rel[1])));
          b = std::max(b, static_cast<int>(rho[ld.var] + ld.rel[1]));
        }
      }
      A[gi] = a;
      B[gi] = b;
      for (const auto& o : G[gi].out)
        if (C.smem_var[o.var]) margin[o.var] = {a, b};
    }
  };
  const long res = ((-goal_so(goal_ti)) % CH + CH) % CH;
  cs = LONG_MAX;
  for (size_t gi = 0; gi < G.size(); ++gi) cs = std::min<long>(cs, G[gi].gmin[1]);
  cs = res + floordiv(cs - res, CH) * CH;
  for (int it = 0;; ++it) {
    margins(cs);
    bool ok = true;
    for (size_t gi = 0; gi < G.size(); ++gi) ok &= G[gi].gmin[1] >= cs + A[gi];
    if (ok) break;
    if (it > 8) return false;
    cs -= CH;
  }
  tw = LONG_MAX;
  for (size_t gi = 0; gi < G.size(); ++gi) tw = std::min<long>(tw, cs + 32L * V - B[gi] - G[gi].gmax[1]);
  tw = tw / CH * CH;
  if (tw < 2 * CH || tw < 4) return false;
  if (const char* e = lfx::option("LF_JIT_RM_TW")) tw = std::min<long>(tw, std::max(CH, std::atoi(e) / CH * CH));
  T1 = NW * tw;  // CTA tile
  inner = (C.N[1] + T1 - 1) / T1;

  return true;
}

bool RMarch::layout() {
  // ---- shared memory: the streamed axioms' rings (TMA boxes of <= 256
  // elements, 128-B multiples), 16-B aligned windows, guard pads for the
  // junk lanes' reads just outside a window
  nbox.assign(nv, 1);
  bw.assign(nv, 0);
  soff.assign(nv, 0);
  long lo_idx = 0, hi_over = 0;
  for (size_t v = 0; v < nv; ++v) {
    if (staged[v] < 0) continue;
    const int w = static_cast<int>(T1) + vmax1[v] - vmin1[v];
    const int al = 128 / eb;
    nbox[v] = (w + 255) / 256;
    bw[v] = ((w + nbox[v] - 1) / nbox[v] + al - 1) / al * al;
    if (bw[v] > 256) nbox[v] += 1, bw[v] = ((w + nbox[v] - 1) / nbox[v] + al - 1) / al * al;
    // lane vectors span [base_al, (NW-1) tw + 32 V + base_al)
    lo_idx = std::min(lo_idx, base_al[v]);
    hi_over = std::max(hi_over, (NW - 1) * tw + 32L * V + base_al[v] - static_cast<long>(nbox[v]) * bw[v]);
  }
  const size_t pad_front = static_cast<size_t>((-lo_idx * eb + 127) / 128 * 128);
  smem = pad_front;
  for (size_t v = 0; v < nv; ++v) {
    if (staged[v] < 0) continue;
    soff[v] = smem;
    smem += (static_cast<size_t>(win[v]) * nbox[v] * bw[v] * eb + 127) / 128 * 128;
  }
  smem += static_cast<size_t>((std::max(0L, hi_over) * eb + 127) / 128 * 128);
  if (smem == pad_front) return false;  // nothing streamed
  if (smem + 16 * NS > 200 * 1024) return false;
  out.rm_smem_bytes = smem + 16 * NS;
  out.rm_threads = 32 * (NW + 1);
  out.rm_inner_tiles = inner;
  out.rm_maps.clear();
  return true;
}

void RMarch::inplace() {
  // in place (config.aliases, the caller passes one buffer): whole (chunk,
  // CTA tile) units that defer their boundary writes.  A unit's cells that a
  // neighbouring unit still reads during the step -- rows within the read
  // reach of an internal chunk boundary, columns within that of an internal
  // tile boundary -- go to band buffers instead of the grid, and a commit
  // kernel copies them in after the step.  So the grid a unit streams from
  // holds the step's input everywhere another unit looks, every row is one
  // TMA box as out of place, and no halo needs patching.  Bands use the plain
  // march's argument slots (row bands full width, [boundary][row][col]; column
  // bands column-major, [boundary][col within the band][row], so an edge lane's
  // writes down the march fill whole sectors).
  ips.clear();
  out.rm_inplace.clear();
  {
    const int nterm = static_cast<int>(C.P.terminals.size());
    for (const auto& [in_ext, out_ext] : C.P.rs.aliases) {
      int ai = -1, gi = -1;
      for (int i = 0; i < nterm; ++i) {
        if (!C.P.terminals[i].is_goal && C.P.terminals[i].name == in_ext) ai = i;
        if (C.P.terminals[i].is_goal && C.P.terminals[i].name == out_ext) gi = i;
      }
      if (ai < 0 || gi < 0) continue;
      const int v = C.P.terminals[ai].var;
      const auto& t = C.P.terminals[ai];
      if (v < 0 || staged[v] < 0 || t.extent != C.P.terminals[gi].extent || t.base != C.P.terminals[gi].base) {
        out.rm_inplace.clear();
        ips.clear();
        break;
      }
      IP ip{static_cast<size_t>(v), ai, gi, nterm + 3 * static_cast<int>(ips.size())};
      if (ip.slot + 3 > 32) {
        out.rm_inplace.clear();
        ips.clear();
        break;
      }
      ips.push_back(ip);
      JitProgram::Inplace q;
      q.ai = ai;
      q.gi = gi;
      q.bh = C.vmax[v][0] - C.vmin[v][0];
      q.bw1 = static_cast<int>(zone_of(C, static_cast<size_t>(v), gi, eb).bw);
      if (T1 < 2 * q.bw1) {  // zones of neighbouring boundaries must not meet
        out.rm_inplace.clear();
        ips.clear();
        break;
      }
      q.e0 = t.extent[0];
      q.e1 = t.extent[1];
      q.t1 = static_cast<int>(T1);
      q.n1 = C.N[1];
      out.rm_inplace.push_back(q);
    }
  }
}

void RMarch::trip_range() {
  // trip range relative to the chunk [r0, r1)
  TS = INT_MAX;
  TE = INT_MIN;
  for (const auto& g : G) {
    TS = std::min(TS, g.gmin[0] - g.shift);
    TE = std::max(TE, g.gmax[0] - g.shift);
  }
  for (size_t v = 0; v < nv; ++v)
    if (staged[v] >= 0) TS = std::min(TS, C.vmin[v][0] - lead[v]);

}

void RMarch::head() {
  int minb = 3;  // <= 72 registers: 3 CTAs of 9 warps per SM (the in-place store path needs 75 uncapped)
  if (const char* e = lfx::option("LF_JIT_RM_MINB")) minb = std::max(1, std::atoi(e));
  emit_prelude(C, src, out.rm_threads, minb, "lf_jit_step_rm");
  src << "  // register march: " << NW << " consumer warps x " << tw << "-column strips, " << V
      << " cells per lane (lane span starts at column " << cs << " of the strip)\n";
  for (size_t v = 0; v < nv; ++v)
    if (staged[v] >= 0)
      src << "  T* __restrict__ v" << v << " = reinterpret_cast<T*>(lf_smem + " << soff[v] << ");  // '"
          << C.P.vars[v].name << "': " << win[v] << " rows x " << nbox[v] * bw[v] << "\n";
  src << "  unsigned long long* lf_full = reinterpret_cast<unsigned long long*>(lf_smem + " << smem << ");\n";
  src << "  unsigned long long* lf_empty = lf_full + " << NS << ";\n";
  src << "  if (threadIdx.x == 0) {\n";
  src << "    for (int i = 0; i < " << NS << "; ++i) { lf_mbar_init(&lf_full[i], 1); lf_mbar_init(&lf_empty[i], " << NW
      << "); }\n";
  src << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n";
  {
    int k = 0;
    for (size_t v = 0; v < nv; ++v)
      if (staged[v] >= 0)
        src << "    asm volatile(\"prefetch.tensormap [%0];\" :: \"l\"(&lf_maps.m[" << k++ << "]) : \"memory\");\n";
  }
  src << "  }\n  __syncthreads();\n";
  src << "  const bool producer = threadIdx.x < 32;\n";
  src << "  if (producer && threadIdx.x != 0) return;\n";
  src << "  const int warp = (int)(threadIdx.x >> 5) - 1, lane = threadIdx.x & 31;\n";
  src << "  const int wl = warp * " << tw << " + lane * " << V << ";  // lane's first cell - lane-span start, CTA tile relative\n";
  src << "  unsigned lf_g = 0;\n";
  for (size_t v = 0; v < nv; ++v)
    if (staged[v] >= 0) src << "  int b" << v << " = 0;\n";
  for (size_t v = 0; v < nv; ++v)
    if (C.smem_var[v]) src << "  T R" << v << "[" << win[v] << "][" << V << "];  // '" << C.P.vars[v].name << "'\n";
  src << "  const int rows = a.row_hi - a.row_lo;\n";
  src << "  const long long units = (long long)((rows + a.chunk - 1) / a.chunk) * " << inner << ";\n";
  src << "  for (long long u = blockIdx.x; u < units; u += gridDim.x) {\n";
  src << "  const int ci = (int)(u / " << inner << "), bt = (int)(u % " << inner << ");\n";
  src << "  const int r0 = a.row_lo + ci * a.chunk, r1 = min(r0 + a.chunk, a.row_hi);\n";
  src << "  const int o1 = bt * " << T1 << ";\n";
  src << "  const int ow = o1 + warp * " << tw << ";  // this warp's strip\n";
  src << "  const bool wact = ow < " << C.N[1] << ";\n";
  // in place: which of this lane's cells fall in a column band, and where in
  // the band they go -- fixed for the unit, so the march only tests a mask
  for (size_t q = 0; q < ips.size(); ++q) {
    const int v = static_cast<int>(ips[q].v);
    const auto& t = C.P.terminals[ips[q].gi];
    const long so0 = -t.base[0] + C.LO[0];
    const Zone z = zone_of(C, ips[q].v, ips[q].gi, eb);
    src << "  unsigned zm" << q << " = 0;\n";
    src << "  long long zb" << q << "[" << V << "];\n";
    src << "  if (a.inplace && (warp == 0 || warp == " << NW - 1 << ")) {\n";
    src << "    #pragma unroll\n";
    src << "    for (int i = 0; i < " << V << "; ++i) {\n";
    src << "      const int c = " << cs << " + lane * " << V << " + i, xi = ow + c;\n";
    src << "      int e = -1;\n";
    src << "      if (c >= 0 && c < " << tw << " && xi < " << C.N[1] << ") {\n";
    src << "        if (o1 > 0 && xi < " << z.ze("o1") << ") e = o1;\n";
    src << "        else if (o1 + " << T1 << " < " << C.N[1] << " && xi >= " << z.zs("o1 + " + std::to_string(T1)) << ") e = o1 + " << T1 << ";\n";
    src << "      }\n";
    src << "      zb" << q << "[i] = e < 0 ? 0 : ((long long)(e / " << T1 << " - 1) * " << z.bw << " + (xi - " << z.zs("e")
        << ")) * " << t.extent[0] << "LL" << plus(so0) << ";\n";
    src << "      if (e >= 0) zm" << q << " |= 1u << i;\n";
    src << "    }\n  }\n";
  }

}

void RMarch::maps() {
  for (size_t v = 0; v < nv; ++v) {
    if (staged[v] < 0) continue;
    const auto& t = C.P.terminals[staged[v]];
    JitProgram::Tma tm;
    tm.term = staged[v];
    tm.rank = 2;
    tm.extent[0] = t.extent[1];
    tm.extent[1] = t.extent[0];
    tm.box[0] = static_cast<unsigned>(bw[v]);
    tm.box[1] = 1;
    out.rm_maps.push_back(tm);
  }

  // register windows rotate by renaming: the trip loop is unrolled U = lcm(W_v)
  // times and copy u keeps the row of logical slot k in R_v[(k + u) % W_v] (no
  // moves); windows whose lcm exceeds 6 shift by moves at the end of each trip
  U = 1;
  for (size_t v = 0; v < nv; ++v)
    if (C.smem_var[v] && win[v] > 1) U = std::lcm(U, win[v]);
  if (U > 6 || (lfx::option("LF_JIT_RM_UNROLL") && std::atoi(lfx::option("LF_JIT_RM_UNROLL")) == 0)) U = 1;
  trip_end = "r1 - 1 + (" + std::to_string(TE) + ")";
}

bool RMarch::trips() {
  if (U == 1) {
    src << "  for (int t = r0 + (" << TS << "); t <= " << trip_end << "; ++t) {\n";
  } else {
    src << "  for (int t0 = r0 + (" << TS << "); t0 <= " << trip_end << "; t0 += " << U << ") {\n";
  }
  for (cu = 0; cu < U; ++cu) {
  if (U > 1) src << "  { const int t = t0 + " << cu << ";  // copy " << cu << "\n  if (t > " << trip_end << ") break;\n";
  src << "    const unsigned stg = lf_g % " << NS << ", par = (lf_g / " << NS << ") & 1;\n";
    producer();
    for (size_t gi = 0; gi < G.size(); ++gi)
      if (!group(gi)) return false;
    copy_tail();
  }
  src << "  }\n";  // trips
  src << "  }\n";  // units
  src << "}\n";
  return true;
}

void RMarch::producer() {
  src << "    if (producer) {\n";
  src << "      if (lf_g >= " << NS << ") lf_mbar_wait(&lf_empty[stg], par ^ 1);\n";
  src << "      unsigned bytes = 0;\n";
  {
    int k = 0;
    for (size_t v = 0; v < nv; ++v) {
      if (staged[v] < 0) continue;
      src << "      const int y" << k << " = t" << plus(lead[v]) << ";\n";
      src << "      const bool in" << k << " = y" << k << " >= r0" << plus(C.vmin[v][0]) << " && y" << k << " <= r1 - 1"
          << plus(C.vmax[v][0]) << ";\n";
      src << "      if (in" << k << ") bytes += " << static_cast<size_t>(nbox[v]) * bw[v] * eb << "u;\n";
      ++k;
    }
  }
  src << "      asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n";
  src << "      lf_mbar_expect(&lf_full[stg], bytes);\n";
  {
    int k = 0;
    for (size_t v = 0; v < nv; ++v) {
      if (staged[v] < 0) continue;
      const int ti = staged[v];
      const auto& t = C.P.terminals[ti];
      const auto ex = C.extra_of(static_cast<int>(v));
      auto so = [&](int d) { return static_cast<long>(ex[d]) - t.base[d] + C.LO[d]; };
      src << "      if (in" << k << ") {\n";
      src << "        T* dst = v" << v << " + " << rowbase(v, lead[v]) << ";\n";
      for (int b = 0; b < nbox[v]; ++b)
        src << "        lf_tma2(dst + " << b * bw[v] << ", &lf_maps.m[" << k << "], &lf_full[stg], o1"
            << plus(vmin1[v] + so(1) + b * bw[v]) << ", y" << k << plus(so(0)) << ");\n";
      src << "      }\n";
      ++k;
    }
  }
  src << "    } else {\n";
  src << "    lf_mbar_wait(&lf_full[stg], par);\n";
  src << "    if (wact) {\n";

}

// one callsite group of the consumer warps
bool RMarch::group(size_t gi) {
  const Grp& g = G[gi];
  const auto& k = C.P.rs.kernels[g.kernel];
  src << "    { // group " << gi << ": kernel '" << k.name << "', lead " << g.shift << ", exact on lane-span cells ["
      << A[gi] << ", " << 32 * V - B[gi] << ")\n";
  src << "      const int y = t" << plus(g.shift) << ";\n";
  src << "      if (y >= r0" << plus(g.gmin[0]) << " && y <= r1 - 1" << plus(g.gmax[0]) << ") {\n";
  // vectors of the streamed rows this group reads
  std::map<std::pair<int, int>, std::string> vec;  // (var, row offset) -> register array
  auto vector_of = [&](int var, int r) {
    auto key = std::make_pair(var, r);
    auto it = vec.find(key);
    if (it != vec.end()) return it->second;
    const std::string nm = "S" + std::to_string(var) + "_" + num(r);
    src << "        T " << nm << "[" << V << "];\n";
    src << "        { const T* p = v" << var << " + " << rowbase(static_cast<size_t>(var), g.shift + r) << " + wl"
        << plus(base_al[var]) << ";\n";
    for (int c = 0; c < V / CH; ++c) {
      src << "          const " << VT << " c" << c << " = *reinterpret_cast<const " << VT << "*>(p + " << c * CH << ");";
      for (int e = 0; e < CH; ++e) src << " " << nm << "[" << c * CH + e << "] = c" << c << "." << comp[e] << ";";
      src << "\n";
    }
    src << "        }\n";
    vec[key] = nm;
    return nm;
  };
  // value of variable `var` at (row r, column i + dr) of this lane: own
  // registers, or a shuffle from the lane that holds it
  std::map<std::tuple<int, int, int>, std::string> elems;
  auto elem = [&](int var, int r, int dr, int i) -> std::string {
    long e;
    std::string arr;
    if (staged[var] >= 0) {
      arr = vector_of(var, r);
      e = rho[var] + i + dr;
    } else if (C.smem_var[var]) {
      const int slot = std::max(0, g.shift + r - old[var] - drop[var]);
      arr = "R" + std::to_string(var) + "[" + std::to_string(phys(var, slot)) + "]";
      e = i + dr;
    } else {
      const int ti = C.terminal_of(var, false);
      if (C.P.terminals[ti].dims.empty()) return "s" + std::to_string(ti);
      std::vector<std::string> pos = {"y" + plus(r), "(ow + " + std::to_string(cs) + " + lane * " + std::to_string(V) +
                                                         plus(i + dr) + ")"};
      return "__ldg(t" + std::to_string(ti) + " + " + C.tidx(ti, pos, C.extra_of(var)) + ")";
    }
    const long q = floordiv(e, V), m = e - q * V;
    const std::string own = arr + "[" + std::to_string(m) + "]";
    if (q == 0) return own;
    auto key = std::make_tuple(var, r, static_cast<int>(e));
    auto it = elems.find(key);
    if (it != elems.end()) return it->second;
    const std::string nm = "X" + std::to_string(var) + "_" + num(r) + "_" + num(e);
    src << "        const T " << nm << " = "
        << (q > 0 ? "__shfl_down_sync(0xffffffffu, " + own + ", " + std::to_string(q) + ")"
                  : "__shfl_up_sync(0xffffffffu, " + own + ", " + std::to_string(-q) + ")")
        << ";\n";
    elems[key] = nm;
    return nm;
  };
  // every operand first (vector loads and shuffles are warp-wide), then the cells
  std::vector<std::vector<std::string>> opnd(V, std::vector<std::string>(g.loads.size()));
  for (int i = 0; i < V; ++i)
    for (size_t li = 0; li < g.loads.size(); ++li)
      opnd[i][li] = elem(g.loads[li].var, g.loads[li].rel[0], g.loads[li].rel[1], i);
  auto load_index = [&](int var, const std::vector<int>& rel) {
    for (size_t li = 0; li < g.loads.size(); ++li)
      if (g.loads[li].var == var && g.loads[li].rel == rel) return static_cast<int>(li);
    return -1;
  };
  std::vector<std::pair<int, const GOut*>> goals;  // (terminal, output)
  for (const auto& o : g.out) {
    const int ti = C.terminal_of(o.var, true);
    if (ti >= 0) {
      goals.emplace_back(ti, &o);
      src << "        T G" << gi << "_" << o.param << "[" << V << "];\n";
    }
  }
  // fp32, opt-in (LF_JIT_RM_PACK=1): cells in pairs on the packed fp32x2
  // pipe when every output (and every inlined producer) has a body.  Exact,
  // but measured slower on the box chain (430 vs 484 G: forming the register
  // pairs costs moves), so scalar cells by default
  bool packed = C.T == "float" && V % 2 == 0 && lfx::option("LF_JIT_RM_PACK") && std::atoi(lfx::option("LF_JIT_RM_PACK")) != 0;
  for (const auto& [op, pat] : k.outputs) packed &= k.bodies.count(op) > 0;
  std::set<std::string> kin;
  for (const auto& [ip, pat] : k.inputs) kin.insert(ip);
  std::vector<std::pair<std::string, std::unique_ptr<lf::Expr>>> bodies;
  for (const auto& [op, pat] : k.outputs) {
    if (!packed) break;
    std::string e2;
    auto e = lf::parse_expr(k.bodies.at(op), e2);
    std::set<std::string> used;
    if (e) lf::expr_vars(*e, used);
    for (const auto& u : used) packed &= kin.count(u) > 0;
    if (!e) packed = false;
    else bodies.emplace_back(op, std::move(e));
  }
  for (const auto& in : g.in)
    if (in.via >= 0)
      for (const auto& o : C.inlined[in.via].out)
        if (o.var == in.var) packed &= C.P.rs.kernels[C.inlined[in.via].kernel].bodies.count(o.param) > 0;
  for (int j = 0; packed && j < V; j += 2) {
    src << "        { // cells " << j << ", " << j + 1 << " (fp32x2)\n";
    auto pair = [&](int li) { return "make_float2(" + opnd[j][li] + ", " + opnd[j + 1][li] + ")"; };
    for (const auto& in : g.in) {
      if (in.via < 0) {
        src << "          const float2 p_" << in.param << " = " << pair(load_index(in.var, in.rel)) << ";\n";
        continue;
      }
      const Grp& pg = C.inlined[in.via];
      const auto& pk = C.P.rs.kernels[pg.kernel];
      std::string oparam;
      std::vector<int> orel(2, 0);
      for (const auto& o : pg.out)
        if (o.var == in.var) {
          oparam = o.param;
          orel = o.rel;
        }
      std::map<std::string, std::string> pv;
      for (const auto& pin : pg.in) {
        std::vector<int> r(2);
        for (int d = 0; d < 2; ++d) r[d] = in.rel[d] - orel[d] + pin.rel[d];
        pv[pin.param] = pair(load_index(pin.var, r));
      }
      std::string e2;
      auto e = lf::parse_expr(pk.bodies.at(oparam), e2);
      if (!e) return (C.error = "kernel '" + pk.name + "': " + e2, false);
      src << "          const float2 p_" << in.param << " = "
          << lf::emit_c2(*e, [&](const std::string& n) { return pv.at(n); }) << ";  // inlined '" << pk.name << "'\n";
    }
    for (const auto& [op, e] : bodies)
      src << "          const float2 q_" << op << " = " << lf::emit_c2(*e, [](const std::string& n) { return "p_" + n; })
          << ";\n";
    for (const auto& o : g.out) {
      for (int h = 0; h < 2; ++h) {
        const char* lane_c = h ? ".y" : ".x";
        if (C.smem_var[o.var])
          src << "          R" << o.var << "[" << phys(o.var, std::max(0, g.shift + o.rel[0] - old[o.var] - drop[o.var])) << "]["
              << j + h << "] = q_" << o.param << lane_c << ";\n";
        if (C.terminal_of(o.var, true) >= 0)
          src << "          G" << gi << "_" << o.param << "[" << j + h << "] = q_" << o.param << lane_c << ";\n";
      }
    }
    src << "        }\n";
  }
  for (int i = 0; i < V && !packed; ++i) {
    src << "        { // cell " << i << "\n";
    for (const auto& in : g.in) {
      if (in.via < 0) {
        src << "          const T p_" << in.param << " = " << opnd[i][load_index(in.var, in.rel)] << ";\n";
        continue;
      }
      const Grp& pg = C.inlined[in.via];
      const auto& pk = C.P.rs.kernels[pg.kernel];
      std::string oparam;
      std::vector<int> orel(2, 0);
      for (const auto& o : pg.out)
        if (o.var == in.var) {
          oparam = o.param;
          orel = o.rel;
        }
      std::map<std::string, std::string> pv;
      for (const auto& pin : pg.in) {
        std::vector<int> r(2);
        for (int d = 0; d < 2; ++d) r[d] = in.rel[d] - orel[d] + pin.rel[d];
        pv[pin.param] = opnd[i][load_index(pin.var, r)];
      }
      std::string e2;
      auto e = lf::parse_expr(pk.bodies.at(oparam), e2);
      if (!e) return (C.error = "kernel '" + pk.name + "': " + e2, false);
      src << "          const T p_" << in.param << " = "
          << lf::emit_c(*e, C.T, [&](const std::string& n) { return pv.at(n); }) << ";  // inlined '" << pk.name
          << "'\n";
    }
    if (!emit_bodies(C, g, src, "          ")) return false;
    for (const auto& o : g.out) {
      if (C.smem_var[o.var])
        src << "          R" << o.var << "[" << phys(o.var, std::max(0, g.shift + o.rel[0] - old[o.var] - drop[o.var])) << "][" << i
            << "] = q_" << o.param << ";\n";
      if (C.terminal_of(o.var, true) >= 0) src << "          G" << gi << "_" << o.param << "[" << i << "] = q_" << o.param << ";\n";
    }
    src << "        }\n";
  }
  store_goals(gi, goals);
  src << "      }\n    }\n";
  return true;
}

// goal rows of group gi: own chunk rows, own strip cells, inside the domain;
// in place, the deferred boundary cells to their bands
void RMarch::store_goals(size_t gi, const std::vector<std::pair<int, const GOut*>>& goals) {
  for (const auto& [ti, o] : goals) {
    const auto& t = C.P.terminals[ti];
    const long so = goal_so(ti);
    const bool vec_ok = ((cs + so) % CH + CH) % CH == 0 && t.extent[1] % CH == 0;
    src << "        { const int yy = y" << plus(o->rel[0]) << ";\n";
    src << "          const int c = " << cs << " + lane * " << V << ", x = ow + c;\n";
    src << "          if (yy >= r0 && yy < r1) {\n";
    src << "            T* gp = t" << ti << " + " << C.tidx(ti, {"yy", "x"}, std::vector<int>(2, 0)) << ";\n";
    const std::string gv = "G" + std::to_string(gi) + "_" + o->param;
    const IP* ip = ip_of_goal(ti);
    if (ip) {
      // in place: deferred boundary writes (row zone: the whole row into the
      // row band; column zone: those cells into the column band)
      const int v = static_cast<int>(ip->v);
      const int lo0 = C.vmin[v][0], hi0 = C.vmax[v][0], lo1 = C.vmin[v][1], hi1 = C.vmax[v][1];
      const size_t q = static_cast<size_t>(ip - ips.data());
      src << "            if (a.inplace) {\n";
      src << "              int br = -1;  // row of the row band (band k - 1 at chunk boundary k)\n";
      src << "              if (r0 > 0 && yy < r0" << plus(hi0) << ") br = (ci - 1) * " << hi0 - lo0 << " + (yy - r0" << plus(-lo0) << ");\n";
      src << "              else if (r1 < N0 && yy >= r1" << plus(lo0) << ") br = ci * " << hi0 - lo0 << " + (yy - r1" << plus(-lo0)
          << ");\n";
      src << "              if (br >= 0) gp = reinterpret_cast<T*>(a.t[" << ip->slot << "]) + (long long)br * " << t.extent[1]
          << "LL + (x" << plus(so) << ");\n";
      src << "              if (br < 0 && zm" << q << ") {  // cells in a column band\n";
      src << "                T* cb = reinterpret_cast<T*>(a.t[" << ip->slot + 1 << "]) + yy;\n";
      src << "                #pragma unroll\n";
      src << "                for (int i = 0; i < " << V << "; ++i) {\n";
      src << "                  if ((zm" << q << " >> i) & 1) cb[zb" << q << "[i]] = " << gv << "[i];\n";
      src << "                  else if (c + i >= 0 && c + i < " << tw << " && x + i < " << C.N[1] << ") gp[i] = " << gv << "[i];\n";
      src << "                }\n";
      src << "                gp = nullptr;\n";
      src << "              }\n";
      src << "            }\n";
      src << "            if (gp)\n";
    }
    if (vec_ok) {
      src << "            if (c >= 0 && c + " << V << " <= " << tw << " && x + " << V << " <= " << C.N[1] << ") {\n";
      for (int c = 0; c < V / CH; ++c) {
        src << "              " << VT << " w" << c << ";";
        for (int e = 0; e < CH; ++e) src << " w" << c << "." << comp[e] << " = " << gv << "[" << c * CH + e << "];";
        src << " *reinterpret_cast<" << VT << "*>(gp + " << c * CH << ") = w" << c << ";\n";
      }
      src << "            } else {\n";
    } else {
      src << "            {\n";
    }
    src << "              #pragma unroll\n";
    src << "              for (int i = 0; i < " << V << "; ++i)\n";
    src << "                if (c + i >= 0 && c + i < " << tw << " && x + i < " << C.N[1] << ") gp[i] = " << gv << "[i];\n";
    src << "            }\n          }\n        }\n";
  }

}

void RMarch::copy_tail() {
  src << "    }\n";  // wact
  src << "    __syncwarp();\n";
  src << "    if (lane == 0) lf_mbar_arrive(&lf_empty[stg]);\n";
  // rotate the register windows: row t + off of trip t is row (t+1) + (off-1)
  for (size_t v = 0; v < nv && U == 1; ++v)
    if (C.smem_var[v] && win[v] > 1)
      src << "    #pragma unroll\n    for (int k = 0; k < " << win[v] - 1 << "; ++k)\n      #pragma unroll\n"
          << "      for (int i = 0; i < " << V << "; ++i) R" << v << "[k][i] = R" << v << "[k + 1][i];\n";
  src << "    }\n";  // consumer
  for (size_t v = 0; v < nv; ++v)
    if (staged[v] >= 0 && win[v] > 1) src << "    b" << v << " = b" << v << " == " << (win[v] - 1) << " ? 0 : b" << v << " + 1;\n";
  src << "    ++lf_g;\n";
  if (U > 1) src << "  }\n";  // copy
}

void RMarch::commit() {
  if (!ips.empty()) {
    std::vector<std::pair<size_t, int>> caps;
    std::vector<int> slots;
    for (const auto& ip : ips) {
      caps.push_back({ip.v, ip.gi});
      slots.push_back(ip.slot);
    }
    emit_commit2(C, "lf_jit_commit_rm", caps, slots, static_cast<int>(T1), src, false);
    // commit + ghost refill in one launch where the refill reads nothing (every
    // iterated goal with zero boundaries, or none)
    bool fill_reads = false;
    for (const auto& it_pair : C.P.rs.iterate) {
      auto it = C.P.rs.boundary.find(it_pair.first);
      if (it == C.P.rs.boundary.end()) it = C.P.rs.boundary.find("*");
      if (it != C.P.rs.boundary.end())
        for (auto m : it->second) fill_reads |= m != lf::Boundary::zero && m != lf::Boundary::none;
    }
    if (out.has_fill && !fill_reads)
      emit_commit2(C, "lf_jit_commit_fill_rm", caps, slots, static_cast<int>(T1), src, true);
  }
}

bool emit_rmarch(Ctx& C, JitProgram& out, std::ostream& src) {
  RMarch m(C, out, src);
  return m.emit();
}

}  // namespace lfx::cg

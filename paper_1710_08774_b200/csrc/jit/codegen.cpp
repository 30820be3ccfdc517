// Generic fused executor, part 1: lowering a planned single-nest chain whose
// kernels carry `body:` expressions (R/SPEC.md:82) to sm_100a CUDA source --
// the role of the reference's missing codegen (R/SPEC.md:449-514), retargeted:
// instead of one serial loop nest with rolling buffers, one CTA per output
// tile evaluates every callsite group in dataflow order over the tile plus the
// halo the planner derived for it, keeping each intermediate in shared memory
// (contraction to a tile-sized window); only terminals touch HBM.
#include <algorithm>
#include <climits>
#include <deque>
#include <map>
#include <sstream>

#include "../planner/dsl.hpp"
#include "jit.hpp"

namespace lfx {

namespace {

std::string elem_type(const std::string& t) {
  if (t.find("double") != std::string::npos) return "double";
  if (t.find("float") != std::string::npos) return "float";
  return "";
}

}  // namespace

bool jit_generate(const lf::Plan& P, JitProgram& out) {
  const auto& rs = P.rs;
  const auto& g = P.dag;
  const int nd = static_cast<int>(rs.loop_order.size());
  auto fail = [&](const std::string& m) {
    out.error = m;
    return false;
  };
  if (nd < 1 || nd > 3) return fail("generic executor handles 1-3 loop dimensions");
  if (!P.one_nest) return fail("chain does not fuse into a single nest (" + std::to_string(P.nests) + " nests, " +
                               std::to_string(P.splits) + " splits)");
  for (const auto& r : rs.ranges)
    if (r.stride != 1) return fail("generic executor needs unit strides");
  // ---- element type: one type for the whole chain
  std::string T;
  for (const auto& t : P.terminals) {
    std::string e = elem_type(t.type);
    if (e.empty()) return fail("unsupported terminal type '" + t.type + "'");
    if (!T.empty() && e != T) return fail("mixed element types in one chain");
    T = e;
  }
  for (const auto& v : P.vars) {
    if (!v.external.empty() || v.alias_of >= 0) continue;
    std::string e = elem_type(v.type);
    if (e.empty() || e != T) return fail("intermediate '" + v.name + "' has type '" + v.type + "'");
    if ((int)v.dims.size() != nd) return fail("intermediate '" + v.name + "' does not span every loop dimension");
  }
  out.type = T;
  out.elem_bytes = T == "double" ? 8 : 4;
  out.nd = nd;
  std::vector<long> N(nd);
  for (int d = 0; d < nd; ++d) N[d] = rs.ranges[d].trips();

  // ---- per-variable term offset ranges (relative to the canonical cell)
  const size_t nv = P.vars.size();
  std::vector<std::vector<int>> vmin(nv, std::vector<int>(nd, INT_MAX)), vmax(nv, std::vector<int>(nd, INT_MIN));
  for (size_t t = 0; t < g.terms.size(); ++t) {
    int v = P.var_of_term[t];
    for (const auto& o : g.terms[t].dims) {
      vmin[v][o.dim] = std::min(vmin[v][o.dim], o.offset);
      vmax[v][o.dim] = std::max(vmax[v][o.dim], o.offset);
    }
  }
  auto canon = [&](int v) {
    while (P.vars[v].alias_of >= 0) v = P.vars[v].alias_of;
    return v;
  };
  // terminal index of a variable (axiom or goal buffer)
  auto terminal_of = [&](int v, bool goal) {
    for (size_t i = 0; i < P.terminals.size(); ++i)
      if (P.terminals[i].var == v && P.terminals[i].is_goal == goal) return static_cast<int>(i);
    return -1;
  };
  // axiom variables: storage displacement extra[d] = ext shift - term offset
  std::map<int, std::vector<int>> axiom_extra;
  for (const auto& r : g.raps) {
    if (r.kind != lf::RapKind::load) continue;
    const auto& term = g.terms[r.out_terms[0]];
    const int v = P.var_of_term[r.out_terms[0]];
    if (axiom_extra.count(v)) continue;
    std::vector<int> ex(nd, 0);
    for (const auto& s : r.ext_slots) {
      if (s.dim < 0) return fail("axioms with constant subscripts are not supported by the generic executor");
      int off = 0;
      for (const auto& o : term.dims)
        if (o.dim == s.dim) off = o.offset;
      ex[s.dim] = s.shift - off;
    }
    axiom_extra[v] = ex;
  }
  // which variables live in shared memory: kernel outputs that some kernel reads
  std::vector<char> read_by_kernel(nv, 0), smem_var(nv, 0);
  for (const auto& r : g.raps)
    if (r.kind == lf::RapKind::kernel)
      for (int t : r.in_terms) read_by_kernel[canon(P.var_of_term[t])] = 1;
  for (size_t v = 0; v < nv; ++v)
    if (read_by_kernel[v] && !P.vars[v].axiom_backed && P.vars[v].alias_of < 0 && !P.vars[v].dims.empty())
      smem_var[v] = 1;

  // ---- kernel groups in dataflow order
  struct GIn {
    std::string param;
    int var;
    std::vector<int> rel;
  };
  struct GOut {
    std::string param;
    int var;
    std::vector<int> rel;
  };
  struct Grp {
    int kernel;
    std::vector<int> gmin, gmax;
    std::vector<GIn> in;
    std::vector<GOut> out;
  };
  std::vector<Grp> groups;
  {
    const int ng = static_cast<int>(P.groups.size());
    std::vector<std::set<int>> adj(ng);
    std::vector<int> indeg(ng, 0);
    for (const auto& e : g.edges) {
      int a = P.group_of[e.from], b = P.group_of[e.to];
      if (a != b && adj[a].insert(b).second) ++indeg[b];
    }
    std::deque<int> q;
    for (int i = 0; i < ng; ++i)
      if (!indeg[i]) q.push_back(i);
    std::vector<int> order;
    while (!q.empty()) {
      int v = q.front();
      q.pop_front();
      order.push_back(v);
      for (int w : adj[v])
        if (--indeg[w] == 0) q.push_back(w);
    }
    for (int gi : order) {
      const auto& cg = P.groups[gi];
      if (cg.kind != lf::RapKind::kernel) continue;
      const auto& k = rs.kernels[cg.kernel];
      if (k.associative) return fail("associative kernels need the reduction path (not in the generic executor)");
      for (const auto& [op, pat] : k.outputs)
        if (!k.bodies.count(op))
          return fail("kernel '" + k.name + "' has no body for output '" + op +
                      "' (the generic executor compiles `body:` expressions)");
      const lf::Rap& rep = g.raps[cg.members[0]];
      std::vector<int> anchor(nd, 0);
      for (const auto& o : g.terms[rep.out_terms[0]].dims) anchor[o.dim] = o.offset;
      Grp G;
      G.kernel = cg.kernel;
      G.gmin = cg.min_disp(nd);
      G.gmax = cg.max_disp(nd);
      for (size_t i = 0; i < k.inputs.size(); ++i) {
        GIn in{k.inputs[i].first, canon(P.var_of_term[rep.in_terms[i]]), std::vector<int>(nd, 0)};
        const auto& term = g.terms[rep.in_terms[i]];
        if (!term.dims.empty() && (int)term.dims.size() != nd)
          return fail("kernel '" + k.name + "' reads a partial-rank term");
        for (const auto& o : term.dims) in.rel[o.dim] = o.offset - anchor[o.dim];
        G.in.push_back(in);
      }
      for (size_t i = 0; i < k.outputs.size(); ++i) {
        GOut o{k.outputs[i].first, canon(P.var_of_term[rep.out_terms[i]]), std::vector<int>(nd, 0)};
        for (const auto& od : g.terms[rep.out_terms[i]].dims) o.rel[od.dim] = od.offset - anchor[od.dim];
        G.out.push_back(o);
      }
      groups.push_back(std::move(G));
    }
  }

  // ---- tile shape and shared-memory layout (shrink the tile until it fits)
  std::vector<int> tile(nd);
  if (nd == 1) tile = {256};
  if (nd == 2) tile = {8, 32};
  if (nd == 3) tile = {4, 4, 32};
  std::vector<size_t> soff(nv, 0);
  size_t smem = 0;
  auto layout = [&] {
    smem = 0;
    for (size_t v = 0; v < nv; ++v) {
      if (!smem_var[v]) continue;
      size_t n = 1;
      for (int d = 0; d < nd; ++d) n *= tile[d] + (vmax[v][d] - vmin[v][d]);
      soff[v] = smem;
      smem += (n * out.elem_bytes + 15) / 16 * 16;
    }
  };
  layout();
  while (smem > 96 * 1024) {
    int d = 0;  // halve the largest outer tile dimension, keep the innermost >= 32
    for (int k = 0; k < nd; ++k)
      if ((k < nd - 1 ? tile[k] : tile[k] / 4) > (d < nd - 1 ? tile[d] : tile[d] / 4)) d = k;
    if (tile[d] <= 1 || (d == nd - 1 && tile[d] <= 32)) break;
    tile[d] /= 2;
    layout();
  }
  if (smem > 200 * 1024) return fail("chain needs too much on-chip storage for one tile");
  out.tile = tile;
  out.smem_bytes = smem;
  out.threads = 256;

  // ---- terminal addressing
  const auto& terms = P.terminals;
  std::ostringstream src;
  auto pitch = [&](const lf::Terminal& t, int slot) {
    long p = 1;
    for (size_t k = slot + 1; k < t.extent.size(); ++k) p *= t.extent[k];
    return p;
  };
  // index expression of terminal `ti` at logical cell x[d] + rel[d] (+ axiom extra)
  auto tindex = [&](int ti, const std::vector<int>& rel, const std::vector<int>& extra) {
    const auto& t = terms[ti];
    std::string e;
    for (size_t s = 0; s < t.dims.size(); ++s) {
      const int d = t.dims[s];
      long off = rel[d] + extra[d] - t.base[s];
      std::string c = "(x" + std::to_string(d) + (off ? (off > 0 ? " + " : " - ") + std::to_string(std::labs(off)) : "") + ")";
      long p = pitch(t, static_cast<int>(s));
      e += (e.empty() ? "" : " + ") + c + (p != 1 ? " * " + std::to_string(p) + "LL" : "");
    }
    return e.empty() ? std::string("0") : e;
  };
  auto sidx = [&](int v, const std::string& rel_expr_prefix, const std::vector<int>& rel) {
    // shared-memory index of variable v at tile-relative cell c + rel
    std::string e;
    for (int d = 0; d < nd; ++d) {
      long width = tile[d] + (vmax[v][d] - vmin[v][d]);
      long off = rel[d] - vmin[v][d];
      std::string c = "(c" + std::to_string(d) + (off ? (off > 0 ? " + " : " - ") + std::to_string(std::labs(off)) : "") + ")";
      if (d == 0)
        e = c;
      else
        e = "(" + e + ") * " + std::to_string(width) + " + " + c;
    }
    (void)rel_expr_prefix;
    return e;
  };

  src << "// generated by loomfuse-b200 (csrc/jit/codegen.cpp) for chain '" << rs.name << "'\n";
  src << "typedef " << T << " T;\n";
  src << "__device__ __forceinline__ T lf_min(T a, T b) { return a < b ? a : b; }\n";
  src << "__device__ __forceinline__ T lf_max(T a, T b) { return a > b ? a : b; }\n";
  // must match lfx::Args in jit.cpp (passed by value)
  src << "struct LfArgs { void* t[32]; long long n0; int row_lo, row_hi, top, bottom; };\n";
  src << "extern \"C\" __global__ void __launch_bounds__(" << out.threads << ") lf_jit_step(const LfArgs a) {\n";
  src << "  extern __shared__ __align__(16) unsigned char lf_smem[];\n";
  // tile origin: innermost dim on blockIdx.x, next on y, outermost on z (or y for 2D)
  const char* bid[3] = {"blockIdx.x", "blockIdx.y", "blockIdx.z"};
  for (int d = 0; d < nd; ++d) {
    const int axis = nd - 1 - d;
    src << "  const long long o" << d << " = " << (d == 0 ? "(long long)a.row_lo + " : "") << "(long long)" << bid[axis]
        << " * " << tile[d] << ";\n";
  }
  src << "  const long long N0 = a.n0;\n";
  for (int d = 1; d < nd; ++d) src << "  const long long N" << d << " = " << N[d] << ";\n";
  for (size_t i = 0; i < terms.size(); ++i) {
    if (terms[i].dims.empty())
      src << "  const T s" << i << " = *reinterpret_cast<const T*>(a.t[" << i << "]);\n";
    else
      src << "  " << (terms[i].is_goal ? "T" : "const T") << "* __restrict__ t" << i << " = reinterpret_cast<"
          << (terms[i].is_goal ? "T" : "const T") << "*>(a.t[" << i << "]);\n";
  }
  for (size_t v = 0; v < nv; ++v)
    if (smem_var[v]) src << "  T* __restrict__ v" << v << " = reinterpret_cast<T*>(lf_smem + " << soff[v] << ");\n";
  auto var_read = [&](int v, const std::vector<int>& rel) -> std::string {
    if (smem_var[v]) return "v" + std::to_string(v) + "[" + sidx(v, "", rel) + "]";
    // terminal: axiom buffer (or a rank-0 scalar)
    int ti = terminal_of(v, false);
    if (ti < 0) return "";
    if (terms[ti].dims.empty()) return "s" + std::to_string(ti);
    return "t" + std::to_string(ti) + "[" + tindex(ti, rel, axiom_extra.count(v) ? axiom_extra[v] : std::vector<int>(nd, 0)) + "]";
  };
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    const Grp& G = groups[gi];
    const auto& k = rs.kernels[G.kernel];
    std::vector<int> ext(nd);
    long cells = 1;
    for (int d = 0; d < nd; ++d) {
      ext[d] = tile[d] + (G.gmax[d] - G.gmin[d]);
      cells *= ext[d];
    }
    src << "  // group " << gi << ": kernel '" << k.name << "' over the tile + [" ;
    for (int d = 0; d < nd; ++d) src << (d ? ", " : "") << G.gmin[d] << ".." << G.gmax[d];
    src << "]\n";
    src << "  for (int idx = threadIdx.x; idx < " << cells << "; idx += blockDim.x) {\n";
    src << "    int rem = idx;\n";
    for (int d = nd - 1; d >= 0; --d) {
      src << "    const int c" << d << " = rem % " << ext[d] << " + (" << G.gmin[d] << ");";
      src << " rem /= " << ext[d] << ";\n";
    }
    for (int d = 0; d < nd; ++d) src << "    const long long x" << d << " = o" << d << " + c" << d << ";\n";
    // the group is needed at cells [gmin, N-1+gmax] of the domain
    src << "    if (";
    for (int d = 0; d < nd; ++d)
      src << (d ? " || " : "") << "x" << d << " < " << G.gmin[d] << " || x" << d << " > N" << d << " - 1 + (" << G.gmax[d]
          << ")";
    src << ") continue;\n";
    std::map<std::string, std::string> pv;
    for (const auto& in : G.in) {
      std::string r = var_read(in.var, in.rel);
      if (r.empty()) return fail("kernel '" + k.name + "' reads '" + in.param + "' from an unsupported source");
      src << "    const T p_" << in.param << " = " << r << ";\n";
      pv[in.param] = "p_" + in.param;
    }
    for (const auto& o : G.out) {
      std::string err;
      auto e = lf::parse_expr(k.bodies.at(o.param), err);
      if (!e) return fail("kernel '" + k.name + "' body of '" + o.param + "': " + err);
      std::set<std::string> used;
      lf::expr_vars(*e, used);
      for (const auto& u : used)
        if (!pv.count(u)) return fail("kernel '" + k.name + "' body of '" + o.param + "' uses unknown name '" + u + "'");
      src << "    const T q_" << o.param << " = "
          << lf::emit_c(*e, T, [&](const std::string& n) { return pv.at(n); }) << ";\n";
    }
    for (const auto& o : G.out) {
      if (smem_var[o.var]) src << "    v" << o.var << "[" << sidx(o.var, "", o.rel) << "] = q_" << o.param << ";\n";
      const int ti = terminal_of(o.var, true);
      if (ti >= 0) {
        // goal: own-tile cells of the computed rows, inside the domain
        src << "    if (";
        for (int d = 0; d < nd; ++d) {
          src << (d ? " && " : "") << "c" << d << " + (" << o.rel[d] << ") >= 0 && c" << d << " + (" << o.rel[d] << ") < "
              << tile[d] << " && x" << d << " + (" << o.rel[d] << ") < N" << d;
          if (d == 0) src << " && x0 + (" << o.rel[0] << ") < a.row_hi";
        }
        src << ") t" << ti << "[" << tindex(ti, o.rel, std::vector<int>(nd, 0)) << "] = q_" << o.param << ";\n";
      }
    }
    src << "  }\n";
    if (gi + 1 < groups.size()) src << "  __syncthreads();\n";
  }
  src << "}\n";

  // ---- ghost refill of iterated goals (boundary modes, between steps)
  out.has_fill = false;
  std::ostringstream fill;
  fill << "extern \"C\" __global__ void lf_jit_fill(const LfArgs a) {\n";
  fill << "  const long long N0 = a.n0;\n";
  for (const auto& [gname, aname] : rs.iterate) {
    int ti = -1;
    for (size_t i = 0; i < terms.size(); ++i)
      if (terms[i].is_goal && terms[i].name == gname) ti = static_cast<int>(i);
    if (ti < 0 || terms[ti].dims.empty()) continue;
    const auto& t = terms[ti];
    if ((int)t.dims.size() != nd) return fail("iterated terminal '" + gname + "' must span every loop dimension");
    auto it = rs.boundary.find(t.name);
    if (it == rs.boundary.end()) it = rs.boundary.find("*");
    std::vector<lf::Boundary> modes(nd, lf::Boundary::none);
    if (it != rs.boundary.end())
      for (int d = 0; d < nd; ++d) modes[d] = it->second.size() == 1 ? it->second[0] : it->second[std::min<size_t>(d, it->second.size() - 1)];
    out.has_fill = true;
    fill << "  {\n    T* b = reinterpret_cast<T*>(a.t[" << ti << "]);\n";
    long cells_inner = 1;
    for (int s = 1; s < nd; ++s) cells_inner *= t.extent[s];
    const long h0 = -t.base[0];
    fill << "    const long long total = (N0 + " << (t.extent[0] - N[0]) << ") * " << cells_inner << "LL;\n";
    fill << "    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total; idx += (long long)gridDim.x * blockDim.x) {\n";
    fill << "      long long rem = idx;\n";
    for (int s = nd - 1; s >= 0; --s) {
      fill << "      const long long y" << s << " = rem % " << (s == 0 ? std::string("(N0 + ") + std::to_string(t.extent[0] - N[0]) + ")" : std::to_string(t.extent[s])) << " + (" << t.base[s] << ");";
      fill << " rem /= " << (s == 0 ? std::string("(N0 + ") + std::to_string(t.extent[0] - N[0]) + ")" : std::to_string(t.extent[s])) << ";\n";
    }
    (void)h0;
    fill << "      bool ghost = false, zero = false; T sign = static_cast<T>(1);\n";
    for (int d = 0; d < nd; ++d) {
      const std::string y = "y" + std::to_string(d), n = "N" + std::string(d == 0 ? "0" : std::to_string(N[d]));
      const std::string nn = d == 0 ? "N0" : std::to_string(N[d]);
      fill << "      long long z" << d << " = " << y << ";\n";
      fill << "      if (" << y << " < 0 || " << y << " >= " << nn << ") {\n";
      if (d == 0) fill << "        if ((" << y << " < 0 && !a.top) || (" << y << " >= " << nn << " && !a.bottom)) continue;\n";
      fill << "        ghost = true;\n";
      switch (modes[d]) {
        case lf::Boundary::zero: fill << "        zero = true;\n"; break;
        case lf::Boundary::periodic: fill << "        z" << d << " = ((" << y << " % " << nn << ") + " << nn << ") % " << nn << ";\n"; break;
        case lf::Boundary::clamp: fill << "        z" << d << " = " << y << " < 0 ? 0 : " << nn << " - 1;\n"; break;
        case lf::Boundary::even:
        case lf::Boundary::odd:
          fill << "        z" << d << " = " << y << " < 0 ? -1 - " << y << " : 2 * " << nn << " - 1 - " << y << ";\n";
          if (modes[d] == lf::Boundary::odd) fill << "        sign = -sign;\n";
          break;
        case lf::Boundary::none: fill << "        continue;\n"; break;
      }
      fill << "      }\n";
    }
    fill << "      if (!ghost) continue;\n";
    std::string dst, srci;
    for (int s = 0; s < nd; ++s) {
      long p = pitch(t, s);
      std::string ps = p != 1 ? " * " + std::to_string(p) + "LL" : "";
      dst += (s ? " + " : "") + std::string("(y") + std::to_string(s) + " - (" + std::to_string(t.base[s]) + "))" + ps;
      srci += (s ? " + " : "") + std::string("(z") + std::to_string(s) + " - (" + std::to_string(t.base[s]) + "))" + ps;
    }
    fill << "      b[" << dst << "] = zero ? static_cast<T>(0) : sign * b[" << srci << "];\n";
    fill << "    }\n  }\n";
  }
  fill << "}\n";
  src << fill.str();
  out.source = src.str();
  return true;
}

}  // namespace lfx

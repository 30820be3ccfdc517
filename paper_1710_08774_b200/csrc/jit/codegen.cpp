// Generic fused executor, part 1: lowering a planned single-nest chain whose
// kernels carry `body:` expressions (R/SPEC.md:82) to sm_100a CUDA source --
// the role of the reference's missing codegen (R/SPEC.md:449-514), retargeted
// to the GPU:
//
//  * 2D/3D chains (`emit_march`): the HFAV schedule itself.  A CTA owns a tile
//    of the inner loop dimensions and marches the outermost one; at trip t
//    callsite group g computes row t + s_g, s_g being the pipeline shift
//    (the recurrence of shifts.cpp:8-79: a producer runs at least as far ahead
//    as its furthest-reading consumer).  Every intermediate lives in a
//    shared-memory rolling window of W_v rows (the contraction of
//    storage.cpp:319-399: W_v = lead of the producer - oldest row any consumer
//    still reads + 1); axioms are streamed into their own windows by cp.async
//    one trip ahead.  Only terminals touch HBM.
//  * 1D chains (`emit_tiled`): one CTA per tile, each group evaluated over the
//    tile plus the halo the planner derived for it.
//
// Ghost refill of iterated goals (`config: boundary:`) is a second kernel that
// visits ghost cells only.
#include <algorithm>
#include <cstring>
#include <cctype>
#include <climits>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <map>
#include <set>
#include <sstream>

#include "../planner/dsl.hpp"
#include "codegen_ctx.hpp"
#include "jit.hpp"

namespace lfx {

namespace cg {

// Kernel evaluation: a `body:` expression per output (R/SPEC.md:82), or a
// call of the function the declaration names (R/PAPER.md:58-62: value
// inputs, outputs by pointer or reference), found in the shipped user-kernel
// headers or in the caller's kernel source.  in(param) is the C expression of
// an input; out(param) the variable an output lands in -- declared here when
// `declare`, assigned otherwise.
bool has_function(const std::string& sources, const std::string& fn) {
  if (fn.empty()) return false;
  size_t pos = 0;
  while ((pos = sources.find(fn, pos)) != std::string::npos) {
    const bool left_ok = pos == 0 || !(std::isalnum(static_cast<unsigned char>(sources[pos - 1])) || sources[pos - 1] == '_');
    size_t e = pos + fn.size();
    while (e < sources.size() && std::isspace(static_cast<unsigned char>(sources[e]))) ++e;
    if (left_ok && e < sources.size() && sources[e] == '(') return true;
    pos += fn.size();
  }
  return false;
}

bool kernel_evaluable(const lf::KernelRule& k, const std::string& sources, std::string& why) {
  bool bodies = true;
  for (const auto& [op, pat] : k.outputs) bodies &= k.bodies.count(op) > 0;
  if (bodies) return true;
  const lf::DeclInfo di = lf::parse_declaration(k.declaration);
  if (has_function(sources, di.function)) return true;
  why = "kernel '" + k.name + "' has no `body:` and its function '" + di.function +
        "' is neither a shipped user kernel nor in the kernel source given to the plan";
  return false;
}

bool emit_kernel(const lf::KernelRule& k, const std::string& T, const std::function<std::string(const std::string&)>& in,
                 const std::function<std::string(const std::string&)>& out, bool declare, std::ostream& src,
                 const std::string& ind, std::string& err) {
  bool bodies = true;
  for (const auto& [op, pat] : k.outputs) bodies &= k.bodies.count(op) > 0;
  std::set<std::string> inputs;
  for (const auto& [ip, pat] : k.inputs) inputs.insert(ip);
  if (bodies) {
    for (const auto& [op, pat] : k.outputs) {
      std::string e2;
      auto e = lf::parse_expr(k.bodies.at(op), e2);
      if (!e) {
        err = "kernel '" + k.name + "' body of '" + op + "': " + e2;
        return false;
      }
      std::set<std::string> used;
      lf::expr_vars(*e, used);
      for (const auto& u : used)
        if (!inputs.count(u)) {
          err = "kernel '" + k.name + "' body of '" + op + "' uses unknown name '" + u + "'";
          return false;
        }
      src << ind << (declare ? "const T " : "") << out(op) << " = " << lf::emit_c(*e, T, in) << ";\n";
    }
    return true;
  }
  const lf::DeclInfo di = lf::parse_declaration(k.declaration);
  std::set<std::string> outputs;
  for (const auto& [op, pat] : k.outputs) outputs.insert(op);
  std::string args;
  std::vector<std::pair<std::string, std::string>> tmps;  // (temp, destination)
  for (const auto& prm : di.params) {
    std::string a;
    if (outputs.count(prm.name)) {
      const std::string tmp = "lf_o_" + prm.name;
      tmps.emplace_back(tmp, out(prm.name));
      a = prm.pointer ? "&" + tmp : tmp;
    } else if (inputs.count(prm.name)) {
      a = in(prm.name);
    } else {
      err = "kernel '" + k.name + "': declaration parameter '" + prm.name + "' is neither an input nor an output";
      return false;
    }
    args += (args.empty() ? "" : ", ") + a;
  }
  if (declare)
    for (const auto& [tmp, dst] : tmps) src << ind << "T " << dst << ";\n";
  src << ind << "{\n";
  for (const auto& [tmp, dst] : tmps) src << ind << "  T " << tmp << ";\n";
  src << ind << "  " << di.function << "(" << args << ");\n";
  for (const auto& [tmp, dst] : tmps) src << ind << "  " << dst << " = " << tmp << ";\n";
  src << ind << "}\n";
  return true;
}

bool analyse(Ctx& C) {
  const lf::Plan& P = C.P;
  const auto& rs = P.rs;
  const auto& g = P.dag;
  const int nd = static_cast<int>(rs.loop_order.size());
  auto fail = [&](const std::string& m) {
    C.error = m;
    return false;
  };
  if (nd < 1 || nd > 3) return fail("generic executor handles 1-3 loop dimensions");
  if (!P.one_nest)
    return fail("chain does not fuse into a single nest (" + std::to_string(P.nests) + " nests, " +
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
  C.T = T;
  C.nd = nd;
  C.N.resize(nd);
  C.LO.resize(nd);
  for (int d = 0; d < nd; ++d) {
    C.N[d] = rs.ranges[d].trips();
    C.LO[d] = rs.ranges[d].lo;
  }

  // ---- per-variable term offset ranges (relative to the canonical cell)
  const size_t nv = P.vars.size();
  C.vmin.assign(nv, std::vector<int>(nd, INT_MAX));
  C.vmax.assign(nv, std::vector<int>(nd, INT_MIN));
  for (size_t t = 0; t < g.terms.size(); ++t) {
    int v = P.var_of_term[t];
    for (const auto& o : g.terms[t].dims) {
      C.vmin[v][o.dim] = std::min(C.vmin[v][o.dim], o.offset);
      C.vmax[v][o.dim] = std::max(C.vmax[v][o.dim], o.offset);
    }
  }
  for (size_t v = 0; v < nv; ++v)
    for (int d = 0; d < nd; ++d)
      if (C.vmin[v][d] == INT_MAX) C.vmin[v][d] = C.vmax[v][d] = 0;
  auto canon = [&](int v) {
    while (P.vars[v].alias_of >= 0) v = P.vars[v].alias_of;
    return v;
  };
  // axiom variables: storage displacement extra[d] = ext shift - term offset
  for (const auto& r : g.raps) {
    if (r.kind != lf::RapKind::load) continue;
    const auto& term = g.terms[r.out_terms[0]];
    const int v = P.var_of_term[r.out_terms[0]];
    if (C.axiom_extra.count(v)) continue;
    std::vector<int> ex(nd, 0);
    for (const auto& s : r.ext_slots) {
      if (s.dim < 0) return fail("axioms with constant subscripts are not supported by the generic executor");
      int off = 0;
      for (const auto& o : term.dims)
        if (o.dim == s.dim) off = o.offset;
      ex[s.dim] = s.shift - off;
    }
    C.axiom_extra[v] = ex;
  }
  // which variables live on chip: kernel outputs that some kernel reads
  std::vector<char> read_by_kernel(nv, 0);
  C.smem_var.assign(nv, 0);
  for (const auto& r : g.raps)
    if (r.kind == lf::RapKind::kernel)
      for (int t : r.in_terms) read_by_kernel[canon(P.var_of_term[t])] = 1;
  for (size_t v = 0; v < nv; ++v)
    if (read_by_kernel[v] && !P.vars[v].axiom_backed && P.vars[v].alias_of < 0 && !P.vars[v].dims.empty())
      C.smem_var[v] = 1;

  // ---- kernel groups in dataflow order
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
    std::string why;
    if (!kernel_evaluable(k, C.sources, why)) return fail(why);
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
      if (!C.smem_var[in.var] && C.terminal_of(in.var, false) < 0)
        return fail("kernel '" + k.name + "' reads '" + in.param + "' from an unsupported source");
      G.in.push_back(in);
    }
    for (size_t i = 0; i < k.outputs.size(); ++i) {
      GOut o{k.outputs[i].first, canon(P.var_of_term[rep.out_terms[i]]), std::vector<int>(nd, 0)};
      for (const auto& od : g.terms[rep.out_terms[i]].dims) o.rel[od.dim] = od.offset - anchor[od.dim];
      G.out.push_back(o);
    }
    C.groups.push_back(std::move(G));
  }
  // ---- inline producers (2D/3D) whose own inputs are not inlined values:
  // cheap ones (a body of at most two operations, read by kernels only at <= 2
  // offsets per output) are recomputed at each read instead of stored -- e.g.
  // the face fluxes u[+1]-u of the 3D heat chain: fewer shared-memory round
  // trips than a window store + two loads, identical arithmetic per term; and
  // any producer whose outputs are each read exactly once (HFAV's scalar
  // contraction, storage.cpp:319-399 with span 1 -- e.g. L2 of the biharmonic
  // chain) is evaluated inside its consumer: no recomputation, no window, one
  // dependency level (and barrier) fewer
  auto ops = [](const lf::Expr& e) {
    std::function<int(const lf::Expr&)> f = [&](const lf::Expr& x) -> int {
      int n = x.kind == lf::Expr::Num || x.kind == lf::Expr::Var ? 0 : 1;
      for (const auto& a : x.args) n += f(*a);
      return n;
    };
    return f(e);
  };
  std::vector<char> inl(C.groups.size(), 0);
  if (nd >= 2 && !lfx::option("LF_JIT_NOINLINE")) {
    for (size_t gi = 0; gi < C.groups.size(); ++gi) {
      const Grp& Pg = C.groups[gi];
      const auto& k = rs.kernels[Pg.kernel];
      bool ok = true;
      int cost = 0;
      for (const auto& [op, pat] : k.outputs) {
        if (!k.bodies.count(op)) {
          ok = false;
          break;
        }
        std::string e2;
        auto e = lf::parse_expr(k.bodies.at(op), e2);
        if (!e) {
          ok = false;
          break;
        }
        cost += ops(*e);
      }
      if (!ok) continue;
      bool once = true;
      for (const auto& o : Pg.out) {
        int reads = 0;
        for (const auto& c : C.groups)
          for (const auto& in : c.in) reads += in.var == o.var;
        once &= reads == 1;
      }
      if (cost > 2 && !once) continue;
      for (const auto& in : Pg.in)
        for (size_t pj = 0; pj < C.groups.size(); ++pj)
          if (inl[pj])
            for (const auto& o2 : C.groups[pj].out) ok &= o2.var != in.var;
      for (const auto& o : Pg.out) {
        if (!C.smem_var[o.var] || C.terminal_of(o.var, true) >= 0) ok = false;
        int reads = 0;
        for (const auto& c : C.groups)
          for (const auto& in : c.in) reads += in.var == o.var;
        if (reads == 0 || reads > 2) ok = false;
      }
      // a producer's input must not itself be an inlined value
      for (size_t pj = 0; pj < C.groups.size() && ok; ++pj)
        if (inl[pj])
          for (const auto& in : C.groups[pj].in)
            for (const auto& o : Pg.out) ok &= in.var != o.var;
      if (ok) inl[gi] = 1;
    }
  }
  {
    std::vector<Grp> kept;
    std::vector<int> new_index(C.groups.size(), -1);
    for (size_t gi = 0; gi < C.groups.size(); ++gi)
      if (inl[gi]) {
        new_index[gi] = static_cast<int>(C.inlined.size());
        C.inlined.push_back(C.groups[gi]);
      }
    for (size_t gi = 0; gi < C.groups.size(); ++gi)
      if (!inl[gi]) kept.push_back(C.groups[gi]);
    for (auto& c : kept)
      for (auto& in : c.in)
        for (size_t pi = 0; pi < C.inlined.size(); ++pi)
          for (const auto& o : C.inlined[pi].out)
            if (o.var == in.var) in.via = static_cast<int>(pi);
    for (const auto& pg : C.inlined)
      for (const auto& o : pg.out) C.smem_var[o.var] = 0;
    C.groups = std::move(kept);
    // effective loads
    for (auto& c : C.groups) {
      auto add = [&](int var, const std::vector<int>& rel) {
        for (const auto& l : c.loads)
          if (l.var == var && l.rel == rel) return;
        c.loads.push_back({var, rel});
      };
      for (const auto& in : c.in) {
        if (in.via < 0) {
          add(in.var, in.rel);
          continue;
        }
        const Grp& pg = C.inlined[in.via];
        std::vector<int> orel(nd, 0);
        for (const auto& o : pg.out)
          if (o.var == in.var) orel = o.rel;
        for (const auto& pin : pg.in) {
          std::vector<int> r(nd);
          for (int d = 0; d < nd; ++d) r[d] = in.rel[d] - orel[d] + pin.rel[d];
          add(pin.var, r);
        }
      }
    }
  }
  // ---- pipeline shifts along dim 0 (reverse dataflow order) and levels
  const int nG = static_cast<int>(C.groups.size());
  for (int gi = nG - 1; gi >= 0; --gi) {
    Grp& G = C.groups[gi];
    bool any = false;
    int s = INT_MIN;
    for (const auto& o : G.out)
      for (int ci = gi + 1; ci < nG; ++ci)
        for (const auto& in : C.groups[ci].loads)
          if (in.var == o.var) {
            s = std::max(s, C.groups[ci].shift + in.rel[0] - o.rel[0]);
            any = true;
          }
    G.shift = any ? s : 0;
  }
  for (int gi = 0; gi < nG; ++gi) {
    Grp& G = C.groups[gi];
    G.level = 1;
    for (const auto& in : G.loads)
      for (int pi = 0; pi < gi; ++pi)
        for (const auto& o : C.groups[pi].out)
          if (o.var == in.var) G.level = std::max(G.level, C.groups[pi].level + 1);
  }
  // one barrier per level: groups of a level are independent of each other
  std::stable_sort(C.groups.begin(), C.groups.end(), [](const Grp& a, const Grp& b) { return a.level < b.level; });
  return true;
}

// body expressions of group G's outputs, p_<param> bound to its inputs
bool emit_bodies(Ctx& C, const Grp& G, std::ostream& src, const char* ind) {
  const auto& k = C.P.rs.kernels[G.kernel];
  std::string err;
  if (!emit_kernel(
          k, C.T, [](const std::string& n) { return "p_" + n; }, [](const std::string& n) { return "q_" + n; }, true,
          src, ind, err)) {
    C.error = err;
    return false;
  }
  return true;
}

void emit_tma_helpers(std::ostream& src) {
  // tensor maps of the streamed axioms (must match lfx::JitMaps in jit.cpp)
  // and the mbarrier / TMA primitives of the warp-specialised marches
  src << R"(struct __align__(64) LfTmap { unsigned long long w[16]; };
struct LfMaps { LfTmap m[)" << kJitMaxMaps << R"(]; };
__device__ __forceinline__ unsigned lf_s32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void lf_mbar_init(unsigned long long* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(lf_s32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void lf_mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(lf_s32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void lf_mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(lf_s32(b)) : "memory");
}
__device__ __forceinline__ void lf_mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile("{\n .reg .pred p;\n LFW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra LFW;\n}\n"
               :: "r"(lf_s32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void lf_tma2(void* dst, const LfTmap* m, unsigned long long* b, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               :: "r"(lf_s32(dst)), "l"(m), "r"(lf_s32(b)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void lf_tma3(void* dst, const LfTmap* m, unsigned long long* b, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
               :: "r"(lf_s32(dst)), "l"(m), "r"(lf_s32(b)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
)";
}

// kernel signature and the terminal pointers.  kernel == nullptr: the first
// kernel of the module (lf_jit_step), preceded by the module prelude; else a
// variant taking the tensor maps of its streamed axioms (emit_tma_helpers
// must precede it)
void emit_prelude(Ctx& C, std::ostream& src, int threads, int min_blocks, const char* kernel) {
  const auto& terms = C.P.terminals;
  if (!kernel) {
    src << "// generated by loomfuse-b200 (csrc/jit/codegen.cpp) for chain '" << C.P.rs.name << "'\n";
    src << "typedef " << C.T << " T;\n";
    src << "__device__ __forceinline__ T lf_min(T a, T b) { return a < b ? a : b; }\n";
    src << "__device__ __forceinline__ T lf_max(T a, T b) { return a > b ? a : b; }\n";
    if (C.T == "float")  // fp32x2 helpers of lf::emit_c2: lanewise, the scalar operations' rounding
      src << R"(__device__ __forceinline__ float2 lf_f2(float c) { return make_float2(c, c); }
__device__ __forceinline__ float2 lf_neg2(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 lf_div2(float2 a, float2 b) { return make_float2(a.x / b.x, a.y / b.y); }
__device__ __forceinline__ float2 lf_sqrt2(float2 a) { return make_float2(sqrtf(a.x), sqrtf(a.y)); }
__device__ __forceinline__ float2 lf_abs2(float2 a) { return make_float2(fabsf(a.x), fabsf(a.y)); }
__device__ __forceinline__ float2 lf_min2(float2 a, float2 b) { return make_float2(lf_min(a.x, b.x), lf_min(a.y, b.y)); }
__device__ __forceinline__ float2 lf_max2(float2 a, float2 b) { return make_float2(lf_max(a.x, b.x), lf_max(a.y, b.y)); }
)";
    // must match lfx::Args in jit.cpp (passed by value)
    src << "struct LfArgs { void* t[32]; long long n0; int row_lo, row_hi, top, bottom, chunk, inplace; };\n";
    src << "extern \"C\" __global__ void __launch_bounds__(" << threads << ", " << min_blocks
        << ") lf_jit_step(const LfArgs a) {\n";
  } else {
    src << "extern \"C\" __global__ void __launch_bounds__(" << threads << ", " << min_blocks << ") " << kernel
        << "(const LfArgs a, const __grid_constant__ LfMaps lf_maps) {\n";
  }
  src << "  extern __shared__ __align__(128) unsigned char lf_smem[];\n";  // one declaration for every march kernel
  src << "  const long long N0 = a.n0;\n";
  for (int d = 1; d < C.nd; ++d) src << "  const long long N" << d << " = " << C.N[d] << ";\n";
  for (size_t i = 0; i < terms.size(); ++i) {
    if (terms[i].dims.empty())
      src << "  const T s" << i << " = *reinterpret_cast<const T*>(a.t[" << i << "]);\n";
    else
      src << "  " << (terms[i].is_goal ? "T" : "const T") << "* __restrict__ t" << i << " = reinterpret_cast<"
          << (terms[i].is_goal ? "T" : "const T") << "*>(a.t[" << i << "]);\n";
  }
}

// In place (config.aliases, one buffer): a kernel copying, before each step,
// the rows at chunk boundaries and the columns at tile boundaries (`tile`: the
// march's inner tile) that one (chunk, tile) unit reads but another writes, for
// each aliased axiom (variable, terminal) into the band buffers a.t[slot],
// a.t[slot + 1], a.t[slot + 2] (rows, dim-1 columns, dim-2 columns)
void emit_capture(Ctx& C, const char* name, const std::vector<std::pair<size_t, int>>& caps,
                  const std::vector<int>& slots, const std::vector<int>& tile, std::ostream& src) {
  const int nd = C.nd;
  src << "extern \"C\" __global__ void " << name << "(const LfArgs a) {\n";
  src << "  const long long N0 = a.n0;\n";
  src << "  const int nch = (int)((N0 + a.chunk - 1) / a.chunk);\n";
  for (size_t q = 0; q < caps.size(); ++q) {
    const size_t v = caps[q].first;
    const int slot = slots[q];
    const auto& t = C.P.terminals[caps[q].second];
    const auto ex = C.extra_of(static_cast<int>(v));
    std::vector<long> so(nd);
    for (int d = 0; d < nd; ++d) so[d] = ex[d] - t.base[d] + C.LO[d];
    const long E0 = t.extent[0], E1 = nd > 1 ? t.extent[1] : 1, E2 = nd > 2 ? t.extent[2] : 1, PL = E1 * E2;
    const long BH = C.vmax[v][0] - C.vmin[v][0];
    const long BW1 = C.vmax[v][1] - C.vmin[v][1], BW2 = nd > 2 ? C.vmax[v][2] - C.vmin[v][2] : 0;
    const long NT1 = (C.N[1] + tile[1] - 1) / tile[1], NT2 = nd > 2 ? (C.N[2] + tile[2] - 1) / tile[2] : 1;
    const long nc1 = (NT1 - 1) * BW1 * E0 * E2, nc2 = nd > 2 ? (NT2 - 1) * BW2 * E0 * E1 : 0;
    src << "  {\n";
    src << "    const T* m = reinterpret_cast<const T*>(a.t[" << caps[q].second << "]);\n";
    src << "    T* rb = reinterpret_cast<T*>(a.t[" << slot << "]);\n";
    src << "    T* c1 = reinterpret_cast<T*>(a.t[" << slot + 1 << "]);\n";
    src << "    T* c2 = reinterpret_cast<T*>(a.t[" << slot + 2 << "]);\n";
    src << "    const long long nrb = (long long)max(0, nch - 1) * " << BH * PL << "LL;\n";
    src << "    const long long tot = nrb + " << (nc1 + nc2) << "LL;\n";
    src << "    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot; idx += (long long)gridDim.x * blockDim.x) {\n";
    src << "      if (idx < nrb) {\n";
    src << "        const long long p = idx % " << PL << "LL, r = idx / " << PL << "LL;\n";
    src << "        const long long y = (r / " << BH << " + 1) * (long long)a.chunk" << plus(C.vmin[v][0]) << " + r % " << BH << ";\n";
    src << "        rb[idx] = m[(y" << plus(so[0]) << ") * " << PL << "LL + p];\n";
    src << "      } else if (idx < nrb + " << nc1 << "LL) {\n";
    src << "        long long j = idx - nrb;\n";
    src << "        const long long z2 = j % " << E2 << "LL; j /= " << E2 << "LL;\n";
    src << "        const long long zy = j % " << E0 << "LL; j /= " << E0 << "LL;\n";
    src << "        const long long x1 = (j / " << std::max(1L, BW1) << " + 1) * " << tile[1] << plus(C.vmin[v][1]) << " + j % "
        << std::max(1L, BW1) << ";\n";
    src << "        c1[idx - nrb] = m[zy * " << PL << "LL + (x1" << plus(so[1]) << ") * " << E2 << "LL + z2];\n";
    if (nd == 3) {
      src << "      } else {\n";
      src << "        long long j = idx - nrb - " << nc1 << "LL;\n";
      src << "        const long long z1 = j % " << E1 << "LL; j /= " << E1 << "LL;\n";
      src << "        const long long zy = j % " << E0 << "LL; j /= " << E0 << "LL;\n";
      src << "        const long long x2 = (j / " << std::max(1L, BW2) << " + 1) * " << tile[2] << plus(C.vmin[v][2]) << " + j % "
          << std::max(1L, BW2) << ";\n";
      src << "        c2[idx - nrb - " << nc1 << "LL] = m[zy * " << PL << "LL + z1 * " << E2 << "LL + (x2" << plus(so[2]) << ")];\n";
    }
    src << "      }\n    }\n  }\n";
  }
  src << "}\n";
}

// ---------------------------------------------------------------------------
// 2D / 3D: march the outermost dimension with rolling windows
// ---------------------------------------------------------------------------
// ws: the warp-specialised variant (lf_jit_step_ws), emitted after the plain
// one with the same tile: one producer warp streams the full-rank axioms by
// TMA into their windows (a ring of PD + 1 trip stages on full / empty
// mbarriers) while 8 consumer warps evaluate the groups; consumers meet only
// at named barriers between dependency levels (intermediate windows one row
// deeper so a trip's writes never hit rows the previous trip still reads), so
// a single-level chain runs with no CTA-wide barrier at all.
//
// The emitter is a class: windows() sizes each variable's rolling window,
// geometry() picks the inner tile and the shared-memory layout, head() writes
// the kernel head and the persistent work order, trips() the per-trip loads
// (cp.async) or producer (TMA), group() one callsite group, tail() the
// window advance; capture() the in-place band copy kernel.
namespace {
class March {
 public:
  March(Ctx& c, JitProgram& o, std::ostream& s, bool w)
      : C(c), out(o), src(s), ws(w), nd(c.nd), eb(o.elem_bytes), al(16 / o.elem_bytes), nv(c.P.vars.size()),
        G(c.groups), saved_vmin(c.vmin) {}
  ~March() { C.vmin = saved_vmin; }  // the ws emission widens streamed windows for itself only
  bool emit() {
    if (!windows() || !geometry()) return false;
    head();
    trips();
    int level = 1;
    for (size_t gi = 0; gi < G.size(); ++gi)
      if (!group(gi, level)) return false;
    tail();
    capture();
    return true;
  }

 private:
  struct IP {
    size_t v;
    int ai, gi, slot;
  };
  struct Rot {
    int K = 1;
    std::vector<int> from;  // load index whose previous-trip value this load takes (-1: load)
    std::vector<char> keep;  // value carried to the next trip
  };
  Ctx& C;
  JitProgram& out;
  std::ostream& src;
  const bool ws;
  const int nd;
  const int NT = 256;
  const int eb;
  const int al;  // elements per 16 B
  const size_t nv;
  std::vector<Grp>& G;
  std::vector<std::vector<int>> saved_vmin;
  // window bookkeeping along dim 0: lead (newest row written at trip t is
  // t + lead) and oldest row read at trip t (t + old)
  std::vector<int> lead, old, win, staged;
  int PD = 3;  // axiom rows are requested PD trips before they are read
  std::vector<int> tile;
  std::vector<size_t> soff;
  size_t smem = 0;
  int TS = 0, TE = 0, cps = 1;
  long inner = 1;
  int STEP = 1, ILP = 1, VEC = 1, NS = 1;
  const char* LANE = "tx";
  bool use_rot = false;
  std::vector<Rot> rot;
  std::vector<IP> ips;
  std::vector<size_t> tv;  // TMA-staged vars, in map order

  bool windows();
  bool geometry();
  void head();
  void trips();
  bool group(size_t gi, int& level);
  void tail();
  void capture();
  void commit3();
  void inplace_masks();
  void emit_load(size_t v, const std::string& row, const std::string& slotexpr, const char* ind);
  // ws: a staged axiom's innermost row is fetched as nbox TMA boxes of bw
  // elements (box rows <= 256 elements, 128-B multiples so every box lands
  // 128-B aligned); its smem row is nbox * bw wide
  void tma_box(size_t v, int& nbox, int& bw) const {
    const int w = tile[nd - 1] + (C.vmax[v][nd - 1] - C.vmin[v][nd - 1]);
    const int al = 128 / eb;
    nbox = (w + 255) / 256;
    bw = ((w + nbox - 1) / nbox + al - 1) / al * al;
    if (bw > 256) nbox = (w + 255) / 256 + 1, bw = ((w + nbox - 1) / nbox + al - 1) / al * al;
  }
  int wdim(size_t v, int d) const {
    int w = tile[d] + (C.vmax[v][d] - C.vmin[v][d]);
    if (ws && staged[v] >= 0 && d == nd - 1) {
      int nb = 1, bw = w;
      tma_box(v, nb, bw);
      w = nb * bw;
    }
    return w;
  }
  int width(size_t v, int d) const { return wdim(v, d); }
  size_t plane(size_t v) const {
    size_t n = 1;
    for (int d = 1; d < nd; ++d) n *= wdim(v, d);
    return n;
  }
  void layout() {
    smem = 0;
    const size_t al = ws ? 128 : 16;
    for (size_t v = 0; v < nv; ++v) {
      if (win[v] <= 0) continue;
      soff[v] = smem;
      smem += (win[v] * plane(v) * eb + al - 1) / al * al;
    }
  }
  // in-plane offset of var v at tile-relative cell (c_d + rel_d)
  std::string inplane(size_t v, const std::vector<int>& rel) const {
    std::string e;
    for (int d = 1; d < nd; ++d) {
      const std::string c = "(c" + std::to_string(d) + plus(rel[d] - C.vmin[v][d]) + ")";
      e = e.empty() ? c : "(" + e + ") * " + std::to_string(width(v, d)) + " + " + c;
    }
    return e;
  }
  // rolling-window slots: b<v> = slot of row t, advanced once per trip; the
  // slot of row t + off is b<v> + (off mod W) with one conditional wrap
  int wrap(size_t v, int off) const { return ((off % win[v]) + win[v]) % win[v]; }
  std::string rowbase(size_t v, int off) const {
    if (win[v] == 1) return "0";
    const int o = wrap(v, off);
    const std::string b = "b" + std::to_string(v);
    const std::string sum = o ? "(" + b + " + " + std::to_string(o) + ")" : b;
    const std::string sl = o ? "(" + sum + " >= " + std::to_string(win[v]) + " ? " + sum + " - " + std::to_string(win[v]) +
                                   " : " + sum + ")"
                             : b;
    return sl + " * " + std::to_string(plane(v));
  }
  const IP* ip_of(size_t v) const {
    for (const auto& ip : ips)
      if (ip.v == v) return &ip;
    return nullptr;
  }
};

bool March::windows() {
  lead.assign(nv, INT_MIN);
  old.assign(nv, INT_MAX);
  win.assign(nv, 0);
  staged.assign(nv, -1);
  // axiom rows are requested PD trips before they are read
  PD = nd == 2 || ws ? 3 : 2;  // measured: 3D plain 2, warp-specialised 3 (324 vs 308 G)
  if (const char* e = lfx::option("LF_JIT_PD")) PD = std::max(1, std::atoi(e));
  for (const auto& g : G)
    for (const auto& in : g.loads) {
      lead[in.var] = std::max(lead[in.var], C.smem_var[in.var] ? INT_MIN : g.shift + in.rel[0]);
      old[in.var] = std::min(old[in.var], g.shift + in.rel[0]);
    }
  for (const auto& g : G)
    for (const auto& o : g.out)
      if (C.smem_var[o.var]) lead[o.var] = g.shift + o.rel[0];
  for (size_t v = 0; v < nv; ++v) {
    if (C.smem_var[v]) {
      win[v] = lead[v] - old[v] + 1 + (ws ? 1 : 0);
    } else if (old[v] != INT_MAX && C.staged_axiom(static_cast<int>(v)) >= 0) {
      staged[v] = C.staged_axiom(static_cast<int>(v));
      win[v] = lead[v] - old[v] + 1 + PD;  // + the rows in flight
    }
    if (win[v] > 0 && (win[v] > 64 || old[v] < -60 || lead[v] > 60))
      return (C.error = "pipeline window deeper than 64 rows", false);
  }
  // fault injection for the differential tests (R/"deliberately
  // corrupted rotation span (span-1) -> mismatch reported"): LF_JIT_FAULT=
  // span:<intermediate> emits that variable's rolling window one row short
  if (const char* f = lfx::option("LF_JIT_FAULT"); f && std::strncmp(f, "span:", 5) == 0)
    for (size_t v = 0; v < nv; ++v)
      if (C.smem_var[v] && win[v] > 1 && C.P.vars[v].name == f + 5) win[v] -= 1;
  // ws: TMA box origins must be 16-B aligned along the contiguous dimension.
  // Tiles are a multiple of `al` elements there, and each streamed axiom's
  // window starts up to al - 1 elements further left (its range is widened
  // for this emission only) so that origin = tile start + a multiple of al.
  // (restored by ~March)
  if (ws)
    for (size_t v = 0; v < nv; ++v) {
      if (staged[v] < 0) continue;
      const auto& t = C.P.terminals[staged[v]];
      const int d = nd - 1;
      const long so = C.extra_of(static_cast<int>(v))[d] - t.base[d] + C.LO[d];
      const long m = ((C.vmin[v][d] + so) % al + al) % al;
      C.vmin[v][d] -= static_cast<int>(m);
    }
  return true;
}

bool March::geometry() {
  // inner tile: cells per plane of the widest window a multiple of the block
  int span_in[3] = {0, 0, 0};
  for (size_t v = 0; v < nv; ++v)
    if (win[v] > 0)
      for (int d = 1; d < nd; ++d) span_in[d] = std::max(span_in[d], C.vmax[v][d] - C.vmin[v][d]);
  for (const auto& g : G)
    for (int d = 1; d < nd; ++d) span_in[d] = std::max(span_in[d], g.gmax[d] - g.gmin[d]);
  tile.assign(nd, 1);
  soff.assign(nv, 0);
  smem = 0;
  // widths: the outermost inner dimension first; defaults sized for >= 2 CTAs/SM
  int wide = eb == 8 ? 512 : 1024;
  int rows_in = 16;
  if (const char* e = lfx::option("LF_JIT_TILE")) {  // experiments: "<rows>x<width>"
    int r = 0, w = 0;
    if (std::sscanf(e, "%dx%d", &r, &w) == 2 && r > 0 && w > 0) rows_in = r, wide = w;
  }
  for (; !ws;) {
    if (nd == 2) {
      tile[1] = std::max(32, wide - span_in[1]);
    } else {
      tile[2] = std::max(16, std::min<int>(64, wide) - span_in[2]);
      tile[1] = std::max(1, rows_in - span_in[1]);
    }
    layout();
    if (smem <= 100 * 1024) break;
    if (nd == 3 && rows_in > 2) {
      rows_in /= 2;
    } else if (wide > 64) {
      wide /= 2;
    } else {
      break;
    }
  }
  if (ws) {
    tile = out.tile;
    if (nd == 3) {
      // TMA stages the halo, so the 64 x 4 consumer lanes need only cover the
      // groups' own extents: a 64-column tile of 16 rows when the groups are
      // pointwise in the plane (e.g. heat3d after inlining), full 32-B sectors
      // per stored row segment and four rows per lane
      int gs[3] = {0, 0, 0};
      for (const auto& g : G)
        for (int d = 1; d < nd; ++d) gs[d] = std::max(gs[d], g.gmax[d] - g.gmin[d]);
      std::vector<int> keep = tile;
      tile[2] = (64 - gs[2]) / al * al;
      tile[1] = std::max(1, 16 - gs[1]);
      layout();
      if (smem > 100 * 1024) tile = keep;
    }
    tile[nd - 1] = std::max(al, tile[nd - 1] / al * al);
    layout();
    if (smem > 200 * 1024) return false;
    out.ws_smem_bytes = smem + 16 * (PD + 1);  // + the stage mbarriers
    out.ws_threads = NT + 32;
  }
  if (smem > 200 * 1024) return (C.error = "chain needs too much on-chip storage for one tile", false);
  if (!ws) {
  out.tile = tile;
  out.tile[0] = 1;
  out.smem_bytes = smem;
  out.threads = NT;
  out.march = true;
  }
  // trip range relative to the chunk [r0, r1): t in [r0 + TS, r1 - 1 + TE]
  TS = INT_MAX;
  TE = INT_MIN;
  for (const auto& g : G) {
    TS = std::min(TS, g.gmin[0] - g.shift);
    TE = std::max(TE, g.gmax[0] - g.shift);
  }
  for (size_t v = 0; v < nv; ++v)
    if (staged[v] >= 0) TS = std::min(TS, C.vmin[v][0] - lead[v]);
  cps = std::max<int>(1, std::min<int>(2048 / NT, static_cast<int>((227 * 1024) / (smem + 1024))));
  inner = 1;
  for (int d = 1; d < nd; ++d) inner *= (C.N[d] + tile[d] - 1) / tile[d];
  if (ws) out.ws_inner_tiles = inner;
  if (!ws) {
    out.prologue = TE - TS;
    out.inner_tiles = inner;
    out.ctas_per_sm = cps;
    out.chunk = nd == 3 ? 64 : 1 << 30;  // rows per chunk of the work order (2D: whole tiles)
  }

  return true;
}

void March::head() {
  int minb = std::min(cps, 2);  // register cap; 2 measured best
  if (const char* e = lfx::option("LF_JIT_MINB")) minb = std::max(1, std::atoi(e));
  emit_prelude(C, src, ws ? NT + 32 : NT, minb, ws ? "lf_jit_step_ws" : nullptr);
  // ws: warp 0 is the producer, consumer thread c = threadIdx.x - 32
  const char* TID = ws ? "((int)threadIdx.x - 32)" : "threadIdx.x";
  if (nd == 3)
    src << "  const int tx = " << TID << " & 63, ty = " << TID << " >> 6;\n";
  else
    src << "  const int tx = " << TID << ";\n";
  for (size_t v = 0; v < nv; ++v)
    if (win[v] > 0)
      src << "  T* __restrict__ v" << v << " = reinterpret_cast<T*>(lf_smem + " << soff[v] << ");  // '"
          << C.P.vars[v].name << "': " << win[v] << " rows x " << plane(v) << "\n";
  // 3D: a 64-wide column per thread x 4 row lanes; 2D: 256 columns per pass
  STEP = nd == 3 ? NT / 64 : NT;
  ILP = 1;  // cells whose operands are loaded before any is evaluated (1 measured best)
  if (const char* e = lfx::option("LF_JIT_ILP")) ILP = std::max(1, std::atoi(e));
  // 2D, opt-in (LF_JIT_VEC=2): adjacent columns per thread sharing their
  // window loads.  Exact, but measured slower (biharm 157 vs 222 G, box 244 vs
  // 274 G): lanes two elements apart make every shared-memory load a 2-way
  // bank conflict and the shared operands cost registers.
  VEC = 1;
  if (const char* e = lfx::option("LF_JIT_VEC")) VEC = std::max(1, std::atoi(e));
  LANE = nd == 3 ? "ty" : "tx";
  // ---- persistent CTAs: each takes an equal share of the (row chunk, inner
  // tile, row) space in that order and marches it as one or more segments,
  // so neighbouring tiles run at the same time and share halos in L2
  for (size_t v = 0; v < nv; ++v)
    if (staged[v] >= 0) src << "  const unsigned sb" << v << " = (unsigned)__cvta_generic_to_shared(v" << v << ");\n";
  // in-place (config.aliases, caller passes one buffer): whole (chunk, tile)
  // units so that every cross-unit read hits a band captured before the step
  ips.clear();
  if (!ws) {
    out.inplace.clear();
    out.inplace_error.clear();
  } else {
    out.ws_inplace.clear();
  }
  const int nterm = static_cast<int>(C.P.terminals.size());
  for (const auto& [in_ext, out_ext] : C.P.rs.aliases) {
    int ai = -1, gi = -1;
    for (int i = 0; i < nterm; ++i) {
      if (!C.P.terminals[i].is_goal && C.P.terminals[i].name == in_ext) ai = i;
      if (C.P.terminals[i].is_goal && C.P.terminals[i].name == out_ext) gi = i;
    }
    if (ai < 0 || gi < 0) continue;
    const int v = C.P.terminals[ai].var;
    if (v < 0 || staged[v] < 0) {
      out.inplace_error = "aliased input '" + in_ext + "' is not a streamed full-rank axiom";
      continue;
    }
    if (C.P.terminals[ai].extent != C.P.terminals[gi].extent || C.P.terminals[ai].base != C.P.terminals[gi].base) {
      out.inplace_error = "aliased buffers '" + in_ext + "' and '" + out_ext + "' have different extents";
      continue;
    }
    IP ip{static_cast<size_t>(v), ai, gi, nterm + 3 * static_cast<int>(ips.size())};
    if (ip.slot + 3 > 32) {
      out.inplace_error = "too many aliased buffers";
      continue;
    }
    ips.push_back(ip);
    const auto& t = C.P.terminals[ai];
    const auto& vm = ws ? saved_vmin : C.vmin;  // the ws emission widens streamed windows for TMA alignment
    JitProgram::Inplace q;
    q.ai = ai;
    q.gi = gi;
    q.bh = C.vmax[v][0] - vm[v][0];
    q.bw1 = nd > 1 ? C.vmax[v][1] - vm[v][1] : 0;
    q.bw2 = nd > 2 ? C.vmax[v][2] - vm[v][2] : 0;
    if (ws && nd == 3) q.bw2 += 2 * (32 / eb - 1);  // deferred column zones widened to whole 32-B sectors
    q.e0 = t.extent[0];
    q.e1 = nd > 1 ? t.extent[1] : 1;
    q.e2 = nd > 2 ? t.extent[2] : 1;
    q.t1 = nd > 1 ? tile[1] : 1;
    q.t2 = nd > 2 ? tile[2] : 1;
    q.n1 = nd > 1 ? C.N[1] : 1;
    q.n2 = nd > 2 ? C.N[2] : 1;
    (ws ? out.ws_inplace : out.inplace).push_back(q);
  }
  for (const auto& ip : ips)
    if (!ws)
    src << "  const T* __restrict__ rb" << ip.slot << " = reinterpret_cast<const T*>(a.t[" << ip.slot
        << "]);  // in-place bands of '" << C.P.vars[ip.v].name << "'\n"
        << "  const T* __restrict__ cb" << ip.slot << "_1 = reinterpret_cast<const T*>(a.t[" << ip.slot + 1 << "]);\n"
        << "  const T* __restrict__ cb" << ip.slot << "_2 = reinterpret_cast<const T*>(a.t[" << ip.slot + 2 << "]);\n";
  // ws: trip-stage ring (full: producer -> consumers, empty: consumers -> producer)
  NS = PD + 1;
  tv.clear();  // TMA-staged vars, in map order
  for (size_t v = 0; v < nv; ++v)
    if (ws && staged[v] >= 0) tv.push_back(v);
  if (ws) {
    src << "  unsigned long long* lf_full = reinterpret_cast<unsigned long long*>(lf_smem + " << smem << ");\n";
    src << "  unsigned long long* lf_empty = lf_full + " << NS << ";\n";
    src << "  if (threadIdx.x == 0) {\n";
    src << "    for (int i = 0; i < " << NS << "; ++i) { lf_mbar_init(&lf_full[i], 1); lf_mbar_init(&lf_empty[i], "
        << NT / 32 << "); }\n";
    src << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n";
    for (size_t k = 0; k < tv.size(); ++k)
      src << "    asm volatile(\"prefetch.tensormap [%0];\" :: \"l\"(&lf_maps.m[" << k << "]) : \"memory\");\n";
    src << "  }\n";
    src << "  __syncthreads();\n";
    src << "  const bool producer = threadIdx.x < 32;\n";
    src << "  if (producer && threadIdx.x != 0) return;\n";
    src << "  unsigned lf_g = 0;  // trip counter across segments: stage lf_g % " << NS << "\n";
    // window slots advance continuously across segments (one ring per variable)
    for (size_t v = 0; v < nv; ++v)
      if (win[v] > 1) src << "  int b" << v << " = 0;\n";
  }
  src << "  const int rows = a.row_hi - a.row_lo;\n";
  src << "  const long long total = (long long)rows * " << inner << ";\n";
  src << "  const long long per = (total + gridDim.x - 1) / gridDim.x;\n";
  src << "  long long s = (long long)blockIdx.x * per;\n";
  src << "  const long long s_end = min(total, s + per);\n";
  // whole (chunk, tile) units dealt round-robin, chunk-major, so the CTAs
  // running at one time hold neighbouring tiles of the same rows: halo rows
  // are fetched once and hit in L2, and the row segments neighbouring tiles
  // write into shared sectors meet in L2 before eviction (LF_JIT_SPAN_ORDER=1:
  // the earlier equal-span order, plain kernel only, for comparison)
  const char* UNITS = ws || !lfx::option("LF_JIT_SPAN_ORDER") ? "true" : "a.inplace";
  src << "  const long long units = " << UNITS << " ? (long long)((rows + a.chunk - 1) / a.chunk) * " << inner
      << " : 0;\n";
  src << "  long long u = blockIdx.x;\n";
  src << "  for (;;) {\n";
  src << "  int bt, r0_, r1_;\n";
  src << "  if (" << UNITS << ") {\n";
  src << "    if (u >= units) break;\n";
  src << "    const int ci = (int)(u / " << inner << ");\n";
  src << "    bt = (int)(u % " << inner << ");\n";
  src << "    r0_ = a.row_lo + ci * a.chunk;\n";
  src << "    r1_ = min(r0_ + a.chunk, a.row_hi);\n";
  src << "    u += gridDim.x;\n";
  src << "  } else {\n";
  src << "    if (s >= s_end) break;\n";
  src << "    const long long cs = (long long)a.chunk * " << inner << ";\n";
  src << "    const int ci = (int)(s / cs);\n";
  src << "    const int rc = min(a.chunk, rows - ci * a.chunk);\n";
  src << "    const long long off = s - ci * cs;\n";
  src << "    bt = (int)(off / rc);\n";
  src << "    r0_ = a.row_lo + ci * a.chunk + (int)(off % rc);\n";
  src << "    r1_ = (int)min((long long)(a.row_lo + ci * a.chunk + rc), r0_ + (s_end - s));\n";
  src << "    s += r1_ - r0_;\n";
  src << "  }\n";
  src << "  const int r0 = r0_, r1 = r1_;\n";
  if (ws && !ips.empty()) src << "  const int ci_ = (r0 - a.row_lo) / a.chunk;  // chunk index (in place: plane bands)\n";
  for (int d = nd - 1; d >= 1; --d) {
    const long nt = (C.N[d] + tile[d] - 1) / tile[d];
    src << "  const int o" << d << " = (bt % " << nt << ") * " << tile[d] << "; bt /= " << nt << ";\n";
  }
  if (!ws)
    for (size_t v = 0; v < nv; ++v)
      if (win[v] > 1) src << "  int b" << v << " = " << wrap(v, TS) << ";\n";
  if (ws && nd == 3 && !ips.empty()) inplace_masks();
  // register windows along the march (opt-in, LF_JIT_ROT=1): a thread keeps
  // its cells for a whole segment, so a window value read at row offset s on
  // trip t+1 is the one it read at s+1 on trip t -- only the newest row of
  // each (variable, in-plane offset) set is loaded, the rest rotate through
  // registers.  Measured slower on the BASELINE chains (biharm 163 vs 178 G,
  // box 171 vs 219 G: the register cost outweighs the shared-memory loads
  // saved), so off by default.
  rot.assign(G.size(), Rot{});
  use_rot = lfx::option("LF_JIT_ROT") && std::atoi(lfx::option("LF_JIT_ROT")) != 0;
  for (size_t gi = 0; gi < G.size(); ++gi) {
    const Grp& g = G[gi];
    Rot& R = rot[gi];
    R.K = (tile[1] + (g.gmax[1] - g.gmin[1]) + STEP - 1) / STEP;
    R.from.assign(g.loads.size(), -1);
    R.keep.assign(g.loads.size(), 0);
    if (!use_rot || ILP != 1) continue;
    for (size_t li = 0; li < g.loads.size(); ++li) {
      const Load& a = g.loads[li];
      if (win[a.var] <= 0) continue;
      for (size_t lj = 0; lj < g.loads.size(); ++lj) {
        const Load& b = g.loads[lj];
        if (b.var != a.var || b.rel[0] != a.rel[0] + 1) continue;
        bool same = true;
        for (int d = 1; d < nd; ++d) same &= a.rel[d] == b.rel[d];
        if (same) {
          R.from[li] = static_cast<int>(lj);
          R.keep[lj] = 1;
        }
      }
    }
    for (size_t lj = 0; lj < g.loads.size(); ++lj)
      if (R.keep[lj]) src << "  T rw" << gi << "_" << lj << "[" << R.K << "];\n";
  }
}

void March::emit_load(size_t v, const std::string& row, const std::string& slotexpr, const char* ind) {
  std::vector<int> ext(nd), lo(nd);
  for (int d = 1; d < nd; ++d) {
    ext[d] = width(v, d);
    lo[d] = C.vmin[v][d];
  }
  const int K = (ext[1] + STEP - 1) / STEP;
  std::string I(ind);
  src << I << "{ const int y = " << row << ";\n";
  src << I << "  if (y >= r0" << plus(C.vmin[v][0]) << " && y <= r1 - 1" << plus(C.vmax[v][0]) << ") {\n";
  src << I << "    const unsigned dst = sb" << v << " + (" << slotexpr << ") * " << eb << ";\n";
  if (nd == 3) {
    src << I << "    const int c2 = tx" << plus(lo[2]) << ";\n";
    src << I << "    const int x2 = o2 + c2;\n";
    src << I << "    if (tx < " << ext[2] << " && x2 <= " << (C.N[2] - 1 + C.vmax[v][2]) << ") {\n";
  } else {
    src << I << "    {\n";
  }
  src << I << "      const int c1hi = min(" << (lo[1] + ext[1] - 1) << ", " << (C.N[1] - 1 + C.vmax[v][1]) << " - o1);\n";
  src << I << "      #pragma unroll\n";
  src << I << "      for (int k = 0; k < " << K << "; ++k) {\n";
  src << I << "        const int c1 = " << LANE << plus(lo[1]) << " + k * " << STEP << ";\n";
  src << I << "        if (c1 <= c1hi) {\n";
  src << I << "          const int x1 = o1 + c1;\n";
  std::vector<std::string> pos = {"y"};
  for (int d = 1; d < nd; ++d) pos.push_back("x" + std::to_string(d));
  src << I << "          const T* sp = t" << staged[v] << " + " << C.tidx(staged[v], pos, C.extra_of(static_cast<int>(v)))
      << ";\n";
  if (const IP* ip = ip_of(v)) {
    // in-place: a cell another unit writes during this step comes from its band
    const auto& t = C.P.terminals[ip->ai];
    const auto ex = C.extra_of(static_cast<int>(v));
    std::vector<long> so(nd);  // storage coordinate = logical + so
    for (int d = 0; d < nd; ++d) so[d] = ex[d] - t.base[d] + C.LO[d];
    const long E0 = t.extent[0], E1 = nd > 1 ? t.extent[1] : 1, E2 = nd > 2 ? t.extent[2] : 1;
    const long BH = C.vmax[v][0] - C.vmin[v][0];
    const std::string sy = "(long long)(y" + plus(so[0]) + ")", sx1 = "(long long)(x1" + plus(so[1]) + ")",
                      sx2 = nd > 2 ? "(long long)(x2" + plus(so[2]) + ")" : "0LL";
    const std::string sl = std::to_string(ip->slot);
    src << I << "          if (a.inplace) {\n";
    src << I << "            if (y < r0 || y >= r1) {\n";
    src << I << "              if (y >= 0 && y < N0) {\n";
    src << I << "                const int b = y < r0 ? r0 : r1;\n";
    src << I << "                sp = rb" << sl << " + ((long long)(b / a.chunk - 1) * " << BH << " + (y - b" << plus(-C.vmin[v][0])
        << ")) * " << (E1 * E2) << "LL + " << sx1 << " * " << E2 << "LL + " << sx2 << ";\n";
    src << I << "              }\n";
    src << I << "            } else if (x1 < o1 || x1 >= o1 + " << tile[1] << ") {\n";
    src << I << "              if (x1 >= 0 && x1 < N1) {\n";
    src << I << "                const int e = x1 < o1 ? o1 : o1 + " << tile[1] << ";\n";
    src << I << "                sp = cb" << sl << "_1 + (((long long)(e / " << tile[1] << " - 1) * "
        << (C.vmax[v][1] - C.vmin[v][1]) << " + (x1 - e" << plus(-C.vmin[v][1]) << ")) * " << E0 << "LL + " << sy
        << ") * " << E2 << "LL + " << sx2 << ";\n";
    src << I << "              }\n";
    if (nd == 3) {
      src << I << "            } else if (x2 < o2 || x2 >= o2 + " << tile[2] << ") {\n";
      src << I << "              if (x2 >= 0 && x2 < N2) {\n";
      src << I << "                const int e = x2 < o2 ? o2 : o2 + " << tile[2] << ";\n";
      src << I << "                sp = cb" << sl << "_2 + (((long long)(e / " << tile[2] << " - 1) * "
          << (C.vmax[v][2] - C.vmin[v][2]) << " + (x2 - e" << plus(-C.vmin[v][2]) << ")) * " << E0 << "LL + " << sy
          << ") * " << E1 << "LL + " << sx1 << ";\n";
      src << I << "              }\n";
    }
    src << I << "            }\n";
    src << I << "          }\n";
  }
  src << I << "          asm volatile(\"cp.async.ca.shared.global [%0], [%1], " << eb << ";\" :: \"r\"(dst + ("
      << inplane(v, std::vector<int>(nd, 0)) << ") * " << eb << "), \"l\"(sp) : \"memory\");\n";
  src << I << "        }\n" << I << "      }\n" << I << "    }\n" << I << "  }\n" << I << "}\n";
}

void March::trips() {
  if (!ws) {
  for (int p = 0; p < PD; ++p) {
    for (size_t v = 0; v < nv; ++v)
      if (staged[v] >= 0)
        emit_load(v, "r0" + plus(TS + p + lead[v]), std::to_string(wrap(v, TS + p + lead[v]) * plane(v)), "  ");
    src << "  asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n";
  }
  src << "  for (int t = r0 + (" << TS << "); t <= r1 - 1 + (" << TE << "); ++t) {\n";
  src << "    asm volatile(\"cp.async.wait_group " << (PD - 1) << ";\" ::: \"memory\");\n";
  src << "    __syncthreads();\n";
  for (size_t v = 0; v < nv; ++v)
    if (staged[v] >= 0) emit_load(v, "t" + plus(PD + lead[v]), rowbase(v, PD + lead[v]), "    ");
  src << "    asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n";
  } else {
  src << "  for (int t = r0 + (" << TS << "); t <= r1 - 1 + (" << TE << "); ++t, ++lf_g) {\n";
  src << "    const unsigned stg = lf_g % " << NS << ", par = (lf_g / " << NS << ") & 1;\n";
  src << "    if (producer) {\n";
  // the stage's previous occupant: trip lf_g - NS, whose window rows this trip's loads overwrite
  src << "      if (lf_g >= " << NS << ") lf_mbar_wait(&lf_empty[stg], par ^ 1);\n";
  src << "      unsigned bytes = 0;\n";
  for (size_t k = 0; k < tv.size(); ++k) {
    const size_t v = tv[k];
    int nb = 1, bw = 1;
    tma_box(v, nb, bw);
    size_t box = static_cast<size_t>(nb) * bw * eb;
    if (nd == 3) box *= width(v, 1);
    src << "      const int y" << k << " = t" << plus(lead[v]) << ";\n";
    src << "      const bool in" << k << " = y" << k << " >= r0" << plus(C.vmin[v][0]) << " && y" << k << " <= r1 - 1"
        << plus(C.vmax[v][0]) << ";\n";
    src << "      if (in" << k << ") bytes += " << box << "u;\n";
  }
  src << "      asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n";
  src << "      lf_mbar_expect(&lf_full[stg], bytes);\n";
  for (size_t k = 0; k < tv.size(); ++k) {
    const size_t v = tv[k];
    const int ti = staged[v];
    const auto& t = C.P.terminals[ti];
    const auto ex = C.extra_of(static_cast<int>(v));
    auto so = [&](int d) { return static_cast<long>(ex[d]) - t.base[d] + C.LO[d]; };  // storage = logical + so
    int nb = 1, bw = 1;
    tma_box(v, nb, bw);
    src << "      if (in" << k << ") {\n";
    src << "        T* dst = v" << v << " + " << rowbase(v, lead[v]) << ";\n";
    if (nd == 3) {
      src << "        lf_tma3(dst, &lf_maps.m[" << k << "], &lf_full[stg], o2" << plus(C.vmin[v][2] + so(2)) << ", o1"
          << plus(C.vmin[v][1] + so(1)) << ", y" << k << plus(so(0)) << ");\n";
    } else {
      for (int b = 0; b < nb; ++b)
        src << "        lf_tma2(dst + " << b * bw << ", &lf_maps.m[" << k << "], &lf_full[stg], o1"
            << plus(C.vmin[v][1] + so(1) + b * bw) << ", y" << k << plus(so(0)) << ");\n";
    }
    src << "      }\n";
    JitProgram::Tma tm;
    tm.term = ti;
    tm.rank = nd;
    for (int d = 0; d < nd; ++d) tm.extent[d] = t.extent[nd - 1 - d];  // innermost first
    tm.box[0] = static_cast<unsigned>(bw);
    tm.box[1] = nd == 3 ? static_cast<unsigned>(width(v, 1)) : 1u;
    tm.box[2] = 1;
    out.ws_maps.push_back(tm);
  }
  src << "    } else {\n";
  src << "    lf_mbar_wait(&lf_full[stg], par);\n";
  }
}

// one callsite group: row t + shift of its outputs, its cells of the tile
bool March::group(size_t gi, int& level) {
  const Grp& g = G[gi];
  const auto& k = C.P.rs.kernels[g.kernel];
  if (g.level != level) {
    src << (ws ? "    asm volatile(\"bar.sync 1, " + std::to_string(NT) + ";\" ::: \"memory\");\n"
               : std::string("    __syncthreads();\n"));
    level = g.level;
  }
  std::vector<int> ext(nd), lo(nd);
  for (int d = 1; d < nd; ++d) {
    ext[d] = tile[d] + (g.gmax[d] - g.gmin[d]);
    lo[d] = g.gmin[d];
  }
  const int K = (ext[1] + STEP - 1) / STEP;
  src << "    { // group " << gi << ": kernel '" << k.name << "', lead " << g.shift << ", level " << g.level << "\n";
  src << "      const int y = t" << plus(g.shift) << ";\n";
  src << "      if (y >= r0" << plus(g.gmin[0]) << " && y <= r1 - 1" << plus(g.gmax[0]) << ") {\n";
  src << "        const bool first = y == r0" << plus(g.gmin[0]) << ";  // segment start: fill the register windows\n";
  std::map<std::pair<int, int>, std::string> rbs;
  auto rb = [&](int v, int r) {
    auto key = std::make_pair(v, r);
    auto it = rbs.find(key);
    if (it != rbs.end()) return it->second;
    std::string nm = "rb" + std::to_string(v) + "_" + (r < 0 ? "m" + std::to_string(-r) : std::to_string(r));
    src << "        const int " << nm << " = " << rowbase(v, g.shift + r) << ";\n";
    rbs[key] = nm;
    return nm;
  };
  for (const auto& in : g.loads)
    if (win[in.var] > 0) rb(in.var, in.rel[0]);
  for (const auto& o : g.out)
    if (C.smem_var[o.var]) rb(o.var, o.rel[0]);
  if (nd == 3) {
    src << "        const int c2 = tx" << plus(lo[2]) << ";\n";
    src << "        const int x2 = o2 + c2;\n";
    src << "        const bool act = tx < " << ext[2] << " && x2 <= " << (C.N[2] - 1 + g.gmax[2]) << ";\n";
  } else {
    src << "        const bool act = true;\n";
  }
  src << "        const int c1hi = min(" << (lo[1] + ext[1] - 1) << ", " << (C.N[1] - 1 + g.gmax[1]) << " - o1);\n";
  auto load_index = [&](int var, const std::vector<int>& rel) {
    for (size_t li = 0; li < g.loads.size(); ++li)
      if (g.loads[li].var == var && g.loads[li].rel == rel) return static_cast<int>(li);
    return -1;
  };
  // evaluation of one cell from its loaded operands l<li>, then its stores
  auto emit_eval = [&](const std::string& I) -> bool {
  for (const auto& in : g.in) {
    if (in.via < 0) {
      src << I << "const T p_" << in.param << " = l" << load_index(in.var, in.rel) << ";\n";
      continue;
    }
    // the inlined producer, evaluated at this read's offset
    const Grp& pg = C.inlined[in.via];
    const auto& pk = C.P.rs.kernels[pg.kernel];
    std::string oparam;
    std::vector<int> orel(nd, 0);
    for (const auto& o : pg.out)
      if (o.var == in.var) {
        oparam = o.param;
        orel = o.rel;
      }
    std::map<std::string, std::string> pv;
    for (const auto& pin : pg.in) {
      std::vector<int> r(nd);
      for (int d = 0; d < nd; ++d) r[d] = in.rel[d] - orel[d] + pin.rel[d];
      pv[pin.param] = "l" + std::to_string(load_index(pin.var, r));
    }
    std::string e2;
    auto e = lf::parse_expr(pk.bodies.at(oparam), e2);
    if (!e) return (C.error = "kernel '" + pk.name + "': " + e2, false);
    src << I << "const T p_" << in.param << " = "
        << lf::emit_c(*e, C.T, [&](const std::string& n) { return pv.at(n); }) << ";  // inlined '" << pk.name
        << "'\n";
  }
  if (!emit_bodies(C, g, src, I.c_str())) return false;
  for (const auto& o : g.out) {
    if (C.smem_var[o.var])
      src << I << "v" << o.var << "[" << rb(o.var, o.rel[0]) << " + " << inplane(o.var, o.rel) << "] = q_"
          << o.param << ";\n";
    const int ti = C.terminal_of(o.var, true);
    if (ti < 0) continue;
    // goal: own chunk rows, own tile cells, inside the domain
    src << I << "if (y" << plus(o.rel[0]) << " >= r0 && y" << plus(o.rel[0]) << " < r1";
    for (int d = 1; d < nd; ++d)
      src << " && c" << d << plus(o.rel[d]) << " >= 0 && c" << d << plus(o.rel[d]) << " < " << tile[d] << " && x" << d
          << plus(o.rel[d]) << " < N" << d;
    std::vector<std::string> pos;
    for (int d = 0; d < nd; ++d) pos.push_back((d == 0 ? std::string("y") : "x" + std::to_string(d)) + plus(o.rel[d]));
    const IP* gip = nullptr;
    for (const auto& ip : ips)
      if (ip.gi == ti) gip = &ip;
    if (ws && nd == 3 && gip) {
      // in place: deferred boundary writes -- plane zone -> plane band, tile-row
      // zone -> row band, sector-aligned tile-column zone -> column band; the
      // addresses are selected, not branched to (every warp holds zone lanes)
      const auto& t = C.P.terminals[ti];
      const size_t v = gip->v;
      const long so1 = -t.base[1] + C.LO[1], so2 = -t.base[2] + C.LO[2];
      const long lo0 = saved_vmin[v][0], hi0 = C.vmax[v][0], lo2 = saved_vmin[v][2], hi2 = C.vmax[v][2];
      const long SE = 32 / eb, E1 = t.extent[1], E2 = t.extent[2], BH = hi0 - lo0, BW2 = hi2 - lo2 + 2 * (SE - 1);
      const std::string yy = "(y" + plus(o.rel[0]) + ")", xx1 = "(x1" + plus(o.rel[1]) + ")", xx2 = "(x2" + plus(o.rel[2]) + ")";
      const std::string nm = std::to_string(gi) + "_" + o.param;
      src << ") {\n";
      src << I << "  T* gp = t" << ti << " + " << C.tidx(ti, pos, std::vector<int>(nd, 0)) << ";\n";
      src << I << "  if (a.inplace) {\n";
      src << I << "    const int pbr = r0 > 0 && " << yy << " < r0" << plus(hi0) << " ? (ci_ - 1) * " << BH << " + (" << yy << " - r0" << plus(-lo0)
          << ") : (r1 < N0 && " << yy << " >= r1" << plus(lo0) << " ? ci_ * " << BH << " + (" << yy << " - r1" << plus(-lo0) << ") : -1);\n";
      src << I << "    T* const pp = reinterpret_cast<T*>(a.t[" << gip->slot << "]) + ((long long)pbr * " << E1 << " + (" << xx1 << plus(so1)
          << ")) * " << E2 << "LL + (" << xx2 << plus(so2) << ");\n";
      src << I << "    T* const rp = reinterpret_cast<T*>(a.t[" << gip->slot + 1 << "]) + rbo" << nm << "[k] + (long long)" << yy << " * " << E2
          << ";\n";
      src << I << "    T* const cp = reinterpret_cast<T*>(a.t[" << gip->slot + 2 << "]) + cbo" << nm << " + ((long long)" << yy << " * " << E1
          << " + " << xx1 << ") * " << BW2 << ";\n";
      src << I << "    gp = pbr >= 0 ? pp : (((rz" << nm << " >> k) & 1u) ? rp : (cz" << nm << " ? cp : gp));\n";
      src << I << "  }\n";
      src << I << "  *gp = q_" << o.param << ";\n";
      src << I << "}\n";
      (void)so1;
      continue;
    }
    src << ") t" << ti << "[" << C.tidx(ti, pos, std::vector<int>(nd, 0)) << "] = q_" << o.param << ";\n";
  }
    return true;
  };
  // 2D: V adjacent columns per thread; window operands are loaded once per
  // distinct (variable, row, column) over the V cells and shared between them
  const int V = nd == 2 && !use_rot && ILP == 1 ? VEC : 1;
  if (V > 1) {
    const int KV = (ext[1] + STEP * V - 1) / (STEP * V);
    src << "        #pragma unroll\n";
    src << "        for (int k = 0; k < " << KV << "; ++k) {\n";
    src << "          const int cb = " << V << " * tx" << plus(lo[1]) << " + k * " << STEP * V << ";\n";
    std::map<std::tuple<int, int, int>, int> need;  // (var, row offset, column offset) -> first cell needing it
    for (const auto& in : g.loads)
      if (win[in.var] > 0)
        for (int v = 0; v < V; ++v) {
          const auto key = std::make_tuple(in.var, in.rel[0], v + in.rel[1]);
          auto it = need.find(key);
          if (it == need.end() || it->second > v) need[key] = v;
        }
    auto uname = [](int var, int r, int u) {
      return "w" + std::to_string(var) + "_" + (r < 0 ? "m" + std::to_string(-r) : std::to_string(r)) + "_" +
             (u < 0 ? "m" + std::to_string(-u) : std::to_string(u));
    };
    for (const auto& [key, v0] : need) {
      const auto [var, r, u] = key;
      src << "          const T " << uname(var, r, u) << " = cb" << plus(v0) << " <= c1hi ? v" << var << "["
          << rb(var, r) << " + cb" << plus(u - C.vmin[var][1]) << "] : T(0);\n";
    }
    for (int v = 0; v < V; ++v) {
      src << "          { const int c1 = cb" << plus(v) << ";\n";
      src << "            const int x1 = o1 + c1;\n";
      src << "            if (c1 <= c1hi) {\n";
      for (size_t li = 0; li < g.loads.size(); ++li) {
        const Load& in = g.loads[li];
        if (win[in.var] > 0) {
          src << "            const T l" << li << " = " << uname(in.var, in.rel[0], v + in.rel[1]) << ";\n";
        } else {
          const int ti = C.terminal_of(in.var, false);
          std::string r;
          if (C.P.terminals[ti].dims.empty()) {
            r = "s" + std::to_string(ti);
          } else {
            std::vector<std::string> pos;
            for (int d = 0; d < nd; ++d)
              pos.push_back((d == 0 ? std::string("y") : "x" + std::to_string(d)) + plus(in.rel[d]));
            r = "__ldg(t" + std::to_string(ti) + " + " + C.tidx(ti, pos, C.extra_of(in.var)) + ")";
          }
          src << "            const T l" << li << " = " << r << ";\n";
        }
      }
      if (!emit_eval("            ")) return false;
      src << "            }\n          }\n";
    }
    src << "        }\n      }\n    }\n";
    return true;
  }
  // phase 1: every operand of the K cells this thread owns (independent loads)
  // in batches of ILP cells (bounded register footprint)
  const int B = std::min(K, ILP);
  src << "        #pragma unroll\n";
  src << "        for (int kb = 0; kb < " << K << "; kb += " << B << ") {\n";
  for (size_t li = 0; li < g.loads.size(); ++li) src << "        T a_l" << li << "[" << B << "];\n";
  src << "        #pragma unroll\n";
  src << "        for (int kk = 0; kk < " << B << "; ++kk) {\n";
  src << "          const int k = kb + kk;\n";
  src << "          const int c1 = " << LANE << plus(lo[1]) << " + k * " << STEP << ";\n";
  src << "          const int x1 = o1 + c1;\n";
  src << "          if (act && c1 <= c1hi) {\n";
  std::vector<std::string> reads(g.loads.size());
  bool any_rot = false;
  for (size_t li = 0; li < g.loads.size(); ++li) {
    const Load& in = g.loads[li];
    std::string r;
    if (win[in.var] > 0) {
      r = "v" + std::to_string(in.var) + "[" + rb(in.var, in.rel[0]) + " + " + inplane(in.var, in.rel) + "]";
    } else {
      const int ti = C.terminal_of(in.var, false);
      if (C.P.terminals[ti].dims.empty()) {
        r = "s" + std::to_string(ti);
      } else {
        std::vector<std::string> pos;
        for (int d = 0; d < nd; ++d) pos.push_back((d == 0 ? std::string("y") : "x" + std::to_string(d)) + plus(in.rel[d]));
        r = "__ldg(t" + std::to_string(ti) + " + " + C.tidx(ti, pos, C.extra_of(in.var)) + ")";
      }
    }
    reads[li] = r;
    any_rot |= rot[gi].from[li] >= 0;
  }
  if (any_rot) {
    // the branch is uniform: the first trip of a segment loads every row
    src << "            if (first) {\n";
    for (size_t li = 0; li < g.loads.size(); ++li) src << "              a_l" << li << "[kk] = " << reads[li] << ";\n";
    src << "            } else {\n";
    for (size_t li = 0; li < g.loads.size(); ++li)
      src << "              a_l" << li << "[kk] = "
          << (rot[gi].from[li] >= 0 ? "rw" + std::to_string(gi) + "_" + std::to_string(rot[gi].from[li]) + "[k]" : reads[li])
          << ";\n";
    src << "            }\n";
  } else {
    for (size_t li = 0; li < g.loads.size(); ++li) src << "            a_l" << li << "[kk] = " << reads[li] << ";\n";
  }
  for (size_t lj = 0; lj < g.loads.size(); ++lj)
    if (rot[gi].keep[lj]) src << "            rw" << gi << "_" << lj << "[k] = a_l" << lj << "[kk];\n";
  src << "          }\n        }\n";
  // phase 2: evaluate and store
  src << "        #pragma unroll\n";
  src << "        for (int kk = 0; kk < " << B << "; ++kk) {\n";
  src << "          const int k = kb + kk;\n";
  src << "          const int c1 = " << LANE << plus(lo[1]) << " + k * " << STEP << ";\n";
  src << "          const int x1 = o1 + c1;\n";
  src << "          if (act && c1 <= c1hi) {\n";
  for (size_t li = 0; li < g.loads.size(); ++li) src << "            const T l" << li << " = a_l" << li << "[kk];\n";
  if (!emit_eval("            ")) return false;
  src << "          }\n        }\n        }\n      }\n    }\n";
  return true;
}

void March::tail() {
  if (ws) {
    // this warp is done with the trip's window rows
    src << "    __syncwarp();\n";
    src << "    if ((threadIdx.x & 31) == 0) lf_mbar_arrive(&lf_empty[stg]);\n";
    src << "    }\n";
  }
  for (size_t v = 0; v < nv; ++v)
    if (win[v] > 1) src << "    b" << v << " = b" << v << " == " << (win[v] - 1) << " ? 0 : b" << v << " + 1;\n";
  src << "  }\n";
  if (!ws) {
    src << "  asm volatile(\"cp.async.wait_group 0;\" ::: \"memory\");\n";
    src << "  __syncthreads();\n";
  }
  src << "  }\n";
  src << "}\n";
}

void March::capture() {
  if (ws) {
    if (!ips.empty() && nd == 3) commit3();
    return;
  }
  // ---- in-place: capture the bands other units read before this step writes
  if (!ips.empty()) {
    std::vector<std::pair<size_t, int>> caps;  // (variable, terminal)
    for (const auto& ip : ips) caps.push_back({ip.v, ip.ai});
    std::vector<int> slots;
    for (const auto& ip : ips) slots.push_back(ip.slot);
    emit_capture(C, "lf_jit_capture", caps, slots, tile, src);
  }
}

// In place, 3D warp-specialised march: which of this thread's cells fall in a
// tile-row or tile-column zone is fixed for the unit -- a bit per row k of the
// cells it owns (rz) and one flag for its column (cz) per in-place goal
// output, so the march tests two bits per store and takes the full routing
// only for the few cells in a zone
void March::inplace_masks() {
  src << "  // in place: where this thread's cells go when they lie in a tile-row /\n"
         "  // tile-column band (fixed for the unit): offsets into the bands less the\n"
         "  // plane term, rz / cz the rows k / the column that do\n";
  for (size_t gi = 0; gi < G.size(); ++gi) {
    const Grp& g = G[gi];
    for (const auto& o : g.out) {
      const int ti = C.terminal_of(o.var, true);
      const IP* gip = nullptr;
      for (const auto& ip : ips)
        if (ip.gi == ti) gip = &ip;
      if (ti < 0 || !gip) continue;
      const auto& t = C.P.terminals[ti];
      const size_t v = gip->v;
      const long so0 = -t.base[0] + C.LO[0], so1 = -t.base[1] + C.LO[1], so2 = -t.base[2] + C.LO[2], SE = 32 / eb;
      const long lo1 = saved_vmin[v][1], hi1 = C.vmax[v][1], lo2 = saved_vmin[v][2], hi2 = C.vmax[v][2];
      const long E0 = t.extent[0], E1 = t.extent[1], E2 = t.extent[2];
      const long BW1 = hi1 - lo1, BW2 = hi2 - lo2 + 2 * (SE - 1);
      const int K = (tile[1] + (g.gmax[1] - g.gmin[1]) + STEP - 1) / STEP;
      auto zs = [&](const std::string& e) {
        return "(((" + e + plus(lo2 + so2) + ") & ~" + std::to_string(SE - 1) + ")" + plus(-so2) + ")";
      };
      auto ze = [&](const std::string& e) {
        return "(((" + e + plus(hi2 + so2 + SE - 1) + ") & ~" + std::to_string(SE - 1) + ")" + plus(-so2) + ")";
      };
      const std::string nm = std::to_string(gi) + "_" + o.param;
      src << "  unsigned rz" << nm << " = 0;\n  bool cz" << nm << " = false;\n";
      src << "  long long rbo" << nm << "[" << K << "], cbo" << nm << " = 0;\n";
      src << "  {\n";
      src << "    const int xx2 = o2 + tx" << plus(g.gmin[2] + o.rel[2]) << ";\n";
      src << "    #pragma unroll\n";
      src << "    for (int k = 0; k < " << K << "; ++k) {\n";
      src << "      const int xx1 = o1 + " << LANE << plus(g.gmin[1] + o.rel[1]) << " + k * " << STEP << ";\n";
      src << "      int e1 = -1;\n";
      src << "      if (o1 > 0 && xx1 < o1" << plus(hi1) << ") e1 = o1;\n";
      src << "      else if (o1 + " << tile[1] << " < N1 && xx1 >= o1 + " << tile[1] << plus(lo1) << ") e1 = o1 + " << tile[1] << ";\n";
      src << "      if (a.inplace && e1 >= 0) rz" << nm << " |= 1u << k;\n";
      src << "      rbo" << nm << "[k] = e1 < 0 ? 0 : (((long long)(e1 / " << tile[1] << " - 1) * " << BW1 << " + (xx1 - e1" << plus(-lo1)
          << ")) * " << E0 << plus(so0) << ") * " << E2 << "LL + (xx2" << plus(so2) << ");\n";
      src << "    }\n";
      src << "    int e2 = -1;\n";
      src << "    if (o2 > 0 && xx2 < " << ze("o2") << ") e2 = o2;\n";
      src << "    else if (o2 + " << tile[2] << " < N2 && xx2 >= " << zs("o2 + " + std::to_string(tile[2])) << ") e2 = o2 + " << tile[2]
          << ";\n";
      src << "    cz" << nm << " = a.inplace && e2 >= 0;\n";
      src << "    cbo" << nm << " = e2 < 0 ? 0 : ((long long)(e2 / " << tile[2] << " - 1) * " << E0 << plus(so0) << ") * " << E1 * BW2
          << "LL + " << so1 * BW2 << "LL + (xx2 - " << zs("e2") << ");\n";
      src << "  }\n";
    }
  }
}

// In place, 3D warp-specialised march: after the step, copy the deferred
// boundary writes into the grid -- plane bands (planes around internal chunk
// boundaries), row bands (tile rows around internal tile-row boundaries,
// outside the plane bands), column bands (sector-aligned tile columns around
// internal tile-column boundaries, outside both, [boundary][plane][row][col])
// -- flat over their cells, four per thread, contiguous on both sides
void March::commit3() {
  src << "extern \"C\" __global__ void __launch_bounds__(256) lf_jit_commit_ws(const LfArgs a) {\n";
  src << "  const int N0 = (int)a.n0;\n";
  src << "  const int nch = (N0 + a.chunk - 1) / a.chunk;\n";
  for (const auto& ip : ips) {
    const auto& t = C.P.terminals[ip.gi];
    const size_t v = ip.v;
    const long so0 = -t.base[0] + C.LO[0], so1 = -t.base[1] + C.LO[1], so2 = -t.base[2] + C.LO[2];
    const long lo0 = saved_vmin[v][0], hi0 = C.vmax[v][0], lo1 = saved_vmin[v][1], hi1 = C.vmax[v][1];
    const long lo2 = saved_vmin[v][2], hi2 = C.vmax[v][2], SE = 32 / eb;
    const long E0 = t.extent[0], E1 = t.extent[1], E2 = t.extent[2];
    const long BH = hi0 - lo0, BW1 = hi1 - lo1, BW2 = hi2 - lo2 + 2 * (SE - 1);
    const long N1 = C.N[1], N2 = C.N[2];
    const long NT1 = (N1 + tile[1] - 1) / tile[1], NT2 = (N2 + tile[2] - 1) / tile[2];
    auto zs = [&](const std::string& e) {
      return "(((" + e + plus(lo2 + so2) + ") & ~" + std::to_string(SE - 1) + ")" + plus(-so2) + ")";
    };
    auto ze = [&](const std::string& e) {
      return "(((" + e + plus(hi2 + so2 + SE - 1) + ") & ~" + std::to_string(SE - 1) + ")" + plus(-so2) + ")";
    };
    src << "  {\n";
    src << "    T* m = reinterpret_cast<T*>(a.t[" << ip.gi << "]);\n";
    src << "    const T* pb = reinterpret_cast<const T*>(a.t[" << ip.slot << "]);\n";
    src << "    const T* b1 = reinterpret_cast<const T*>(a.t[" << ip.slot + 1 << "]);\n";
    src << "    const T* b2 = reinterpret_cast<const T*>(a.t[" << ip.slot + 2 << "]);\n";
    src << "    const long long np = (long long)max(0, nch - 1) * " << BH * N1 * N2 << "LL;\n";
    src << "    const long long n1 = (long long)N0 * " << (NT1 - 1) * BW1 * N2 << "LL;\n";
    src << "    const long long n2 = (long long)N0 * " << (NT2 - 1) * BW2 * N1 << "LL;\n";
    src << "    #pragma unroll\n";
    src << "    for (int j = 0; j < 4; ++j) {\n";
    src << "      long long p = (long long)blockIdx.x * 1024 + j * 256 + threadIdx.x;\n";
    src << "      if (p < np) {\n";
    src << "        const long long r = p / " << N1 * N2 << "LL, q = p - r * " << N1 * N2 << "LL;\n";
    src << "        const int x1 = (int)(q / " << N2 << "), x2 = (int)(q % " << N2 << ");\n";
    src << "        const int y = (int)(r / " << BH << " + 1) * a.chunk" << plus(lo0) << " + (int)(r % " << BH << ");\n";
    src << "        if (y >= 0 && y < N0) m[((long long)(y" << plus(so0) << ") * " << E1 << " + (x1" << plus(so1) << ")) * " << E2
        << "LL + (x2" << plus(so2) << ")] = pb[(r * " << E1 << " + (x1" << plus(so1) << ")) * " << E2 << "LL + (x2" << plus(so2) << ")];\n";
    src << "        continue;\n";
    src << "      }\n";
    src << "      p -= np;\n";
    src << "      if (p < n1) {\n";
    src << "        const long long kr = p / ((long long)N0 * " << N2 << "), q = p - kr * ((long long)N0 * " << N2 << ");\n";
    src << "        const int y = (int)(q / " << N2 << "), x2 = (int)(q % " << N2 << ");\n";
    src << "        const int x1 = (int)(kr / " << BW1 << " + 1) * " << tile[1] << plus(lo1) << " + (int)(kr % " << BW1 << ");\n";
    src << "        const int bb = (y" << plus(-lo0) << ") / a.chunk * a.chunk;\n";
    src << "        if (bb > 0 && bb < N0 && y < bb" << plus(hi0) << ") continue;  // with the plane bands\n";
    src << "        if (x1 >= 0 && x1 < " << N1 << ") m[((long long)(y" << plus(so0) << ") * " << E1 << " + (x1" << plus(so1) << ")) * " << E2
        << "LL + (x2" << plus(so2) << ")] = b1[(kr * " << E0 << " + (y" << plus(so0) << ")) * " << E2 << "LL + (x2" << plus(so2) << ")];\n";
    src << "        continue;\n";
    src << "      }\n";
    src << "      p -= n1;\n";
    src << "      if (p < n2) {\n";
    // column bands [boundary][plane][row][column]: a band row is one or two
    // whole 32-B sectors of the grid row, read and written contiguously
    src << "        const int c = (int)(p % " << BW2 << ");\n";
    src << "        const long long rr = p / " << BW2 << ";\n";
    src << "        const int x1 = (int)(rr % " << N1 << "), y = (int)((rr / " << N1 << ") % N0);\n";
    src << "        const int k = (int)(rr / ((long long)N0 * " << N1 << "));\n";
    src << "        const int e2 = (k + 1) * " << tile[2] << ", x2 = " << zs("e2") << " + c;\n";
    src << "        const int bb = (y" << plus(-lo0) << ") / a.chunk * a.chunk;\n";
    src << "        if (bb > 0 && bb < N0 && y < bb" << plus(hi0) << ") continue;  // with the plane bands\n";
    src << "        const int b1_ = (x1" << plus(-lo1) << ") / " << tile[1] << " * " << tile[1] << ";\n";
    src << "        if (b1_ > 0 && b1_ < " << N1 << " && x1 < b1_" << plus(hi1) << ") continue;  // with the row bands\n";
    src << "        if (x2 >= 0 && x2 < " << N2 << " && x2 < " << ze("e2") << ") m[((long long)(y" << plus(so0) << ") * " << E1 << " + (x1"
        << plus(so1) << ")) * " << E2 << "LL + (x2" << plus(so2) << ")] = b2[(((long long)k * " << E0 << " + (y" << plus(so0) << ")) * "
        << E1 << " + (x1" << plus(so1) << ")) * " << BW2 << "LL + c];\n";
    src << "      }\n";
    src << "    }\n  }\n";
  }
  src << "}\n";
}
}  // namespace

bool emit_march(Ctx& C, JitProgram& out, std::ostream& src, bool ws = false) {
  March m(C, out, src, ws);
  return m.emit();
}

// ---------------------------------------------------------------------------
// 1D: one CTA per tile, every group over tile + halo in shared memory
// ---------------------------------------------------------------------------
bool emit_tiled(Ctx& C, JitProgram& out, std::ostream& src) {
  const int NT = 256;
  const int eb = out.elem_bytes;
  const size_t nv = C.P.vars.size();
  const int tile = 1024;
  std::vector<size_t> soff(nv, 0);
  size_t smem = 0;
  for (size_t v = 0; v < nv; ++v) {
    if (!C.smem_var[v]) continue;
    soff[v] = smem;
    smem += ((tile + C.vmax[v][0] - C.vmin[v][0]) * eb + 15) / 16 * 16;
  }
  if (smem > 200 * 1024) return (C.error = "chain needs too much on-chip storage for one tile", false);
  out.tile = {tile};
  out.smem_bytes = smem;
  out.threads = NT;
  out.march = false;
  out.inplace.clear();
  out.inplace_error = C.P.rs.aliases.empty() ? "" : "in-place runs need a 2D/3D chain (the 1D path reads axioms in place)";
  emit_prelude(C, src, NT, 1, nullptr);
  src << "  const long long o0 = (long long)a.row_lo + (long long)blockIdx.x * " << tile << ";\n";
  for (size_t v = 0; v < nv; ++v)
    if (C.smem_var[v]) src << "  T* __restrict__ v" << v << " = reinterpret_cast<T*>(lf_smem + " << soff[v] << ");\n";
  for (size_t gi = 0; gi < C.groups.size(); ++gi) {
    const Grp& g = C.groups[gi];
    const long cells = tile + g.gmax[0] - g.gmin[0];
    src << "  for (int idx = threadIdx.x; idx < " << cells << "; idx += " << NT << ") {\n";
    src << "    const int c0 = idx" << plus(g.gmin[0]) << ";\n";
    src << "    const long long x0 = o0 + c0;\n";
    src << "    if (x0 < " << g.gmin[0] << " || x0 > N0 - 1" << plus(g.gmax[0]) << ") continue;\n";
    for (const auto& in : g.in) {
      std::string r;
      if (C.smem_var[in.var]) {
        r = "v" + std::to_string(in.var) + "[c0" + plus(in.rel[0] - C.vmin[in.var][0]) + "]";
      } else {
        const int ti = C.terminal_of(in.var, false);
        r = C.P.terminals[ti].dims.empty()
                ? "s" + std::to_string(ti)
                : "t" + std::to_string(ti) + "[" + C.tidx(ti, {"x0" + plus(in.rel[0])}, C.extra_of(in.var)) + "]";
      }
      src << "    const T p_" << in.param << " = " << r << ";\n";
    }
    if (!emit_bodies(C, g, src, "    ")) return false;
    for (const auto& o : g.out) {
      if (C.smem_var[o.var])
        src << "    v" << o.var << "[c0" << plus(o.rel[0] - C.vmin[o.var][0]) << "] = q_" << o.param << ";\n";
      const int ti = C.terminal_of(o.var, true);
      if (ti >= 0)
        src << "    if (c0" << plus(o.rel[0]) << " >= 0 && c0" << plus(o.rel[0]) << " < " << tile << " && x0"
            << plus(o.rel[0]) << " < a.row_hi) t" << ti << "[" << C.tidx(ti, {"x0" + plus(o.rel[0])}, {0}) << "] = q_"
            << o.param << ";\n";
    }
    src << "  }\n";
    if (gi + 1 < C.groups.size()) src << "  __syncthreads();\n";
  }
  src << "}\n";
  return true;
}

// ---------------------------------------------------------------------------
// ghost refill of iterated goals (boundary modes), ghost cells only: region d
// holds the cells whose outermost ghost dimension is d (dims < d interior)
// ---------------------------------------------------------------------------
bool emit_fill(Ctx& C, JitProgram& out, std::ostream& fill) {
  const auto& rs = C.P.rs;
  const auto& terms = C.P.terminals;
  const int nd = C.nd;
  out.has_fill = false;
  // the body as a device function: lf_jit_fill runs it alone, the in-place
  // register march's commit kernel may run it after its own work
  fill << "__device__ __forceinline__ void lf_fill_body(const LfArgs& a) {\n";
  fill << "  const long long N0 = a.n0;\n";
  for (const auto& [gname, aname] : rs.iterate) {
    int ti = -1;
    for (size_t i = 0; i < terms.size(); ++i)
      if (terms[i].is_goal && terms[i].name == gname) ti = static_cast<int>(i);
    if (ti < 0 || terms[ti].dims.empty()) continue;
    const auto& t = terms[ti];
    if ((int)t.dims.size() != nd)
      return (C.error = "iterated terminal '" + gname + "' must span every loop dimension", false);
    auto it = rs.boundary.find(t.name);
    if (it == rs.boundary.end()) it = rs.boundary.find("*");
    std::vector<lf::Boundary> modes(nd, lf::Boundary::none);
    if (it != rs.boundary.end())
      for (int d = 0; d < nd; ++d) modes[d] = it->second[std::min<size_t>(d, it->second.size() - 1)];
    bool any = false;
    for (auto m : modes) any |= m != lf::Boundary::none;
    if (!any) continue;
    out.has_fill = true;
    std::vector<long> lo(nd), hi(nd), E(nd);  // ghost widths below / above the interior, extents
    for (int d = 0; d < nd; ++d) {
      lo[d] = C.LO[d] - t.base[d];
      E[d] = t.extent[d];
      hi[d] = E[d] - C.N[d] - lo[d];
    }
    auto nn = [&](int d) { return d == 0 ? std::string("N0") : std::to_string(C.N[d]); };
    fill << "  {\n    T* b = reinterpret_cast<T*>(a.t[" << ti << "]);\n";
    // region sizes
    fill << "    long long rs[" << nd << "];\n";
    for (int d = 0; d < nd; ++d) {
      fill << "    rs[" << d << "] = ";
      if (d == 0)
        fill << "(long long)((a.top ? " << lo[0] << " : 0) + (a.bottom ? " << hi[0] << " : 0))";
      else
        fill << "(long long)(a.row_hi - a.row_lo)";
      for (int k = 1; k < d; ++k) fill << " * " << C.N[k];
      if (d > 0) fill << " * " << (lo[d] + hi[d]);
      for (int k = d + 1; k < nd; ++k) fill << " * " << E[k];
      fill << ";\n";
    }
    fill << "    long long total = 0; for (int r = 0; r < " << nd << "; ++r) total += rs[r];\n";
    fill << "    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total; idx += (long long)gridDim.x * blockDim.x) {\n";
    fill << "      long long rem = idx; int reg = 0;\n";
    fill << "      while (rem >= rs[reg]) rem -= rs[reg++];\n";
    for (int d = 0; d < nd; ++d) fill << "      long long y" << d << ";\n";
    for (int d = 0; d < nd; ++d) {
      fill << "      " << (d ? "else " : "") << "if (reg == " << d << ") {\n";
      // dims > d: anything in the extent (innermost fastest)
      for (int k = nd - 1; k > d; --k)
        fill << "        y" << k << " = rem % " << E[k] << " - " << lo[k] << "; rem /= " << E[k] << ";\n";
      if (d == 0) {
        fill << "        { const long long g = rem; const long long nt = a.top ? " << lo[0] << " : 0;\n";
        fill << "          y0 = g < nt ? g - " << lo[0] << " : N0 + (g - nt); }\n";
      } else {
        fill << "        { const long long g = rem % " << (lo[d] + hi[d]) << "; rem /= " << (lo[d] + hi[d]) << ";\n";
        fill << "          y" << d << " = g < " << lo[d] << " ? g - " << lo[d] << " : " << C.N[d] << " + (g - " << lo[d] << "); }\n";
        for (int k = d - 1; k >= 1; --k) fill << "        y" << k << " = rem % " << C.N[k] << "; rem /= " << C.N[k] << ";\n";
        fill << "        y0 = a.row_lo + rem;\n";
      }
      fill << "      }\n";
    }
    fill << "      bool zero = false; T sign = static_cast<T>(1);\n";
    for (int d = 0; d < nd; ++d) {
      const std::string y = "y" + std::to_string(d), n = nn(d);
      fill << "      long long z" << d << " = " << y << ";\n";
      fill << "      if (" << y << " < 0 || " << y << " >= " << n << ") {\n";
      switch (modes[d]) {
        case lf::Boundary::zero: fill << "        zero = true;\n"; break;
        case lf::Boundary::periodic: fill << "        z" << d << " = ((" << y << " % " << n << ") + " << n << ") % " << n << ";\n"; break;
        case lf::Boundary::clamp: fill << "        z" << d << " = " << y << " < 0 ? 0 : " << n << " - 1;\n"; break;
        case lf::Boundary::even:
        case lf::Boundary::odd:
          fill << "        z" << d << " = " << y << " < 0 ? -1 - " << y << " : 2 * " << n << " - 1 - " << y << ";\n";
          if (modes[d] == lf::Boundary::odd) fill << "        sign = -sign;\n";
          break;
        case lf::Boundary::none: fill << "        continue;\n"; break;
      }
      fill << "      }\n";
    }
    std::string dst, srci;
    for (int s = 0; s < nd; ++s) {
      const long p = C.pitch(t, s);
      const std::string ps = p != 1 ? " * " + std::to_string(p) + "LL" : "";
      dst += (s ? " + " : "") + std::string("(y") + std::to_string(s) + plus(C.LO[s] - t.base[s]) + ")" + ps;
      srci += (s ? " + " : "") + std::string("(z") + std::to_string(s) + plus(C.LO[s] - t.base[s]) + ")" + ps;
    }
    fill << "      b[" << dst << "] = zero ? static_cast<T>(0) : sign * b[" << srci << "];\n";
    fill << "    }\n  }\n";
  }
  fill << "}\n";
  fill << "extern \"C\" __global__ void lf_jit_fill(const LfArgs a) {\n  lf_fill_body(a);\n}\n";
  return true;
}

// ---------------------------------------------------------------------------
// Multi-nest plans (reductions / broadcast splits, fusion.cpp:8-95; the
// paper's section 3.4): one kernel per fused nest, in nest dataflow order.
// Terms produced in one nest and read in another are materialised in
// plan-owned buffers with the variable's buffer extents (storage.cpp:403-427);
// everything else is recomputed per cell from the reference DAG's rule
// applications.  A nest holding associative kernels is a reduction nest:
// one warp per cell of its parallel dims, the reduced dims marched in loop
// order 32 elements at a time -- lanes evaluate the elements, then the
// accumulation runs in element order, so the result equals run_naive's
// sequential sweep bit for bit (no reassociation needed).
// ---------------------------------------------------------------------------
bool emit_nests(const lf::Plan& P, const std::string& sources, JitProgram& out, std::ostream& src, std::string& err) {
  const auto& rs = P.rs;
  const auto& g = P.dag;
  const int nd = static_cast<int>(rs.loop_order.size());
  auto fail = [&](const std::string& m) {
    err = m;
    return false;
  };
  if (nd < 1 || nd > 3) return fail("generic executor handles 1-3 loop dimensions");
  for (const auto& r : rs.ranges)
    if (r.stride != 1) return fail("generic executor needs unit strides");
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
  }
  out.type = T;
  out.elem_bytes = T == "double" ? 8 : 4;
  out.nd = nd;
  std::vector<long> N(nd), LO(nd);
  for (int d = 0; d < nd; ++d) {
    N[d] = rs.ranges[d].trips();
    LO[d] = rs.ranges[d].lo;
  }
  const int nr = static_cast<int>(g.raps.size());
  auto nest_of = [&](int r) { return P.vertex_of_group[P.group_of[r]]; };
  auto term_axes = [&](int t) {
    std::set<int> a;
    for (const auto& o : g.terms[t].dims) a.insert(o.dim);
    return a;
  };
  auto term_off = [&](int t, int d) {
    for (const auto& o : g.terms[t].dims)
      if (o.dim == d) return o.offset;
    return 0;
  };
  for (int r = 0; r < nr; ++r)
    if (g.raps[r].kind == lf::RapKind::kernel) {
      std::string why;
      if (!kernel_evaluable(rs.kernels[g.raps[r].kernel], sources, why)) return fail(why);
    }
  // ---- nests in dataflow order (kernel and store raps; loads go where read)
  std::set<int> nest_ids;
  for (int r = 0; r < nr; ++r)
    if (g.raps[r].kind != lf::RapKind::load) nest_ids.insert(nest_of(r));
  std::map<int, std::set<int>> nadj;
  std::map<int, int> nindeg;
  for (int v : nest_ids) nindeg[v] = 0;
  for (const auto& e : g.edges) {
    if (g.raps[e.from].kind == lf::RapKind::load) continue;
    const int a = nest_of(e.from), b = nest_of(e.to);
    if (a != b && nadj[a].insert(b).second) ++nindeg[b];
  }
  std::vector<int> norder;
  {
    std::deque<int> q;
    for (int v : nest_ids)
      if (!nindeg[v]) q.push_back(v);
    while (!q.empty()) {
      int v = q.front();
      q.pop_front();
      norder.push_back(v);
      for (int w : nadj[v])
        if (--nindeg[w] == 0) q.push_back(w);
    }
    if (norder.size() != nest_ids.size()) return fail("cyclic nest dataflow");
  }
  const std::vector<int> topo = g.topo_order();
  // ---- materialised terms: kernel outputs read by a rap of another nest
  std::map<int, int> mat_of_var;  // var -> materialised buffer index
  std::vector<int> mat_vars;
  std::vector<char> term_mat(g.terms.size(), 0);
  for (const auto& e : g.edges) {
    const auto& from = g.raps[e.from];
    if (from.kind != lf::RapKind::kernel) continue;
    if (nest_of(e.from) == nest_of(e.to)) continue;
    term_mat[e.term] = 1;
    const int v = P.var_of_term[e.term];
    if (!mat_of_var.count(v)) {
      mat_of_var[v] = static_cast<int>(mat_vars.size());
      mat_vars.push_back(v);
    }
  }
  const int nterm = static_cast<int>(P.terminals.size());
  if (nterm + (int)mat_vars.size() > 32) return fail("more than 32 terminal and materialised buffers");
  out.mat_bytes.clear();
  for (int v : mat_vars) {
    size_t n = out.elem_bytes;
    for (const auto& [ext, base] : P.vars[v].extents) n *= static_cast<size_t>(ext);
    out.mat_bytes.push_back(n);
  }
  auto terminal_of = [&](const std::string& name, bool goal) {
    for (size_t i = 0; i < P.terminals.size(); ++i)
      if (P.terminals[i].name == name && P.terminals[i].is_goal == goal) return static_cast<int>(i);
    return -1;
  };
  auto pitch = [&](const std::vector<long>& ext, size_t slot) {
    long p = 1;
    for (size_t k = slot + 1; k < ext.size(); ++k) p *= ext[k];
    return p;
  };
  // index of terminal `ti` for a load / store rap (slot coordinate = x + shift - base)
  auto slot_index = [&](int ti, const std::vector<lf::ExtSlot>& slots) {
    const auto& t = P.terminals[ti];
    std::string e;
    for (size_t s = 0; s < slots.size(); ++s) {
      const long c0 = slots[s].shift - t.base[s] + (slots[s].dim >= 0 ? LO[slots[s].dim] : 0);
      std::string c = slots[s].dim >= 0 ? "(long long)(x" + std::to_string(slots[s].dim) + plus(c0) + ")"
                                        : std::to_string(c0) + "LL";
      const long p = pitch(t.extent, s);
      e += (e.empty() ? "" : " + ") + c + (p != 1 ? " * " + std::to_string(p) + "LL" : "");
    }
    return e.empty() ? std::string("0") : e;
  };
  // index of materialised var buffer for term t at the current cell
  auto mat_index = [&](int t) {
    const int v = P.var_of_term[t];
    const auto& var = P.vars[v];
    std::vector<long> ext;
    for (const auto& [e, b] : var.extents) ext.push_back(e);
    std::string e;
    for (size_t s = 0; s < var.dims.size(); ++s) {
      const int d = var.dims[s];
      const long c0 = term_off(t, d) + LO[d] - var.extents[s].second;
      const std::string c = "(long long)(x" + std::to_string(d) + plus(c0) + ")";
      const long p = pitch(ext, s);
      e += (e.empty() ? "" : " + ") + c + (p != 1 ? " * " + std::to_string(p) + "LL" : "");
    }
    return "m" + std::to_string(mat_of_var.at(v)) + "[" + (e.empty() ? std::string("0") : e) + "]";
  };

  src << "// generated by loomfuse-b200 (csrc/jit/codegen.cpp, multi-nest) for chain '" << rs.name << "'\n";
  src << "typedef " << T << " T;\n";
  src << "__device__ __forceinline__ T lf_min(T a, T b) { return a < b ? a : b; }\n";
  src << "__device__ __forceinline__ T lf_max(T a, T b) { return a > b ? a : b; }\n";
  src << "struct LfArgs { void* t[32]; long long n0; int row_lo, row_hi, top, bottom, chunk, inplace; };\n";
  auto pointers = [&](std::ostream& o) {
    for (int i = 0; i < nterm; ++i) {
      const auto& t = P.terminals[i];
      if (t.dims.empty())
        o << "  const T s" << i << " = *reinterpret_cast<const T*>(a.t[" << i << "]);\n";
      else
        o << "  " << (t.is_goal ? "T" : "const T") << "* __restrict__ t" << i << " = reinterpret_cast<"
          << (t.is_goal ? "T" : "const T") << "*>(a.t[" << i << "]);\n";
    }
    for (size_t m = 0; m < mat_vars.size(); ++m)
      o << "  T* __restrict__ m" << m << " = reinterpret_cast<T*>(a.t[" << (nterm + m) << "]);  // '"
        << P.vars[mat_vars[m]].name << "'\n";
  };
  // value expression of an input term of a rap in nest `nv` (computed locally or loaded)
  std::vector<char> done;  // per term: already defined in the current scope
  // `guard`: condition on the stores (terminal and materialised) of this rap
  auto emit_rap = [&](int r, int nv, std::ostream& o, const std::string& ind, bool& okk, const std::string& guard) {
    const std::string G = guard.empty() ? std::string() : "if (" + guard + ") ";
    const auto& rap = g.raps[r];
    auto need = [&](int t) {
      if (done[t]) return;
      const int pr = g.producer[t];
      if (pr >= 0 && g.raps[pr].kind == lf::RapKind::kernel && nest_of(pr) != nv) {
        o << ind << "const T v" << t << " = " << mat_index(t) << ";\n";
        done[t] = 1;
      }
    };
    if (rap.kind == lf::RapKind::load) {
      const int ti = terminal_of(rap.external, false);
      if (ti < 0) {
        okk = false;
        err = "axiom '" + rap.external + "' not found";
        return;
      }
      const int t = rap.out_terms[0];
      if (P.terminals[ti].dims.empty() && rap.ext_slots.empty())
        o << ind << "const T v" << t << " = s" << ti << ";\n";
      else
        // axioms are read-only on the multi-nest path (no in-place runs here): the
        // non-coherent load lets the compiler hoist the loads of an unrolled element
        // loop above the materialising stores between them
        o << ind << "const T v" << t << " = __ldg(&t" << ti << "[" << slot_index(ti, rap.ext_slots) << "]);\n";
      done[t] = 1;
    } else if (rap.kind == lf::RapKind::store) {
      const int ti = terminal_of(rap.external, true);
      if (ti < 0) {
        okk = false;
        err = "goal '" + rap.external + "' not found";
        return;
      }
      need(rap.in_terms[0]);
      o << ind << G << "t" << ti << "[" << slot_index(ti, rap.ext_slots) << "] = v" << rap.in_terms[0] << ";\n";
    } else {
      const auto& k = rs.kernels[rap.kernel];
      for (int t : rap.in_terms) need(t);
      std::map<std::string, std::string> pv, ov;
      for (size_t j = 0; j < k.inputs.size(); ++j) pv[k.inputs[j].first] = "v" + std::to_string(rap.in_terms[j]);
      for (size_t j = 0; j < k.outputs.size(); ++j) ov[k.outputs[j].first] = "v" + std::to_string(rap.out_terms[j]);
      if (!emit_kernel(
              k, T, [&](const std::string& n) { return pv.at(n); }, [&](const std::string& n) { return ov.at(n); },
              true, o, ind, err)) {
        okk = false;
        return;
      }
      for (int t : rap.out_terms) {
        done[t] = 1;
        if (term_mat[t]) o << ind << G << mat_index(t) << " = v" << t << ";\n";
      }
    }
  };
  out.nest_kernels.clear();
  int kid = 0;
  for (int nv : norder) {
    // raps of this nest (kernels, stores) plus the loads they read
    std::vector<char> in_nest(nr, 0);
    for (int r = 0; r < nr; ++r)
      if (g.raps[r].kind != lf::RapKind::load && nest_of(r) == nv) in_nest[r] = 1;
    for (int r = 0; r < nr; ++r)
      if (in_nest[r])
        for (int t : g.raps[r].in_terms) {
          const int pr = g.producer[t];
          if (pr >= 0 && g.raps[pr].kind == lf::RapKind::load) in_nest[pr] = 1;
        }
    std::set<int> space;
    for (int r = 0; r < nr; ++r)
      if (in_nest[r] && g.raps[r].kind != lf::RapKind::load)
        for (int d : P.groups[P.group_of[r]].space) space.insert(d);
    // reductions
    std::vector<int> reds;
    std::set<int> R;
    for (int r = 0; r < nr; ++r)
      if (in_nest[r] && g.raps[r].kind == lf::RapKind::kernel && rs.kernels[g.raps[r].kernel].associative) {
        std::set<int> rd;
        const auto oax = term_axes(g.raps[r].out_terms[0]);
        for (int d : P.groups[P.group_of[r]].space)
          if (!oax.count(d)) rd.insert(d);
        if (rd.empty()) return fail("associative kernel '" + rs.kernels[g.raps[r].kernel].name + "' reduces nothing");
        if (!reds.empty() && rd != R) return fail("reductions over different dimensions in one nest");
        R = rd;
        reds.push_back(r);
      }
    const std::string fn = "lf_nest" + std::to_string(kid++);
    done.assign(g.terms.size(), 0);
    bool okk = true;
    std::ostringstream body;
    NestLaunch nl;
    nl.fn = fn;
    if (reds.empty()) {
      // ---- cell-parallel nest
      long long cells = 1;
      for (int d : space) cells *= N[d];
      nl.reduction = false;
      nl.units = cells;
      src << "extern \"C\" __global__ void __launch_bounds__(256) " << fn << "(const LfArgs a) {\n";
      pointers(src);
      src << "  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < " << cells
          << "LL; idx += (long long)gridDim.x * blockDim.x) {\n";
      src << "    long long rem = idx;\n";
      for (int d = nd - 1; d >= 0; --d) {
        if (space.count(d))
          src << "    const int x" << d << " = (int)(rem % " << N[d] << "); rem /= " << N[d] << ";\n";
        else
          src << "    const int x" << d << " = 0;\n";
      }
      for (int r : topo)
        if (in_nest[r]) emit_rap(r, nv, src, "    ", okk, "");
      src << "  }\n}\n";
    } else {
      // ---- reduction nest: warp per parallel cell, reduced dims in order
      int LFB = 2;  // element blocks of 32 in flight per warp (LF_JIT_RED_BLOCKS; 104 -> 117 G at 2, no gain beyond)
      if (const char* e = lfx::option("LF_JIT_RED_BLOCKS")) LFB = std::max(1, std::atoi(e));
      std::set<int> Pd;
      for (int d : space)
        if (!R.count(d)) Pd.insert(d);
      long long pcells = 1, rcount = 1;
      for (int d : Pd) pcells *= N[d];
      for (int d : R) rcount *= N[d];
      nl.reduction = true;
      nl.units = pcells;
      // classify raps: element (depends on the reduced dims), post (after a reduction), pre
      std::vector<int> cls(nr, 0);  // 0 pre, 1 element, 2 reduction, 3 post
      for (int r : topo) {
        if (!in_nest[r]) continue;
        const auto& rap = g.raps[r];
        if (std::find(reds.begin(), reds.end(), r) != reds.end()) {
          cls[r] = 2;
          continue;
        }
        int c = 0;
        for (int t : rap.in_terms) {
          const int pr = g.producer[t];
          if (pr >= 0 && in_nest[pr]) c = std::max(c, cls[pr] == 2 ? 3 : cls[pr]);
        }
        if (rap.kind == lf::RapKind::load) {
          const auto ax = term_axes(rap.out_terms[0]);
          for (int d : R)
            if (ax.count(d)) c = std::max(c, 1);
        } else if (rap.kind == lf::RapKind::store) {
          const auto ax = term_axes(rap.in_terms[0]);
          for (int d : R)
            if (ax.count(d)) c = std::max(c, 1);
        } else {
          for (int d : P.groups[P.group_of[r]].space)
            if (R.count(d)) c = std::max(c, 1);
        }
        if (c == 3 && rap.kind != lf::RapKind::store) {
          for (int d : P.groups[P.group_of[r]].space)
            if (R.count(d)) return fail("broadcast of a reduction inside its own nest (needs a split)");
        }
        cls[r] = c;
      }
      // elements operands of each reduction (the non-carry inputs)
      std::vector<std::vector<int>> elem_t(reds.size());
      for (size_t m = 0; m < reds.size(); ++m) {
        const auto& rap = g.raps[reds[m]];
        const auto& k = rs.kernels[rap.kernel];
        if (k.inputs.size() > 2) return fail("associative kernel '" + k.name + "' with more than one element input");
        for (size_t i = 0; i < rap.in_terms.size(); ++i) {
          const auto& to = g.terms[rap.out_terms[0]];
          const auto& ti = g.terms[rap.in_terms[i]];
          if (!(ti.ident == to.ident && ti.dims == to.dims && !(ti == to))) elem_t[m].push_back(static_cast<int>(i));
        }
      }
      // carry term of each reduction
      std::vector<int> carry_t(reds.size(), -1);
      for (size_t m = 0; m < reds.size(); ++m) {
        const auto& rap = g.raps[reds[m]];
        for (size_t i = 0; i < rap.in_terms.size(); ++i) {
          const auto& ti = g.terms[rap.in_terms[i]];
          const auto& to = g.terms[rap.out_terms[0]];
          if (ti.ident == to.ident && ti.dims == to.dims && !(ti == to)) carry_t[m] = rap.in_terms[i];
        }
        if (carry_t[m] < 0) return fail("associative kernel '" + rs.kernels[rap.kernel].name + "' has no carry input");
      }
      // opt-in (LF_JIT_RED_TILED=1): exact, but measured slower on the 8192^2
      // normalization (nest 0: 606 vs 350 us) -- 32 cells per CTA leave too few
      // CTAs (256) to keep HBM busy
      const bool tiled = pcells >= 32 && lfx::option("LF_JIT_RED_TILED") && std::atoi(lfx::option("LF_JIT_RED_TILED")) != 0;
      if (tiled) {
        // ---- transposed: a CTA owns 32 parallel cells, lane c of warp 0
        // accumulates cell c (one ordered chain per lane, none redundant); all
        // 256 threads evaluate the element operands of a 32 x EB tile into
        // shared memory (double-buffered: warp 0 accumulates tile k while the
        // others evaluate tile k+1).  Consecutive threads take consecutive
        // elements when the innermost loop dimension is reduced (row sums),
        // consecutive cells otherwise (column sums): coalesced either way.
        // CPC cells per CTA: 8 or 16 while 32 would leave fewer than six CTAs per SM
        // (8192 rows: 1024 CTAs of 8 rows) -- a filler warp keeps only a few loads
        // in flight, so HBM bandwidth comes from resident CTAs; EB elements of each
        // cell per tile.
        // Warp 0 only accumulates (lane c < CPC owns cell c); warps 1..8 fill.
        const int CPC = pcells < 16LL * 888 ? 8 : (pcells < 32LL * 888 ? 16 : 32);  // >= 6 CTAs per SM where the cells allow
        const int EB = CPC == 32 ? 64 : 128;
        const bool elemfast = R.count(nd - 1) > 0;
        nl.cells_per_cta = CPC;
        nl.threads = 288;
        src << "extern \"C\" __global__ void __launch_bounds__(288) " << fn << "(const LfArgs a) {\n";
        pointers(src);
        src << "  __shared__ T lf_t[2][" << reds.size() << "][" << CPC << "][" << EB + 1 << "];\n";
        src << "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = (int)threadIdx.x - 32;\n";
        src << "  for (long long cb = blockIdx.x * " << CPC << "LL; cb < " << pcells << "LL; cb += gridDim.x * " << CPC
            << "LL) {\n";
        // warp 0: carries of its cell
        for (size_t m = 0; m < reds.size(); ++m) src << "    T acc" << m << " = T(0);\n";
        auto cell_coords = [&](std::ostream& o, const std::string& pcexpr, const std::string& ind) {
          o << ind << "long long rem = " << pcexpr << ";\n";
          for (int d = nd - 1; d >= 0; --d)
            if (Pd.count(d)) o << ind << "const int x" << d << " = (int)(rem % " << N[d] << "); rem /= " << N[d] << ";\n";
        };
        const std::string mine = "warp == 0 && lane < " + std::to_string(CPC) + " && cb + lane < " + std::to_string(pcells) + "LL";
        src << "    if (" << mine << ") {\n";
        cell_coords(src, "cb + lane", "      ");
        for (int d = 0; d < nd; ++d)
          if (!Pd.count(d)) src << "      const int x" << d << " = 0;\n";
        done.assign(g.terms.size(), 0);
        for (int r : topo)
          if (in_nest[r] && cls[r] == 0) emit_rap(r, nv, src, "      ", okk, "true");
        for (size_t m = 0; m < reds.size(); ++m) {
          const int ct = carry_t[m];
          const int pr = g.producer[ct];
          if (pr >= 0 && g.raps[pr].kind == lf::RapKind::kernel && nest_of(pr) != nv && !done[ct]) {
            src << "      const T v" << ct << " = " << mat_index(ct) << ";\n";
            done[ct] = 1;
          }
          src << "      acc" << m << " = v" << ct << ";\n";
        }
        src << "    }\n";
        src << "    for (long long rb = 0, kt = 0; rb < " << rcount << "LL; rb += " << EB << ", ++kt) {\n";
        src << "      const int buf = (int)(kt & 1);\n";
        src << "      if (warp > 0) {\n";
        // Two unrolled passes over the thread's elements of the tile: the first
        // only loads, evaluates and fills the shared tile -- no global store sits
        // between its loads, so all of them (8 x the operands at EB = 64) are in
        // flight together instead of one round trip per element; the second
        // re-evaluates (the non-coherent loads are the first pass's: same
        // addresses, the compiler keeps the values) and issues the stores of the
        // variables materialised for later nests.
        for (int pass = 0; pass < 2; ++pass) {
          src << "      #pragma unroll\n";
          src << "      for (int q = tid; q < " << CPC * EB << "; q += 256) {\n";
          src << "        const int c = " << (elemfast ? "q / " + std::to_string(EB) : "q % " + std::to_string(CPC))
              << ", j = " << (elemfast ? "q % " + std::to_string(EB) : "q / " + std::to_string(CPC)) << ";\n";
          src << "        const bool ok = cb + c < " << pcells << "LL && rb + j < " << rcount << "LL;\n";
          std::ostringstream ev;
          cell_coords(ev, "ok ? cb + c : 0LL", "        ");
          ev << "        long long rr = ok ? rb + j : 0LL;\n";
          for (int d = nd - 1; d >= 0; --d)
            if (R.count(d)) ev << "        const int x" << d << " = (int)(rr % " << N[d] << "); rr /= " << N[d] << ";\n";
          for (int d = 0; d < nd; ++d)
            if (!Pd.count(d) && !R.count(d)) ev << "        const int x" << d << " = 0;\n";
          done.assign(g.terms.size(), 0);
          for (int r : topo)
            if (in_nest[r] && cls[r] == 0) emit_rap(r, nv, ev, "        ", okk, "false");
          for (int r : topo)
            if (in_nest[r] && cls[r] == 1) emit_rap(r, nv, ev, "        ", okk, pass == 0 ? "false" : "ok");
          for (size_t m = 0; m < reds.size(); ++m) {
            const auto& rap = g.raps[reds[m]];
            for (int i : elem_t[m]) {
              const int t = rap.in_terms[i];
              const int pr = g.producer[t];
              if (pr >= 0 && g.raps[pr].kind == lf::RapKind::kernel && nest_of(pr) != nv && !done[t]) {
                ev << "        const T v" << t << " = " << mat_index(t) << ";\n";
                done[t] = 1;
              }
              if (pass == 0) ev << "        lf_t[buf][" << m << "][c][j] = v" << t << ";\n";
            }
          }
          src << ev.str();
          if (pass == 0) src << "      }\n";
        }
        src << "      }\n";
        src << "      }\n";  // warp > 0
        src << "      __syncthreads();\n";
        src << "      if (warp == 0 && lane < " << CPC << ") {\n";
        src << "        const int cnt = (int)min((long long)" << EB << ", " << rcount << "LL - rb);\n";
        // full tiles: the element values are loaded from shared memory ahead of the
        // ordered chain (no exit test between them), so the chain advances at the
        // operation's own latency; the last, partial tile takes the counted loop
        for (int full = 1; full >= 0; --full) {
          if (full) {
            src << "        if (cnt == " << EB << ") {\n";
            src << "        #pragma unroll 32\n";
            src << "        for (int e = 0; e < " << EB << "; ++e) {\n";
          } else {
            src << "        } else {\n";
            src << "        for (int e = 0; e < cnt; ++e) {\n";
          }
          for (size_t m = 0; m < reds.size(); ++m) {
            const auto& rap = g.raps[reds[m]];
            const auto& k = rs.kernels[rap.kernel];
            std::map<std::string, std::string> pv;
            for (size_t i = 0; i < k.inputs.size(); ++i) {
              const bool is_elem = std::find(elem_t[m].begin(), elem_t[m].end(), (int)i) != elem_t[m].end();
              pv[k.inputs[i].first] =
                  is_elem ? "lf_t[buf][" + std::to_string(m) + "][lane][e]" : "acc" + std::to_string(m);
            }
            if (!emit_kernel(
                    k, T, [&](const std::string& n) { return pv.at(n); },
                    [&](const std::string&) { return "acc" + std::to_string(m); }, false, src, "          ", err))
              return false;
          }
          src << "        }\n";
        }
        src << "        }\n";
        src << "      }\n";
        src << "    }\n";
        // warp 0: reduction outputs and the raps after them, per cell
        src << "    if (" << mine << ") {\n";
        cell_coords(src, "cb + lane", "      ");
        for (int d = 0; d < nd; ++d)
          if (!Pd.count(d)) src << "      const int x" << d << " = 0;\n";
        done.assign(g.terms.size(), 0);
        for (int r : topo)
          if (in_nest[r] && cls[r] == 0) emit_rap(r, nv, src, "      ", okk, "false");
        for (size_t m = 0; m < reds.size(); ++m) {
          const int ot = g.raps[reds[m]].out_terms[0];
          src << "      const T v" << ot << " = acc" << m << ";\n";
          done[ot] = 1;
          if (term_mat[ot]) src << "      " << mat_index(ot) << " = v" << ot << ";\n";
        }
        for (int r : topo)
          if (in_nest[r] && cls[r] == 3) emit_rap(r, nv, src, "      ", okk, "");
        src << "    }\n";
        src << "    __syncthreads();\n";
        src << "  }\n}\n";
        if (!okk) return false;
        out.nest_kernels.push_back(nl);
        continue;
      }
      src << "extern \"C\" __global__ void __launch_bounds__(256) " << fn << "(const LfArgs a) {\n";
      pointers(src);
      src << "  __shared__ T lf_red[8][" << 2 * LFB << "][" << reds.size() << "][32];\n";
      src << "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n";
      src << "  for (long long pc = blockIdx.x * 8LL + warp; pc < " << pcells << "LL; pc += gridDim.x * 8LL) {\n";
      src << "    long long rem = pc;\n";
      for (int d = nd - 1; d >= 0; --d)
        if (Pd.count(d)) src << "    const int x" << d << " = (int)(rem % " << N[d] << "); rem /= " << N[d] << ";\n";
      for (int d = 0; d < nd; ++d)
        if (!Pd.count(d) && !R.count(d)) src << "    const int x" << d << " = 0;\n";
      // pre raps (every lane)
      for (int r : topo)
        if (in_nest[r] && cls[r] == 0) emit_rap(r, nv, src, "    ", okk, "lane == 0");
      // carries
      for (size_t m = 0; m < reds.size(); ++m) {
        const auto& rap = g.raps[reds[m]];
        const auto& k = rs.kernels[rap.kernel];
        const int ot = rap.out_terms[0];
        int carry = -1;
        for (size_t i = 0; i < rap.in_terms.size(); ++i) {
          const auto& ti = g.terms[rap.in_terms[i]];
          const auto& to = g.terms[ot];
          if (ti.ident == to.ident && ti.dims == to.dims && !(ti == to)) carry = static_cast<int>(i);
        }
        if (carry < 0) return fail("associative kernel '" + k.name + "' has no carry input");
        const int ct = rap.in_terms[carry];
        const int pr = g.producer[ct];
        if (pr >= 0 && g.raps[pr].kind == lf::RapKind::kernel && nest_of(pr) != nv && !done[ct]) {
          src << "    const T v" << ct << " = " << mat_index(ct) << ";\n";
          done[ct] = 1;
        }
        src << "    T acc" << m << " = v" << ct << ";\n";
      }
      // element loop, LFB blocks of 32 elements per iteration: the element code
      // (global loads) of every block is issued before the ordered
      // accumulation of the first, so a warp keeps LFB blocks of loads in
      // flight instead of idling on memory after each 32-element accumulation
      std::ostringstream stage;  // one block's elements into lf_red[warp][LFBUF]
      stage << "      const bool ok = rb + lane < " << rcount << "LL;\n";
      stage << "      long long rr = ok ? rb + lane : " << (rcount - 1) << "LL;\n";
      for (int d = nd - 1; d >= 0; --d)
        if (R.count(d)) stage << "      const int x" << d << " = (int)(rr % " << N[d] << "); rr /= " << N[d] << ";\n";
      std::ostringstream el;
      for (int r : topo)
        if (in_nest[r] && cls[r] == 1) emit_rap(r, nv, el, "      ", okk, "ok");
      stage << el.str();
      // element operands of each reduction into shared memory, then the ordered accumulation
      std::vector<std::vector<int>> elem_in(reds.size());
      for (size_t m = 0; m < reds.size(); ++m) {
        const auto& rap = g.raps[reds[m]];
        const auto& k = rs.kernels[rap.kernel];
        if (k.inputs.size() > 2) return fail("associative kernel '" + k.name + "' with more than one element input");
        for (size_t i = 0; i < rap.in_terms.size(); ++i) {
          const int t = rap.in_terms[i];
          const auto& to = g.terms[rap.out_terms[0]];
          const auto& ti = g.terms[t];
          if (ti.ident == to.ident && ti.dims == to.dims && !(ti == to)) continue;
          const int pr = g.producer[t];
          if (pr >= 0 && g.raps[pr].kind == lf::RapKind::kernel && nest_of(pr) != nv && !done[t]) {
            stage << "      const T v" << t << " = " << mat_index(t) << ";\n";
            done[t] = 1;
          }
          stage << "      ev" << "LFBUF_" << m << " = v" << t << ";\n";
          elem_in[m].push_back(static_cast<int>(i));
        }
      }
      const std::string stage_text = stage.str();
      // software pipeline over groups of LFB blocks: the element code (global
      // loads) of group i+1 is issued before group i is accumulated and its
      // values stored to the other half of the buffer after it, so the loads
      // are in flight during the ordered chain
      auto stage_group = [&](const std::string& base) {
        for (int h = 0; h < LFB; ++h) {
          std::string t = stage_text;
          for (size_t pos; (pos = t.find("LFBUF")) != std::string::npos;) t.replace(pos, 5, std::to_string(h));
          src << "      if (" << base << " + " << 32 * h << " < " << rcount << "LL) {\n";
          src << "      const long long rb = " << base << " + " << 32 * h << ";\n";
          src << t;
          src << "      }\n";
        }
      };
      auto store_group = [&](const std::string& half) {
        for (int h = 0; h < LFB; ++h)
          for (size_t m = 0; m < reds.size(); ++m)
            src << "      lf_red[warp][" << half << " + " << h << "][" << m << "][lane] = ev" << h << "_" << m << ";\n";
      };
      auto declare_ev = [&]() {
        for (int h = 0; h < LFB; ++h)
          for (size_t m = 0; m < reds.size(); ++m) src << "      T ev" << h << "_" << m << " = T(0);\n";
      };
      src << "    {\n";
      declare_ev();
      stage_group("0LL");
      store_group("0");
      src << "    }\n";
      src << "    for (long long rb0 = 0, it = 0; rb0 < " << rcount << "LL; rb0 += " << 32 * LFB << ", ++it) {\n";
      src << "      const int cur = (int)(it & 1) * " << LFB << ", nxt = " << LFB << " - cur;\n";
      src << "      __syncwarp();\n";
      declare_ev();
      stage_group("rb0 + " + std::to_string(32 * LFB));
      src << "      for (int h = 0; h < " << LFB << "; ++h) {\n";
      src << "      const long long rb = rb0 + 32 * h;\n";
      src << "      const int cnt = (int)max(0LL, min(32LL, " << rcount << "LL - rb));\n";
      // full blocks unrolled
      src << "      #pragma unroll 32\n";
      src << "      for (int e = 0; e < 32; ++e) {\n";
      src << "        if (e >= cnt) break;\n";
      for (size_t m = 0; m < reds.size(); ++m) {
        const auto& rap = g.raps[reds[m]];
        const auto& k = rs.kernels[rap.kernel];
        std::map<std::string, std::string> pv;
        for (size_t i = 0; i < k.inputs.size(); ++i) {
          const bool is_elem = std::find(elem_in[m].begin(), elem_in[m].end(), (int)i) != elem_in[m].end();
          pv[k.inputs[i].first] = is_elem ? "lf_red[warp][cur + h][" + std::to_string(m) + "][e]" : "acc" + std::to_string(m);
        }
        if (!emit_kernel(
                k, T, [&](const std::string& n) { return pv.at(n); },
                [&](const std::string&) { return "acc" + std::to_string(m); }, false, src, "        ", err))
          return false;
      }
      src << "      }\n";
      src << "      }\n";
      src << "      __syncwarp();\n";
      store_group("nxt");
      src << "    }\n";
      // reduction outputs, post raps, P-level stores (lane 0 writes)
      for (size_t m = 0; m < reds.size(); ++m) {
        const int ot = g.raps[reds[m]].out_terms[0];
        src << "    const T v" << ot << " = acc" << m << ";\n";
        done[ot] = 1;
        if (term_mat[ot]) src << "    if (lane == 0) " << mat_index(ot) << " = v" << ot << ";\n";
      }
      for (int r : topo)
        if (in_nest[r] && cls[r] == 3) emit_rap(r, nv, src, "    ", okk, "lane == 0");
      src << "  }\n}\n";
    }
    if (!okk) return false;
    out.nest_kernels.push_back(nl);
  }
  return true;
}

}  // namespace cg

using namespace cg;

// Programmatic dependent launch (jit.cpp launches with programmatic stream
// serialization): every generated kernel first waits for the previous grid of
// the stream (its inputs written, its outputs free).  The persistent march
// kernels then let the next launch (the light ghost fill / in-place commit) be
// scheduled at once; the other kernels only wait: a multi-wave nest kernel's
// dependents would take the slots of its later waves (normalization 117 ->
// 110 G), and early-launched march CTAs behind a fill or capture cost the 3D
// in-place chain 9 % (136 -> 124 G).  Inserted as each kernel's first statement.
static std::string with_pdl(const std::string& src, std::string& err) {
  std::string out =
      "__device__ __forceinline__ void lf_pdl_wait() { asm volatile(\"griddepcontrol.wait;\" ::: \"memory\"); }\n"
      "__device__ __forceinline__ void lf_pdl() {\n"
      "  lf_pdl_wait();\n"
      "  asm volatile(\"griddepcontrol.launch_dependents;\" ::: \"memory\");\n"
      "}\n";
  size_t pos = 0;
  for (;;) {
    const size_t k = src.find("__global__ void", pos);
    if (k == std::string::npos) break;
    const size_t brace = src.find(") {\n", k);
    if (brace == std::string::npos) break;
    if (src.find('\n', k) < brace) {  // every generated kernel opens its body at the end of its signature line
      err = "internal error: generated kernel signature not followed by its body on the same line";
      break;
    }
    const bool march = src.substr(k, brace - k).find(" lf_jit_step") != std::string::npos;
    out += src.substr(pos, brace + 4 - pos);
    out += march ? "  lf_pdl();\n" : "  lf_pdl_wait();\n";
    pos = brace + 4;
  }
  out += src.substr(pos);
  return out;
}

bool jit_generate(const lf::Plan& P, JitProgram& out, const std::string& sources) {
  bool multi = !P.one_nest;
  for (const auto& k : P.rs.kernels) multi |= k.associative;
  if (multi) {
    std::ostringstream src;
    std::string err;
    if (!emit_nests(P, sources, out, src, err)) {
      out.error = err;
      return false;
    }
    // ghost refill of iterated goals: the same kernel as the single-nest path
    Ctx C(P);
    C.nd = out.nd;
    C.T = out.type;
    C.N.resize(C.nd);
    C.LO.resize(C.nd);
    for (int d = 0; d < C.nd; ++d) {
      C.N[d] = P.rs.ranges[d].trips();
      C.LO[d] = P.rs.ranges[d].lo;
    }
    if (!emit_fill(C, out, src)) {
      out.error = C.error;
      return false;
    }
    std::string perr;
    out.source = sources + with_pdl(src.str(), perr);
    out.march = false;
    if (!perr.empty()) {
      out.error = perr;
      return false;
    }
    return true;
  }
  Ctx C(P);
  C.sources = sources;
  if (!analyse(C)) {
    out.error = C.error;
    return false;
  }
  out.type = C.T;
  out.elem_bytes = C.T == "double" ? 8 : 4;
  out.nd = C.nd;
  std::ostringstream src;
  const bool ok = C.nd >= 2 ? emit_march(C, out, src) : emit_tiled(C, out, src);
  if (!ok || !emit_fill(C, out, src)) {
    out.error = C.error;
    return false;
  }
  // the warp-specialised variant, where every streamed axiom can be fetched by
  // TMA: a dense terminal in loop-dimension order with 16-B row pitches, no
  // in-place aliases (those keep the band-capturing loader)
  bool tma_ok = C.nd >= 2 && !(lfx::option("LF_JIT_WS") && std::atoi(lfx::option("LF_JIT_WS")) == 0);
  int nstaged = 0;
  for (size_t v = 0; tma_ok && v < C.P.vars.size(); ++v) {
    const int ti = C.staged_axiom(static_cast<int>(v));
    if (ti < 0) continue;
    ++nstaged;
    const auto& t = C.P.terminals[ti];
    for (int d = 0; d < C.nd; ++d) tma_ok &= t.dims[d] == d;
    tma_ok &= (t.extent[C.nd - 1] * out.elem_bytes) % 16 == 0;
  }
  tma_ok &= nstaged > 0 && nstaged <= kJitMaxMaps;
  if (tma_ok) {
    std::string variants;
    std::ostringstream ws;
    out.ws_maps.clear();
    // in place: 2D chains take the register march below; 3D chains the
    // warp-specialised march with deferred boundary writes
    if ((C.P.rs.aliases.empty() || C.nd == 3) && emit_march(C, out, ws, true) && !out.ws_maps.empty() &&
        static_cast<int>(out.ws_maps.size()) <= kJitMaxMaps) {
      out.has_ws = true;
      variants += ws.str();
    } else {
      out.ws_maps.clear();
    }
    // 2D: the register march (LF_JIT_RM=0: off)
    std::ostringstream rm;
    const bool rm_off = lfx::option("LF_JIT_RM") && std::atoi(lfx::option("LF_JIT_RM")) == 0;
    if (C.nd == 2 && !rm_off && emit_rmarch(C, out, rm) && !out.rm_maps.empty() &&
        static_cast<int>(out.rm_maps.size()) <= kJitMaxMaps) {
      out.has_rm = true;
      variants += rm.str();
    } else {
      out.rm_maps.clear();  // the chain keeps the marches above
      out.has_rm = false;
    }
    if (!variants.empty()) {
      emit_tma_helpers(src);
      src << variants;
    }
  }
  std::string perr;
  out.source = sources + with_pdl(src.str(), perr);
  if (!perr.empty()) {
    out.error = perr;
    return false;
  }
  return true;
}

}  // namespace lfx

// Generic executor code generation: the analysis context shared by the
// emitters (codegen.cpp: plain / warp-specialised smem-window marches, 1D
// tiles, multi-nest plans; codegen_rm.cpp: the register march of 2D chains).
#pragma once

#include <functional>
#include <map>
#include <ostream>
#include <string>
#include <vector>

#include "../planner/planner.hpp"
#include "jit.hpp"

namespace lfx::cg {

inline std::string elem_type(const std::string& t) {
  if (t.find("double") != std::string::npos) return "double";
  if (t.find("float") != std::string::npos) return "float";
  return "";
}

inline std::string plus(long off) {
  if (!off) return "";
  return (off > 0 ? " + " : " - ") + std::to_string(std::labs(off));
}

struct GIn {
  std::string param;
  int var;
  std::vector<int> rel;
  int via = -1;  // index into Ctx::inlined: the value is that producer recomputed in place
};
struct GOut {
  std::string param;
  int var;
  std::vector<int> rel;
};
struct Load {
  int var;
  std::vector<int> rel;
};
struct Grp {
  int kernel;
  std::vector<int> gmin, gmax;
  std::vector<GIn> in;
  std::vector<GOut> out;
  std::vector<Load> loads;  // distinct (variable, offset) reads, inlined producers expanded
  int shift = 0;  // lead along the outermost dimension (march schedule)
  int level = 1;  // dependency level (groups of one level share a barrier)
};

// everything the emitters share
struct Ctx {
  const lf::Plan& P;
  std::string sources;  // user-kernel sources the generated code is compiled with
  int nd = 0;
  std::vector<long> LO;  // range lower bounds: loop index = LO + trip
  std::string T;
  std::vector<long> N;
  std::vector<std::vector<int>> vmin, vmax;  // per var, per dim: term offset range
  std::map<int, std::vector<int>> axiom_extra;
  std::vector<char> smem_var;  // kernel outputs read by some kernel
  std::vector<Grp> groups;     // kernel groups, dataflow order
  std::vector<Grp> inlined;    // cheap producers recomputed inside their consumers
  std::string error;

  explicit Ctx(const lf::Plan& p) : P(p) {}

  int terminal_of(int v, bool goal) const {
    for (size_t i = 0; i < P.terminals.size(); ++i)
      if (P.terminals[i].var == v && P.terminals[i].is_goal == goal) return static_cast<int>(i);
    return -1;
  }
  long pitch(const lf::Terminal& t, size_t slot) const {
    long p = 1;
    for (size_t k = slot + 1; k < t.extent.size(); ++k) p *= t.extent[k];
    return p;
  }
  // flat index of terminal `ti` at term-frame position pos[d] (+ extra[d])
  std::string tidx(int ti, const std::vector<std::string>& pos, const std::vector<int>& extra) const {
    const auto& t = P.terminals[ti];
    std::string e;
    for (size_t s = 0; s < t.dims.size(); ++s) {
      const int d = t.dims[s];
      const long off = extra[d] - t.base[s] + LO[d];
      const std::string c = "(long long)(" + pos[d] + plus(off) + ")";
      const long p = pitch(t, s);
      e += (e.empty() ? "" : " + ") + c + (p != 1 ? " * " + std::to_string(p) + "LL" : "");
    }
    return e.empty() ? std::string("0") : e;
  }
  std::vector<int> extra_of(int v) const {
    auto it = axiom_extra.find(v);
    return it == axiom_extra.end() ? std::vector<int>(nd, 0) : it->second;
  }
  // full-rank axiom terminal backing variable v (or -1)
  int staged_axiom(int v) const {
    const int ti = terminal_of(v, false);
    if (ti < 0 || (int)P.terminals[ti].dims.size() != nd) return -1;
    return ti;
  }
};

bool emit_kernel(const lf::KernelRule& k, const std::string& T, const std::function<std::string(const std::string&)>& in,
                 const std::function<std::string(const std::string&)>& out, bool declare, std::ostream& src,
                 const std::string& ind, std::string& err);
// body expressions of group G's outputs, p_<param> bound to its inputs, q_<param> declared
bool emit_bodies(Ctx& C, const Grp& G, std::ostream& src, const char* ind);
// kernel signature and terminal pointers (kernel == nullptr: lf_jit_step and the module prelude)
void emit_prelude(Ctx& C, std::ostream& src, int threads, int min_blocks, const char* kernel);
// mbarrier / TMA device helpers and the tensor-map parameter block (emitted
// once, before the first kernel that takes LfMaps)
void emit_tma_helpers(std::ostream& src);
// in place: the band-capture kernel `name` for the aliased axioms caps =
// (variable, terminal), band buffers at a.t[slots[q] .. slots[q] + 2], inner tile `tile`
void emit_capture(Ctx& C, const char* name, const std::vector<std::pair<size_t, int>>& caps,
                  const std::vector<int>& slots, const std::vector<int>& tile, std::ostream& src);
// 2D register march (lf_jit_step_rm); false when the chain does not fit it
bool emit_rmarch(Ctx& C, JitProgram& out, std::ostream& src);

}  // namespace lfx::cg

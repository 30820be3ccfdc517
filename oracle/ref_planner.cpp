// BOOKKEEPING ORACLE -- test infrastructure only.
//
// Links the reference's own planning modules, compiled from the sources
// where they lie (/root/reference/proj/src/{inference,nests,fusion,shifts,
// storage}.cpp; recipe in oracle/Makefile, outputs only in oracle/_ref/), and
// prints their verdict on a `.lf` file as JSON so tests can pin the
// loomfuse-b200 planner's terminal extents/bases, windows and footprints
// against the reference.
//
// rulespec.cpp itself does not build here (yaml-cpp is absent and
// rulespec.cpp:147 is ill-formed), so this driver
//   * parses the file with loomfuse-b200's own parser and converts the result
//     to loomfuse::RuleSet, and
//   * provides the four rulespec.cpp symbols the other modules call
//     (RuleSet::dim_of, TermPattern::str, DeclInfo::param, parse_declaration),
//     restated from rulespec.cpp:13-48 and 493-548.
#include <cctype>
#include <fstream>
#include <iostream>
#include <sstream>

#include "loomfuse/storage.hpp"
#include "planner/planner.hpp"

namespace loomfuse {

std::string TermPattern::str() const {
  std::string s;
  if (!tag.empty()) s += tag + "(";
  s += ident;
  for (const auto& o : subscripts) {
    s += "[" + o.var;
    if (o.displacement > 0) s += "+" + std::to_string(o.displacement);
    if (o.displacement < 0) s += std::to_string(o.displacement);
    s += "]";
  }
  if (!tag.empty()) s += ")";
  return s;
}

int RuleSet::dim_of(const std::string& var) const {
  for (size_t i = 0; i < loop_order.size(); ++i)
    if (loop_order[i] == var) return static_cast<int>(i);
  return -1;
}

const DeclParam* DeclInfo::param(const std::string& name) const {
  for (const auto& p : params)
    if (p.name == name) return &p;
  return nullptr;
}

DeclInfo parse_declaration(const std::string& decl) {
  lf::DeclInfo d = lf::parse_declaration(decl);
  DeclInfo out;
  out.function = d.function;
  for (const auto& p : d.params) out.params.push_back({p.type, p.name, p.pointer, p.reference});
  return out;
}

}  // namespace loomfuse

namespace {

loomfuse::SourceLoc conv(const lf::SourceLoc& l) { return {l.file, l.line, l.column}; }

loomfuse::TermPattern conv(const lf::TermPattern& p) {
  loomfuse::TermPattern t;
  t.tag = p.tag;
  t.ident = p.ident;
  for (const auto& s : p.subscripts) t.subscripts.push_back({s.var, s.displacement});
  t.loc = conv(p.loc);
  return t;
}

loomfuse::ExternalDecl conv(const lf::ExternalDecl& e) {
  loomfuse::ExternalDecl x;
  x.type = e.type;
  x.name = e.name;
  for (const auto& s : e.subscripts) x.subscripts.push_back({s.var, s.displacement});
  x.loc = conv(e.loc);
  return x;
}

loomfuse::RuleSet conv(const lf::RuleSet& r) {
  loomfuse::RuleSet rs;
  rs.name = r.name;
  for (const auto& k : r.kernels) {
    loomfuse::KernelRule kr;
    kr.name = k.name;
    kr.declaration = k.declaration;
    kr.associative = k.associative;
    kr.params = k.params;
    for (const auto& [p, t] : k.inputs) kr.inputs.emplace_back(p, conv(t));
    for (const auto& [p, t] : k.outputs) kr.outputs.emplace_back(p, conv(t));
    kr.bodies = k.bodies;
    kr.loc = conv(k.loc);
    rs.kernels.push_back(std::move(kr));
  }
  for (const auto& a : r.axioms) rs.axioms.push_back({conv(a.external), conv(a.term)});
  for (const auto& g : r.goals) rs.goals.push_back({conv(g.term), conv(g.external)});
  rs.loop_order = r.loop_order;
  for (const auto& rg : r.ranges) rs.ranges.push_back({rg.lo, rg.hi, rg.stride});
  rs.aliases = r.aliases;
  rs.vector_length = r.vector_length;
  rs.backend = r.backend;
  return rs;
}

const char* scheme(loomfuse::Scheme s) {
  switch (s) {
    case loomfuse::Scheme::full: return "full";
    case loomfuse::Scheme::inner_circular: return "inner_circular";
    case loomfuse::Scheme::outer_rotate: return "outer_rotate";
    case loomfuse::Scheme::vector_expanded: return "vector_expanded";
  }
  return "?";
}

std::string q(const std::string& s) { return "\"" + s + "\""; }

}  // namespace

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    if (c == '\n') {
      o += "\\n";
      continue;
    }
    o += c;
  }
  return o + "\"";
}

// --dag: the reference's inference DAG plus the rule bodies, for the generic
// run_naive in oracle/generic.py
void dump_dag(const lf::RuleSet& mine, const loomfuse::RuleSet& rs, const loomfuse::DataflowDAG& dag,
              const loomfuse::StoragePlan& sp) {
  std::ostringstream os;
  os << "{\"loop_order\":[";
  for (size_t d = 0; d < rs.loop_order.size(); ++d) os << (d ? "," : "") << jstr(rs.loop_order[d]);
  os << "],\"ranges\":[";
  for (size_t d = 0; d < rs.ranges.size(); ++d) os << (d ? "," : "") << "[" << rs.ranges[d].lo << "," << rs.ranges[d].hi << "]";
  os << "],\"terms\":[";
  for (size_t t = 0; t < dag.terms.size(); ++t) {
    const auto& ct = dag.terms[t];
    os << (t ? "," : "") << "{\"tag\":" << jstr(ct.tag) << ",\"ident\":" << jstr(ct.ident) << ",\"dims\":[";
    for (size_t k = 0; k < ct.dims.size(); ++k) os << (k ? "," : "") << "[" << ct.dims[k].dim << "," << ct.dims[k].offset << "]";
    os << "]}";
  }
  os << "],\"raps\":[";
  for (size_t r = 0; r < dag.raps.size(); ++r) {
    const auto& rp = dag.raps[r];
    const char* kind = rp.kind == loomfuse::RapKind::kernel ? "kernel" : rp.kind == loomfuse::RapKind::load ? "load" : "store";
    os << (r ? "," : "") << "{\"kind\":\"" << kind << "\",\"kernel\":" << jstr(rp.kind == loomfuse::RapKind::kernel ? rs.kernels[rp.kernel].name : "")
       << ",\"external\":" << jstr(rp.external) << ",\"in\":[";
    for (size_t k = 0; k < rp.in_terms.size(); ++k) os << (k ? "," : "") << rp.in_terms[k];
    os << "],\"out\":[";
    for (size_t k = 0; k < rp.out_terms.size(); ++k) os << (k ? "," : "") << rp.out_terms[k];
    os << "],\"slots\":[";
    for (size_t k = 0; k < rp.ext_slots.size(); ++k) os << (k ? "," : "") << "[" << rp.ext_slots[k].dim << "," << rp.ext_slots[k].shift << "]";
    os << "]}";
  }
  os << "],\"topo\":[";
  auto order = dag.topo_order();
  for (size_t k = 0; k < order.size(); ++k) os << (k ? "," : "") << order[k];
  os << "],\"kernels\":{";
  for (size_t k = 0; k < mine.kernels.size(); ++k) {
    const auto& kr = mine.kernels[k];
    os << (k ? "," : "") << jstr(kr.name) << ":{\"declaration\":" << jstr(kr.declaration)
       << ",\"associative\":" << (kr.associative ? "true" : "false") << ",\"inputs\":[";
    for (size_t i = 0; i < kr.inputs.size(); ++i) os << (i ? "," : "") << jstr(kr.inputs[i].first);
    os << "],\"outputs\":[";
    for (size_t i = 0; i < kr.outputs.size(); ++i) os << (i ? "," : "") << jstr(kr.outputs[i].first);
    os << "],\"bodies\":{";
    size_t b = 0;
    for (const auto& [pn, e] : kr.bodies) os << (b++ ? "," : "") << jstr(pn) << ":" << jstr(e);
    os << "}}";
  }
  os << "},\"externals\":{";
  size_t e = 0;
  for (const auto& v : sp.vars.vars) {
    if (v.alias_of >= 0 || !v.terminal()) continue;
    auto ext = loomfuse::buffer_extents(v.id, sp.vars, dag, rs);
    os << (e++ ? "," : "") << jstr(v.backing->external) << ":{\"type\":" << jstr(v.type) << ",\"axiom\":" << (v.axiom_backed ? "true" : "false")
       << ",\"extents\":[";
    for (size_t k = 0; k < ext.size(); ++k) os << (k ? "," : "") << "[" << ext[k].first << "," << ext[k].second << "]";
    os << "]}";
  }
  os << "},\"axioms\":[";
  for (size_t a = 0; a < mine.axioms.size(); ++a) os << (a ? "," : "") << jstr(mine.axioms[a].external.name);
  os << "],\"goals\":[";
  for (size_t a = 0; a < mine.goals.size(); ++a) os << (a ? "," : "") << jstr(mine.goals[a].external.name);
  os << "],\"iterate\":[";
  for (size_t a = 0; a < mine.iterate.size(); ++a) os << (a ? "," : "") << "[" << jstr(mine.iterate[a].first) << "," << jstr(mine.iterate[a].second) << "]";
  os << "],\"boundary\":{";
  size_t bcount = 0;
  for (const auto& [ext, modes] : mine.boundary) {
    os << (bcount++ ? "," : "") << jstr(ext) << ":[";
    for (size_t k = 0; k < modes.size(); ++k) os << (k ? "," : "") << jstr(lf::boundary_name(modes[k]));
    os << "]";
  }
  os << "}}";
  std::cout << os.str() << "\n";
}

int main(int argc, char** argv) {
  bool want_dag = argc == 3 && std::string(argv[1]) == "--dag";
  if (argc != 2 && !want_dag) {
    std::cerr << "usage: refplan [--dag] <spec.lf>\n";
    return 2;
  }
  if (want_dag) argv[1] = argv[2];
  std::ifstream f(argv[1]);
  std::stringstream ss;
  ss << f.rdbuf();
  lf::DiagList d;
  auto mine = lf::parse_spec(ss.str(), argv[1], d);
  if (!mine) {
    std::cerr << d.str();
    return 1;
  }
  try {
    loomfuse::RuleSet rs = conv(*mine);
    loomfuse::DiagList diags;
    auto idag = loomfuse::infer_idag(rs, diags);
    if (!idag) {
      std::cerr << diags.str();
      return 1;
    }
    loomfuse::DataflowDAG dag = loomfuse::rap_dual(*idag);
    loomfuse::GroupingResult grouping = loomfuse::group_callsites(dag);
    loomfuse::InestDAG inest = loomfuse::build_inest_dag(dag, grouping, rs);
    loomfuse::FusionResult fusion = loomfuse::fuse_inest_dag(inest, dag, grouping, rs);
    loomfuse::StoragePlan sp = loomfuse::analyze_storage(rs, dag, grouping, fusion, rs.vector_length);
    if (want_dag) {
      dump_dag(*mine, rs, dag, sp);
      return 0;
    }

    std::ostringstream os;
    os << "{\"terms\":" << dag.terms.size() << ",\"raps\":" << dag.raps.size() << ",\"edges\":" << dag.edges.size()
       << ",\"groups\":" << grouping.groups.size() << ",\"nests\":" << fusion.dag.vertices.size()
       << ",\"splits\":" << fusion.splits.size() << ",\"footprint\":" << q(sp.footprint.str(rs)) << ",\"shifts\":[";
    for (size_t g = 0; g < grouping.groups.size(); ++g) {
      const auto& cg = grouping.groups[g];
      std::string nm = cg.kind == loomfuse::RapKind::kernel ? rs.kernels[cg.kernel].name
                       : cg.kind == loomfuse::RapKind::load ? "load " + cg.external
                                                            : "store " + cg.external;
      os << (g ? "," : "") << "{\"name\":" << q(nm) << ",\"members\":" << cg.members.size() << ",\"shift\":[";
      for (size_t k = 0; k < sp.shifts.shift[g].size(); ++k) os << (k ? "," : "") << sp.shifts.shift[g][k];
      os << "]}";
    }
    os << "],\"variables\":[";
    bool first = true;
    for (const auto& v : sp.vars.vars) {
      if (v.alias_of >= 0) continue;
      const auto& sd = sp.descriptors[v.id];
      auto ext = loomfuse::buffer_extents(v.id, sp.vars, dag, rs);
      os << (first ? "" : ",") << "{\"name\":" << q(v.name) << ",\"ident\":" << q(v.ident)
         << ",\"type\":" << q(v.type) << ",\"terminal\":" << (v.terminal() ? "true" : "false")
         << ",\"external\":" << q(v.terminal() ? v.backing->external : "") << ",\"scheme\":" << q(scheme(sd.scheme))
         << ",\"span\":" << sd.span() << ",\"extents\":[";
      for (size_t k = 0; k < ext.size(); ++k) os << (k ? "," : "") << "[" << ext[k].first << "," << ext[k].second << "]";
      os << "]}";
      first = false;
    }
    os << "],\"alias\":[";
    for (size_t k = 0; k < sp.alias.entries.size(); ++k) {
      const auto& e = sp.alias.entries[k];
      const auto& wg = grouping.groups[e.writer_group];
      std::string wn = wg.kind == loomfuse::RapKind::kernel ? rs.kernels[wg.kernel].name
                       : wg.kind == loomfuse::RapKind::load ? "load " + wg.external
                                                            : "store " + wg.external;
      os << (k ? "," : "") << "{\"input\":" << q(e.input_external) << ",\"output\":" << q(e.output_external)
         << ",\"var\":" << q(sp.vars.vars[e.var].name) << ",\"writer\":" << q(wn) << ",\"writer_shift\":[";
      for (size_t d = 0; d < e.writer_shift.size(); ++d) os << (d ? "," : "") << e.writer_shift[d];
      os << "],\"offsets\":[";
      for (size_t o = 0; o < e.offsets.size(); ++o) {
        os << (o ? "," : "") << "[";
        for (size_t d = 0; d < e.offsets[o].size(); ++d) os << (d ? "," : "") << e.offsets[o][d];
        os << "]";
      }
      const auto& sh = sp.shadows[k];
      os << "],\"shadow\":{\"scheme\":" << q(scheme(sh.scheme)) << ",\"spans\":[";
      for (size_t d = 0; d < sh.dims.size(); ++d) os << (d ? "," : "") << sh.dims[d].span;
      os << "]}}";
    }
    os << "]}";
    std::cout << os.str() << "\n";
  } catch (const std::exception& e) {
    std::cerr << "reference planner threw: " << e.what() << "\n";
    return 3;
  }
  return 0;
}

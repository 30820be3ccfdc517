// Planner analysis: callsite grouping, the single-nest check, pipeline
// shifts, storage contraction windows, terminal extents, footprint and the
// canonical chain signature used to dispatch to a fused sm_100a executor.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <deque>
#include <functional>
#include <sstream>

#include "fusion.hpp"
#include "planner.hpp"

namespace lf {

const char* scheme_name(Scheme s) {
  switch (s) {
    case Scheme::full: return "full";
    case Scheme::inner_circular: return "inner_circular";
    case Scheme::outer_rotate: return "outer_rotate";
    case Scheme::scalar: return "scalar";
    case Scheme::terminal: return "terminal";
  }
  return "?";
}

std::vector<int> CallsiteGroup::min_disp(size_t nd) const {
  std::vector<int> m(nd, 0);
  for (size_t d = 0; d < nd && !member_disp.empty(); ++d) {
    m[d] = member_disp[0][d];
    for (const auto& md : member_disp) m[d] = std::min(m[d], md[d]);
  }
  return m;
}
std::vector<int> CallsiteGroup::max_disp(size_t nd) const {
  std::vector<int> m(nd, 0);
  for (size_t d = 0; d < nd && !member_disp.empty(); ++d) {
    m[d] = member_disp[0][d];
    for (const auto& md : member_disp) m[d] = std::max(m[d], md[d]);
  }
  return m;
}

namespace {

// anchor displacement of a callsite: first output term (kernels, loads) or
// first input term (stores), nests.cpp:113-126
std::vector<int> displacement(const Rap& r, const DataflowDAG& g, size_t nd) {
  std::vector<int> d(nd, 0);
  int anchor = !r.out_terms.empty() ? r.out_terms[0] : (!r.in_terms.empty() ? r.in_terms[0] : -1);
  if (anchor >= 0)
    for (const auto& o : g.terms[anchor].dims) d[o.dim] = o.offset;
  return d;
}

// Shape key: callsites that differ only by a spatial displacement share it
// (R/SPEC.md:204-214, nests.cpp:117-143).  Unlike nests.cpp:134-141 only
// identifier bindings enter the key -- a loop variable bound at zero
// displacement does not -- so all instances of one kernel group together
// (fixes SURVEY.md Appendix B-1, which made the reference recompute lap1
// three times per cell).
std::string shape_key(const Rap& r, const DataflowDAG& g, size_t nd) {
  auto base = displacement(r, g, nd);
  std::ostringstream os;
  os << static_cast<int>(r.kind) << "|" << r.kernel << "|" << r.external;
  auto term = [&](int t) {
    const auto& ct = g.terms[t];
    os << "|" << ct.tag << ":" << ct.ident;
    for (const auto& o : ct.dims) os << "," << o.dim << "@" << (o.offset - base[o.dim]);
  };
  for (int t : r.in_terms) term(t);
  os << "|>";
  for (int t : r.out_terms) term(t);
  if (r.kind != RapKind::kernel) {
    os << "|ext";
    for (const auto& s : r.ext_slots) os << "," << s.dim << "@" << (s.dim >= 0 ? s.shift - base[s.dim] : s.shift);
  }
  for (const auto& [v, b] : r.binding)
    if (b.is_ident) os << "|b:" << v << "=" << b.ident;
  return os.str();
}

bool quotient_acyclic(const DataflowDAG& g, const std::vector<int>& gof, int ng) {
  std::vector<std::set<int>> adj(ng);
  std::vector<int> indeg(ng, 0);
  for (const auto& e : g.edges) {
    int a = gof[e.from], b = gof[e.to];
    if (a == b) {
      if (e.from != e.to) return false;
      continue;
    }
    if (adj[a].insert(b).second) ++indeg[b];
  }
  std::deque<int> q;
  for (int i = 0; i < ng; ++i)
    if (!indeg[i]) q.push_back(i);
  int seen = 0;
  while (!q.empty()) {
    int v = q.front();
    q.pop_front();
    ++seen;
    for (int w : adj[v])
      if (--indeg[w] == 0) q.push_back(w);
  }
  return seen == ng;
}

std::string hex64(uint64_t h) {
  char buf[17];
  std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(h));
  return buf;
}

struct Fnv {
  uint64_t h = 1469598103934665603ull;
  void add(const std::string& s) {
    for (unsigned char c : s) {
      h ^= c;
      h *= 1099511628211ull;
    }
    h ^= 0xff;
    h *= 1099511628211ull;
  }
  void add(long v) { add(std::to_string(v)); }
};

std::string json_str(const std::string& s) {
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

int elem_bytes_of(const std::string& type) {
  if (type.find("double") != std::string::npos) return 8;
  if (type.find("float") != std::string::npos) return 4;
  if (type.find("int64") != std::string::npos || type.find("long") != std::string::npos) return 8;
  if (type.find("int") != std::string::npos) return 4;
  return 8;
}

}  // namespace

std::optional<Plan> make_plan(const RuleSet& rs_in, DiagList& diags) {
  Plan P;
  P.rs = rs_in;
  const RuleSet& rs = P.rs;
  for (auto& d : validate_rules(rs)) diags.items.push_back(d);
  if (diags.has_errors()) return std::nullopt;
  auto dag = infer(rs, diags);
  if (!dag) return std::nullopt;
  P.dag = std::move(*dag);
  const DataflowDAG& g = P.dag;
  const size_t nd = rs.loop_order.size();

  // ---- grouping (nests.cpp:172-242 with the B-1 fix) ------------------------
  std::map<std::string, int> bucket_of;
  std::vector<std::vector<int>> buckets;
  for (const auto& r : g.raps) {
    std::string key = shape_key(r, g, nd);
    auto [it, fresh] = bucket_of.emplace(key, static_cast<int>(buckets.size()));
    if (fresh)
      buckets.push_back({r.id});
    else
      buckets[it->second].push_back(r.id);
  }
  auto assign = [&](std::vector<int>& gof) {
    gof.assign(g.raps.size(), -1);
    for (size_t b = 0; b < buckets.size(); ++b)
      for (int r : buckets[b]) gof[r] = static_cast<int>(b);
  };
  assign(P.group_of);
  while (!quotient_acyclic(g, P.group_of, static_cast<int>(buckets.size()))) {
    // degrade a multi-member bucket to singletons (R/SPEC.md:251)
    bool changed = false;
    for (size_t b = 0; b < buckets.size() && !changed; ++b) {
      if (buckets[b].size() < 2) continue;
      std::vector<std::vector<int>> nb;
      for (size_t h = 0; h < buckets.size(); ++h) {
        if (h == b)
          for (int r : buckets[h]) nb.push_back({r});
        else
          nb.push_back(buckets[h]);
      }
      buckets = std::move(nb);
      changed = true;
    }
    if (!changed) throw internal_error("grouping: cyclic quotient with singleton groups");
    assign(P.group_of);
  }
  for (size_t b = 0; b < buckets.size(); ++b) {
    CallsiteGroup cg;
    cg.id = static_cast<int>(b);
    const Rap& f = g.raps[buckets[b][0]];
    cg.kind = f.kind;
    cg.kernel = f.kernel;
    cg.external = f.external;
    cg.members = buckets[b];
    std::set<int> dims;
    for (int r : buckets[b]) {
      cg.member_disp.push_back(displacement(g.raps[r], g, nd));
      for (int t : g.raps[r].in_terms)
        for (const auto& o : g.terms[t].dims) dims.insert(o.dim);
      for (int t : g.raps[r].out_terms)
        for (const auto& o : g.terms[t].dims) dims.insert(o.dim);
    }
    cg.space.assign(dims.begin(), dims.end());
    P.groups.push_back(std::move(cg));
  }
  const size_t ng = P.groups.size();

  // ---- nest fusion (nests.cpp:294-315, fusion.cpp:8-372) --------------------
  const FusionResult fr = fuse_groups(rs, g, P.groups, P.group_of);
  P.nests = fr.nests;
  P.splits = fr.splits;
  P.one_nest = fr.nests == 1 && fr.splits == 0;
  P.vertex_of_group = fr.vertex_of_group;
  auto vertex_of_rap = [&](int rap) { return fr.vertex_of_group[P.group_of[rap]]; };

  // ---- pipeline shifts (shifts.cpp:8-79) --------------------------------------
  P.shifts.assign(ng, std::vector<int>(nd, 0));
  for (size_t gi = 0; gi < ng; ++gi) {
    if (P.groups[gi].kind == RapKind::load) continue;
    auto mx = P.groups[gi].max_disp(nd);
    for (size_t d = 0; d < nd; ++d) P.shifts[gi][d] = std::max(0, mx[d]);
  }
  auto member_delta = [&](int rap) {
    const auto& cg = P.groups[P.group_of[rap]];
    for (size_t m = 0; m < cg.members.size(); ++m)
      if (cg.members[m] == rap) return cg.member_disp[m];
    throw internal_error("rap missing from its group");
  };
  {
    std::vector<std::set<int>> gadj(ng);
    for (const auto& e : g.edges) {
      int gp = P.group_of[e.from], gc = P.group_of[e.to];
      if (gp == gc || g.raps[e.from].kind == RapKind::load) continue;
      if (vertex_of_rap(e.from) != vertex_of_rap(e.to)) continue;  // only intra-nest edges constrain
      gadj[gp].insert(gc);
    }
    std::vector<int> indeg(ng, 0);
    for (size_t gi = 0; gi < ng; ++gi)
      for (int c : gadj[gi]) ++indeg[c];
    std::deque<int> q;
    for (size_t gi = 0; gi < ng; ++gi)
      if (!indeg[gi]) q.push_back(static_cast<int>(gi));
    std::vector<int> order;
    while (!q.empty()) {
      int v = q.front();
      q.pop_front();
      order.push_back(v);
      for (int w : gadj[v])
        if (--indeg[w] == 0) q.push_back(w);
    }
    if (order.size() != ng) throw internal_error("cyclic group graph in shift computation");
    for (auto it = order.rbegin(); it != order.rend(); ++it) {
      int gi = *it;
      if (P.groups[gi].kind == RapKind::load) continue;
      for (const auto& e : g.edges) {
        if (P.group_of[e.from] != gi) continue;
        int gc = P.group_of[e.to];
        if (gc == gi) continue;
        if (vertex_of_rap(e.from) != vertex_of_rap(e.to)) continue;
        auto delta = member_delta(e.to);
        for (const auto& o : g.terms[e.term].dims) {
          int r = o.offset - delta[o.dim];
          P.shifts[gi][o.dim] = std::max(P.shifts[gi][o.dim], P.shifts[gc][o.dim] + r);
        }
      }
    }
  }

  // ---- variables, extents, contraction (storage.cpp:18-107, 206-427) ------------
  std::map<std::pair<std::string, std::string>, int> var_of;
  std::set<std::string> taken;
  for (const auto& a : rs.axioms) taken.insert(a.external.name);
  for (const auto& gl : rs.goals) taken.insert(gl.external.name);
  auto get_var = [&](const ConcreteTerm& t) {
    auto key = std::make_pair(t.tag, t.ident);
    auto it = var_of.find(key);
    if (it != var_of.end()) return it->second;
    Variable v;
    v.id = static_cast<int>(P.vars.size());
    v.tag = t.tag;
    v.ident = t.ident;
    std::string base = t.tag.empty() ? t.ident : t.tag + "_" + t.ident;
    v.name = base;
    for (int k = 2; taken.count(v.name); ++k) v.name = base + "_v" + std::to_string(k);
    taken.insert(v.name);
    v.type = "double";
    for (const auto& d : t.dims) v.dims.push_back(d.dim);
    var_of.emplace(key, v.id);
    P.vars.push_back(v);
    return v.id;
  };
  for (const auto& t : g.terms) P.var_of_term.push_back(get_var(t));
  for (const auto& r : g.raps) {
    if (r.kind == RapKind::load) {
      Variable& v = P.vars[get_var(g.terms[r.out_terms[0]])];
      if (v.external.empty()) {
        v.external = r.external;
        v.axiom_backed = true;
        for (const auto& ax : rs.axioms)
          if (ax.external.name == r.external) v.type = ax.external.type;
      }
    } else if (r.kind == RapKind::store) {
      Variable& v = P.vars[get_var(g.terms[r.in_terms[0]])];
      if (v.external.empty()) {
        v.external = r.external;  // write-through by the producer (storage.cpp:64-76)
        for (const auto& gl : rs.goals)
          if (gl.external.name == r.external) v.type = gl.external.type;
      }
    } else {
      const KernelRule& k = rs.kernels[r.kernel];
      DeclInfo decl = parse_declaration(k.declaration);
      for (size_t oi = 0; oi < k.outputs.size(); ++oi) {
        Variable& v = P.vars[get_var(g.terms[r.out_terms[oi]])];
        v.producer_group = P.group_of[r.id];
        if (v.external.empty())
          if (const DeclParam* p = decl.param(k.outputs[oi].first)) v.type = p->type;
      }
    }
  }
  // associative carry: the carry input and the output share one buffer
  // (storage.cpp:93-105)
  for (const auto& r : g.raps) {
    if (r.kind != RapKind::kernel || !rs.kernels[r.kernel].associative) continue;
    const ConcreteTerm& out = g.terms[r.out_terms[0]];
    const int vo = var_of.at({out.tag, out.ident});
    for (int t : r.in_terms) {
      const ConcreteTerm& ti = g.terms[t];
      if (ti.ident == out.ident && ti.dims == out.dims && !(ti == out)) {
        int vi = var_of.at({ti.tag, ti.ident});
        while (P.vars[vi].alias_of >= 0) vi = P.vars[vi].alias_of;
        int vc = vo;
        while (P.vars[vc].alias_of >= 0) vc = P.vars[vc].alias_of;
        if (vi != vc) P.vars[vi].alias_of = vc;
      }
    }
  }
  for (auto& v : P.vars) {
    std::vector<long> mn(nd, LONG_MAX), mx(nd, LONG_MIN), rmn(nd, LONG_MAX), rmx(nd, LONG_MIN);
    bool writes = false;
    std::set<int> vertices;  // fused nests touching the variable
    for (const auto& t : g.terms) {
      if (var_of.at({t.tag, t.ident}) != v.id) continue;
      for (const auto& o : t.dims) {
        mn[o.dim] = std::min<long>(mn[o.dim], o.offset);
        mx[o.dim] = std::max<long>(mx[o.dim], o.offset);
      }
    }
    // per-trip window of touched cells, shift-adjusted (storage.cpp:206-271)
    for (const auto& r : g.raps) {
      auto touch = [&](int t) {
        if (var_of.at({g.terms[t].tag, g.terms[t].ident}) != v.id) return;
        auto delta = member_delta(r.id);
        for (const auto& o : g.terms[t].dims) {
          long rel = P.shifts[P.group_of[r.id]][o.dim] + (o.offset - delta[o.dim]);
          rmn[o.dim] = std::min(rmn[o.dim], rel);
          rmx[o.dim] = std::max(rmx[o.dim], rel);
        }
      };
      for (int t : r.out_terms)
        if (var_of.at({g.terms[t].tag, g.terms[t].ident}) == v.id) vertices.insert(vertex_of_rap(r.id));
      for (int t : r.in_terms)
        if (var_of.at({g.terms[t].tag, g.terms[t].ident}) == v.id) vertices.insert(vertex_of_rap(r.id));
      if (r.kind == RapKind::load) continue;
      for (int t : r.in_terms) touch(t);
      for (int t : r.out_terms) {
        if (var_of.at({g.terms[t].tag, g.terms[t].ident}) == v.id) writes = true;
        touch(t);
      }
    }
    {
      // a is visited before b iff offset(a) >lex offset(b): the path is the
      // distinct read offsets in descending lexicographic order
      std::set<std::vector<int>> reads;
      for (const auto& r : g.raps)
        for (int t : r.in_terms) {
          const auto& ct = g.terms[t];
          if (var_of.at({ct.tag, ct.ident}) != v.id) continue;
          std::vector<int> off(nd, 0);
          for (const auto& o : ct.dims) off[o.dim] = o.offset;
          reads.insert(off);
        }
      std::string path;
      for (auto it = reads.rbegin(); it != reads.rend(); ++it) {
        if (!path.empty()) path += " -> ";
        path += "(";
        for (size_t k = it->size(); k-- > 0;) {
          path += ((*it)[k] > 0 ? "+" : "") + std::to_string((*it)[k]);
          if (k) path += ",";
        }
        path += ")";
      }
      v.reuse_path = path;
    }
    v.extents.clear();
    v.spans.clear();
    for (int d : v.dims) {
      long lo = mn[d] == LONG_MAX ? 0 : mn[d], hi = mx[d] == LONG_MIN ? 0 : mx[d];
      v.extents.emplace_back(rs.ranges[d].trips() + (hi - lo), rs.ranges[d].lo + lo);
      long agg = hi - lo + 1;
      long win = rmn[d] == LONG_MAX ? 1 : rmx[d] - rmn[d] + 1;
      v.spans.push_back(std::max(agg, win));
    }
    if (!v.external.empty()) {
      v.scheme = Scheme::terminal;
    } else if (!writes || vertices.size() > 1) {
      v.scheme = Scheme::full;  // crosses a split: lives across nests (storage.cpp:325-329)
    } else {
      v.rotating_dim = -1;
      for (size_t k = 0; k < v.dims.size(); ++k)
        if (v.spans[k] > 1) {
          v.rotating_dim = v.dims[k];
          v.span = v.spans[k];
          break;
        }
      if (v.rotating_dim < 0) {
        v.scheme = Scheme::scalar;
      } else {
        bool inner_full = false;
        for (size_t k = 0; k < v.dims.size(); ++k)
          if (v.dims[k] > v.rotating_dim) inner_full = true;
        v.scheme = inner_full ? Scheme::outer_rotate : Scheme::inner_circular;
      }
    }
  }

  // ---- terminals (axioms then goals: the emitted function's parameter order,
  // R/SPEC.md:500) ---------------------------------------------------------------
  auto add_terminal = [&](const ExternalDecl& e, const TermPattern& term, bool goal) {
    Terminal T;
    T.name = e.name;
    T.type = e.type;
    T.is_goal = goal;
    T.elem_bytes = elem_bytes_of(e.type);
    for (const auto& v : P.vars)
      if (v.external == e.name && (goal ? !v.axiom_backed : v.axiom_backed)) T.var = v.id;
    if (T.var < 0)  // declared but unused axiom: its own pattern's ident
      for (const auto& v : P.vars)
        if (v.ident == term.ident && v.tag == term.tag) T.var = v.id;
    for (const auto& s : e.subscripts) {
      int d = rs.dim_of(s.base_name());
      if (d < 0 && s.is_free()) {
        // axiom subscripts bind through the term pattern's free variables
        for (size_t k = 0; k < term.subscripts.size(); ++k)
          if (term.subscripts[k].var == s.var) d = rs.dim_of(term.subscripts[k].base_name());
      }
      T.dims.push_back(d);
    }
    if (T.var >= 0) {
      const Variable& v = P.vars[T.var];
      for (int d : T.dims) {
        long ext = d >= 0 ? rs.ranges[d].trips() : 1, base = d >= 0 ? rs.ranges[d].lo : 0;
        for (size_t k = 0; k < v.dims.size(); ++k)
          if (v.dims[k] == d) {
            ext = v.extents[k].first;
            base = v.extents[k].second;
          }
        T.extent.push_back(ext);
        T.base.push_back(base);
      }
    }
    P.terminals.push_back(std::move(T));
  };
  for (const auto& a : rs.axioms) add_terminal(a.external, a.term, false);
  for (const auto& gl : rs.goals) add_terminal(gl.external, gl.term, true);
  // iterated goals take their axiom's layout so the two buffers ping-pong
  for (const auto& [gname, aname] : rs.iterate) {
    Terminal* gt = nullptr;
    const Terminal* at = nullptr;
    for (auto& t : P.terminals) {
      if (t.is_goal && t.name == gname) gt = &t;
      if (!t.is_goal && t.name == aname) at = &t;
    }
    if (!gt || !at) continue;
    if (gt->dims != at->dims || gt->elem_bytes != at->elem_bytes) {
      diags.error({}, "iterate pair [" + gname + ", " + aname + "] has mismatched dimensions or element types");
      return std::nullopt;
    }
    gt->extent = at->extent;
    gt->base = at->base;
  }
  P.halo_lo.assign(nd, 0);
  P.halo_hi.assign(nd, 0);
  for (const auto& t : P.terminals) {
    if (t.is_goal) continue;
    for (size_t k = 0; k < t.dims.size(); ++k) {
      int d = t.dims[k];
      if (d < 0) continue;
      long lo = rs.ranges[d].lo - t.base[k];
      long hi = (t.base[k] + t.extent[k]) - (rs.ranges[d].lo + rs.ranges[d].trips());
      P.halo_lo[d] = std::max<int>(P.halo_lo[d], static_cast<int>(lo));
      P.halo_hi[d] = std::max<int>(P.halo_hi[d], static_cast<int>(hi));
    }
  }

  // ---- alias chain and shadow windows (storage.cpp:453-524, 544-594) ----------
  for (const auto& [in_ext, out_ext] : rs.aliases) {
    std::set<int> start, target;
    for (const auto& r : g.raps) {
      if (r.kind == RapKind::load && r.external == in_ext) start.insert(r.id);
      if (r.kind == RapKind::store && r.external == out_ext) target.insert(r.id);
    }
    if (start.empty() || target.empty()) continue;
    std::set<int> reach;
    std::vector<int> stack(start.begin(), start.end());
    while (!stack.empty()) {
      const int r = stack.back();
      stack.pop_back();
      if (!reach.insert(r).second) continue;
      for (int w : g.out_adj[r]) stack.push_back(w);
    }
    bool interdependent = false;
    for (int t : target) interdependent |= reach.count(t) > 0;
    if (!interdependent) continue;
    for (int t : target) {
      const Rap& st = g.raps[t];
      const auto& sterm = g.terms[st.in_terms[0]];
      const int sv = var_of.at({sterm.tag, sterm.ident});
      // write-through producer, or the store itself when it materialises a copy
      const int writer = (P.vars[sv].external == out_ext && !P.vars[sv].axiom_backed && P.vars[sv].producer_group >= 0)
                             ? P.vars[sv].producer_group
                             : P.group_of[t];
      const auto& sw = P.shifts[writer];
      AliasEntry e;
      e.input = in_ext;
      e.output = out_ext;
      e.writer_group = writer;
      e.writer_shift = sw;
      std::set<std::vector<int>> offs;
      for (const auto& r : g.raps) {
        if (r.kind == RapKind::load) continue;
        for (int in : r.in_terms) {
          const auto& ct = g.terms[in];
          const int rv = var_of.at({ct.tag, ct.ident});
          if (!P.vars[rv].axiom_backed || P.vars[rv].external != in_ext) continue;
          e.var = rv;
          const auto delta = member_delta(r.id);
          const auto& sc = P.shifts[P.group_of[r.id]];
          std::vector<int> eff(nd, 0);
          for (const auto& o : ct.dims) eff[o.dim] = sc[o.dim] + (o.offset - delta[o.dim]) - sw[o.dim];
          if (eff <= std::vector<int>(nd, 0)) offs.insert(eff);  // read at or after the write trip
        }
      }
      if (e.var < 0 || offs.empty()) continue;
      e.offsets.assign(offs.rbegin(), offs.rend());
      // shadow covering the clobbered window
      Shadow sh;
      sh.var = e.var;
      const auto& vd = P.vars[e.var].dims;
      std::map<int, std::pair<int, int>> win;
      for (int d : vd) win[d] = {0, 0};
      for (const auto& o : e.offsets)
        for (int d : vd) {
          win[d].first = std::min(win[d].first, o[d]);
          win[d].second = std::max(win[d].second, o[d]);
        }
      int rot = -1;
      for (int d : vd)
        if (win[d].second - win[d].first + 1 > 1) {
          rot = d;
          break;
        }
      for (int d : vd) sh.spans.push_back(win[d].second - win[d].first + 1);
      sh.dims = vd;
      sh.rotating = rot;
      if (rot < 0) {
        sh.scheme = vd.empty() ? Scheme::full : Scheme::inner_circular;
        if (!vd.empty()) sh.spans.back() = 1;
      } else {
        bool inner_full = false;
        for (int d : vd) inner_full |= d > rot;
        sh.scheme = inner_full ? Scheme::outer_rotate : Scheme::inner_circular;
      }
      P.alias.push_back(std::move(e));
      P.shadows.push_back(std::move(sh));
    }
  }

  // ---- footprint polynomial (storage.cpp:161-190, 596-626) --------------------
  {
    std::map<std::vector<int>, long> terms;
    std::set<std::string> counted;
    for (const auto& v : P.vars) {
      if (v.alias_of >= 0) continue;
      std::vector<int> mono;
      long coeff = 1;
      if (v.scheme == Scheme::terminal) {
        if (!counted.insert(v.external).second) continue;
        mono = v.dims;
      } else if (v.scheme == Scheme::full) {
        mono = v.dims;
      } else if (v.scheme == Scheme::scalar) {
      } else {
        for (size_t k = 0; k < v.dims.size(); ++k) {
          if (v.dims[k] == v.rotating_dim)
            coeff *= v.spans[k];
          else if (v.dims[k] > v.rotating_dim)
            mono.push_back(v.dims[k]);
        }
      }
      std::sort(mono.begin(), mono.end());
      terms[mono] += coeff;
    }
    // shadow windows of in-place aliases (storage.cpp:617-625)
    for (const auto& sh : P.shadows) {
      std::vector<int> mono;
      long coeff = 1;
      for (size_t k = 0; k < sh.dims.size(); ++k) {
        if (sh.dims[k] == sh.rotating) coeff *= sh.spans[k];
        else if (sh.rotating >= 0 && sh.dims[k] > sh.rotating) mono.push_back(sh.dims[k]);
      }
      std::sort(mono.begin(), mono.end());
      terms[mono] += coeff;
    }
    std::vector<std::pair<std::vector<int>, long>> ord(terms.begin(), terms.end());
    std::sort(ord.begin(), ord.end(), [](const auto& a, const auto& b) {
      if (a.first.size() != b.first.size()) return a.first.size() > b.first.size();
      return a.first < b.first;
    });
    std::string s;
    for (const auto& [mono, c] : ord) {
      if (!c) continue;
      if (!s.empty()) s += " + ";
      std::string m;
      for (int d : mono) m += (m.empty() ? "" : "*") + std::string("N_") + rs.loop_order[d];
      s += m.empty() ? std::to_string(c) : (c == 1 ? m : std::to_string(c) + "*" + m);
    }
    P.footprint = s.empty() ? "0" : s;
  }

  // ---- canonical chain signature ---------------------------------------------
  // Hash of the computation independent of rule/variable/terminal names: each
  // intermediate is named by its producing function, output slot and the
  // canonical names of its inputs with offsets relative to the producer's
  // anchor; terminals by position and element type.
  {
    std::vector<std::string> canon(P.vars.size());
    std::vector<char> busy(P.vars.size(), 0);
    std::function<std::string(int)> name_of = [&](int vid) -> std::string {
      if (!canon[vid].empty()) return canon[vid];
      if (busy[vid]) throw internal_error("cyclic variable derivation in signature");
      busy[vid] = 1;
      const Variable& v = P.vars[vid];
      Fnv h;
      if (v.axiom_backed) {
        int idx = 0;
        for (size_t a = 0; a < rs.axioms.size(); ++a)
          if (rs.axioms[a].external.name == v.external) idx = static_cast<int>(a);
        h.add("A");
        h.add(idx);
        h.add(v.type);
        for (int d : v.dims) h.add(d);
      } else {
        // any producing rap (all instances share the shape)
        const Rap* pr = nullptr;
        size_t oslot = 0;
        for (const auto& r : g.raps) {
          if (r.kind != RapKind::kernel) continue;
          for (size_t oi = 0; oi < r.out_terms.size(); ++oi)
            if (var_of.at({g.terms[r.out_terms[oi]].tag, g.terms[r.out_terms[oi]].ident}) == vid) {
              pr = &r;
              oslot = oi;
            }
          if (pr) break;
        }
        if (!pr) throw internal_error("variable without producer in signature");
        const KernelRule& k = rs.kernels[pr->kernel];
        DeclInfo di = parse_declaration(k.declaration);
        h.add("K");
        h.add(di.function);
        for (const auto& p : di.params) h.add(p.type + (p.pointer ? "*" : "") + (p.reference ? "&" : ""));
        h.add(static_cast<long>(oslot));
        h.add(v.type);
        auto anchor = displacement(*pr, g, nd);
        for (int t : pr->in_terms) {
          const auto& ct = g.terms[t];
          h.add(name_of(var_of.at({ct.tag, ct.ident})));
          for (const auto& o : ct.dims) {
            h.add(o.dim);
            h.add(static_cast<long>(o.offset - anchor[o.dim]));
          }
        }
      }
      busy[vid] = 0;
      canon[vid] = hex64(h.h);
      return canon[vid];
    };
    Fnv h;
    h.add(static_cast<long>(nd));
    for (const auto& t : P.terminals) {
      h.add(t.is_goal ? "G" : "A");
      h.add(t.type);
      h.add(static_cast<long>(t.dims.size()));
      for (int d : t.dims) h.add(d);
      if (t.var >= 0 && t.is_goal) h.add(name_of(t.var));
    }
    for (const auto& [gname, aname] : rs.iterate) {
      h.add("I");
      for (size_t i = 0; i < P.terminals.size(); ++i)
        if (P.terminals[i].name == gname || P.terminals[i].name == aname) h.add(static_cast<long>(i));
    }
    for (const auto& t : P.terminals) {
      auto it = rs.boundary.find(t.name);
      if (it == rs.boundary.end()) it = rs.boundary.find("*");
      h.add("B");
      if (it != rs.boundary.end())
        for (Boundary b : it->second) h.add(boundary_name(b));
    }
    P.signature = hex64(h.h);
  }
  return P;
}

std::string Plan::report_json() const {
  std::ostringstream os;
  const size_t nd = rs.loop_order.size();
  os << "{\"name\":" << json_str(rs.name) << ",\"loop_order\":[";
  for (size_t d = 0; d < nd; ++d) os << (d ? "," : "") << json_str(rs.loop_order[d]);
  os << "],\"ranges\":[";
  for (size_t d = 0; d < nd; ++d)
    os << (d ? "," : "") << "[" << rs.ranges[d].lo << "," << rs.ranges[d].hi << "," << rs.ranges[d].stride << "]";
  size_t nk = 0, nl = 0, ns = 0;
  for (const auto& r : dag.raps) (r.kind == RapKind::kernel ? nk : r.kind == RapKind::load ? nl : ns)++;
  os << "],\"terms\":" << dag.terms.size() << ",\"raps\":" << dag.raps.size() << ",\"kernel_raps\":" << nk
     << ",\"load_raps\":" << nl << ",\"store_raps\":" << ns << ",\"edges\":" << dag.edges.size()
     << ",\"groups\":[";
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    const auto& cg = groups[gi];
    std::string nm = cg.kind == RapKind::kernel ? rs.kernels[cg.kernel].name
                                                : (cg.kind == RapKind::load ? "load " : "store ") + cg.external;
    os << (gi ? "," : "") << "{\"name\":" << json_str(nm) << ",\"members\":" << cg.members.size()
       << ",\"nest\":" << (gi < vertex_of_group.size() ? vertex_of_group[gi] : -1) << ",\"space\":[";
    for (size_t k = 0; k < cg.space.size(); ++k) os << (k ? "," : "") << cg.space[k];
    os << "],\"shift\":[";
    for (size_t d = 0; d < nd; ++d) os << (d ? "," : "") << shifts[gi][d];
    os << "]}";
  }
  os << "],\"nests\":" << nests << ",\"splits\":" << splits << ",\"one_nest\":" << (one_nest ? "true" : "false")
     << ",\"variables\":[";
  for (size_t i = 0; i < vars.size(); ++i) {
    const auto& v = vars[i];
    os << (i ? "," : "") << "{\"name\":" << json_str(v.name) << ",\"type\":" << json_str(v.type)
       << ",\"scheme\":" << json_str(scheme_name(v.scheme)) << ",\"span\":" << v.span << ",\"rotating_dim\":"
       << v.rotating_dim << ",\"alias_of\":" << v.alias_of << ",\"reuse_path\":" << json_str(v.reuse_path)
       << ",\"external\":" << json_str(v.external)
       << ",\"extents\":[";
    for (size_t k = 0; k < v.extents.size(); ++k)
      os << (k ? "," : "") << "[" << v.extents[k].first << "," << v.extents[k].second << "]";
    os << "],\"spans\":[";
    for (size_t k = 0; k < v.spans.size(); ++k) os << (k ? "," : "") << v.spans[k];
    os << "]}";
  }
  os << "],\"terminals\":[";
  for (size_t i = 0; i < terminals.size(); ++i) {
    const auto& t = terminals[i];
    os << (i ? "," : "") << "{\"name\":" << json_str(t.name) << ",\"type\":" << json_str(t.type)
       << ",\"goal\":" << (t.is_goal ? "true" : "false") << ",\"elem_bytes\":" << t.elem_bytes << ",\"dims\":[";
    for (size_t k = 0; k < t.dims.size(); ++k) os << (k ? "," : "") << t.dims[k];
    os << "],\"extent\":[";
    for (size_t k = 0; k < t.extent.size(); ++k) os << (k ? "," : "") << t.extent[k];
    os << "],\"base\":[";
    for (size_t k = 0; k < t.base.size(); ++k) os << (k ? "," : "") << t.base[k];
    os << "]}";
  }
  os << "],\"halo_lo\":[";
  for (size_t d = 0; d < nd; ++d) os << (d ? "," : "") << halo_lo[d];
  os << "],\"halo_hi\":[";
  for (size_t d = 0; d < nd; ++d) os << (d ? "," : "") << halo_hi[d];
  os << "],\"alias\":[";
  for (size_t k = 0; k < alias.size(); ++k) {
    const auto& e = alias[k];
    const auto& wg = groups[e.writer_group];
    std::string wn = wg.kind == RapKind::kernel ? rs.kernels[wg.kernel].name
                                                : (wg.kind == RapKind::load ? "load " : "store ") + wg.external;
    os << (k ? "," : "") << "{\"input\":" << json_str(e.input) << ",\"output\":" << json_str(e.output)
       << ",\"var\":" << json_str(vars[e.var].name) << ",\"writer\":" << json_str(wn) << ",\"writer_shift\":[";
    for (size_t d = 0; d < e.writer_shift.size(); ++d) os << (d ? "," : "") << e.writer_shift[d];
    os << "],\"offsets\":[";
    for (size_t o = 0; o < e.offsets.size(); ++o) {
      os << (o ? "," : "") << "[";
      for (size_t d = 0; d < e.offsets[o].size(); ++d) os << (d ? "," : "") << e.offsets[o][d];
      os << "]";
    }
    os << "],\"shadow\":{\"scheme\":" << json_str(scheme_name(shadows[k].scheme)) << ",\"spans\":[";
    for (size_t d = 0; d < shadows[k].spans.size(); ++d) os << (d ? "," : "") << shadows[k].spans[d];
    os << "]}}";
  }
  os << "],\"footprint\":" << json_str(footprint) << ",\"signature\":" << json_str(signature) << "}";
  return os.str();
}

}  // namespace lf

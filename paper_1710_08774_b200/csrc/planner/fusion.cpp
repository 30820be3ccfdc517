// Iteration nests and their fusion -- the reference's nests + fusion modules
// restated (nests.cpp:294-315, fusion.cpp:8-372; R/PAPER.md:211-252 Listings
// `code:inest-dag-fusion` / `code:inest-fusion`; R/SPEC.md:268-347).
//
// One perfect nest per callsite group; nests are fused along the quotient of
// the dataflow DAG in topological order, a pair at a time, until a fixed
// point.  Equal-rank nests fuse phase by phase under the four dataflow
// guards; a lower-rank nest fuses into the higher one's prologue (preferred)
// or epilogue.  A reduction whose value is broadcast back up (concave
// dataflow) forces a split; a failed fusion severs the edges into everything
// downstream of the candidate.
#include <algorithm>
#include <climits>
#include <deque>
#include <functional>
#include <map>

#include "fusion.hpp"

namespace lf {

namespace {

NestP leaf(std::vector<int> raps) {
  auto n = std::make_shared<Nest>();
  n->leaf = true;
  n->body = std::move(raps);
  return n;
}

NestP loop(int dim, Range r, NestP pro, NestP steady, NestP epi) {
  if (!steady) throw internal_error("loop nest requires a steady-state child");
  auto n = std::make_shared<Nest>();
  n->dim = dim;
  n->range = r;
  n->pro = std::move(pro);
  n->steady = std::move(steady);
  n->epi = std::move(epi);
  return n;
}

void collect(const NestP& n, std::set<int>& out) {
  if (!n) return;
  if (n->leaf) {
    out.insert(n->body.begin(), n->body.end());
    return;
  }
  collect(n->pro, out);
  collect(n->steady, out);
  collect(n->epi, out);
}

std::set<int> raps_of(const NestP& n) {
  std::set<int> s;
  collect(n, s);
  return s;
}

std::set<int> minus(std::set<int> a, const std::set<int>& b) {
  for (int x : b) a.erase(x);
  return a;
}

int rank_of(const NestP& n, int nd) { return (!n || n->leaf) ? -1 : nd - 1 - n->dim; }

}  // namespace

RapClass classify_rap(const Rap& r, const DataflowDAG& g) {
  if (r.in_terms.empty()) return RapClass::pointwise;
  int out_rank = 0, in_max = 0, in_min = INT_MAX;
  for (int t : r.out_terms) out_rank = std::max<int>(out_rank, g.terms[t].dims.size());
  for (int t : r.in_terms) {
    in_max = std::max<int>(in_max, g.terms[t].dims.size());
    in_min = std::min<int>(in_min, g.terms[t].dims.size());
  }
  if (in_max > out_rank) return RapClass::reduction;
  if (in_min < out_rank) return RapClass::broadcast;
  return RapClass::pointwise;
}

// Pairwise fusion (fusion.cpp:113-167).
NestP fuse_nests(const NestP& a, const NestP& b, const DataflowDAG& g, int nd) {
  if (!a) return b;
  if (!b) return a;
  if (a->leaf && b->leaf) {  // one trip's statements; order fixed at lowering
    std::vector<int> body = a->body;
    body.insert(body.end(), b->body.begin(), b->body.end());
    return leaf(std::move(body));
  }
  const int ra = rank_of(a, nd), rb = rank_of(b, nd);
  if (ra == rb) {
    if (!(a->range == b->range)) return nullptr;
    const auto sa = raps_of(a->steady), sb = raps_of(b->steady);
    const auto pa = minus(raps_of(a->pro), sa), pb = minus(raps_of(b->pro), sb);
    const auto ea = minus(raps_of(a->epi), sa), eb = minus(raps_of(b->epi), sb);
    if (!(dataflow_le(pa, sb, g) && dataflow_le(pb, sa, g) && dataflow_le(sa, eb, g) && dataflow_le(sb, ea, g)))
      return nullptr;
    NestP p = fuse_nests(a->pro, b->pro, g, nd);
    if (a->pro && b->pro && !p) return nullptr;
    NestP s = fuse_nests(a->steady, b->steady, g, nd);
    if (!s) return nullptr;
    NestP e = fuse_nests(a->epi, b->epi, g, nd);
    if (a->epi && b->epi && !e) return nullptr;
    return loop(a->dim, a->range, p, s, e);
  }
  // differing ranks: the lower nest joins the higher one's prologue (preferred)
  // or epilogue, as dataflow allows
  const NestP lo = ra < rb ? a : b, hi = ra < rb ? b : a;
  const auto lset = raps_of(lo);
  const bool before = dataflow_le(lset, raps_of(hi->steady), g);
  const bool after = dataflow_le(raps_of(hi->epi), lset, g) && dataflow_le(raps_of(hi->steady), lset, g);
  if (before)
    if (NestP p = fuse_nests(hi->pro, lo, g, nd)) return loop(hi->dim, hi->range, p, hi->steady, hi->epi);
  if (after)
    if (NestP e = fuse_nests(hi->epi, lo, g, nd)) return loop(hi->dim, hi->range, hi->pro, hi->steady, e);
  return nullptr;
}

FusionResult fuse_groups(const RuleSet& rs, const DataflowDAG& g, const std::vector<CallsiteGroup>& groups,
                         const std::vector<int>& group_of) {
  const int nd = static_cast<int>(rs.loop_order.size());
  const int nv = static_cast<int>(groups.size());
  // ---- initial nests: one perfect nest per group over its space (nests.cpp:294-315)
  std::vector<NestP> nest(nv);
  for (int v = 0; v < nv; ++v) {
    NestP n = leaf(groups[v].members);
    for (auto it = groups[v].space.rbegin(); it != groups[v].space.rend(); ++it)
      n = loop(*it, rs.ranges[*it], nullptr, n, nullptr);
    nest[v] = n;
  }
  struct Edge {
    int from, to;
    std::set<int> terms;
  };
  std::vector<Edge> edges;
  {
    std::map<std::pair<int, int>, std::set<int>> q;
    for (const auto& e : g.edges) {
      int a = group_of[e.from], b = group_of[e.to];
      if (a != b) q[{a, b}].insert(e.term);
    }
    for (auto& [k, t] : q) edges.push_back({k.first, k.second, t});
  }

  // ---- concave splits: reductions broadcast back up (fusion.cpp:23-95)
  FusionResult res;
  std::set<size_t> severed;
  std::set<std::pair<int, int>> forbidden;  // initial vertex pairs kept apart
  {
    std::vector<std::vector<int>> adj(nv);
    for (const auto& e : edges) adj[e.from].push_back(e.to);
    auto out_rank = [&](const Rap& r) {
      int m = 0;
      for (int t : r.out_terms) m = std::max<int>(m, g.terms[t].dims.size());
      return m;
    };
    for (const auto& red : g.raps) {
      if (classify_rap(red, g) != RapClass::reduction) continue;
      const int reduced = out_rank(red);
      std::vector<char> seen(g.raps.size(), 0);
      std::vector<int> st(g.out_adj[red.id].begin(), g.out_adj[red.id].end()), bcast;
      while (!st.empty()) {
        int v = st.back();
        st.pop_back();
        if (seen[v]) continue;
        seen[v] = 1;
        if (classify_rap(g.raps[v], g) == RapClass::broadcast && out_rank(g.raps[v]) > reduced) bcast.push_back(v);
        for (int w : g.out_adj[v]) st.push_back(w);
      }
      if (bcast.empty()) continue;
      std::vector<char> down(nv, 0);
      std::vector<int> vs;
      for (int b : bcast) vs.push_back(group_of[b]);
      while (!vs.empty()) {
        int v = vs.back();
        vs.pop_back();
        if (down[v]) continue;
        down[v] = 1;
        for (int w : adj[v]) vs.push_back(w);
      }
      ++res.splits;
      for (size_t i = 0; i < edges.size(); ++i)
        if (!down[edges[i].from] && down[edges[i].to]) {
          severed.insert(i);
          forbidden.insert({edges[i].from, edges[i].to});
        }
    }
  }

  // ---- fixed-point driver over the quotient DAG (fusion.cpp:171-372)
  std::vector<int> parent(nv);
  for (int v = 0; v < nv; ++v) parent[v] = v;
  std::function<int(int)> find = [&](int v) { return parent[v] == v ? v : parent[v] = find(parent[v]); };
  struct QEdge {
    int from, to;
    int first_term;
    std::vector<size_t> orig;
  };
  auto quotient = [&] {
    std::map<std::pair<int, int>, size_t> idx;
    std::vector<QEdge> q;
    for (size_t i = 0; i < edges.size(); ++i) {
      int a = find(edges[i].from), b = find(edges[i].to);
      if (a == b) continue;
      auto [it, fresh] = idx.emplace(std::make_pair(a, b), q.size());
      if (fresh) q.push_back({a, b, INT_MAX, {}});
      q[it->second].first_term = std::min(q[it->second].first_term, *edges[i].terms.begin());
      q[it->second].orig.push_back(i);
    }
    return q;
  };
  auto topo = [&](const std::vector<QEdge>& q) {
    std::set<int> roots;
    for (int v = 0; v < nv; ++v) roots.insert(find(v));
    std::map<int, int> indeg;
    std::map<int, std::vector<int>> adj;
    for (int r : roots) indeg[r] = 0;
    for (const auto& e : q) {
      adj[e.from].push_back(e.to);
      ++indeg[e.to];
    }
    std::deque<int> ready;
    for (int r : roots)
      if (!indeg[r]) ready.push_back(r);
    std::vector<int> order;
    while (!ready.empty()) {
      int v = ready.front();
      ready.pop_front();
      order.push_back(v);
      for (int w : adj[v])
        if (--indeg[w] == 0) ready.push_back(w);
    }
    if (order.size() != roots.size()) throw internal_error("fusion introduced a cycle in the iteration nest DAG");
    return order;
  };
  auto reaches = [&](int from, int to, const std::vector<QEdge>& q, int skip_direct_to) {
    std::map<int, std::vector<int>> adj;
    for (const auto& e : q) adj[e.from].push_back(e.to);
    std::vector<int> st;
    for (int w : adj[from])
      if (w != skip_direct_to) st.push_back(w);
    std::set<int> seen;
    while (!st.empty()) {
      int v = st.back();
      st.pop_back();
      if (!seen.insert(v).second) continue;
      if (v == to) return true;
      for (int w : adj[v]) st.push_back(w);
    }
    return false;
  };
  auto pair_forbidden = [&](int a, int b) {
    for (const auto& [x, y] : forbidden) {
      int fx = find(x), fy = find(y);
      if ((fx == a && fy == b) || (fx == b && fy == a)) return true;
    }
    return false;
  };
  bool changed = true;
  while (changed) {
    changed = false;
    const auto q = quotient();
    const auto order = topo(q);
    std::map<int, int> tix;
    for (size_t i = 0; i < order.size(); ++i) tix[order[i]] = static_cast<int>(i);
    for (int vert : order) {
      std::vector<const QEdge*> in;
      for (const auto& e : q)
        if (e.to == vert) in.push_back(&e);
      std::sort(in.begin(), in.end(), [&](const QEdge* x, const QEdge* y) {
        if (tix[x->from] != tix[y->from]) return tix[x->from] < tix[y->from];
        return x->first_term < y->first_term;
      });
      for (const QEdge* e : in) {
        const int src = find(e->from), dst = find(vert);
        if (src == dst) continue;
        bool cut = false;
        for (size_t i : e->orig) cut |= severed.count(i) > 0;
        if (cut || pair_forbidden(src, dst)) continue;
        if (reaches(src, dst, q, dst)) continue;  // merging would close a cycle: stays an edge
        NestP f = fuse_nests(nest[dst], nest[src], g, nd);
        if (!f) {
          // unfusable: sever every edge into the subgraph below the candidate
          std::map<int, std::vector<int>> adj;
          for (const auto& qe : q) adj[qe.from].push_back(qe.to);
          std::set<int> down;
          std::vector<int> st{dst};
          while (!st.empty()) {
            int v = st.back();
            st.pop_back();
            if (!down.insert(v).second) continue;
            for (int w : adj[v]) st.push_back(w);
          }
          for (size_t i = 0; i < edges.size(); ++i) {
            int a = find(edges[i].from), b = find(edges[i].to);
            if (a != b && !down.count(a) && down.count(b)) {
              severed.insert(i);
              forbidden.insert({edges[i].from, edges[i].to});
            }
          }
          continue;
        }
        parent[src] = dst;
        nest[dst] = f;
        changed = true;
        break;
      }
      if (changed) break;
    }
  }
  const auto q = quotient();
  const auto order = topo(q);
  std::map<int, int> fin;
  for (size_t i = 0; i < order.size(); ++i) fin[order[i]] = static_cast<int>(i);
  for (int r : order) res.vertices.push_back(nest[r]);
  res.vertex_of_group.resize(nv);
  for (int v = 0; v < nv; ++v) res.vertex_of_group[v] = fin[find(v)];
  res.nests = static_cast<int>(order.size());
  return res;
}

bool is_perfect(const NestP& n) {
  if (!n || n->leaf) return true;
  return !n->pro && !n->epi && is_perfect(n->steady);
}

}  // namespace lf

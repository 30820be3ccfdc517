// loomfuse-b200 host planner: the reference's rules/axioms/goals front end and
// the bookkeeping half of its analysis pipeline, restated in C++20 for the
// B200 executors.  Behaviour follows the reference module by module; every
// function cites the reference code it mirrors.  No CUDA in here.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

namespace lf {

// ---------------------------------------------------------------- diagnostics
// Position-annotated diagnostics, as diag.hpp:10-64 of the reference.
struct SourceLoc {
  std::string file;
  int line = 0;
  int column = 0;
  std::string str() const;
};

struct Diagnostic {
  bool error = true;
  SourceLoc loc;
  std::string message;
  std::string str() const;
};

struct DiagList {
  std::vector<Diagnostic> items;
  void error(SourceLoc loc, std::string msg) { items.push_back({true, std::move(loc), std::move(msg)}); }
  void warning(SourceLoc loc, std::string msg) { items.push_back({false, std::move(loc), std::move(msg)}); }
  bool has_errors() const;
  std::string str() const;
};

// Contract violations (reference: `internal_error`, diag.hpp:68-70).
struct internal_error : std::logic_error {
  using std::logic_error::logic_error;
};

// ------------------------------------------------------------- YAML subset
// yaml-cpp is absent from this image; the rule format only
// needs block maps, block sequences, `|` literals, flow sequences/maps and
// plain/quoted scalars.
struct YNode {
  enum Kind { Null, Scalar, Map, Seq } kind = Null;
  std::string scalar;
  std::vector<std::pair<std::string, YNode>> map;
  std::vector<YNode> seq;
  int line = 0;    // 1-based line of the node's first character
  int column = 0;  // 1-based
  bool literal = false;  // came from a `|` block scalar
  const YNode* get(const std::string& key) const;
};

std::optional<YNode> yaml_parse(const std::string& text, const std::string& file, DiagList& diags);

// ------------------------------------------------------------- rule spec
// Types mirror rulespec.hpp:13-128.
struct OffsetExpr {
  std::string var;  // keeps the trailing '?' of free variables
  int displacement = 0;
  bool is_free() const { return !var.empty() && var.back() == '?'; }
  std::string base_name() const { return is_free() ? var.substr(0, var.size() - 1) : var; }
  bool operator==(const OffsetExpr&) const = default;
};

struct TermPattern {
  std::string tag;
  std::string ident;
  std::vector<OffsetExpr> subscripts;
  SourceLoc loc;
  bool ident_is_free() const { return !ident.empty() && ident.back() == '?'; }
  std::string str() const;
  bool operator==(const TermPattern& o) const {
    return tag == o.tag && ident == o.ident && subscripts == o.subscripts;
  }
};

struct KernelRule {
  std::string name;
  std::string declaration;
  bool associative = false;
  std::vector<std::string> params;
  std::vector<std::pair<std::string, TermPattern>> inputs;
  std::vector<std::pair<std::string, TermPattern>> outputs;
  std::map<std::string, std::string> bodies;
  SourceLoc loc;
  const TermPattern* input_of(const std::string& p) const;
  const TermPattern* output_of(const std::string& p) const;
};

struct ExternalDecl {
  std::string type;
  std::string name;
  std::vector<OffsetExpr> subscripts;
  SourceLoc loc;
};

struct Axiom {
  ExternalDecl external;
  TermPattern term;
};
struct Goal {
  TermPattern term;
  ExternalDecl external;
};

struct Range {
  long lo = 0, hi = 0, stride = 1;
  long trips() const { return (hi - lo) / stride; }
  bool operator==(const Range&) const = default;
};

// Ghost-cell refill between iterated steps (extension; the reference parser
// ignores unknown `config` keys, rulespec.cpp:416-472).
enum class Boundary { none, zero, periodic, clamp, even, odd };
const char* boundary_name(Boundary b);

struct RuleSet {
  std::string name;
  std::vector<KernelRule> kernels;
  std::vector<Axiom> axioms;
  std::vector<Goal> goals;
  std::vector<std::string> loop_order;
  std::vector<Range> ranges;
  std::vector<std::pair<std::string, std::string>> aliases;
  int vector_length = 1;
  std::string backend = "c99";
  // --- loomfuse-b200 extensions -------------------------------------------
  // boundary[external][dim] (dims outermost first); missing = none
  std::map<std::string, std::vector<Boundary>> boundary;
  // (goal external, axiom external): goal of step s feeds axiom of step s+1
  std::vector<std::pair<std::string, std::string>> iterate;

  int dim_of(const std::string& var) const;
  const KernelRule* kernel(const std::string& name) const;
};

struct DeclParam {
  std::string type;
  std::string name;
  bool pointer = false;
  bool reference = false;
};
struct DeclInfo {
  std::string function;
  std::vector<DeclParam> params;
  const DeclParam* param(const std::string& name) const;
};

DeclInfo parse_declaration(const std::string& decl);
std::optional<RuleSet> parse_spec(const std::string& text, const std::string& file, DiagList& diags);
std::vector<Diagnostic> validate_rules(const RuleSet& rs);
std::string print_spec(const RuleSet& rs);
bool structurally_equal(const RuleSet& a, const RuleSet& b);

// ------------------------------------------------------------- inference
// Types mirror inference.hpp:14-114.
struct DimOffset {
  int dim = 0;
  int offset = 0;
  auto operator<=>(const DimOffset&) const = default;
};

struct ConcreteTerm {
  std::string tag;
  std::string ident;
  std::vector<DimOffset> dims;  // sorted by dim
  auto operator<=>(const ConcreteTerm&) const = default;
  std::string str(const RuleSet& rs) const;
};

enum class RapKind { kernel, load, store };

struct ExtSlot {
  int dim = -1;
  int shift = 0;
  auto operator<=>(const ExtSlot&) const = default;
};

struct Bound {  // value of a free variable inside one rule application
  bool is_ident = false;
  std::string ident;
  int dim = -1;
  int offset = 0;
  bool operator==(const Bound&) const = default;
};

struct Rap {
  int id = -1;
  RapKind kind = RapKind::kernel;
  int kernel = -1;
  std::vector<int> in_terms;
  std::vector<int> out_terms;
  std::vector<std::pair<std::string, Bound>> binding;
  std::string external;
  std::vector<ExtSlot> ext_slots;
  std::string label(const RuleSet& rs) const;
};

struct DataflowEdge {
  int from = -1, to = -1, term = -1;
  auto operator<=>(const DataflowEdge&) const = default;
};

struct DataflowDAG {
  std::vector<ConcreteTerm> terms;
  std::vector<Rap> raps;
  std::vector<int> producer;  // term -> rap
  std::vector<DataflowEdge> edges;
  std::vector<std::vector<int>> out_adj, in_adj;
  std::vector<int> goal_terms;
  void build_adjacency();
  std::vector<int> topo_order() const;  // throws internal_error on a cycle
};

// Backward chaining from the goals (inference.cpp:404-453) followed by the
// RAP dual (inference.cpp:455-472).
std::optional<DataflowDAG> infer(const RuleSet& rs, DiagList& diags);
bool dataflow_le(const std::set<int>& R, const std::set<int>& S, const DataflowDAG& dag);

// ------------------------------------------------------------- analysis
struct CallsiteGroup {
  int id = -1;
  RapKind kind = RapKind::kernel;
  int kernel = -1;
  std::string external;
  std::vector<int> members;
  std::vector<std::vector<int>> member_disp;  // per member, per loop dim
  std::vector<int> space;                     // loop dims, outermost first
  std::vector<int> min_disp(size_t nd) const;
  std::vector<int> max_disp(size_t nd) const;
};

enum class Scheme { full, inner_circular, outer_rotate, scalar, terminal };
const char* scheme_name(Scheme s);

struct Variable {
  int id = -1;
  std::string tag, ident, name, type;
  std::vector<int> dims;
  int producer_group = -1;
  int alias_of = -1;     // associative carry unified with the output (storage.cpp:93-105)
  std::string external;  // backing terminal ("" for intermediates)
  bool axiom_backed = false;
  // buffer_extents (storage.cpp:403-427): per variable dim {extent, base}
  std::vector<std::pair<long, long>> extents;
  // contraction (storage.cpp:319-399)
  Scheme scheme = Scheme::full;
  int rotating_dim = -1;
  long span = 1;
  std::vector<long> spans;  // per variable dim
  // reuse Hamiltonian path (storage.cpp:124-141, R/SPEC.md:387-395): distinct
  // read offsets, first visit first, rendered innermost dim first
  std::string reuse_path;
};

struct Terminal {
  std::string name;
  std::string type;       // element type text from the declaration
  bool is_goal = false;
  int var = -1;
  std::vector<int> dims;  // loop dims of the buffer, outermost first
  std::vector<long> extent;
  std::vector<long> base;
  int elem_bytes = 8;
};

// alias_chain (storage.cpp:453-524): reads of an aliased input that happen at
// or after the trip that overwrites them, relative to the writer's shift
struct AliasEntry {
  std::string input, output;            // [input buffer, output buffer] from config.aliases
  int var = -1;                         // the axiom-backed variable read
  int writer_group = -1;                // group writing the output (write-through producer)
  std::vector<int> writer_shift;
  std::vector<std::vector<int>> offsets;  // clobbered read offsets, descending lexicographic
};
// shadow window of an alias entry (storage.cpp:544-594)
struct Shadow {
  int var = -1;
  Scheme scheme = Scheme::full;
  std::vector<int> dims;    // the variable's loop dims
  std::vector<long> spans;  // per variable dim
  int rotating = -1;        // first dim with a window > 1 (-1: a single cell)
};

struct Plan {
  RuleSet rs;
  DataflowDAG dag;
  std::vector<CallsiteGroup> groups;
  std::vector<int> group_of;
  std::vector<int> vertex_of_group;      // group -> fused nest (fusion.cpp:171-372)
  std::vector<std::vector<int>> shifts;  // group -> per dim (shifts.cpp:8-79)
  std::vector<Variable> vars;
  std::vector<int> var_of_term;     // term -> variable
  std::vector<Terminal> terminals;  // axioms (declaration order) then goals
  int nests = 0;
  int splits = 0;
  bool one_nest = false;
  std::string footprint;
  std::vector<int> halo_lo, halo_hi;  // per loop dim: max terminal read reach
  std::string signature;             // canonical chain signature for dispatch
  std::vector<AliasEntry> alias;     // in-place safety plan (empty without config.aliases)
  std::vector<Shadow> shadows;       // one per alias entry
  std::string report_json() const;
};

// Runs inference + grouping + one-nest check + shifts + storage bookkeeping.
std::optional<Plan> make_plan(const RuleSet& rs, DiagList& diags);

}  // namespace lf

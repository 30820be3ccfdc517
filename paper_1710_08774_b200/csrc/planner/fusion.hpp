// Iteration nests and nest fusion (reference: nests.hpp:10-86, fusion.hpp:8-50).
#pragma once

#include <memory>

#include "planner.hpp"

namespace lf {

struct Nest;
using NestP = std::shared_ptr<const Nest>;

// Leaf = ordered callsites of one trip; loop = one iteration variable with
// prologue / steady-state / epilogue phases (R/SPEC.md:189-195).
struct Nest {
  bool leaf = false;
  std::vector<int> body;
  int dim = -1;
  Range range;
  NestP pro, steady, epi;
};

enum class RapClass { pointwise, reduction, broadcast };

struct FusionResult {
  std::vector<NestP> vertices;       // fused nests in topological order
  std::vector<int> vertex_of_group;  // callsite group -> fused vertex
  int nests = 0;
  int splits = 0;                    // concave (reduction -> broadcast) splits
};

RapClass classify_rap(const Rap& r, const DataflowDAG& g);
NestP fuse_nests(const NestP& a, const NestP& b, const DataflowDAG& g, int ndims);
FusionResult fuse_groups(const RuleSet& rs, const DataflowDAG& g, const std::vector<CallsiteGroup>& groups,
                         const std::vector<int>& group_of);
bool is_perfect(const NestP& n);

}  // namespace lf

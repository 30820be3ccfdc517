// Registry of fused sm_100a executors.  A plan dispatches to the executor
// whose embedded reference spec has the same canonical chain signature
// (planner.hpp: Plan::signature), i.e. the same user kernels wired with the
// same offsets, terminal types, iterate pairs and boundary modes.  Sizes come
// from the user's plan (config ranges), not from the embedded spec.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../../include/loomfuse_b200.h"
#include "../planner/planner.hpp"

namespace lfx {

struct ExecArgs {
  const lf::Plan* plan = nullptr;
  void* const* terms = nullptr;  // device pointers, axioms then goals
  int steps = 1;
  cudaStream_t stream = nullptr;
  const lf_slab* slab = nullptr;  // nullptr: the whole domain
  void* const* scratch = nullptr;  // per iterated goal, same layout (steps > 1)
};

struct Executor {
  const char* name;
  const char* spec_file;   // specs/<file>.lf embedded at build time
  int launches_per_step;   // kernel launches one step issues
  double bytes_per_cell;   // compulsory HBM bytes per cell-update
  // size / layout constraints of the kernel; fills `why` when unsupported
  bool (*supports)(const lf::Plan&, std::string& why);
  // run `steps` steps (ping-pong for steps > 1); returns an LF_* status
  int (*run)(const ExecArgs&, std::string& err);
};

// all executors compiled into this library
const std::vector<Executor>& executors();

// embedded spec text by file name ("" if unknown); generated at build time
const char* embedded_spec(const char* file);

// helpers shared by the executors
int cuda_status(cudaError_t e, const char* what, std::string& err);

}  // namespace lfx

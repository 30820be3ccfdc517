// Registry of fused sm_100a executors.  A plan dispatches to the executor
// whose embedded reference spec has the same canonical chain signature
// (planner.hpp: Plan::signature), i.e. the same user kernels wired with the
// same offsets, terminal types, iterate pairs and boundary modes.  Sizes come
// from the user's plan (config ranges), not from the embedded spec.
#pragma once

#include <cuda_runtime.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../../include/loomfuse_b200.h"
#include "../planner/planner.hpp"

namespace lfx {

// LF_* tuning switch: the lf_set_option override if one is set, else the
// environment (options.cpp)
const char* option(const char* name);
// value == nullptr: the switch reads as unset whatever the environment says;
// clear: drop the override (the environment applies again)
int set_option(const char* name, const char* value, int clear);

// Plan-owned device memory an executor may keep between runs (grow-only; the
// caller holds the plan lock; freed with the plan).
struct ExecMem {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t need) {
    if (need <= bytes) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&ptr, need);
    if (e == cudaSuccess) bytes = need;
    return e;
  }
  ~ExecMem() {
    if (ptr) cudaFree(ptr);
  }
};

// In-place band memory with guard zones (LF_BAND_GUARD=1; compute-sanitizer is
// not available on every pool): `need` bytes for the executor at the returned
// pointer, kBandGuard bytes of a canary before and after it.  band_guard_check
// -- after the run's last launch; synchronises -- fails with LF_ERR_INTERNAL
// when a band store went outside [ptr, ptr + need).  Without the switch:
// a plain ensure(), and the check returns LF_OK at once.
constexpr size_t kBandGuard = 4096;
int band_memory(ExecMem& mem, size_t need, cudaStream_t stream, void** ptr, std::string& err);
int band_guard_check(const ExecMem& mem, size_t need, cudaStream_t stream, std::string& err);

struct ExecArgs {
  const lf::Plan* plan = nullptr;
  void* const* terms = nullptr;  // device pointers, axioms then goals
  int steps = 1;
  cudaStream_t stream = nullptr;
  const lf_slab* slab = nullptr;  // nullptr: the whole domain
  void* const* scratch = nullptr;  // per iterated goal, same layout (steps > 1)
  bool whole_domain_parts = false;  // slab = the whole domain, computed in row parts (pipelined host run)
  // max_reduce executors under a slab driver: the rank-0 iterated axioms hold
  // the previous step's (combined) raw maxima, not final values
  bool raw_max_input = false;
  // every iterated goal shares its axiom's buffer (config.aliases): run in
  // place on that one buffer; only executors with `inplace` set are asked to
  bool inplace = false;
  ExecMem* mem = nullptr;  // set with `inplace`
  // In-place row parts of a whole domain (whole_domain_parts), launched in
  // ascending order within a step (pipelined host runs): part p's last halo
  // rows are still read by part p+1's launch, so phase 0 (the step) defers
  // them into row-band slot `inplace_slot` of `inplace_slots`, and phase 1
  // -- issued after part p+1's step -- copies them in.
  int inplace_phase = 0;
  int inplace_slot = 0, inplace_slots = 1;
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
  // passes over the grid `steps` steps take (temporal blocking fuses several
  // steps into one pass); nullptr: one pass per step
  int (*passes)(const lf::Plan&, int steps, bool slab) = nullptr;
  // rank-0 iterated goals are per-step MAX reductions over the cells (the
  // CFL time step): under a slab driver they are zeroed before each step,
  // combined across ranks after it (MAX), and `finalize` turns the last raw
  // maximum into the goal's value; a whole-domain run() does all of it itself
  bool max_reduce = false;
  int (*finalize)(const ExecArgs&, std::string& err) = nullptr;
  // runs whole-domain steps (and ordered row parts, see ExecArgs) in place when
  // every iterated goal is passed on its aliased axiom's buffer (ExecArgs::inplace)
  bool inplace = false;
  // ... and also whole slabs (lf_run_slabs) and ordered row parts (pipelined host runs)
  bool inplace_parts = false;
};

// all executors compiled into this library
const std::vector<Executor>& executors();

// embedded spec text by file name ("" if unknown); generated at build time
const char* embedded_spec(const char* file);
// the shipped user-kernel headers (userkernels/*.h), concatenated
const std::string& embedded_userkernels();

// helpers shared by the executors
int cuda_status(cudaError_t e, const char* what, std::string& err);

// Device-dependent launch setup of one kernel -- its dynamic shared-memory
// attribute and the number of CTAs resident at once (SMs x occupancy, capped
// at `occ_cap` per SM when > 0) -- done once per device ordinal, thread-safe.
// A process may drive several GPUs (one per host thread or in turn).
constexpr int kMaxDevices = 64;
struct LaunchCache {
  std::once_flag once[kMaxDevices];
  int slots[kMaxDevices] = {};
  cudaError_t err[kMaxDevices] = {};
};
int resident_slots(LaunchCache& cache, const void* kernel, int threads, int smem, int occ_cap, const char* what,
                   int* slots, std::string& err);

// rows of the outer dimension one launch computes (slab-local; whole slab when
// no part is given) and the slab's row count
struct RowPart {
  int rows;      // rows of this launch's domain (slab or whole grid)
  int lo, hi;    // rows to compute
  bool top, bottom;  // domain edge is a global boundary
};
inline RowPart row_part(const ExecArgs& a, int global_rows) {
  RowPart r{global_rows, 0, global_rows, true, true};
  if (a.slab) {
    r.rows = (int)(a.slab->hi - a.slab->lo);
    r.top = a.slab->lo == 0;
    r.bottom = a.slab->hi == a.slab->global;
    r.lo = 0;
    r.hi = r.rows;
    if (a.slab->part_hi > a.slab->part_lo) {
      r.lo = (int)a.slab->part_lo;
      r.hi = (int)a.slab->part_hi;
    }
  }
  return r;
}

}  // namespace lfx

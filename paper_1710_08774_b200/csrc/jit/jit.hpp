// Generic fused executor: `body:` chains lowered to CUDA (codegen.cpp) and
// compiled for sm_100a at plan creation with NVRTC (jit.cpp).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../exec/exec.hpp"
#include "../planner/planner.hpp"

namespace lfx {

struct NestLaunch {
  std::string fn;          // kernel name
  bool reduction = false;  // warp per parallel cell (true) or thread per cell
  long long units = 0;     // parallel cells
  int cells_per_cta = 0;   // reduction kernels: parallel cells a CTA owns (0: one per warp, 8)
  int threads = 256;       // CTA size
};

// streamed axioms the warp-specialised march can fetch by TMA (tensor maps
// passed by value next to the argument block)
constexpr int kJitMaxMaps = 8;

struct JitProgram {
  // config.aliases pairs the executor can run in place (one buffer):
  // row bands at chunk boundaries and column bands at tile boundaries
  struct Inplace {
    int ai = -1, gi = -1;      // axiom / goal terminal indices
    int bh = 0, bw1 = 0, bw2 = 0;  // band widths (dim 0, 1, 2)
    long e0 = 1, e1 = 1, e2 = 1;   // storage extents
    int t1 = 1, t2 = 1;        // inner tile sizes
    long n1 = 1, n2 = 1;       // inner trip counts
  };
  std::vector<Inplace> inplace;
  std::string inplace_error;   // why declared aliases cannot run in place
  std::string source;
  std::string type;  // "double" / "float"
  int elem_bytes = 8;
  int nd = 0;
  std::vector<int> tile;  // per loop dim, outermost first
  size_t smem_bytes = 0;
  int threads = 256;
  bool has_fill = false;
  bool march = false;       // 2D/3D rolling-window schedule (outer dim chunked over blockIdx.y)
  int prologue = 0;         // extra trips per chunk (pipeline fill)
  long inner_tiles = 1;     // CTAs across the inner dimensions
  int ctas_per_sm = 1;      // resident CTAs per SM the shared-memory footprint allows
  int chunk = 64;           // rows per chunk of the persistent work order
  // multi-nest plans: one kernel per nest, materialised cross-nest variables
  std::vector<NestLaunch> nest_kernels;
  std::vector<size_t> mat_bytes;
  // warp-specialised march (lf_jit_step_ws): one TMA map per streamed axiom,
  // extents innermost first (the outermost one is the launch domain's at run time)
  struct Tma {
    int term = -1;
    // >= 0: an in-place row-band buffer a.t[band] instead of a terminal; its
    // rows are band_rows per internal chunk boundary (known at launch)
    int band = -1;
    int band_rows = 0;
    int rank = 0;
    uint64_t extent[3] = {1, 1, 1};
    unsigned box[3] = {1, 1, 1};
  };
  bool has_ws = false;
  std::vector<Tma> ws_maps;
  size_t ws_smem_bytes = 0;
  long ws_inner_tiles = 1;  // the variant's own inner tiling
  int ws_threads = 288;
  std::vector<Inplace> ws_inplace;  // 3D in place on the warp-specialised march (deferred writes)
  // 2D register march (lf_jit_step_rm, codegen_rm.cpp): warp strips, register
  // windows, no CTA barriers; preferred over lf_jit_step_ws where it compiles
  bool has_rm = false;
  std::vector<Tma> rm_maps;
  std::vector<Inplace> rm_inplace;  // as `inplace`, for the register march's tile
  size_t rm_smem_bytes = 0;
  long rm_inner_tiles = 1;
  int rm_threads = 288;
  std::string error;  // why the chain is not supported
};

// `sources`: user-kernel code (the shipped headers + the caller's) prepended
// to the generated kernels; chains may name its functions instead of bodies
bool jit_generate(const lf::Plan& plan, JitProgram& out, const std::string& sources);

// kernel argument block, passed by value; must match `struct LfArgs` in the
// generated source (codegen.cpp)
struct JitArgs {
  void* t[32];  // terminals, then materialised variables / in-place bands
  long long n0;
  int row_lo, row_hi, top, bottom, chunk, inplace;
};

// tensor maps of the warp-specialised march, passed by value as its second
// kernel parameter (`struct LfMaps` in the generated source)
struct alignas(64) JitMap {
  unsigned long long w[16];
};
struct JitMaps {
  JitMap m[kJitMaxMaps];
};

// A compiled chain; owned by one plan.
class JitKernel {
 public:
  static std::shared_ptr<JitKernel> build(const lf::Plan& plan, std::string& why, const std::string& kernel_source = "");
  int run(const ExecArgs& a, std::string& err);
  const JitProgram& program() const { return prog_; }
  ~JitKernel();

 private:
  JitProgram prog_;
  void* module_ = nullptr;  // CUmodule, loaded into the context of device_ at the first run
  int device_ = -1;
  void* step_ = nullptr;    // CUfunction
  void* step_ws_ = nullptr; // warp-specialised variant (TMA producer warp)
  void* step_rm_ = nullptr; // 2D register march (TMA producer warp, warp strips)
  void* fill_ = nullptr;
  void* capture_ = nullptr;
  std::vector<void*> bands_;        // in-place band copies
  std::vector<size_t> band_bytes_;
  int resident_ = 0;  // CTAs resident at once (occupancy x SMs)
  int resident_ws_ = 0;
  int resident_rm_ = 0;
  std::vector<void*> nest_fns_;
  std::vector<void*> mats_;  // device buffers of materialised variables
  std::vector<char> cubin_;
  int launch(void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st, void* args, std::string& err,
             void* args2 = nullptr);
  int run_nests(const ExecArgs& a, std::string& err);
  // bufs: the launch's argument slots (terminals, then in-place bands);
  // boundaries: internal chunk boundaries of an in-place launch (band rows)
  bool tma_maps(const std::vector<JitProgram::Tma>& list, const std::vector<void*>& bufs, long rows, JitMaps& maps,
                long boundaries = 0);
  void* commit_rm_ = nullptr;  // in-place register march: deferred boundary writes into the grid
  void* commit_fill_rm_ = nullptr;  // the same plus the ghost refill (zero boundaries)
  void* commit_ws_ = nullptr;  // in-place 3D warp-specialised march: the same
  int bands_for(const std::vector<JitProgram::Inplace>& list, long nch, long nt_of_tile1, std::string& err);
  long plan_rows_ = 0;  // trips of the outermost loop dimension (whole domain)
  int run_inplace(const ExecArgs& a, JitArgs& args, std::string& err);
};

}  // namespace lfx

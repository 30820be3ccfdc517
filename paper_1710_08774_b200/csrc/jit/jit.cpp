// Generic fused executor, part 2: NVRTC compilation for sm_100a (libnvrtc is
// opened at first use, so the library still loads where NVRTC is absent) and
// module loading / launching through the driver entry points the runtime
// exposes (no -lcuda).  Same numerics contract as the hand-written
// executors: -fmad=false, IEEE division and square root.
#include "jit.hpp"

#include "../exec/common.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace lfx {

namespace {

// ---- NVRTC through dlopen ----------------------------------------------------
typedef int nvrtcResult_t;
struct Nvrtc {
  void* h = nullptr;
  int (*create)(void**, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
  int (*compile)(void*, int, const char* const*) = nullptr;
  int (*log_size)(void*, size_t*) = nullptr;
  int (*log)(void*, char*) = nullptr;
  int (*cubin_size)(void*, size_t*) = nullptr;
  int (*cubin)(void*, char*) = nullptr;
  int (*destroy)(void**) = nullptr;
  std::string error;
};

const Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"};
    for (const char* nm : names)
      if ((n.h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
    if (!n.h) {
      n.error = "libnvrtc.so.12 not found";
      return;
    }
    auto sym = [&](const char* s) { return dlsym(n.h, s); };
    n.create = reinterpret_cast<decltype(n.create)>(sym("nvrtcCreateProgram"));
    n.compile = reinterpret_cast<decltype(n.compile)>(sym("nvrtcCompileProgram"));
    n.log_size = reinterpret_cast<decltype(n.log_size)>(sym("nvrtcGetProgramLogSize"));
    n.log = reinterpret_cast<decltype(n.log)>(sym("nvrtcGetProgramLog"));
    n.cubin_size = reinterpret_cast<decltype(n.cubin_size)>(sym("nvrtcGetCUBINSize"));
    n.cubin = reinterpret_cast<decltype(n.cubin)>(sym("nvrtcGetCUBIN"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(sym("nvrtcDestroyProgram"));
    if (!n.create || !n.compile || !n.cubin || !n.destroy) n.error = "libnvrtc symbols missing";
  });
  return n;
}

// ---- driver entry points -------------------------------------------------------
struct Drv {
  PFN_cuModuleLoadData_v2000 load = nullptr;
  PFN_cuModuleGetFunction_v2000 get = nullptr;
  PFN_cuLaunchKernel_v4000 launch = nullptr;
  PFN_cuLaunchKernelEx_v11060 launch_ex = nullptr;
  PFN_cuFuncSetAttribute_v9000 attr = nullptr;
  PFN_cuModuleUnload_v2000 unload = nullptr;
  PFN_cuOccupancyMaxActiveBlocksPerMultiprocessor_v6050 occupancy = nullptr;
  bool ok = false;
};

const Drv& drv() {
  static Drv d;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, void** p) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess;
    };
    d.ok = get("cuModuleLoadData", reinterpret_cast<void**>(&d.load)) &&
           get("cuModuleGetFunction", reinterpret_cast<void**>(&d.get)) &&
           get("cuLaunchKernel", reinterpret_cast<void**>(&d.launch)) &&
           get("cuFuncSetAttribute", reinterpret_cast<void**>(&d.attr)) &&
           get("cuModuleUnload", reinterpret_cast<void**>(&d.unload)) &&
           get("cuOccupancyMaxActiveBlocksPerMultiprocessor", reinterpret_cast<void**>(&d.occupancy));
    if (!get("cuLaunchKernelEx", reinterpret_cast<void**>(&d.launch_ex))) d.launch_ex = nullptr;
  });
  return d;
}

}  // namespace

std::shared_ptr<JitKernel> JitKernel::build(const lf::Plan& plan, std::string& why, const std::string& kernel_source) {
  auto k = std::shared_ptr<JitKernel>(new JitKernel);
  if (plan.terminals.size() > 32) {
    why = "more than 32 terminals";
    return nullptr;
  }
  const std::string sources = embedded_userkernels() + (kernel_source.empty() ? "" : "// ---- kernel source given to the plan\n" + kernel_source + "\n");
  if (!jit_generate(plan, k->prog_, sources)) {
    why = k->prog_.error;
    return nullptr;
  }
  // compile now (plan creation) so errors surface early; loading waits for a device
  const Nvrtc& n = nvrtc();
  if (!n.error.empty()) {
    why = "generic executor unavailable: " + n.error;
    return nullptr;
  }
  void* prog = nullptr;
  if (n.create(&prog, k->prog_.source.c_str(), "lf_chain.cu", 0, nullptr, nullptr) != 0) {
    why = "nvrtcCreateProgram failed";
    return nullptr;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-fmad=false", "-prec-div=true", "-prec-sqrt=true",
                        "-std=c++17", "-lineinfo"};
  const int rc = n.compile(prog, 6, opts);
  if (rc != 0) {
    size_t ls = 0;
    n.log_size(prog, &ls);
    std::string log(ls, '\0');
    if (ls) n.log(prog, log.data());
    n.destroy(&prog);
    why = "NVRTC failed to compile the generated chain:\n" + log;
    return nullptr;
  }
  size_t cs = 0;
  n.cubin_size(prog, &cs);
  k->cubin_.resize(cs);
  n.cubin(prog, k->cubin_.data());
  n.destroy(&prog);
  return k;
}

JitKernel::~JitKernel() {
  for (void* p : mats_) cudaFree(p);
  for (void* p : bands_) cudaFree(p);
  if (module_ && drv().ok) drv().unload(static_cast<CUmodule>(module_));
}

// In place (config.aliases with one buffer for the axiom and its goal): whole
// (chunk, tile) units; before each step lf_jit_capture copies the rows at
// chunk boundaries and the columns at tile boundaries that a unit reads but
// another unit writes, and the step reads those cells from the copies.  The
// copies are O(surface) -- the grid itself is never duplicated.
static long pick_chunk(long rows, long inner, long resident, long fill, long max_chunk);

// band buffers of an in-place launch: per aliased axiom, the rows at the nch-1
// internal chunk boundaries and the columns at the internal boundaries of the
// inner tiles the descriptors name
int JitKernel::bands_for(const std::vector<JitProgram::Inplace>& list, long nch, long, std::string& err) {
  const size_t eb = static_cast<size_t>(prog_.elem_bytes);
  std::vector<size_t> need;
  for (const auto& q : list) {
    const long nt1 = (q.n1 + q.t1 - 1) / q.t1, nt2 = (q.n2 + q.t2 - 1) / q.t2;
    need.push_back(std::max<long>(0, nch - 1) * q.bh * q.e1 * q.e2 * eb);
    need.push_back(std::max<long>(0, nt1 - 1) * q.bw1 * q.e0 * q.e2 * eb);
    need.push_back(prog_.nd == 3 ? std::max<long>(0, nt2 - 1) * q.bw2 * q.e0 * q.e1 * eb : 0);
  }
  if (band_bytes_ != need) {
    for (void* p : bands_) cudaFree(p);
    bands_.assign(need.size(), nullptr);
    for (size_t k = 0; k < need.size(); ++k) {
      cudaError_t e = cudaMalloc(&bands_[k], std::max<size_t>(need[k], 16));
      if (e != cudaSuccess) {
        err = std::string("cudaMalloc(in-place bands): ") + cudaGetErrorString(e);
        band_bytes_.clear();
        return LF_ERR_CUDA;
      }
    }
    band_bytes_ = need;
  }
  return LF_OK;
}

int JitKernel::run_inplace(const ExecArgs& a, JitArgs& args, std::string& err) {
  const auto& rs = a.plan->rs;
  const auto& T = a.plan->terminals;
  if (a.slab && (a.slab->lo != 0 || a.slab->hi != a.slab->global || a.slab->part_hi > a.slab->part_lo)) {
    err = "in-place runs cover the whole domain (no slabs)";
    return LF_ERR_UNSUPPORTED;
  }
  if (!capture_) {
    err = "in-place capture kernel missing";
    return LF_ERR_INTERNAL;
  }
  const long rows = rs.ranges[0].trips();
  args.n0 = rows;
  args.row_lo = 0;
  args.row_hi = static_cast<int>(rows);
  args.top = args.bottom = 1;
  args.inplace = 1;
  // the register march (2D), when it covers every aliased pair: units defer
  // their boundary writes to the bands, lf_jit_commit_rm copies them in after
  // the step (codegen_rm.cpp)
  if (step_rm_ && commit_rm_ && prog_.rm_inplace.size() == prog_.inplace.size()) {
    long chunk = pick_chunk(rows, prog_.rm_inner_tiles, resident_rm_, prog_.prologue, rows);
    long bh = 1;
    for (const auto& q : prog_.rm_inplace) bh = std::max<long>(bh, q.bh);
    chunk = std::min(rows, std::max({chunk, 8L * std::max(1, prog_.prologue), bh}));
    if (const char* e = lfx::option("LF_JIT_CHUNK")) chunk = std::max(bh, std::min<long>(rows, std::atol(e)));
    const long nch = (rows + chunk - 1) / chunk;
    int st = bands_for(prog_.rm_inplace, nch, 0, err);
    if (st != LF_OK) return st;
    args.chunk = static_cast<int>(chunk);
    for (size_t i = 0; i < T.size(); ++i) args.t[i] = a.terms[i];
    for (size_t k = 0; k < bands_.size(); ++k) args.t[T.size() + k] = bands_[k];
    JitMaps maps;
    bool goals_aligned = true;
    for (size_t i = 0; i < T.size(); ++i)
      if (T[i].is_goal) goals_aligned &= reinterpret_cast<uintptr_t>(a.terms[i]) % 16 == 0;
    std::vector<void*> bufs(a.terms, a.terms + T.size());
    if (goals_aligned && tma_maps(prog_.rm_maps, bufs, rows, maps)) {
      const long units = nch * prog_.rm_inner_tiles;
      const dim3 grid(static_cast<unsigned>(std::max<long>(1, std::min<long>(resident_rm_, units))));
      long band_cells = 1;  // the commit kernel's flat index space (largest aliased pair)
      for (const auto& q : prog_.rm_inplace)
        band_cells = std::max(band_cells, (nch - 1) * q.bh * q.n1 + rows * ((q.n1 + q.t1 - 1) / q.t1 - 1) * q.bw1);
      const unsigned commit_blocks = static_cast<unsigned>((band_cells + 1023) / 1024);
      for (int s = 0; s < a.steps; ++s) {
        st = launch(step_rm_, grid, dim3(prog_.rm_threads), prog_.rm_smem_bytes, a.stream, &args, err, &maps);
        if (st != LF_OK) return st;
        if (commit_fill_rm_ && fill_ && prog_.has_fill) {  // commit and ghost refill in one launch
          st = launch(commit_fill_rm_, dim3(std::max(commit_blocks, 592u)), dim3(256), 0, a.stream, &args, err);
          if (st != LF_OK) return st;
          continue;
        }
        st = launch(commit_rm_, dim3(commit_blocks), dim3(256), 0, a.stream, &args, err);
        if (st != LF_OK) return st;
        if (fill_ && prog_.has_fill) {
          st = launch(fill_, dim3(592), dim3(256), 0, a.stream, &args, err);
          if (st != LF_OK) return st;
        }
      }
      return LF_OK;
    }
  }
  // 3D: the warp-specialised march with deferred boundary writes (the same
  // scheme; codegen.cpp March::commit3)
  if (step_ws_ && commit_ws_ && prog_.ws_inplace.size() == prog_.inplace.size() && !prog_.ws_inplace.empty()) {
    long chunk = pick_chunk(rows, prog_.ws_inner_tiles, resident_ws_, prog_.prologue, prog_.chunk);
    long bh = 1;
    for (const auto& q : prog_.ws_inplace) bh = std::max<long>(bh, q.bh);
    chunk = std::min(rows, std::max(chunk, bh));
    if (const char* e = lfx::option("LF_JIT_CHUNK")) chunk = std::max(bh, std::min<long>(rows, std::atol(e)));
    const long nch = (rows + chunk - 1) / chunk;
    int st = bands_for(prog_.ws_inplace, nch, 0, err);
    if (st != LF_OK) return st;
    args.chunk = static_cast<int>(chunk);
    for (size_t i = 0; i < T.size(); ++i) args.t[i] = a.terms[i];
    for (size_t k = 0; k < bands_.size(); ++k) args.t[T.size() + k] = bands_[k];
    JitMaps maps;
    std::vector<void*> bufs(a.terms, a.terms + T.size());
    if (tma_maps(prog_.ws_maps, bufs, rows, maps)) {
      const long units = nch * prog_.ws_inner_tiles;
      const dim3 grid(static_cast<unsigned>(std::max<long>(1, std::min<long>(resident_ws_, units))));
      long band_cells = 1;  // the commit kernel's flat index space (largest aliased pair)
      for (const auto& q : prog_.ws_inplace) {
        const long nt1 = (q.n1 + q.t1 - 1) / q.t1, nt2 = (q.n2 + q.t2 - 1) / q.t2;
        band_cells = std::max(band_cells, (nch - 1) * q.bh * q.n1 * q.n2 + rows * (nt1 - 1) * q.bw1 * q.n2 +
                                              rows * (nt2 - 1) * q.bw2 * q.n1);
      }
      const unsigned commit_blocks = static_cast<unsigned>((band_cells + 1023) / 1024);
      for (int s = 0; s < a.steps; ++s) {
        st = launch(step_ws_, grid, dim3(prog_.ws_threads), prog_.ws_smem_bytes, a.stream, &args, err, &maps);
        if (st != LF_OK) return st;
        st = launch(commit_ws_, dim3(commit_blocks), dim3(256), 0, a.stream, &args, err);
        if (st != LF_OK) return st;
        if (fill_ && prog_.has_fill) {
          st = launch(fill_, dim3(592), dim3(256), 0, a.stream, &args, err);
          if (st != LF_OK) return st;
        }
      }
      return LF_OK;
    }
  }
  // chunk: about two units per resident CTA, at least 8 pipeline depths
  long chunk = (rows * prog_.inner_tiles + 2L * resident_ - 1) / (2L * resident_);
  chunk = std::min(rows, std::max(chunk, 8L * std::max(1, prog_.prologue)));
  if (const char* e = lfx::option("LF_JIT_CHUNK")) chunk = std::max(1L, std::min<long>(rows, std::atol(e)));
  const long nch = (rows + chunk - 1) / chunk;
  int bst = bands_for(prog_.inplace, nch, 0, err);
  if (bst != LF_OK) return bst;
  args.chunk = static_cast<int>(chunk);
  for (size_t i = 0; i < T.size(); ++i) args.t[i] = a.terms[i];
  for (size_t k = 0; k < bands_.size(); ++k) args.t[T.size() + k] = bands_[k];
  const long units = nch * prog_.inner_tiles;
  const dim3 grid(static_cast<unsigned>(std::max<long>(1, std::min<long>(resident_, units))));
  for (int s = 0; s < a.steps; ++s) {
    int st = launch(capture_, dim3(592), dim3(256), 0, a.stream, &args, err);
    if (st != LF_OK) return st;
    st = launch(step_, grid, dim3(prog_.threads), prog_.smem_bytes, a.stream, &args, err);
    if (st != LF_OK) return st;
    if (fill_ && prog_.has_fill) {
      st = launch(fill_, dim3(592), dim3(256), 0, a.stream, &args, err);
      if (st != LF_OK) return st;
    }
  }
  return LF_OK;
}

// multi-nest plans: the nests in dataflow order each step; whole domain only
int JitKernel::run_nests(const ExecArgs& a, std::string& err) {
  const auto& rs = a.plan->rs;
  const auto& T = a.plan->terminals;
  if (a.slab && (a.slab->lo != 0 || a.slab->hi != a.slab->global || a.slab->part_hi > a.slab->part_lo)) {
    err = "multi-nest plans (reductions) run on the whole domain only, not on slabs";
    return LF_ERR_UNSUPPORTED;
  }
  if (mats_.empty())
    for (size_t b : prog_.mat_bytes) {
      void* p = nullptr;
      cudaError_t e = cudaMalloc(&p, std::max<size_t>(b, 16));
      if (e != cudaSuccess) {
        err = std::string("cudaMalloc(materialised variable): ") + cudaGetErrorString(e);
        return LF_ERR_CUDA;
      }
      mats_.push_back(p);
    }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  JitArgs args;
  std::memset(&args, 0, sizeof args);
  const long rows = rs.ranges[0].trips();
  args.n0 = rows;
  args.row_lo = 0;
  args.row_hi = static_cast<int>(rows);
  args.top = args.bottom = 1;
  std::vector<int> iter_axiom(T.size(), -1);
  for (const auto& [gname, aname] : rs.iterate) {
    int gi = -1, ai = -1;
    for (size_t i = 0; i < T.size(); ++i) {
      if (T[i].is_goal && T[i].name == gname) gi = static_cast<int>(i);
      if (!T[i].is_goal && T[i].name == aname) ai = static_cast<int>(i);
    }
    if (gi >= 0 && ai >= 0) iter_axiom[gi] = ai;
  }
  int scratch_idx = 0;
  std::vector<void*> scratch(T.size(), nullptr);
  for (size_t i = 0; i < T.size(); ++i)
    if (iter_axiom[i] >= 0 && a.steps > 1) scratch[i] = a.scratch[scratch_idx++];
  std::vector<void*> cur(a.terms, a.terms + T.size());
  for (int s = 0; s < a.steps; ++s) {
    const bool to_goal = ((a.steps - 1 - s) % 2) == 0;
    std::vector<void*> bufs = cur;
    for (size_t i = 0; i < T.size(); ++i)
      if (T[i].is_goal) bufs[i] = (to_goal || iter_axiom[i] < 0) ? a.terms[i] : scratch[i];
    for (size_t i = 0; i < T.size(); ++i) args.t[i] = bufs[i];
    for (size_t m = 0; m < mats_.size(); ++m) args.t[T.size() + m] = mats_[m];
    for (size_t k = 0; k < prog_.nest_kernels.size(); ++k) {
      const auto& nk = prog_.nest_kernels[k];
      const long long per_cta = nk.cells_per_cta > 0 ? nk.cells_per_cta : (nk.reduction ? 8 : 256);
      const long long want = (nk.units + per_cta - 1) / per_cta;
      const unsigned ctas = static_cast<unsigned>(std::max<long long>(1, std::min<long long>(want, 32LL * sms)));
      int st = launch(nest_fns_[k], dim3(ctas), dim3(nk.threads), 0, a.stream, &args, err);
      if (st != LF_OK) return st;
    }
    if (fill_ && prog_.has_fill) {
      int st = launch(fill_, dim3(592), dim3(256), 0, a.stream, &args, err);
      if (st != LF_OK) return st;
    }
    for (size_t i = 0; i < T.size(); ++i)
      if (iter_axiom[i] >= 0) cur[iter_axiom[i]] = bufs[i];
  }
  return LF_OK;
}

// Rows per (chunk, tile) unit of the round-robin work order: the chunk count n
// minimising waves(n) x (rows per chunk + pipeline fill), waves(n) =
// ceil(n * inner / resident) -- a unit count just above a multiple of the
// resident CTAs would otherwise leave a nearly empty last wave (Hydro2D named
// kernels: 306 units on 296 CTAs ran at half speed).  max_chunk caps the rows
// of a unit (3D: L2 locality of the planes a unit streams).
static long pick_chunk(long rows, long inner, long resident, long fill, long max_chunk) {
  long best_n = 1;
  double best = -1;
  const long n_lo = std::max(1L, (rows + max_chunk - 1) / max_chunk);
  const long n_hi = std::max(n_lo, std::min(rows, n_lo + 4 * std::max(1L, resident)));
  for (long n = n_lo; n <= n_hi; ++n) {
    const long chunk = (rows + n - 1) / n;
    const long units = (rows + chunk - 1) / chunk * inner;
    const long waves = (units + resident - 1) / resident;
    const double t = static_cast<double>(waves) * static_cast<double>(chunk + fill);
    if (best < 0 || t < best - 1e-9) {
      best = t;
      best_n = n;
    }
  }
  return (rows + best_n - 1) / best_n;
}

// tensor maps of the streamed axioms for this launch's buffers; false (plain
// kernel) when a buffer is not 16-B aligned or the driver refuses a map
bool JitKernel::tma_maps(const std::vector<JitProgram::Tma>& list, const std::vector<void*>& bufs, long rows,
                         JitMaps& maps, long boundaries) {
  const bool off = lfx::option("LF_JIT_WS") && std::atoi(lfx::option("LF_JIT_WS")) == 0;
  if (off) return false;
  const CUtensorMapDataType dt = prog_.elem_bytes == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const long n0 = plan_rows_;
  for (size_t k = 0; k < list.size(); ++k) {
    const auto& m = list[k];
    const void* base = bufs[m.band >= 0 ? m.band : m.term];
    if (reinterpret_cast<uintptr_t>(base) % 16) return false;
    uint64_t dims[3] = {m.extent[0], m.extent[1], m.extent[2]};
    if (m.band >= 0)  // in-place row bands: band_rows per internal chunk boundary
      dims[m.rank - 1] = static_cast<uint64_t>(std::max(1L, boundaries * m.band_rows));
    else  // outermost extent of the launch domain: a slab holds rows + the terminal's halo rows
      dims[m.rank - 1] = static_cast<uint64_t>(static_cast<long>(m.extent[m.rank - 1]) - n0 + rows);
    std::string e;
    if (!make_tensor_map(reinterpret_cast<CUtensorMap*>(&maps.m[k]), base, dt, prog_.elem_bytes, m.rank, dims, m.box, e))
      return false;
  }
  return true;
}

int JitKernel::launch(void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st, void* args, std::string& err,
                      void* args2) {
  void* params[] = {args, args2};
  // programmatic dependent launch: every generated kernel starts with
  // griddepcontrol.wait + launch_dependents (lf_pdl), so the next launch of
  // the step (ghost fill, commit, the next step) is set up while this one
  // drains (LF_NO_PDL=1: plain stream order)
  const bool no_pdl = lfx::option("LF_NO_PDL") != nullptr;
  CUresult r;
  if (drv().launch_ex && !no_pdl) {
    CUlaunchAttribute attr;
    std::memset(&attr, 0, sizeof attr);
    attr.id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr.value.programmaticStreamSerializationAllowed = 1;
    CUlaunchConfig cfg;
    std::memset(&cfg, 0, sizeof cfg);
    cfg.gridDimX = grid.x;
    cfg.gridDimY = grid.y;
    cfg.gridDimZ = grid.z;
    cfg.blockDimX = block.x;
    cfg.blockDimY = block.y;
    cfg.blockDimZ = block.z;
    cfg.sharedMemBytes = static_cast<unsigned>(smem);
    cfg.hStream = reinterpret_cast<CUstream>(st);
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    r = drv().launch_ex(&cfg, static_cast<CUfunction>(fn), params, nullptr);
  } else {
    r = drv().launch(static_cast<CUfunction>(fn), grid.x, grid.y, grid.z, block.x, block.y, block.z,
                     static_cast<unsigned>(smem), reinterpret_cast<CUstream>(st), params, nullptr);
  }
  if (r != CUDA_SUCCESS) {
    err = "cuLaunchKernel failed with CUresult " + std::to_string(static_cast<int>(r));
    return LF_ERR_CUDA;
  }
  return LF_OK;
}

int JitKernel::run(const ExecArgs& a, std::string& err) {
  const Drv& d = drv();
  if (!d.ok) {
    err = "CUDA driver entry points unavailable";
    return LF_ERR_CUDA;
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    err = "cudaGetDevice failed";
    return LF_ERR_CUDA;
  }
  if (module_ && dev != device_) {
    // the module, its functions and the plan-owned device buffers belong to
    // the context they were created in
    err = "this plan's generated kernels are loaded on device " + std::to_string(device_) +
          "; create one plan per device (current device " + std::to_string(dev) + ")";
    return LF_ERR_UNSUPPORTED;
  }
  if (!module_) {
    cudaFree(nullptr);  // make sure the primary context exists
    device_ = dev;
    CUmodule m;
    CUresult r = d.load(&m, cubin_.data());
    if (r != CUDA_SUCCESS) {
      err = "cuModuleLoadData failed with CUresult " + std::to_string(static_cast<int>(r));
      return LF_ERR_CUDA;
    }
    module_ = m;
    CUfunction f;
    if (d.get(&f, m, "lf_jit_fill") == CUDA_SUCCESS) fill_ = f;
    if (d.get(&f, m, "lf_jit_capture") == CUDA_SUCCESS) capture_ = f;
    if (d.get(&f, m, "lf_jit_commit_rm") == CUDA_SUCCESS) commit_rm_ = f;
    if (d.get(&f, m, "lf_jit_commit_fill_rm") == CUDA_SUCCESS) commit_fill_rm_ = f;
    if (d.get(&f, m, "lf_jit_commit_ws") == CUDA_SUCCESS) commit_ws_ = f;
    if (!prog_.nest_kernels.empty()) {
      for (const auto& nk : prog_.nest_kernels) {
        if (d.get(&f, m, nk.fn.c_str()) != CUDA_SUCCESS) {
          err = "generated kernel " + nk.fn + " missing";
          return LF_ERR_INTERNAL;
        }
        nest_fns_.push_back(f);
      }
    } else {
      if (d.get(&f, m, "lf_jit_step") != CUDA_SUCCESS) {
        err = "generated kernel missing";
        return LF_ERR_INTERNAL;
      }
      step_ = f;
      d.attr(static_cast<CUfunction>(step_), CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
             static_cast<int>(prog_.smem_bytes));
      if (prog_.has_ws && d.get(&f, m, "lf_jit_step_ws") == CUDA_SUCCESS) {
        step_ws_ = f;
        d.attr(static_cast<CUfunction>(step_ws_), CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
               static_cast<int>(prog_.ws_smem_bytes));
      }
      if (prog_.has_rm && d.get(&f, m, "lf_jit_step_rm") == CUDA_SUCCESS) {
        step_rm_ = f;
        d.attr(static_cast<CUfunction>(step_rm_), CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
               static_cast<int>(prog_.rm_smem_bytes));
      }
    }
  }
  if (!prog_.nest_kernels.empty()) return run_nests(a, err);
  const auto& rs = a.plan->rs;
  const auto& T = a.plan->terminals;
  const RowPart rp = row_part(a, (int)rs.ranges[0].trips());
  plan_rows_ = rs.ranges[0].trips();
  JitArgs args;
  std::memset(&args, 0, sizeof args);
  args.n0 = rp.rows;
  args.row_lo = rp.lo;
  args.row_hi = rp.hi;
  // ghost rows of dim 0 (the fill kernel's top/bottom regions): refilled by
  // the part that computes the face rows they mirror -- except a periodic
  // dim 0, whose images are the far face: on a slab they arrive by the
  // caller's halo exchange, on a whole domain computed in row parts they are
  // filled once the last part is done
  bool periodic0 = false;
  for (const auto& [gname, mode] : rs.boundary)
    if (!mode.empty() && mode[0] == lf::Boundary::periodic) periodic0 = true;
  const bool first_part = rp.lo == 0, last_part = rp.hi == rp.rows;
  if (!periodic0) {
    args.top = rp.top && first_part;
    args.bottom = rp.bottom && last_part;
  } else if (!a.slab || a.whole_domain_parts) {
    args.top = args.bottom = last_part;
  } else {
    args.top = args.bottom = 0;
  }
  dim3 grid(1, 1, 1);
  const long rows = rp.hi - rp.lo;
  if (rows <= 0) return LF_OK;
  if (prog_.march) {
    // persistent: one wave of resident CTAs, each an equal share of the
    // (chunk, tile, row) space; tiny grids keep >= 16 rows per CTA
    if (!resident_) {
      int dev = 0, sms = 0, occ = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (d.occupancy(&occ, static_cast<CUfunction>(step_), prog_.threads, prog_.smem_bytes) != CUDA_SUCCESS || occ < 1)
        occ = prog_.ctas_per_sm;
      resident_ = std::max(1, sms) * std::max(1, occ);
      if (step_ws_) {
        int ows = 0;
        // keep the plain kernel when the variant cannot be resident, or fits a
        // single CTA per SM where the plain one fits more (its deeper windows
        // cost shared memory, and one CTA cannot hide its own level barriers:
        // the 12-kernel Hydro2D chain runs 2.0 G cell-steps/s warp-specialised
        // at 1 CTA/SM against 3.6 G plain at 2; heat3d, 2 vs 3 CTAs/SM, is
        // faster warp-specialised: 310 vs 276 G)
        if (d.occupancy(&ows, static_cast<CUfunction>(step_ws_), prog_.ws_threads, prog_.ws_smem_bytes) != CUDA_SUCCESS ||
            ows < 1 || (ows < 2 && occ >= 2))
          step_ws_ = nullptr;
        else
          resident_ws_ = std::max(1, sms) * ows;
      }
      if (step_rm_) {
        int orm = 0;
        if (d.occupancy(&orm, static_cast<CUfunction>(step_rm_), prog_.rm_threads, prog_.rm_smem_bytes) != CUDA_SUCCESS ||
            orm < 1)
          step_rm_ = nullptr;
        else
          resident_rm_ = std::max(1, sms) * orm;
      }
    }
    // whole (chunk, tile) units round-robin over the resident CTAs
    const bool span_order = lfx::option("LF_JIT_SPAN_ORDER") != nullptr;
    long chunk = pick_chunk(rows, prog_.inner_tiles, resident_, prog_.prologue, prog_.nd == 3 ? prog_.chunk : rows);
    if (span_order) chunk = std::min<long>(prog_.chunk, rows);
    if (const char* e = lfx::option("LF_JIT_CHUNK")) chunk = std::max(1L, std::min<long>(rows, std::atol(e)));
    const long total = rows * prog_.inner_tiles;
    args.chunk = static_cast<int>(chunk);
    const long units = (rows + chunk - 1) / chunk * prog_.inner_tiles;
    grid.x = static_cast<unsigned>(std::max<long>(1, std::min<long>(resident_, span_order ? total / 16 : units)));
  } else {
    grid.x = static_cast<unsigned>((rows + prog_.tile[0] - 1) / prog_.tile[0]);
  }
  // one buffer passed as an aliased axiom and goal: run in place
  for (size_t i = 0; i < T.size(); ++i)
    for (size_t j = 0; j < T.size(); ++j)
      if (!T[i].is_goal && T[j].is_goal && a.terms[i] && a.terms[i] == a.terms[j] && !T[i].dims.empty()) {
        for (const auto& q : prog_.inplace)
          if (q.ai == (int)i && q.gi == (int)j) return run_inplace(a, args, err);
        err = "axiom '" + T[i].name + "' and goal '" + T[j].name + "' share one buffer but " +
              (prog_.inplace_error.empty() ? std::string("config.aliases does not declare them")
                                           : prog_.inplace_error);
        return LF_ERR_UNSUPPORTED;
      }
  // ping-pong as the built-in executors: goals of the last step land in the
  // goal buffers, intermediate states in plan-owned scratch, axioms untouched
  std::vector<void*> src(a.terms, a.terms + T.size());
  std::vector<int> iter_axiom(T.size(), -1);  // goal terminal -> paired axiom terminal
  for (const auto& [gname, aname] : rs.iterate) {
    int gi = -1, ai = -1;
    for (size_t i = 0; i < T.size(); ++i) {
      if (T[i].is_goal && T[i].name == gname) gi = static_cast<int>(i);
      if (!T[i].is_goal && T[i].name == aname) ai = static_cast<int>(i);
    }
    if (gi >= 0 && ai >= 0) iter_axiom[gi] = ai;
  }
  int scratch_idx = 0;
  std::vector<void*> scratch(T.size(), nullptr);
  for (size_t i = 0; i < T.size(); ++i)
    if (iter_axiom[i] >= 0 && a.steps > 1) scratch[i] = a.scratch[scratch_idx++];
  std::vector<void*> cur = src;
  for (int s = 0; s < a.steps; ++s) {
    const bool to_goal = ((a.steps - 1 - s) % 2) == 0;
    std::vector<void*> bufs = cur;
    for (size_t i = 0; i < T.size(); ++i)
      if (T[i].is_goal) bufs[i] = (to_goal || iter_axiom[i] < 0) ? a.terms[i] : scratch[i];
    for (size_t i = 0; i < T.size(); ++i) args.t[i] = bufs[i];
    int st = LF_OK;
    JitMaps maps;
    // the register march stores its goal rows in 16-B vectors
    bool goals_aligned = true;
    for (size_t i = 0; i < T.size(); ++i)
      if (T[i].is_goal) goals_aligned &= reinterpret_cast<uintptr_t>(bufs[i]) % 16 == 0;
    if (prog_.march && step_rm_ && goals_aligned && tma_maps(prog_.rm_maps, bufs, rp.rows, maps)) {
      JitArgs wa = args;
      long chunk = pick_chunk(rows, prog_.rm_inner_tiles, resident_rm_, prog_.prologue, rows);
      if (const char* e = lfx::option("LF_JIT_CHUNK")) chunk = std::max(1L, std::min<long>(rows, std::atol(e)));
      wa.chunk = static_cast<int>(chunk);
      const long units = (rows + chunk - 1) / chunk * prog_.rm_inner_tiles;
      dim3 grm(static_cast<unsigned>(std::max<long>(1, std::min<long>(resident_rm_, units))));
      st = launch(step_rm_, grm, dim3(prog_.rm_threads), prog_.rm_smem_bytes, a.stream, &wa, err, &maps);
    } else if (prog_.march && step_ws_ && tma_maps(prog_.ws_maps, bufs, rp.rows, maps)) {
      // whole (chunk, tile) units round-robin over the resident CTAs
      JitArgs wa = args;
      long chunk = pick_chunk(rows, prog_.ws_inner_tiles, resident_ws_, prog_.prologue,
                              prog_.nd == 3 ? prog_.chunk : rows);
      if (const char* e = lfx::option("LF_JIT_CHUNK")) chunk = std::max(1L, std::min<long>(rows, std::atol(e)));
      wa.chunk = static_cast<int>(chunk);
      const long units = (rows + chunk - 1) / chunk * prog_.ws_inner_tiles;
      dim3 gws(static_cast<unsigned>(std::max<long>(1, std::min<long>(resident_ws_, units))));
      st = launch(step_ws_, gws, dim3(prog_.ws_threads), prog_.ws_smem_bytes, a.stream, &wa, err, &maps);
    } else {
      st = launch(step_, grid, dim3(prog_.threads), prog_.smem_bytes, a.stream, &args, err);
    }
    if (st != LF_OK) return st;
    if (fill_ && prog_.has_fill) {
      st = launch(fill_, dim3(592), dim3(256), 0, a.stream, &args, err);
      if (st != LF_OK) return st;
    }
    // the goals just written feed the paired axioms of the next step
    for (size_t i = 0; i < T.size(); ++i)
      if (iter_axiom[i] >= 0) cur[iter_axiom[i]] = bufs[i];
  }
  return LF_OK;
}

}  // namespace lfx

// extern "C" boundary of loomfuse-b200 (include/loomfuse_b200.h).
// Maps the reference's pipeline entry (parse_spec -> analysis, rulespec.cpp:550,
// storage.cpp:526) and its emitted per-goal-set function (R/SPEC.md:500) onto
// plan objects and fused sm_100a executors.  No exception crosses this file.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <dlfcn.h>
#include <nccl.h>
#include <memory>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/loomfuse_b200.h"
#include "exec/exec.hpp"
#include "jit/jit.hpp"
#include "planner/planner.hpp"

namespace {

thread_local std::string g_err;

int fail(int code, std::string msg) {
  g_err = std::move(msg);
  return code;
}

struct Signed {
  const lfx::Executor* exec;
  std::string signature;
  std::string error;  // embedded spec failed to plan (build bug)
};

const std::vector<Signed>& signed_executors() {
  static std::vector<Signed> v;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const auto& e : lfx::executors()) {
      Signed s{&e, "", ""};
      const char* text = lfx::embedded_spec(e.spec_file);
      lf::DiagList d;
      auto rs = lf::parse_spec(text ? text : "", e.spec_file, d);
      std::optional<lf::Plan> p;
      if (rs) p = lf::make_plan(*rs, d);
      if (p)
        s.signature = p->signature;
      else
        s.error = d.str();
      v.push_back(std::move(s));
    }
  });
  return v;
}

}  // namespace

struct lf_plan {
  lf::Plan plan;
  const lfx::Executor* exec = nullptr;
  std::shared_ptr<lfx::JitKernel> jit;  // generic executor when no built-in matches
  std::string unsupported;  // why no executor applies
  std::string report;
  std::mutex mu;            // guards the device caches below
  std::vector<void*> dev;   // lf_run_host device terminals
  std::vector<void*> scratch;  // per goal; iterated goals only
  lfx::ExecMem exec_mem;       // the built-in executor's own buffers (in-place bands)
  cudaStream_t stream = nullptr;
  cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams of the pipelined host path
  cudaStream_t comm = nullptr;                // halo-exchange stream of lf_run_slabs
  cudaStream_t comm2 = nullptr;               // second face stream (parallel schedule)
  std::vector<void*> slab_scratch;            // lf_run_slabs ping-pong buffers (slab-sized)
  std::vector<int64_t> slab_scratch_bytes;
  ~lf_plan() {
    for (void* p : dev)
      if (p) cudaFree(p);
    for (void* p : scratch)
      if (p) cudaFree(p);
    if (stream) cudaStreamDestroy(stream);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
    if (comm) cudaStreamDestroy(comm);
    if (comm2) cudaStreamDestroy(comm2);
    for (void* p : slab_scratch)
      if (p) cudaFree(p);
  }
};

namespace {

// ---- NCCL through dlopen: no link-time dependency; the process's copy (e.g.
// the one PyTorch loaded) is reused when present
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static NcclApi n;
  static std::once_flag once;
  std::call_once(once, [] {
    n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!n.h) n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!n.h) {
      n.error = "libnccl.so.2 not found";
      return;
    }
    auto sym = [&](const char* name) { return dlsym(n.h, name); };
    n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
    n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
    n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(sym("ncclAllReduce"));
    n.unique_id = reinterpret_cast<decltype(n.unique_id)>(sym("ncclGetUniqueId"));
    n.init_rank = reinterpret_cast<decltype(n.init_rank)>(sym("ncclCommInitRank"));
    n.init_all = reinterpret_cast<decltype(n.init_all)>(sym("ncclCommInitAll"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(sym("ncclCommDestroy"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
    if (!n.group_start || !n.group_end || !n.send || !n.recv || !n.unique_id || !n.init_rank || !n.init_all ||
        !n.destroy || !n.all_reduce)
      n.error = "libnccl.so.2 lacks the point-to-point / all-reduce API";
  });
  return n;
}

int nccl_status(ncclResult_t r, const char* what, std::string& err) {
  if (r == ncclSuccess) return LF_OK;
  const NcclApi& n = nccl();
  err = std::string(what) + ": " + (n.error_string ? n.error_string(r) : ("ncclResult " + std::to_string(r)));
  return LF_ERR_CUDA;
}

// ---- slab runs (lf_run_slabs): halo geometry and the overlapped schedule ----

// Per terminal: the iterate pairing (goal -> axiom index) and, along the
// outermost dim, the storage row size and the ghost rows below/above the
// slab's own rows; whether dim 0 wraps (periodic boundary).
struct SlabGeom {
  std::vector<int> paired;
  std::vector<int64_t> rb;
  std::vector<long> below, above;
  std::vector<char> periodic;
  std::vector<int64_t> elem;       // element bytes per terminal
  long halo_lo = 0, halo_hi = 0;  // max ghost rows below / above over the iterated terminals
  long n0 = 0;
  int world = 1;                   // ranks of the whole decomposition
};

SlabGeom slab_geom(const lf::Plan& P) {
  const auto& T = P.terminals;
  const auto& rs = P.rs;
  SlabGeom g;
  g.n0 = rs.ranges[0].trips();
  const long lo0 = rs.ranges[0].lo;
  g.paired.assign(T.size(), -1);
  g.rb.assign(T.size(), 0);
  g.below.assign(T.size(), 0);
  g.above.assign(T.size(), 0);
  g.periodic.assign(T.size(), 0);
  g.elem.assign(T.size(), 0);
  for (size_t i = 0; i < T.size(); ++i) g.elem[i] = T[i].elem_bytes;
  for (const auto& [gname, aname] : rs.iterate)
    for (size_t i = 0; i < T.size(); ++i)
      for (size_t a = 0; a < T.size(); ++a)
        if (T[i].is_goal && T[i].name == gname && !T[a].is_goal && T[a].name == aname) g.paired[i] = (int)a;
  for (size_t i = 0; i < T.size(); ++i) {
    const auto& t = T[i];
    if (t.extent.empty()) continue;
    int64_t rb = t.elem_bytes;
    for (size_t k = 1; k < t.extent.size(); ++k) rb *= t.extent[k];
    g.rb[i] = rb;
    g.below[i] = lo0 - t.base[0];
    g.above[i] = t.extent[0] - g.n0 - g.below[i];
    auto it = rs.boundary.find(t.name);
    if (it == rs.boundary.end()) it = rs.boundary.find("*");
    g.periodic[i] = it != rs.boundary.end() && !it->second.empty() && it->second[0] == lf::Boundary::periodic;
    if (g.paired[i] >= 0) {
      g.halo_lo = std::max(g.halo_lo, g.below[i]);
      g.halo_hi = std::max(g.halo_hi, g.above[i]);
    }
  }
  return g;
}

struct RankState {
  int rank = 0;
  long lo = 0, hi = 0;
  void* const* terms = nullptr;
  std::vector<void*> scratch;    // per terminal; iterated goals only
  std::vector<void*> cur, bufs;  // this step's inputs / outputs
};

// in place: the slab-sized pairs share their buffers; only rank-0 pairs (per-step
// reduction slots) still alternate
std::vector<int64_t> scratch_need(const SlabGeom& g, const RankState& r, bool inplace = false) {
  std::vector<int64_t> need(g.paired.size(), 0);
  for (size_t i = 0; i < g.paired.size(); ++i)
    if (g.paired[i] >= 0 && !(inplace && g.rb[i]))
      need[i] = g.rb[i] ? g.rb[i] * (r.hi - r.lo + g.below[i] + g.above[i]) : g.elem[i];
  return need;
}

int alloc_list(const std::vector<int64_t>& need, std::vector<void*>& out, std::string& err) {
  out.assign(need.size(), nullptr);
  for (size_t i = 0; i < need.size(); ++i)
    if (need[i]) {
      cudaError_t e = cudaMalloc(&out[i], need[i]);
      if (e != cudaSuccess) {
        for (void* q : out)
          if (q) cudaFree(q);
        out.clear();
        return lfx::cuda_status(e, "cudaMalloc(slab scratch)", err);
      }
    }
  return LF_OK;
}

int make_side_stream(cudaStream_t* s, std::string& err) {
  int lowp = 0, highp = 0;
  cudaDeviceGetStreamPriorityRange(&lowp, &highp);
  cudaError_t e = cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, highp);
  return e == cudaSuccess ? LF_OK : lfx::cuda_status(e, "cudaStreamCreate", err);
}

int slab_check(const lf_plan* plan, const SlabGeom& g, int world, std::string& err) {
  if (plan->plan.rs.ranges.empty()) {
    err = "slab runs need a loop dimension";
    return LF_ERR_UNSUPPORTED;
  }
  if (plan->jit && !plan->jit->program().nest_kernels.empty()) {
    err = "multi-nest plans (reductions) run on the whole domain only";
    return LF_ERR_UNSUPPORTED;
  }
  if (g.n0 < world) {
    err = "more ranks than rows along the outer dimension";
    return LF_ERR_SPEC;
  }
  // every rank must own at least as many rows as a neighbour's ghost band:
  // the exchange sends a rank's own outermost rows (single hop)
  const long need = std::max(g.halo_lo, g.halo_hi);
  if (g.n0 / world < need) {
    err = "slabs of " + std::to_string(g.n0 / world) + " row(s) are thinner than the " + std::to_string(need) +
          "-row halo exchanged with each neighbour (use fewer ranks)";
    return LF_ERR_SPEC;
  }
  return LF_OK;
}

// The overlapped schedule of every step, for each local rank: first the
// output rows its neighbours need -- [0, halo_hi) and [rows - halo_lo, rows),
// the two faces launched side by side on the high-priority streams `side` and
// `side2` -- then the exchange on `side`, overlapped with the interior rows on
// `stream`; the next step waits for both.  Iterated goals ping-pong between the
// goal buffers and the rank's scratch so the last step lands in the goals.
// LF_SLAB_SCHEDULE selects the variant (tools/slab_probe.py measures them):
//   parallel (default)  faces side by side, then the interior next to the exchange;
//   serial              both faces on `stream`, then the interior;
//   concurrent          faces and exchange on `side` while the interior already
//                       runs on `stream` (disjoint output rows, same inputs) --
//                       best for thin slabs, but the faces then compete with the
//                       interior for SM slots and HBM (heat3d 512^3: 0.79 of
//                       the single-domain rate, against 0.96 for serial).
// Executors with per-step MAX reductions (Executor::max_reduce, the adaptive
// CFL time step): the rank-0 iterated goal slots are zeroed before each step
// (the local ranks of one device share one slot), `combine` merges the ranks'
// maxima after the step (NCCL MAX all-reduce; nullptr when the ranks share
// the slot), and the executor finalises the last one into every rank's goal.
int run_slabs_core(lf_plan* plan, const SlabGeom& g, std::vector<RankState>& R, int steps, cudaStream_t stream,
                   cudaStream_t side,
                   const std::function<int(std::vector<RankState>&, cudaStream_t, std::string&)>& exchange,
                   std::string& err,
                   const std::function<int(void* slot, cudaStream_t, std::string&)>& combine = nullptr,
                   bool inplace = false) {
  const size_t nt = g.paired.size();
  const bool mr = plan->exec && plan->exec->max_reduce;
  std::vector<size_t> scalars;  // rank-0 iterated goals
  if (mr)
    for (size_t i = 0; i < nt; ++i)
      if (g.paired[i] >= 0 && !g.rb[i]) scalars.push_back(i);
  for (auto& r : R) r.cur.assign(r.terms, r.terms + nt);
  cudaEvent_t faces_done, exchanged;
  cudaEventCreateWithFlags(&faces_done, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&exchanged, cudaEventDisableTiming);
  int step_no = 0;
  auto launch = [&](RankState& r, long plo, long phi, cudaStream_t on) {
    lf_slab slab{r.lo, r.hi, g.n0, plo, phi};
    lfx::ExecArgs ea;
    ea.plan = &plan->plan;
    ea.terms = r.bufs.data();
    ea.steps = 1;
    ea.stream = on;
    ea.slab = &slab;
    ea.raw_max_input = mr && step_no > 0;
    if (inplace) {  // every iterated goal on its axiom's slab buffer (whole-slab launches only)
      ea.inplace = true;
      ea.mem = &plan->exec_mem;
    }
    return plan->exec ? plan->exec->run(ea, err) : plan->jit->run(ea, err);
  };
  // LF_SLAB_SCHEDULE: parallel (default) | serial | concurrent -- see above
  const int sched_env = [] {
    const char* e = lfx::option("LF_SLAB_SCHEDULE");
    if (e && std::string(e) == "serial") return 1;
    if (e && std::string(e) == "concurrent") return 2;
    if (e && std::string(e) == "whole") return 3;
    if (e && std::string(e) == "parallel") return 0;
    return -1;
  }();
  // default: `whole` (one launch per rank and step, then the exchange) when a
  // step's compute dwarfs the face launches it would otherwise split off --
  // a pipeline fill of a few rows per launch and a partly idle grid -- i.e.
  // for slabs of many rows; `parallel` for thin slabs, whose exchange is worth
  // hiding behind the interior (tools/slab_probe.py, profiles/r02_slab_schedules.txt)
  long min_rows = g.n0;
  for (const auto& r : R) min_rows = std::min(min_rows, r.hi - r.lo);
  // no rank has a neighbour to exchange with (one rank, no periodic outer
  // dimension): every step is one launch per rank, nothing else
  bool peers = R.size() > 1 || g.world > 1;
  for (size_t i = 0; i < g.paired.size(); ++i) peers |= g.paired[i] >= 0 && g.periodic[i];
  // in place: one launch per rank and step (the face / interior split would need ordered parts)
  const int sched = (!peers || inplace) ? 3 : (sched_env >= 0 ? sched_env : (min_rows >= 1024 ? 3 : 0));
  cudaStream_t side2 = side;
  if (sched == 0) {
    if (!plan->comm2 && make_side_stream(&plan->comm2, err) != LF_OK) return LF_ERR_CUDA;
    side2 = plan->comm2;
  }
  cudaEvent_t mark, face2;
  cudaEventCreateWithFlags(&mark, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&face2, cudaEventDisableTiming);
  // the side streams start after whatever the caller queued before the run
  cudaEventRecord(mark, stream);
  cudaStreamWaitEvent(side, mark, 0);
  if (side2 != side) cudaStreamWaitEvent(side2, mark, 0);
  int st = LF_OK;
  for (int s = 0; s < steps && st == LF_OK; ++s) {
    step_no = s;
    const bool to_goal = ((steps - 1 - s) % 2) == 0;
    for (auto& r : R) {
      r.bufs = r.cur;
      for (size_t i = 0; i < nt; ++i)
        if (plan->plan.terminals[i].is_goal)
          r.bufs[i] = (to_goal || g.paired[i] < 0 || (inplace && g.rb[i])) ? r.terms[i] : r.scratch[i];
    }
    if (!scalars.empty()) {
      for (size_t i : scalars) {
        for (auto& r : R) r.bufs[i] = R[0].bufs[i];  // one accumulation slot per device
        if (cudaMemsetAsync(R[0].bufs[i], 0, g.elem[i], stream) != cudaSuccess) {
          err = "cudaMemsetAsync(reduction slot) failed";
          st = LF_ERR_CUDA;
        }
      }
      cudaEventRecord(mark, stream);  // the faces start after the zeroing
      cudaStreamWaitEvent(side, mark, 0);
      if (side2 != side) cudaStreamWaitEvent(side2, mark, 0);
    }
    if (sched == 3) {  // whole: one launch per rank, then the exchange on the same stream, the next step after it
      for (size_t k = 0; k < R.size() && st == LF_OK; ++k) st = launch(R[k], 0, R[k].hi - R[k].lo, stream);
      if (st != LF_OK) break;
      if (peers && (st = exchange(R, stream, err)) != LF_OK) break;
      if (combine)
        for (size_t i : scalars)
          if (st == LF_OK) st = combine(R[0].bufs[i], stream, err);
      for (auto& r : R)
        for (size_t i = 0; i < nt; ++i)
          if (g.paired[i] >= 0) r.cur[g.paired[i]] = r.bufs[i];
      continue;
    }
    std::vector<char> split(R.size());
    const cudaStream_t top = sched == 1 ? stream : side, bottom = sched == 1 ? stream : side2;
    for (size_t k = 0; k < R.size() && st == LF_OK; ++k) {
      const long rows = R[k].hi - R[k].lo;
      split[k] = rows > g.halo_lo + g.halo_hi && (g.halo_lo || g.halo_hi);
      if (!split[k]) {
        st = launch(R[k], 0, rows, top);
        continue;
      }
      if (g.halo_hi) st = launch(R[k], 0, g.halo_hi, top);
      if (st == LF_OK && g.halo_lo) st = launch(R[k], rows - g.halo_lo, rows, bottom);
    }
    if (st != LF_OK) break;
    if (sched == 1) {  // faces done on the main stream: hand them to the exchange
      cudaEventRecord(faces_done, stream);
      cudaStreamWaitEvent(side, faces_done, 0);
    } else if (side2 != side) {  // both face streams joined on `side`
      cudaEventRecord(face2, side2);
      cudaStreamWaitEvent(side, face2, 0);
    }
    cudaEventRecord(faces_done, side);
    if ((st = exchange(R, side, err)) != LF_OK) break;
    cudaEventRecord(exchanged, side);
    if (sched == 0) cudaStreamWaitEvent(stream, faces_done, 0);  // interior after the faces, next to the exchange
    for (size_t k = 0; k < R.size() && st == LF_OK; ++k)
      if (split[k]) st = launch(R[k], g.halo_hi, R[k].hi - R[k].lo - g.halo_lo, stream);
    cudaStreamWaitEvent(stream, exchanged, 0);
    if (combine)
      for (size_t i : scalars)
        if (st == LF_OK) st = combine(R[0].bufs[i], stream, err);
    if (sched != 1) {  // next step's faces: after this step's interior (input rows, ping-pong buffer)
      cudaEventRecord(mark, stream);
      cudaStreamWaitEvent(side, mark, 0);
      if (side2 != side) cudaStreamWaitEvent(side2, mark, 0);
    }
    for (auto& r : R)
      for (size_t i = 0; i < nt; ++i)
        if (g.paired[i] >= 0) r.cur[g.paired[i]] = r.bufs[i];
  }
  if (st == LF_OK && !scalars.empty()) {
    // the last step wrote the goal slot of rank 0: finalise, then hand every
    // other local rank its copy
    lfx::ExecArgs ea;
    ea.plan = &plan->plan;
    ea.terms = R[0].terms;
    ea.stream = stream;
    if (plan->exec->finalize) st = plan->exec->finalize(ea, err);
    for (size_t k = 1; k < R.size() && st == LF_OK; ++k)
      for (size_t i : scalars)
        if (cudaMemcpyAsync(R[k].terms[i], R[0].terms[i], g.elem[i], cudaMemcpyDeviceToDevice, stream) !=
            cudaSuccess) {
          err = "cudaMemcpyAsync(reduction result) failed";
          st = LF_ERR_CUDA;
        }
  }
  cudaEventDestroy(mark);
  cudaEventDestroy(face2);
  cudaEventDestroy(faces_done);
  cudaEventDestroy(exchanged);
  return st;
}

int64_t terminal_bytes(const lf::Terminal& t) {
  int64_t n = t.elem_bytes;
  for (long e : t.extent) n *= e;
  return n;
}

int ensure_scratch(lf_plan* p, std::string& err) {
  const auto& T = p->plan.terminals;
  if (p->scratch.size() == T.size()) return LF_OK;
  p->scratch.assign(T.size(), nullptr);
  for (size_t i = 0; i < T.size(); ++i) {
    if (!T[i].is_goal) continue;
    bool iterated = false;
    for (const auto& [g, a] : p->plan.rs.iterate) iterated |= g == T[i].name;
    if (!iterated) continue;
    cudaError_t e = cudaMalloc(&p->scratch[i], terminal_bytes(T[i]));
    if (e != cudaSuccess) return lfx::cuda_status(e, "cudaMalloc(scratch)", err);
  }
  return LF_OK;
}

// scratch pointers ordered like the executors expect: one per iterated goal,
// in goal order
std::vector<void*> scratch_list(lf_plan* p) {
  std::vector<void*> s;
  for (size_t i = 0; i < p->plan.terminals.size(); ++i)
    if (p->scratch[i]) s.push_back(p->scratch[i]);
  return s;
}

int check_run_args(const lf_plan* plan, void* const* terms, int nterm, int steps) {
  if (!plan) return fail(LF_ERR_SPEC, "plan is NULL");
  if (!plan->exec && !plan->jit)
    return fail(LF_ERR_UNSUPPORTED, "no fused sm_100a executor for chain '" + plan->plan.rs.name +
                                        "' (signature " + plan->plan.signature + "): " + plan->unsupported);
  if (nterm != static_cast<int>(plan->plan.terminals.size()))
    return fail(LF_ERR_SPEC, "expected " + std::to_string(plan->plan.terminals.size()) + " terminal buffers, got " +
                                 std::to_string(nterm));
  if (!terms) return fail(LF_ERR_SPEC, "terminal array is NULL");
  for (int i = 0; i < nterm; ++i)
    if (!terms[i]) return fail(LF_ERR_SPEC, "terminal " + plan->plan.terminals[i].name + " is NULL");
  if (steps < 1) return fail(LF_ERR_SPEC, "steps must be >= 1");
  if (steps > 1 && plan->plan.rs.iterate.empty())
    return fail(LF_ERR_SPEC, "steps > 1 needs `iterate:` pairs in the rule file's config");
  return LF_OK;
}

}  // namespace

extern "C" {

const char* lf_last_error(void) { return g_err.c_str(); }

const char* lf_version(void) { return "loomfuse-b200 0.1 (sm_100a)"; }

int lf_set_option(const char* name, const char* value) {
  if (lfx::set_option(name, value, value ? 0 : 1) != 0)
    return fail(LF_ERR_SPEC, std::string("lf_set_option: '") + (name ? name : "(null)") + "' is not an LF_* switch");
  return LF_OK;
}

int lf_plan_create(const char* spec_text, size_t len, const char* filename, lf_plan** out) {
  return lf_plan_create_ex(spec_text, len, filename, nullptr, 0, out);
}

int lf_plan_create_ex(const char* spec_text, size_t len, const char* filename, const char* kernel_source,
                      size_t kernel_len, lf_plan** out) {
  try {
    g_err.clear();
    if (!out) return fail(LF_ERR_SPEC, "out is NULL");
    *out = nullptr;
    if (!spec_text) return fail(LF_ERR_SPEC, "spec_text is NULL");
    std::string text(spec_text, len);
    std::string file = filename ? filename : "<input>";
    lf::DiagList d;
    auto rs = lf::parse_spec(text, file, d);
    if (!rs) return fail(LF_ERR_SPEC, d.str());
    auto plan = lf::make_plan(*rs, d);
    if (!plan) return fail(LF_ERR_SPEC, d.str());
    auto* p = new lf_plan;
    p->plan = std::move(*plan);
    p->report = p->plan.report_json();
    std::string why = "no built-in executor implements this chain";
    // LF_NO_BUILTIN=1: skip the hand-written executors (A/B runs of the generic one)
    const bool no_builtin = lfx::option("LF_NO_BUILTIN") && std::atoi(lfx::option("LF_NO_BUILTIN")) != 0;
    for (const auto& s : signed_executors()) {
      if (no_builtin) break;
      if (!s.error.empty()) {
        why = std::string("embedded spec ") + s.exec->spec_file + " failed to plan: " + s.error;
        continue;
      }
      if (s.signature != p->plan.signature) continue;
      std::string w;
      if (s.exec->supports(p->plan, w)) {
        p->exec = s.exec;
        break;
      }
      why = std::string(s.exec->name) + ": " + w;
    }
    if (!p->exec) {
      // generic path: `body:` chains compiled for sm_100a with NVRTC
      std::string jwhy;
      p->jit = lfx::JitKernel::build(p->plan, jwhy,
                                     kernel_source ? std::string(kernel_source, kernel_len) : std::string());
      if (!p->jit) p->unsupported = why + "; generic executor: " + jwhy;
    }
    *out = p;
    return LF_OK;
  } catch (const std::exception& e) {
    return fail(LF_ERR_INTERNAL, std::string("internal error: ") + e.what());
  }
}

int lf_spec_print(const char* spec_text, size_t len, const char* filename, char* buf, size_t cap,
                  size_t* needed) {
  try {
    g_err.clear();
    if (!spec_text) return fail(LF_ERR_SPEC, "spec_text is NULL");
    lf::DiagList d;
    auto rs = lf::parse_spec(std::string(spec_text, len), filename ? filename : "<input>", d);
    if (!rs) return fail(LF_ERR_SPEC, d.str());
    std::string text = lf::print_spec(*rs);
    if (needed) *needed = text.size() + 1;
    if (buf && cap) {
      size_t n = std::min(cap - 1, text.size());
      std::memcpy(buf, text.data(), n);
      buf[n] = '\0';
    }
    return LF_OK;
  } catch (const std::exception& e) {
    return fail(LF_ERR_INTERNAL, std::string("internal error: ") + e.what());
  }
}

void lf_plan_destroy(lf_plan* plan) { delete plan; }

int lf_plan_num_terminals(const lf_plan* plan) {
  return plan ? static_cast<int>(plan->plan.terminals.size()) : 0;
}

int lf_plan_terminal(const lf_plan* plan, int idx, lf_terminal* out) {
  if (!plan || !out) return fail(LF_ERR_SPEC, "NULL argument");
  if (idx < 0 || idx >= static_cast<int>(plan->plan.terminals.size()))
    return fail(LF_ERR_SPEC, "terminal index out of range");
  const auto& t = plan->plan.terminals[idx];
  if (t.dims.size() > LF_MAX_DIMS) return fail(LF_ERR_SPEC, "terminal rank exceeds LF_MAX_DIMS");
  std::memset(out, 0, sizeof *out);
  std::strncpy(out->name, t.name.c_str(), sizeof out->name - 1);
  std::strncpy(out->type, t.type.c_str(), sizeof out->type - 1);
  out->is_goal = t.is_goal;
  out->elem_bytes = t.elem_bytes;
  out->ndim = static_cast<int32_t>(t.dims.size());
  for (size_t k = 0; k < t.dims.size(); ++k) {
    out->loop_dim[k] = t.dims[k];
    out->extent[k] = t.extent.size() > k ? t.extent[k] : 1;
    out->base[k] = t.base.size() > k ? t.base[k] : 0;
  }
  out->bytes = terminal_bytes(t);
  return LF_OK;
}

int lf_plan_report(const lf_plan* plan, char* buf, size_t cap, size_t* needed) {
  if (!plan) return fail(LF_ERR_SPEC, "plan is NULL");
  if (needed) *needed = plan->report.size() + 1;
  if (buf && cap) {
    size_t n = std::min(cap - 1, plan->report.size());
    std::memcpy(buf, plan->report.data(), n);
    buf[n] = '\0';
  }
  return LF_OK;
}

const char* lf_plan_executor(const lf_plan* plan) {
  if (!plan) return "";
  if (plan->exec) return plan->exec->name;
  if (!plan->jit) return "";
  const auto& pg = plan->jit->program();
  return !pg.nest_kernels.empty() ? "jit_nests_fused" : (pg.march ? "jit_window_fused" : "jit_tiled_fused");
}

int lf_plan_launches_per_step(const lf_plan* plan) {
  if (!plan) return 0;
  if (plan->exec) return plan->exec->launches_per_step;
  if (!plan->jit) return 0;
  const auto& pg = plan->jit->program();
  return static_cast<int>(std::max<size_t>(1, pg.nest_kernels.size())) + (pg.has_fill ? 1 : 0);
}

int lf_plan_grid_passes(const lf_plan* plan, int steps) {
  if (!plan || steps < 1) return 0;
  if (plan->exec && plan->exec->passes) return plan->exec->passes(plan->plan, steps, false);
  return steps;
}

int lf_plan_launches(const lf_plan* plan, int steps) {
  if (!plan || steps < 1) return 0;
  if (plan->exec) return lf_plan_grid_passes(plan, steps) * plan->exec->launches_per_step;
  return steps * lf_plan_launches_per_step(plan);
}

double lf_plan_compulsory_bytes_per_cell(const lf_plan* plan) {
  if (!plan) return 0.0;
  if (plan->exec) return plan->exec->bytes_per_cell;
  if (!plan->jit) return 0.0;
  double b = 0;  // every non-scalar terminal read or written once per cell
  for (const auto& t : plan->plan.terminals)
    if (!t.dims.empty()) b += t.elem_bytes;
  return b;
}

const char* lf_plan_source(const lf_plan* plan) {
  return plan && plan->jit ? plan->jit->program().source.c_str() : "";
}

// an axiom buffer passed again as a goal (in-place run)
static bool shares_buffer(const lf_plan* plan, void* const* terms) {
  const auto& T = plan->plan.terminals;
  for (size_t i = 0; i < T.size(); ++i)
    for (size_t j = 0; j < T.size(); ++j)
      if (!T[i].is_goal && T[j].is_goal && terms[i] && terms[i] == terms[j]) return true;
  return false;
}

// In-place run of a built-in executor: every iterated full-rank goal sits on
// its axiom's buffer, the pair is declared in config.aliases (the reference's
// contract for in-place updates, storage.cpp:453-524), and nothing else is
// shared.  `share[g]` = axiom index for such goals.
static int exec_inplace_pairs(const lf_plan* plan, void* const* terms, std::vector<int>& share, std::string& err) {
  const auto& T = plan->plan.terminals;
  const auto& rs = plan->plan.rs;
  share.assign(T.size(), -1);
  if (!plan->exec->inplace) {
    err = std::string(plan->exec->name) +
          " ping-pongs between distinct buffers; in-place runs (config.aliases) use the generic executor";
    return LF_ERR_UNSUPPORTED;
  }
  for (size_t i = 0; i < T.size(); ++i)
    for (size_t j = 0; j < T.size(); ++j) {
      if (T[i].is_goal || !T[j].is_goal || !terms[i] || terms[i] != terms[j]) continue;
      bool iterated = false, declared = false;
      for (const auto& [gname, aname] : rs.iterate) iterated |= gname == T[j].name && aname == T[i].name;
      for (const auto& [in, out] : rs.aliases) declared |= in == T[i].name && out == T[j].name;
      if (!iterated || !declared) {
        err = "axiom '" + T[i].name + "' and goal '" + T[j].name + "' share one buffer but " +
              (iterated ? "config.aliases does not declare them" : "are not an iterate pair");
        return LF_ERR_UNSUPPORTED;
      }
      share[j] = static_cast<int>(i);
    }
  for (const auto& [gname, aname] : rs.iterate)
    for (size_t j = 0; j < T.size(); ++j)
      if (T[j].is_goal && T[j].name == gname && !T[j].dims.empty() && share[j] < 0) {
        err = "in-place runs take every iterated goal on its axiom's buffer ('" + gname + "' has its own)";
        return LF_ERR_UNSUPPORTED;
      }
  return LF_OK;
}


// Slab runs in place: the rank passes every iterated slab-sized goal on its
// axiom's slab buffer (declared in config.aliases) and the built-in executor
// runs whole-slab launches in place; the generic executor's in-place runs
// cover the whole domain only.
static int slab_inplace(const lf_plan* plan, void* const* terms, bool& inplace, std::string& err) {
  inplace = shares_buffer(plan, terms);
  if (!inplace) return LF_OK;
  if (!plan->exec || !plan->exec->inplace_parts) {
    err = std::string("slab runs of ") + (plan->exec ? plan->exec->name : "the generic executor") +
          " need distinct axiom and goal buffers (its in-place runs cover the whole domain)";
    return LF_ERR_UNSUPPORTED;
  }
  std::vector<int> share;
  if (int st = exec_inplace_pairs(plan, terms, share, err)) return st;
  const auto& T = plan->plan.terminals;
  for (size_t j = 0; j < T.size(); ++j)
    if (share[j] >= 0 && T[j].dims.empty()) {  // per-step reduction slots alternate between goal and scratch
      err = "slab runs need a separate buffer for the rank-0 goal '" + T[j].name + "'";
      return LF_ERR_UNSUPPORTED;
    }
  return LF_OK;
}

int lf_run(const lf_plan* cplan, void* const* terms, int nterm, int steps, void* cuda_stream) {
  try {
    g_err.clear();
    int st = check_run_args(cplan, terms, nterm, steps);
    if (st != LF_OK) return st;
    lf_plan* plan = const_cast<lf_plan*>(cplan);
    std::lock_guard<std::mutex> lk(plan->mu);
    std::string err;
    const bool inplace = shares_buffer(plan, terms);
    if (inplace && plan->exec) {
      std::vector<int> share;
      if ((st = exec_inplace_pairs(plan, terms, share, err)) != LF_OK) return fail(st, err);
    }
    std::vector<void*> scratch;
    if (steps > 1 && !inplace) {
      if ((st = ensure_scratch(plan, err)) != LF_OK) return fail(st, err);
      scratch = scratch_list(plan);
    }
    lfx::ExecArgs a;
    a.plan = &plan->plan;
    a.terms = terms;
    a.steps = steps;
    a.stream = static_cast<cudaStream_t>(cuda_stream);
    a.scratch = scratch.data();
    a.inplace = inplace && plan->exec;
    a.mem = &plan->exec_mem;
    st = plan->exec ? plan->exec->run(a, err) : plan->jit->run(a, err);
    if (st != LF_OK) return fail(st, err);
    return LF_OK;
  } catch (const std::exception& e) {
    return fail(LF_ERR_INTERNAL, std::string("internal error: ") + e.what());
  }
}

// Host runs of large grids, pipelined: the outer dimension is cut into parts.
// The FIRST step computes part p as soon as its input rows (and the halo above
// them) have come up on one copy stream; the LAST step sends part p's finished
// rows down on a second copy stream while part p+1 is computed; the steps in
// between are whole-domain launches.  So the PCIe transfers overlap the first
// and the last step's compute (for one step: both directions and the SMs at
// once) instead of preceding and following the whole run.  Every executor
// computes row parts (lf_slab part ranges); iterated state ping-pongs through
// the plan's scratch so the last step lands in the goals; ghost rows of the
// goals are copied once all parts are done.
// In place (`inplace`: every iterated goal on its axiom's device buffer, an
// executor that runs ordered row parts in place): only the wavefront applies
// -- parts of a step in ascending order, each part's last halo rows committed
// after the next part's launch has read them (ExecArgs::inplace_phase) -- and
// kNotPipelined is returned, before anything is issued, when it does not.
constexpr int kNotPipelined = -1;
static int run_host_pipelined(lf_plan* plan, void* const* terms, const std::vector<void*>& dterms, int parts,
                              int steps, std::string& err, bool inplace = false) {
  const auto& T = plan->plan.terminals;
  const long n0 = plan->plan.rs.ranges[0].trips();
  const long lo0 = plan->plan.rs.ranges[0].lo;
  for (cudaStream_t* s : {&plan->h2d, &plan->d2h})
    if (!*s) {
      cudaError_t e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
      if (e != cudaSuccess) return lfx::cuda_status(e, "cudaStreamCreate", err);
    }
  auto chunked = [&](const lf::Terminal& t) { return !t.dims.empty() && t.dims[0] == 0; };
  auto row_bytes = [&](const lf::Terminal& t) {
    int64_t b = t.elem_bytes;
    for (size_t k = 1; k < t.extent.size(); ++k) b *= t.extent[k];
    return b;
  };
  // Multi-step runs of chains whose outer dimension does not wrap run as a
  // wavefront over (step, part) -- see below -- in parts of >= 8 M cells (a part
  // launch costs host time and a pipeline fill per row segment: Hydro2D 4096^2 x20
  // runs 54 ms per run whole-domain, 57 / 70 ms as a wavefront of 16 / 32 parts),
  // and only where that gives >= 16 parts; 32768^2 x10: 2188 ms first/last-step
  // pipelined, 1376 / 1289 / 1274 ms as a wavefront of 32 / 64 / 96-128 parts.
  // LF_HOST_WAVEFRONT=1 / 0 forces it on / off, LF_HOST_PARTS fixes the parts.
  bool periodic0 = false;
  for (const auto& [gname, mode] : plan->plan.rs.boundary)
    if (!mode.empty() && mode[0] == lf::Boundary::periodic) periodic0 = true;
  long halo0 = 0;
  for (const auto& t : T)
    if (chunked(t)) halo0 = std::max({halo0, lo0 - t.base[0], t.extent[0] - n0 - (lo0 - t.base[0])});
  long cells = 1;
  for (const auto& r : plan->plan.rs.ranges) cells *= r.trips();
  const int wparts = lfx::option("LF_HOST_PARTS") ? parts : static_cast<int>(std::min<long>(128, cells / (8L << 20)));
  bool wavefront = wparts >= 16;
  if (const char* e = lfx::option("LF_HOST_WAVEFRONT")) wavefront = std::atoi(e) != 0;
  wavefront = wavefront && steps > 1 && !periodic0 && wparts >= 2 && n0 / wparts >= std::max(1L, halo0);
  // per-step MAX reductions over the whole grid (Executor::max_reduce, the CFL time
  // step): step s+1 needs step s's complete maximum, so no wavefront -- the first
  // and the last step still run in parts under the copies; each step's goal slot
  // is zeroed before its launches and the last one finalised (as lf_run_slabs does)
  const bool mr = plan->exec && plan->exec->max_reduce;
  if (mr) wavefront = false;
  if (wavefront) parts = wparts;
  if (inplace && (!wavefront || n0 / parts < 2 * std::max(1L, halo0))) return kNotPipelined;  // parts of >= 2 halos
  auto copy = [&](void* dst, const void* src, int64_t bytes, cudaMemcpyKind kind, cudaStream_t st) {
    if (bytes <= 0) return LF_OK;
    return lfx::cuda_status(cudaMemcpyAsync(dst, src, bytes, kind, st), "cudaMemcpyAsync(pipelined)", err);
  };
  // iterate pairs: goal terminal -> axiom terminal
  std::vector<int> axiom_of(T.size(), -1);
  for (const auto& [gname, aname] : plan->plan.rs.iterate)
    for (size_t i = 0; i < T.size(); ++i)
      for (size_t a = 0; a < T.size(); ++a)
        if (T[i].is_goal && T[i].name == gname && !T[a].is_goal && T[a].name == aname) axiom_of[i] = (int)a;
  // device buffers of step s: inputs = the previous step's outputs for the
  // iterated axioms; outputs = goals or scratch, alternating so that the last
  // step writes the goals
  std::vector<void*> cur(dterms);
  auto step_bufs = [&](int s) {
    std::vector<void*> b(cur);
    const bool to_goal = ((steps - 1 - s) % 2) == 0;
    for (size_t i = 0; i < T.size(); ++i)
      if (T[i].is_goal && axiom_of[i] >= 0 && !to_goal && !inplace) b[i] = plan->scratch[i];
    return b;
  };
  auto advance = [&](const std::vector<void*>& b) {
    for (size_t i = 0; i < T.size(); ++i)
      if (axiom_of[i] >= 0) cur[axiom_of[i]] = b[i];
  };
  // in place: (step, part) and the phase (0 the step, 1 the commit of the part's deferred last rows)
  auto run_part = [&](std::vector<void*>& b, long a, long e, bool whole, int s = 0, int p = 0, int phase = 0) {
    lf_slab slab{0, n0, n0, a, e};
    lfx::ExecArgs ea;
    ea.plan = &plan->plan;
    ea.terms = b.data();
    ea.steps = 1;
    ea.stream = plan->stream;
    if (!whole) {
      ea.slab = &slab;
      ea.whole_domain_parts = true;
    } else if (mr) {  // one step of a driver's schedule: the executor neither zeroes nor finalises
      slab.part_lo = slab.part_hi = 0;
      ea.slab = &slab;
      ea.whole_domain_parts = true;
    }
    ea.raw_max_input = mr && s > 0;
    if (inplace) {
      ea.inplace = true;
      ea.mem = &plan->exec_mem;
      ea.inplace_phase = phase;
      // a part's rows wait through one launch of the same step: two slots per
      // step, reused once the step that far ahead cannot overlap (tau = p + 2s:
      // step s + ring/2 starts after tau >= 2s + ring > p + 1 + 2s)
      const int ring = std::min(2 * steps, (parts + 5) / 2 * 2);
      ea.inplace_slots = ring;
      ea.inplace_slot = (2 * s + (p & 1)) % ring;
    }
    return plan->exec ? plan->exec->run(ea, err) : plan->jit->run(ea, err);
  };
  std::vector<cudaEvent_t> up(parts), done(parts);
  for (int p = 0; p < parts; ++p) {
    cudaEventCreateWithFlags(&up[p], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&done[p], cudaEventDisableTiming);
  }
  int st = LF_OK;
  // inputs that do not span the outer dimension go up first, whole
  for (size_t i = 0; i < T.size() && st == LF_OK; ++i)
    if (!T[i].is_goal && !chunked(T[i])) st = copy(dterms[i], terms[i], terminal_bytes(T[i]), cudaMemcpyHostToDevice, plan->h2d);
  auto part_rows = [&](int p) { return std::make_pair(n0 * p / parts, n0 * (p + 1) / parts); };
  // max_reduce: this step's reduction slots (rank-0 iterated goals) start from zero
  auto zero_reductions = [&](const std::vector<void*>& b) {
    if (!mr) return;
    for (size_t i = 0; i < T.size() && st == LF_OK; ++i)
      if (T[i].is_goal && axiom_of[i] >= 0 && T[i].dims.empty() &&
          cudaMemsetAsync(b[i], 0, terminal_bytes(T[i]), plan->stream) != cudaSuccess) {
        err = "cudaMemsetAsync(reduction slot) failed";
        st = LF_ERR_CUDA;
      }
  };
  auto send_down = [&](const std::vector<void*>& b, int p) {
    const auto [a, e] = part_rows(p);
    cudaEventRecord(done[p], plan->stream);
    cudaStreamWaitEvent(plan->d2h, done[p], 0);
    for (size_t i = 0; i < T.size() && st == LF_OK; ++i) {
      if (!T[i].is_goal || !chunked(T[i])) continue;
      const long below = lo0 - T[i].base[0];
      const int64_t rb = row_bytes(T[i]);
      st = copy(static_cast<char*>(terms[i]) + (a + below) * rb, static_cast<const char*>(b[i]) + (a + below) * rb,
                (e - a) * rb, cudaMemcpyDeviceToHost, plan->d2h);
    }
  };
  // a multi-step run of a chain whose outer dimension does not wrap runs as a
  // wavefront over (step, part): part p of step s needs step s-1's parts p-1..p+1
  // (its input rows and halo) and overwrites the buffer step s-1 read its own
  // parts p-1..p+1 from (ping-pong), so in stream order tau = p + 2s every
  // dependence comes first.  Then every step trails the input rows up and the
  // last one sends each part down as it finishes: PCIe in both directions
  // overlaps the whole run, not only its first and last step.
  if (wavefront) {
    std::vector<std::vector<void*>> B(steps);
    for (int s = 0; s < steps; ++s) {
      B[s] = step_bufs(s);
      advance(B[s]);
    }
    std::vector<long> copied(T.size(), 0);
    for (int tau = 0; tau <= parts - 1 + 2 * (steps - 1) && st == LF_OK; ++tau)
      for (int s = 0; s < steps && st == LF_OK; ++s) {
        const int p = tau - 2 * s;
        if (p < 0 || p >= parts) continue;
        const auto [a, e] = part_rows(p);
        if (s == 0) {  // this part's input rows (and the halo above them)
          for (size_t i = 0; i < T.size() && st == LF_OK; ++i) {
            if (T[i].is_goal || !chunked(T[i])) continue;
            const long e0 = T[i].extent[0], below = lo0 - T[i].base[0], above = e0 - n0 - below;
            const long need = p == parts - 1 ? e0 : std::min(e0, e + below + above);
            if (need > copied[i]) {
              const int64_t rb = row_bytes(T[i]);
              st = copy(static_cast<char*>(dterms[i]) + copied[i] * rb,
                        static_cast<const char*>(terms[i]) + copied[i] * rb, (need - copied[i]) * rb,
                        cudaMemcpyHostToDevice, plan->h2d);
              copied[i] = need;
            }
          }
          if (st != LF_OK) break;
          cudaEventRecord(up[p], plan->h2d);
          cudaStreamWaitEvent(plan->stream, up[p], 0);
        }
        if (!inplace) {
          if ((st = run_part(B[s], a, e, false)) != LF_OK) break;
          if (s == steps - 1) send_down(B[s], p);
          continue;
        }
        if ((st = run_part(B[s], a, e, false, s, p, 0)) != LF_OK) break;
        if (p > 0) {  // part p-1's last rows: this launch was their last reader
          const auto [pa, pe] = part_rows(p - 1);
          if ((st = run_part(B[s], pa, pe, false, s, p - 1, 1)) != LF_OK) break;
          if (s == steps - 1) send_down(B[s], p - 1);
        }
        if (s == steps - 1 && p == parts - 1) send_down(B[s], p);
      }
  }
  // ---- first step: parts as their rows arrive
  if (!wavefront) {
    std::vector<void*> b = step_bufs(0);
    std::vector<long> copied(T.size(), 0);  // storage rows already sent, per axiom
    zero_reductions(b);
    for (int p = 0; p < parts && st == LF_OK; ++p) {
      const auto [a, e] = part_rows(p);
      // rows of every chunked axiom up to this part's last row plus the ghost/halo rows above it
      for (size_t i = 0; i < T.size() && st == LF_OK; ++i) {
        if (T[i].is_goal || !chunked(T[i])) continue;
        const long e0 = T[i].extent[0], below = lo0 - T[i].base[0], above = e0 - n0 - below;
        const long need = p == parts - 1 ? e0 : std::min(e0, e + below + above);
        if (need > copied[i]) {
          const int64_t rb = row_bytes(T[i]);
          st = copy(static_cast<char*>(dterms[i]) + copied[i] * rb, static_cast<const char*>(terms[i]) + copied[i] * rb,
                    (need - copied[i]) * rb, cudaMemcpyHostToDevice, plan->h2d);
          copied[i] = need;
        }
      }
      if (st != LF_OK) break;
      cudaEventRecord(up[p], plan->h2d);
      cudaStreamWaitEvent(plan->stream, up[p], 0);
      if ((st = run_part(b, a, e, false)) != LF_OK) break;
      if (steps == 1) send_down(b, p);
    }
    advance(b);
  }
  // ---- the steps in between: whole-domain launches
  for (int s = 1; s < steps - 1 && st == LF_OK && !wavefront; ++s) {
    std::vector<void*> b = step_bufs(s);
    zero_reductions(b);
    if (st == LF_OK) st = run_part(b, 0, n0, true, s);
    advance(b);
  }
  // ---- last step: parts, each sent down as soon as it is done
  if (steps > 1 && st == LF_OK && !wavefront) {
    std::vector<void*> b = step_bufs(steps - 1);
    zero_reductions(b);
    for (int p = 0; p < parts && st == LF_OK; ++p) {
      const auto [a, e] = part_rows(p);
      if ((st = run_part(b, a, e, false, steps - 1)) != LF_OK) break;
      send_down(b, p);
    }
  }
  if (mr && st == LF_OK && plan->exec->finalize) {  // the last raw maximum becomes the goal's value
    lfx::ExecArgs ea;
    ea.plan = &plan->plan;
    ea.terms = const_cast<void* const*>(dterms.data());
    ea.stream = plan->stream;
    st = plan->exec->finalize(ea, err);
    cudaEventRecord(done[parts - 1], plan->stream);  // the scalar goals go down after it
  }
  // once every part is done: ghost rows of the goals, and goals without an outer dimension
  if (st == LF_OK) {
    cudaStreamWaitEvent(plan->d2h, done[parts - 1], 0);
    for (size_t i = 0; i < T.size() && st == LF_OK; ++i) {
      if (!T[i].is_goal) continue;
      if (!chunked(T[i])) {
        st = copy(terms[i], dterms[i], terminal_bytes(T[i]), cudaMemcpyDeviceToHost, plan->d2h);
        continue;
      }
      const long e0 = T[i].extent[0], below = lo0 - T[i].base[0];
      const int64_t rb = row_bytes(T[i]);
      st = copy(terms[i], dterms[i], below * rb, cudaMemcpyDeviceToHost, plan->d2h);
      if (st == LF_OK)
        st = copy(static_cast<char*>(terms[i]) + (n0 + below) * rb, static_cast<const char*>(dterms[i]) + (n0 + below) * rb,
                  (e0 - n0 - below) * rb, cudaMemcpyDeviceToHost, plan->d2h);
    }
  }
  cudaError_t e1 = cudaStreamSynchronize(plan->h2d);
  cudaError_t e2 = cudaStreamSynchronize(plan->stream);
  cudaError_t e3 = cudaStreamSynchronize(plan->d2h);
  for (int p = 0; p < parts; ++p) {
    cudaEventDestroy(up[p]);
    cudaEventDestroy(done[p]);
  }
  if (st != LF_OK) return st;
  for (cudaError_t e : {e1, e2, e3})
    if (e != cudaSuccess) return lfx::cuda_status(e, "cudaStreamSynchronize(pipelined)", err);
  return LF_OK;
}

int lf_run_host(const lf_plan* cplan, void* const* terms, int nterm, int steps) {
  try {
    g_err.clear();
    int st = check_run_args(cplan, terms, nterm, steps);
    if (st != LF_OK) return st;
    lf_plan* plan = const_cast<lf_plan*>(cplan);
    std::lock_guard<std::mutex> lk(plan->mu);
    std::string err;
    const auto& T = plan->plan.terminals;
    if (!plan->stream) {
      cudaError_t e = cudaStreamCreateWithFlags(&plan->stream, cudaStreamNonBlocking);
      if (e != cudaSuccess) return fail(lfx::cuda_status(e, "cudaStreamCreate", err), err);
    }
    // a host buffer passed as an aliased axiom and goal stays one device buffer
    // when the executor can run the pair in place (half the device footprint)
    std::vector<int> share(T.size(), -1);
    if (plan->jit)
      for (const auto& q : plan->jit->program().inplace)
        if (terms[q.ai] && terms[q.ai] == terms[q.gi]) share[q.gi] = q.ai;
    if (plan->exec && shares_buffer(plan, terms))
      if ((st = exec_inplace_pairs(plan, terms, share, err)) != LF_OK) return fail(st, err);
    bool inplace = false;
    for (int s2 : share) inplace |= s2 >= 0;
    if (plan->dev.size() != T.size()) plan->dev.assign(T.size(), nullptr);
    for (size_t i = 0; i < T.size(); ++i) {
      if (share[i] >= 0 || plan->dev[i]) continue;
      cudaError_t e = cudaMalloc(&plan->dev[i], terminal_bytes(T[i]));
      if (e != cudaSuccess) return fail(lfx::cuda_status(e, "cudaMalloc(terminal)", err), err);
    }
    std::vector<void*> dterms(plan->dev);
    for (size_t i = 0; i < T.size(); ++i)
      if (share[i] >= 0) dterms[i] = plan->dev[share[i]];
    std::vector<void*> scratch;
    if (steps > 1 && !inplace) {
      if ((st = ensure_scratch(plan, err)) != LF_OK) return fail(st, err);
      scratch = scratch_list(plan);
    }
    // large grids: the copies overlap the first and the last step's compute
    {
      const long n0 = plan->plan.rs.ranges[0].trips();
      const bool nests = plan->jit && !plan->jit->program().nest_kernels.empty();
      int parts = static_cast<int>(std::min<long>(32, n0 / 512));  // 32: measured best for the 16384^2 box pass
      if (const char* e = lfx::option("LF_HOST_PARTS")) parts = std::atoi(e);
      const bool reduces = plan->exec && plan->exec->max_reduce;
      const bool inplace_parts = inplace && plan->exec && plan->exec->inplace_parts;
      if ((!inplace || inplace_parts) && !nests && !(reduces && inplace) && parts >= 2) {
        st = run_host_pipelined(plan, terms, dterms, parts, steps, err, inplace);
        if (st != kNotPipelined) {
          if (st != LF_OK) return fail(st, err);
          return LF_OK;
        }
      }
    }
    for (size_t i = 0; i < T.size(); ++i) {
      if (T[i].is_goal) continue;
      cudaError_t e = cudaMemcpyAsync(plan->dev[i], terms[i], terminal_bytes(T[i]), cudaMemcpyHostToDevice,
                                      plan->stream);
      if (e != cudaSuccess) return fail(lfx::cuda_status(e, "cudaMemcpyAsync(H2D)", err), err);
    }
    lfx::ExecArgs a;
    a.plan = &plan->plan;
    a.terms = dterms.data();
    a.steps = steps;
    a.stream = plan->stream;
    a.scratch = scratch.data();
    a.inplace = inplace && plan->exec;
    a.mem = &plan->exec_mem;
    st = plan->exec ? plan->exec->run(a, err) : plan->jit->run(a, err);
    if (st != LF_OK) return fail(st, err);
    for (size_t i = 0; i < T.size(); ++i) {
      if (!T[i].is_goal) continue;
      cudaError_t e = cudaMemcpyAsync(terms[i], dterms[i], terminal_bytes(T[i]), cudaMemcpyDeviceToHost,
                                      plan->stream);
      if (e != cudaSuccess) return fail(lfx::cuda_status(e, "cudaMemcpyAsync(D2H)", err), err);
    }
    cudaError_t e = cudaStreamSynchronize(plan->stream);
    if (e != cudaSuccess) return fail(lfx::cuda_status(e, "cudaStreamSynchronize", err), err);
    return LF_OK;
  } catch (const std::exception& e) {
    return fail(LF_ERR_INTERNAL, std::string("internal error: ") + e.what());
  }
}

int lf_run_slab(const lf_plan* cplan, void* const* terms, int nterm, const lf_slab* slab, void* cuda_stream) {
  try {
    g_err.clear();
    int st = check_run_args(cplan, terms, nterm, 1);
    if (st != LF_OK) return st;
    if (!slab || slab->lo < 0 || slab->hi <= slab->lo || slab->hi > slab->global)
      return fail(LF_ERR_SPEC, "invalid slab");
    if (slab->part_lo < 0 || slab->part_hi < slab->part_lo || slab->part_hi > slab->hi - slab->lo)
      return fail(LF_ERR_SPEC, "invalid slab part");
    if (slab->part_hi == slab->part_lo && slab->part_lo != 0) return LF_OK;  // empty part
    if (shares_buffer(cplan, terms))
      return fail(LF_ERR_UNSUPPORTED, "slab runs need distinct axiom and goal buffers (in-place runs cover the whole domain)");
    if (cplan->exec && cplan->exec->max_reduce)
      return fail(LF_ERR_UNSUPPORTED, "this chain reduces over the whole grid every step (" +
                                          std::string(cplan->exec->name) +
                                          "): run its slabs through lf_run_slabs / lf_run_slabs_local");
    // the generic executor's lazily created state (module, bands) is per plan
    std::lock_guard<std::mutex> lk(const_cast<lf_plan*>(cplan)->mu);
    lfx::ExecArgs a;
    a.plan = &cplan->plan;
    a.terms = terms;
    a.steps = 1;
    a.stream = static_cast<cudaStream_t>(cuda_stream);
    a.slab = slab;
    std::string err;
    st = cplan->exec ? cplan->exec->run(a, err) : cplan->jit->run(a, err);
    if (st != LF_OK) return fail(st, err);
    return LF_OK;
  } catch (const std::exception& e) {
    return fail(LF_ERR_INTERNAL, std::string("internal error: ") + e.what());
  }
}

// ---- native multi-GPU: slabs of the outer dimension, NCCL halo exchange ----

int lf_nccl_unique_id(char id[128]) {
  g_err.clear();
  const NcclApi& n = nccl();
  if (!n.error.empty()) return fail(LF_ERR_UNSUPPORTED, n.error);
  ncclUniqueId u;
  std::string err;
  int st = nccl_status(n.unique_id(&u), "ncclGetUniqueId", err);
  if (st != LF_OK) return fail(st, err);
  static_assert(sizeof(u.internal) == 128, "NCCL unique id size");
  std::memcpy(id, u.internal, 128);
  return LF_OK;
}

int lf_nccl_comm_init_rank(void** comm, int world, const char id[128], int rank) {
  g_err.clear();
  const NcclApi& n = nccl();
  if (!n.error.empty()) return fail(LF_ERR_UNSUPPORTED, n.error);
  if (!comm || world < 1 || rank < 0 || rank >= world) return fail(LF_ERR_SPEC, "invalid communicator arguments");
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  ncclComm_t c = nullptr;
  std::string err;
  int st = nccl_status(n.init_rank(&c, world, u, rank), "ncclCommInitRank", err);
  if (st != LF_OK) return fail(st, err);
  *comm = c;
  return LF_OK;
}

int lf_nccl_comm_init_single(void** comm) {
  g_err.clear();
  const NcclApi& n = nccl();
  if (!n.error.empty()) return fail(LF_ERR_UNSUPPORTED, n.error);
  int dev = 0;
  cudaGetDevice(&dev);
  ncclComm_t c = nullptr;
  std::string err;
  int st = nccl_status(n.init_all(&c, 1, &dev), "ncclCommInitAll", err);
  if (st != LF_OK) return fail(st, err);
  *comm = c;
  return LF_OK;
}

int lf_nccl_comm_destroy(void* comm) {
  g_err.clear();
  const NcclApi& n = nccl();
  if (!n.error.empty()) return fail(LF_ERR_UNSUPPORTED, n.error);
  std::string err;
  int st = nccl_status(n.destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy", err);
  return st == LF_OK ? LF_OK : fail(st, err);
}

int lf_run_slabs(const lf_plan* cplan, void* comm, int rank, int world, void* const* terms, int nterm, int steps,
                 void* cuda_stream) {
  try {
    g_err.clear();
    int st = check_run_args(cplan, terms, nterm, steps);
    if (st != LF_OK) return st;
    const NcclApi& n = nccl();
    if (!n.error.empty()) return fail(LF_ERR_UNSUPPORTED, n.error);
    if (!comm || world < 1 || rank < 0 || rank >= world) return fail(LF_ERR_SPEC, "invalid communicator arguments");
    lf_plan* plan = const_cast<lf_plan*>(cplan);
    std::lock_guard<std::mutex> lk(plan->mu);
    std::string err;
    bool inplace = false;
    if ((st = slab_inplace(plan, terms, inplace, err)) != LF_OK) return fail(st, err);
    SlabGeom g = slab_geom(plan->plan);
    g.world = world;
    if ((st = slab_check(plan, g, world, err)) != LF_OK) return fail(st, err);
    cudaStream_t stream = static_cast<cudaStream_t>(cuda_stream);
    if (!plan->comm && (st = make_side_stream(&plan->comm, err)) != LF_OK) return fail(st, err);
    std::vector<RankState> R(1);
    R[0].rank = rank;
    R[0].lo = g.n0 * rank / world;
    R[0].hi = g.n0 * (rank + 1) / world;
    R[0].terms = terms;
    if (steps > 1) {
      std::vector<int64_t> need = scratch_need(g, R[0], inplace);
      if (plan->slab_scratch_bytes != need) {
        for (void* q : plan->slab_scratch)
          if (q) cudaFree(q);
        plan->slab_scratch.clear();
        plan->slab_scratch_bytes.clear();
        std::vector<void*> fresh;
        if ((st = alloc_list(need, fresh, err)) != LF_OK) return fail(st, err);
        plan->slab_scratch = fresh;
        plan->slab_scratch_bytes = need;
      }
      R[0].scratch = plan->slab_scratch;
    }
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    auto exchange = [&](std::vector<RankState>& rs, cudaStream_t side, std::string& e) {
      RankState& r = rs[0];
      const long rows = r.hi - r.lo;
      int s2 = nccl_status(n.group_start(), "ncclGroupStart", e);
      for (size_t i = 0; i < g.paired.size() && s2 == LF_OK; ++i) {
        if (g.paired[i] < 0) continue;
        const int64_t rb = g.rb[i];
        const long below = g.below[i], above = g.above[i];
        const int up = r.rank + 1 < world ? r.rank + 1 : (g.periodic[i] ? 0 : -1);
        const int down = r.rank > 0 ? r.rank - 1 : (g.periodic[i] ? world - 1 : -1);
        char* d = static_cast<char*>(r.bufs[i]);
        if (up >= 0 && below)  // my last `below` rows -> up's lower ghosts
          s2 = nccl_status(n.send(d + rows * rb, below * rb, ncclUint8, up, c, side), "ncclSend", e);
        if (s2 == LF_OK && down >= 0 && below)  // my lower ghosts <- down's last rows
          s2 = nccl_status(n.recv(d, below * rb, ncclUint8, down, c, side), "ncclRecv", e);
        if (s2 == LF_OK && down >= 0 && above)  // my first `above` rows -> down's upper ghosts
          s2 = nccl_status(n.send(d + below * rb, above * rb, ncclUint8, down, c, side), "ncclSend", e);
        if (s2 == LF_OK && up >= 0 && above)  // my upper ghosts <- up's first rows
          s2 = nccl_status(n.recv(d + (below + rows) * rb, above * rb, ncclUint8, up, c, side), "ncclRecv", e);
      }
      int s3 = nccl_status(n.group_end(), "ncclGroupEnd", e);
      return s2 != LF_OK ? s2 : s3;
    };
    // per-step MAX reductions (the adaptive CFL time step): one all-reduce of
    // the rank's raw maximum, in place, before the next step reads it
    auto combine = [&](void* slot, cudaStream_t on, std::string& e) {
      return nccl_status(n.all_reduce(slot, slot, 1, ncclFloat64, ncclMax, c, on), "ncclAllReduce", e);
    };
    st = run_slabs_core(plan, g, R, steps, stream, plan->comm, exchange, err, combine, inplace);
    if (st != LF_OK) return fail(st, err);
    return LF_OK;
  } catch (const std::exception& e) {
    return fail(LF_ERR_INTERNAL, std::string("internal error: ") + e.what());
  }
}

int lf_run_slabs_local(const lf_plan* cplan, int world, void* const* terms, int nterm, int steps, void* cuda_stream) {
  try {
    g_err.clear();
    if (!cplan) return fail(LF_ERR_SPEC, "null plan");
    if (world < 1 || !terms) return fail(LF_ERR_SPEC, "invalid rank count");
    for (int r = 0; r < world; ++r) {
      int st = check_run_args(cplan, terms + (size_t)r * nterm, nterm, steps);
      if (st != LF_OK) return st;
    }
    lf_plan* plan = const_cast<lf_plan*>(cplan);
    std::lock_guard<std::mutex> lk(plan->mu);
    std::string err;
    bool inplace = false;
    for (int r = 0; r < world; ++r) {  // every rank in place, or none
      bool ip = false;
      int st = slab_inplace(plan, terms + (size_t)r * nterm, ip, err);
      if (st != LF_OK) return fail(st, err);
      if (r > 0 && ip != inplace) return fail(LF_ERR_SPEC, "some ranks share axiom and goal buffers, some do not");
      inplace = ip;
    }
    SlabGeom g = slab_geom(plan->plan);
    g.world = world;
    int st = slab_check(plan, g, world, err);
    if (st != LF_OK) return fail(st, err);
    cudaStream_t stream = static_cast<cudaStream_t>(cuda_stream);
    if (!plan->comm && (st = make_side_stream(&plan->comm, err)) != LF_OK) return fail(st, err);
    std::vector<RankState> R(world);
    std::vector<void*> owned;
    for (int r = 0; r < world && st == LF_OK; ++r) {
      R[r].rank = r;
      R[r].lo = g.n0 * r / world;
      R[r].hi = g.n0 * (r + 1) / world;
      R[r].terms = terms + (size_t)r * nterm;
      if (steps > 1) {
        st = alloc_list(scratch_need(g, R[r], inplace), R[r].scratch, err);
        for (void* q : R[r].scratch) owned.push_back(q);
      }
    }
    // the exchange as device copies between the ranks' slabs (all on this GPU)
    auto exchange = [&](std::vector<RankState>& rs, cudaStream_t side, std::string& e) {
      for (int r = 0; r < world; ++r)
        for (size_t i = 0; i < g.paired.size(); ++i) {
          if (g.paired[i] < 0) continue;
          const int64_t rb = g.rb[i];
          const long below = g.below[i], above = g.above[i];
          const int up = r + 1 < world ? r + 1 : (g.periodic[i] ? 0 : -1);
          const int down = r > 0 ? r - 1 : (g.periodic[i] ? world - 1 : -1);
          char* d = static_cast<char*>(rs[r].bufs[i]);
          const long rows = rs[r].hi - rs[r].lo;
          cudaError_t ce = cudaSuccess;
          if (down >= 0 && below) {
            const long drows = rs[down].hi - rs[down].lo;
            ce = cudaMemcpyAsync(d, static_cast<char*>(rs[down].bufs[i]) + drows * rb, below * rb,
                                 cudaMemcpyDeviceToDevice, side);
          }
          if (ce == cudaSuccess && up >= 0 && above)
            ce = cudaMemcpyAsync(d + (below + rows) * rb, static_cast<char*>(rs[up].bufs[i]) + below * rb,
                                 above * rb, cudaMemcpyDeviceToDevice, side);
          if (ce != cudaSuccess) return lfx::cuda_status(ce, "cudaMemcpyAsync(halo)", e);
        }
      return LF_OK;
    };
    if (st == LF_OK) st = run_slabs_core(plan, g, R, steps, stream, plan->comm, exchange, err, nullptr, inplace);
    if (!owned.empty()) {
      cudaStreamSynchronize(stream);
      for (void* q : owned)
        if (q) cudaFree(q);
    }
    if (st != LF_OK) return fail(st, err);
    return LF_OK;
  } catch (const std::exception& e) {
    return fail(LF_ERR_INTERNAL, std::string("internal error: ") + e.what());
  }
}

}  // extern "C"

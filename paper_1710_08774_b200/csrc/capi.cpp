// extern "C" boundary of loomfuse-b200 (include/loomfuse_b200.h).
// Maps the reference's pipeline entry (parse_spec -> analysis, rulespec.cpp:550,
// storage.cpp:526) and its emitted per-goal-set function (R/SPEC.md:500) onto
// plan objects and fused sm_100a executors.  No exception crosses this file.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
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
  cudaStream_t stream = nullptr;
  cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams of the pipelined host path
  ~lf_plan() {
    for (void* p : dev)
      if (p) cudaFree(p);
    for (void* p : scratch)
      if (p) cudaFree(p);
    if (stream) cudaStreamDestroy(stream);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
  }
};

namespace {

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
    static const bool no_builtin = std::getenv("LF_NO_BUILTIN") && std::atoi(std::getenv("LF_NO_BUILTIN")) != 0;
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

int lf_run(const lf_plan* cplan, void* const* terms, int nterm, int steps, void* cuda_stream) {
  try {
    g_err.clear();
    int st = check_run_args(cplan, terms, nterm, steps);
    if (st != LF_OK) return st;
    lf_plan* plan = const_cast<lf_plan*>(cplan);
    std::lock_guard<std::mutex> lk(plan->mu);
    std::string err;
    const bool inplace = shares_buffer(plan, terms);
    if (inplace && plan->exec)
      return fail(LF_ERR_UNSUPPORTED, std::string(plan->exec->name) +
                                          " ping-pongs between distinct buffers; in-place runs (config.aliases) "
                                          "use the generic executor");
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
    st = plan->exec ? plan->exec->run(a, err) : plan->jit->run(a, err);
    if (st != LF_OK) return fail(st, err);
    return LF_OK;
  } catch (const std::exception& e) {
    return fail(LF_ERR_INTERNAL, std::string("internal error: ") + e.what());
  }
}

// Single-step host runs, pipelined: the outer dimension is cut into parts;
// part p's input rows go up on one copy stream, the part is computed on the
// plan's stream as soon as they (and the halo) have landed, and its finished
// output rows come down on a second copy stream -- both PCIe directions and
// the SMs busy at once instead of one after the other.  Every executor
// computes row parts (lf_slab part ranges); ghost rows of the goals are
// copied once all parts are done.
static int run_host_pipelined(lf_plan* plan, void* const* terms, const std::vector<void*>& dterms, int parts,
                              std::string& err) {
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
  auto copy = [&](void* dst, const void* src, int64_t bytes, cudaMemcpyKind kind, cudaStream_t st) {
    if (bytes <= 0) return LF_OK;
    return lfx::cuda_status(cudaMemcpyAsync(dst, src, bytes, kind, st), "cudaMemcpyAsync(pipelined)", err);
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
  std::vector<long> copied(T.size(), 0);  // storage rows already sent, per axiom
  for (int p = 0; p < parts && st == LF_OK; ++p) {
    const long a = n0 * p / parts, b = n0 * (p + 1) / parts;
    // rows of every chunked axiom up to this part's last row plus the ghost/halo rows above it
    for (size_t i = 0; i < T.size() && st == LF_OK; ++i) {
      if (T[i].is_goal || !chunked(T[i])) continue;
      const long e0 = T[i].extent[0], below = lo0 - T[i].base[0], above = e0 - n0 - below;
      const long need = p == parts - 1 ? e0 : std::min(e0, b + below + above);
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
    lf_slab slab{0, n0, n0, a, b};
    lfx::ExecArgs ea;
    ea.plan = &plan->plan;
    ea.terms = dterms.data();
    ea.steps = 1;
    ea.stream = plan->stream;
    ea.slab = &slab;
    ea.whole_domain_parts = true;
    st = plan->exec ? plan->exec->run(ea, err) : plan->jit->run(ea, err);
    if (st != LF_OK) break;
    cudaEventRecord(done[p], plan->stream);
    cudaStreamWaitEvent(plan->d2h, done[p], 0);
    // this part's interior output rows
    for (size_t i = 0; i < T.size() && st == LF_OK; ++i) {
      if (!T[i].is_goal || !chunked(T[i])) continue;
      const long below = lo0 - T[i].base[0];
      const int64_t rb = row_bytes(T[i]);
      st = copy(static_cast<char*>(terms[i]) + (a + below) * rb, static_cast<const char*>(dterms[i]) + (a + below) * rb,
                (b - a) * rb, cudaMemcpyDeviceToHost, plan->d2h);
    }
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
    // single steps of large grids: copies in both directions overlap the parts' compute
    {
      const long n0 = plan->plan.rs.ranges[0].trips();
      const bool nests = plan->jit && !plan->jit->program().nest_kernels.empty();
      int parts = static_cast<int>(std::min<long>(32, n0 / 512));  // 32: measured best for the 16384^2 box pass
      if (const char* e = std::getenv("LF_HOST_PARTS")) parts = std::atoi(e);
      if (steps == 1 && !inplace && !nests && parts >= 2) {
        st = run_host_pipelined(plan, terms, dterms, parts, err);
        if (st != LF_OK) return fail(st, err);
        return LF_OK;
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

}  // extern "C"

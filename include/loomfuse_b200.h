/*
 * loomfuse-b200 -- C ABI of the B200-native fused stencil-chain executor.
 *
 * Drop-in boundary for the reference's fused path.  In the reference the user
 * writes a rule file (`.lf`: kernels / globals / config, R/SPEC.md:88,
 * R/PAPER.md:358-375) and the code generator emits "one function per goal
 * set, taking terminal buffers as parameters" (R/SPEC.md:500), with the
 * prototype in `<name>.h` (R/SPEC.md:507) and buffers ordered axioms then
 * goals.  That emitted function is the hot path this library replaces:
 *
 *   reference (emitted, host)            loomfuse-b200
 *   ----------------------------------   ---------------------------------------
 *   parse_spec + analysis pipeline        lf_plan_create        (rulespec.cpp:550,
 *     (rulespec/inference/nests/fusion/                          inference.cpp:404,
 *      shifts/storage)                                           storage.cpp:526)
 *   buffer_extents / storage report       lf_plan_terminal, lf_plan_report
 *                                                               (storage.cpp:403-427,
 *                                                                R/SPEC.md:440)
 *   void <name>(axioms..., goals...)      lf_run_host  (host buffers, same order)
 *                                         lf_run       (device buffers + stream)
 *   outer-level parallelism (external,    lf_run_slab  (one row/plane slab of a
 *     R/PAPER.md:499)                                   domain split across GPUs)
 *   DiagList / internal_error /           int status codes below + lf_last_error()
 *     CLI exit codes (diag.hpp:37-70,     (thread-local message, `file:line:col`
 *     R/SPEC.md:596)                       prefixes as SourceLoc::str)
 *
 * No exceptions cross this boundary; every entry point returns a status.
 * Plans are immutable after creation and may be shared between threads;
 * execution is stream-ordered.
 */
#ifndef LOOMFUSE_B200_H
#define LOOMFUSE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (R/SPEC.md:596: 0 ok / 1 user error / 2 verify mismatch) */
#define LF_OK 0
#define LF_ERR_SPEC 1        /* rule-file or argument error (diagnostics in lf_last_error) */
#define LF_ERR_MISMATCH 2    /* reserved: verification mismatch */
#define LF_ERR_INTERNAL 3    /* contract violation inside the planner/executor */
#define LF_ERR_CUDA 4        /* CUDA runtime / driver failure */
#define LF_ERR_UNSUPPORTED 5 /* valid chain, but no fused sm_100a executor for it */

#define LF_MAX_DIMS 4

typedef struct lf_plan lf_plan;

/* One terminal buffer (axiom or goal) as the reference's storage analysis
 * sizes it: extent = trips + offset spread, base = logical coordinate of
 * index 0 (storage.cpp:403-427).  Dims are outermost first; buffers are dense
 * and row-major.  For iterated chains (config `iterate:`) the goal buffer
 * takes its paired axiom's layout so the two can ping-pong. */
typedef struct {
  char name[64];
  char type[32];      /* element type text from the declaration, e.g. "double" */
  int32_t is_goal;
  int32_t elem_bytes;
  int32_t ndim;
  int32_t loop_dim[LF_MAX_DIMS]; /* index into loop-order; -1 for none */
  int64_t extent[LF_MAX_DIMS];
  int64_t base[LF_MAX_DIMS];
  int64_t bytes;      /* elem_bytes * prod(extent) */
} lf_terminal;

/* A slab of the outermost loop dimension owned by one rank (lf_run_slab):
 * rows [lo, hi) of the global range [0, global).  Terminal buffers of a slab
 * are sized for that slab (the planner's extents with `hi-lo` trips along the
 * outermost dim).  Ghost rows on an internal face are filled by the caller's
 * halo exchange before each step; ghost rows on a global face are refilled by
 * the executor from the chain's boundary mode.  [part_lo, part_hi) (slab-local
 * rows; 0,0 = all) restricts one call to part of the slab, so a caller can
 * compute the face rows first, start their exchange, and overlap it with the
 * interior rows. */
typedef struct {
  int64_t lo;
  int64_t hi;
  int64_t global;
  int64_t part_lo;
  int64_t part_hi;
} lf_slab;

/* Parse, validate, infer and analyse a rule file.  `filename` is only used in
 * diagnostics.  On LF_ERR_SPEC the diagnostics are in lf_last_error(). */
int lf_plan_create(const char* spec_text, size_t len, const char* filename, lf_plan** out);

/* As lf_plan_create, plus CUDA C source defining the user kernels the rule
 * file names in `declaration:` (R/PAPER.md:58-62: value inputs, outputs by
 * pointer or reference), as `__device__` (or __host__ __device__) functions.
 * A chain that no built-in executor implements is lowered by the generic
 * executor and compiled for sm_100a together with this source and the shipped
 * user-kernel headers (the userkernels/ directory), so kernels need no `body:`.
 * kernel_source may be NULL. */
int lf_plan_create_ex(const char* spec_text, size_t len, const char* filename, const char* kernel_source,
                      size_t kernel_len, lf_plan** out);

/* Canonical text of a rule file (print_spec, rulespec.cpp:668-705): parsing
 * the output again yields a structurally equal rule set.  Same buffer
 * convention as lf_plan_report. */
int lf_spec_print(const char* spec_text, size_t len, const char* filename, char* buf, size_t cap,
                  size_t* needed);

/* Release a plan and the device scratch it owns. */
void lf_plan_destroy(lf_plan* plan);

/* Number of terminals (axioms in declaration order, then goals). */
int lf_plan_num_terminals(const lf_plan* plan);

/* Describe terminal `idx`. */
int lf_plan_terminal(const lf_plan* plan, int idx, lf_terminal* out);

/* Analysis report as JSON (groups + shifts, variables + storage schemes and
 * windows, terminals, nests/splits, footprint polynomial, chain signature).
 * Writes at most `cap` bytes including the NUL; returns the full length via
 * *needed when non-NULL. */
int lf_plan_report(const lf_plan* plan, char* buf, size_t cap, size_t* needed);

/* Name of the fused executor the plan dispatches to, or "" if none: a
 * hand-written sm_100a executor whose chain signature matches and whose size
 * constraints hold ("heat3d_fused_tma", "biharm2d_fused_tma",
 * "box2x_fused_tma", "hydro2d_fused_tma"), else the generic executor, which
 * lowers the chain to CUDA and compiles it for sm_100a with NVRTC at plan
 * creation: "jit_window_fused" (2D/3D march with rolling windows),
 * "jit_tiled_fused" (1D), "jit_nests_fused" (multi-nest plans: reductions and
 * broadcast splits). */
const char* lf_plan_executor(const lf_plan* plan);

/* CUDA source the generic executor generated for this plan ("" otherwise). */
const char* lf_plan_source(const lf_plan* plan);

/* Run the chain `steps` times on DEVICE buffers (axioms then goals, sized per
 * lf_plan_terminal), stream-ordered on `cuda_stream` (a cudaStream_t, NULL =
 * legacy default stream).  steps == 1 is exactly the reference's emitted
 * function.  steps > 1 requires `iterate:` pairs: the goal of step s is the
 * axiom of step s+1, ghost cells are refilled from `boundary:` after every
 * step, and the final state is left in the goal buffers.  Intermediate states
 * ping-pong between the goal buffer and a plan-owned scratch buffer, so the
 * axiom buffers are never written -- except in place: passing ONE buffer for
 * an axiom and its goal that `config: aliases:` declares runs the chain in
 * place, on the generic executor or on the hand-written Hydro2D (all four
 * state pairs together) and biharmonic executors; LF_ERR_UNSUPPORTED
 * otherwise.  One multi-step run per plan at a time (the ping-pong scratch
 * and the in-place bands are plan-owned); create one plan per concurrent
 * stream. */
int lf_run(const lf_plan* plan, void* const* terminals, int nterm, int steps, void* cuda_stream);

/* Same on HOST buffers: copies axioms host->device, runs, copies goals
 * device->host, synchronises.  This is the drop-in for the emitted host
 * function <name>(terminals...) of R/SPEC.md:500.  Device buffers are owned
 * and cached by the plan.  Pinned host memory gives full copy bandwidth;
 * large grids are pipelined over row parts (host->device copies, compute and
 * device->host copies overlap): the first and the last step, or -- multi-step
 * runs of chains whose outer dimension does not wrap -- every step, as a
 * wavefront over (step, part).  A host array passed as an aliased axiom AND
 * its goal (config.aliases) keeps ONE device buffer and runs in place, where
 * the executor can (as lf_run). */
int lf_run_host(const lf_plan* plan, void* const* terminals, int nterm, int steps);

/* One step on a slab of the outermost loop dimension (multi-GPU row/plane
 * slabs).  Buffers are device buffers sized for the slab. */
int lf_run_slab(const lf_plan* plan, void* const* terminals, int nterm, const lf_slab* slab,
                void* cuda_stream);

/* Native multi-GPU run: `steps` steps of rank `rank`'s slab
 * of a `world`-rank decomposition of the outermost loop dimension -- rows
 * [n*rank/world, n*(rank+1)/world) -- on device buffers sized for that slab
 * (the planner's extents with the slab's row count along dim 0).  `nccl_comm`
 * is an ncclComm_t of `world` ranks, one per GPU.  Every step computes the
 * output rows the neighbours need first (the two faces side by side on two
 * library-owned high-priority streams), exchanges them by NCCL send/recv on
 * one of them (ring-wrapped when the boundary of dim 0 is periodic) while the
 * interior rows are computed on `cuda_stream`, and orders the next step after
 * both.  Iterated state ping-pongs through
 * slab-sized plan scratch; the final state is left in the goal buffers.  A
 * rank that passes its slab-sized goals on its aliased axioms' buffers runs
 * its slab in place instead (built-in Hydro2D executors: one launch per step,
 * then the exchange; no slab scratch; every rank must do the same).  NCCL
 * is loaded at run time (libnccl.so.2; the process's copy when one is
 * loaded).  Replaces the reference's external outer-level parallelism
 * (R/PAPER.md:499). */
int lf_run_slabs(const lf_plan* plan, void* nccl_comm, int rank, int world, void* const* terminals, int nterm,
                 int steps, void* cuda_stream);

/* The same decomposition with all `world` ranks on the current GPU, the
 * exchange done by device copies: `terminals` holds world * nterm device
 * pointers, rank-major.  Same geometry and schedule as lf_run_slabs, for
 * testing the slab path on one GPU. */
int lf_run_slabs_local(const lf_plan* plan, int world, void* const* terminals, int nterm, int steps,
                       void* cuda_stream);

/* NCCL communicator helpers for lf_run_slabs (the handles are ncclComm_t):
 * a 128-byte unique id made on one rank and shared out of band, one rank's
 * communicator from it, a one-rank communicator on the current device, and
 * destruction. */
int lf_nccl_unique_id(char id[128]);
int lf_nccl_comm_init_rank(void** nccl_comm, int world, const char id[128], int rank);
int lf_nccl_comm_init_single(void** nccl_comm);
int lf_nccl_comm_destroy(void* nccl_comm);

/* Bench accounting.  lf_plan_launches_per_step: kernel launches of one
 * single-step pass; lf_plan_compulsory_bytes_per_cell: algorithmic HBM bytes
 * per cell of one pass over the grid (terminals read once + written once);
 * lf_plan_grid_passes: passes lf_run(plan, ..., steps) makes over a whole
 * domain (fewer than `steps` where the executor fuses time steps, e.g. the
 * 3D heat chain's two-step passes); lf_plan_launches: kernel launches it
 * issues (out of place; an in-place run adds one per step, the band commit
 * or capture kernel). */
int lf_plan_launches_per_step(const lf_plan* plan);
double lf_plan_compulsory_bytes_per_cell(const lf_plan* plan);
int lf_plan_grid_passes(const lf_plan* plan, int steps);
int lf_plan_launches(const lf_plan* plan, int steps);

/* Tuning / A-B switches (names LF_*): set `value` as the
 * in-process value of switch `name`, overriding the environment variable of
 * that name; value == NULL drops the override.  A switch takes effect where it
 * is read -- plan creation (code generation, executor choice) or the next run.
 * No switch changes results (every variant is bit-exact).  Returns
 * LF_ERR_SPEC for a name outside the LF_ namespace.  (No reference
 * counterpart: the reference has no executor to tune.) */
int lf_set_option(const char* name, const char* value);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* lf_last_error(void);

/* Library version string. */
const char* lf_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LOOMFUSE_B200_H */

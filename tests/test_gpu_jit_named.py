"""Chains that name user-kernel functions (no `body:`) on the generic
executor: the shipped kernels (userkernels/*.h) at sizes outside the
hand-written executors' constraints, and caller-supplied kernel source
(lf_plan_create_ex) -- bit-exact against the oracles."""
import numpy as np
import pytest

import oracle
from oracle import generic
import paper_1710_08774_b200 as lf
from paper_1710_08774_b200 import inputs

pytestmark = pytest.mark.gpu
SPECS = lf.PKG_DIR.parent / "tests" / "specs"


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def run(plan, axioms, steps):
    import torch
    ax = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in axioms]
    dt = {8: torch.float64, 4: torch.float32}
    goals = [torch.full(t.extent, float("nan"), dtype=dt[t.elem_bytes], device="cuda") for t in plan.goals]
    plan.run(ax + goals, steps=steps)
    torch.cuda.synchronize()
    return [g.cpu().numpy() for g in goals]


def inner(a, h):
    return a[tuple(slice(h, -h) for _ in range(a.ndim))]


@pytest.mark.parametrize("shape,steps", [((10, 20, 50), 3), ((5, 33, 70), 2)])
def test_heat3d_outside_kernel_constraints(shape, steps):
    plan = lf.Plan.with_ranges("heat3d", shape)
    assert plan.executor == "jit_window_fused"
    u = inputs.heat3d_input(*shape, seed=4, sigma=3.0)
    (got,) = run(plan, [u], steps)
    assert np.array_equal(bits(inner(got, 1)), bits(inner(oracle.heat3d(u, steps), 1)))


@pytest.mark.parametrize("shape,steps", [((30, 100), 3), ((57, 203), 2)])
def test_biharm_outside_kernel_constraints(shape, steps):
    plan = lf.Plan.with_ranges("biharmonic2d", shape)
    assert plan.executor == "jit_window_fused"
    u = inputs.biharm_input(*shape, seed=5)
    (got,) = run(plan, [u], steps)
    assert np.array_equal(bits(got), bits(oracle.biharm(u, steps)))


def test_box_outside_kernel_constraints():
    plan = lf.Plan.with_ranges("box2x", (30, 100))
    assert plan.executor == "jit_window_fused"
    img = inputs.box_input(30, 100, seed=6)
    (got,) = run(plan, [img], 1)
    assert np.array_equal(bits(got), bits(oracle.box(img)))


@pytest.mark.parametrize("shape,steps", [((30, 101), 2), ((17, 67), 1)])
def test_hydro_outside_kernel_constraints(shape, steps):
    plan = lf.Plan.with_ranges("hydro2d", shape)
    assert plan.executor == "jit_window_fused"
    st, dtdx = inputs.hydro_input(*shape, seed=9)
    got = run(plan, st + [np.array([dtdx])], steps)
    ref = oracle.hydro(st, dtdx, steps)
    for v in range(4):
        assert np.array_equal(bits(inner(got[v], 2)), bits(inner(ref[v], 2))), v


KERNELS = r"""
__device__ void mylap(double w, double e, double s, double n, double c, double* o) {
  *o = w + e + s + n - 4.0 * c;
}
__device__ void myupd(double c, double l2, double& o) { o = c - 0.01 * l2; }
"""


def test_caller_kernel_source():
    """The body-form biharmonic spec with its bodies removed and myupd's output
    made a reference: the functions come from the caller's CUDA source."""
    text = (SPECS / "biharm_body.lf").read_text()
    lines = []
    skip = False
    for ln in text.splitlines():
        if ln.strip().startswith("body:"):
            skip = True
            continue
        if skip and ln.startswith("      "):
            continue
        skip = False
        lines.append(ln)
    named = "\n".join(lines).replace("double l2, double* o)", "double l2, double& o)")
    with pytest.raises(lf.LoomfuseError):
        lf.Plan(named, "named.lf").run([0, 0])  # no functions without the source
    plan = lf.Plan(named, "named.lf", kernel_source=KERNELS)
    assert plan.executor == "jit_window_fused"
    assert "__device__ void mylap" in plan.source
    u = inputs.biharm_input(40, 72, seed=10)
    (got,) = run(plan, [u], 2)
    ref = generic.run_naive(SPECS / "biharm_body.lf", {"g_u": u}, steps=2)["g_unew"]
    assert np.array_equal(bits(got), bits(ref))


# the user's own kernels of the paper's normalization example (R/PAPER.md:66),
# passed as CUDA source with the plan (the rule file only names them)
NORMALIZATION_KERNELS = """
__device__ void flux(double a, double b, double* f) { *f = (b - a) * (b - a); }
__device__ void accinit(double z, double* a) { *a = z; }
__device__ void accum(double c, double f, double* o) { *o = c + f; }
__device__ void root(double t, double* r) { *r = sqrt(t); }
__device__ void normalize(double f, double r, double* o) { *o = f / r; }
"""


@pytest.mark.parametrize("shape", [(64, 128), (37, 300), (5, 1000)])
def test_paper_normalization_as_written(shape, tmp_path):
    """tests/specs/normalization.lf exactly as the paper writes it -- five
    declaration-only kernels, a reduction over i, its root and a broadcast
    divide: 2 nests, 1 split (R/SPEC.md:633) -- runs on the generic
    executor's multi-nest path with the caller's kernel source, bit-exact
    against run_naive over the reference's DAG of the same rules (their
    `body:` twins in normalization_body.lf)."""
    named = lf.set_ranges((SPECS / "normalization.lf").read_text(), shape)
    plan = lf.Plan(named, "normalization.lf", kernel_source=NORMALIZATION_KERNELS)
    r = plan.report()
    assert (r["nests"], r["splits"]) == (2, 1)
    assert plan.executor == "jit_nests_fused"
    rng = np.random.default_rng(shape[1])
    q = rng.random((shape[0], shape[1] + 1))
    z = np.zeros(shape[0])
    got = run(plan, [q, z], 1)[0]
    body = tmp_path / "normalization_body.lf"
    body.write_text(lf.set_ranges((SPECS / "normalization_body.lf").read_text(), shape))
    ref = generic.run_naive(body, {"g_q": q, "g_zero": z}, steps=1)["g_out"]
    assert np.array_equal(bits(got), bits(ref))

"""Degenerate grids (one or a few cells per dimension) through whichever
executor the dispatcher picks -- bit-exact against the C oracles."""
import numpy as np
import pytest

import oracle
import paper_1710_08774_b200 as lf
from paper_1710_08774_b200 import inputs

pytestmark = pytest.mark.gpu


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


@pytest.mark.parametrize("shape", [(1, 1), (1, 7), (5, 1), (2, 3)])
def test_biharm_tiny(shape):
    plan = lf.Plan.with_ranges("biharmonic2d", shape)
    assert plan.executor
    u = inputs.biharm_input(*shape, seed=1)
    (got,) = run(plan, [u], 3)
    assert np.array_equal(bits(got), bits(oracle.biharm(u, 3)))


@pytest.mark.parametrize("shape", [(1, 1, 1), (2, 3, 5), (1, 16, 64)])
def test_heat3d_tiny(shape):
    plan = lf.Plan.with_ranges("heat3d", shape)
    assert plan.executor
    u = inputs.heat3d_input(*shape, seed=2, sigma=1.0)
    (got,) = run(plan, [u], 3)
    assert np.array_equal(bits(inner(got, 1)), bits(inner(oracle.heat3d(u, 3), 1)))


@pytest.mark.parametrize("shape", [(1, 1), (3, 7), (2, 128)])
def test_box_tiny(shape):
    plan = lf.Plan.with_ranges("box2x", shape)
    assert plan.executor
    img = inputs.box_input(*shape, seed=3)
    (got,) = run(plan, [img], 1)
    assert np.array_equal(bits(got), bits(oracle.box(img)))


@pytest.mark.parametrize("shape", [(2, 3), (4, 5), (1, 9)])
def test_hydro_tiny(shape):
    plan = lf.Plan.with_ranges("hydro2d", shape)
    assert plan.executor
    st, dtdx = inputs.hydro_input(*shape, seed=4)
    got = run(plan, st + [np.array([dtdx])], 2)
    ref = oracle.hydro(st, dtdx, 2)
    for v in range(4):
        assert np.array_equal(bits(inner(got[v], 2)), bits(inner(ref[v], 2))), v


SPECS = lf.PKG_DIR.parent / "tests" / "specs"


@pytest.mark.parametrize("name,shape", [("laplace3_body", (1,)), ("laplace3_body", (2,)), ("laplace3_body", (1025,)),
                                        ("biharm_body", (1, 1)), ("heat3d_body", (1, 2, 3)),
                                        ("normalization_body", (1, 1)), ("normalization_body", (3, 33)),
                                        ("colsum_body", (1, 5)), ("multi_body", (1, 3))])
def test_generic_tiny(name, shape):
    from oracle import generic
    text = lf.set_ranges((SPECS / f"{name}.lf").read_text(), shape)
    path = SPECS / f"_tiny_{name}_{'x'.join(map(str, shape))}.lf"
    path.write_text(text)
    try:
        plan = lf.Plan(text, path.name)
        assert plan.executor.startswith("jit_")
        rng = np.random.default_rng(5)
        ax = {}
        for t in plan.axioms:
            ax[t.name] = rng.random(t.extent) if t.extent else np.array([0.5])
        got = run(plan, [ax[t.name] for t in plan.axioms], 1)
        ref = generic.run_naive(path, ax, steps=1)
    finally:
        path.unlink()
    for g, t in zip(got, plan.goals):
        assert np.array_equal(bits(g), bits(ref[t.name])), t.name

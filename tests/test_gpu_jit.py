"""Generic NVRTC-compiled executor (jit_tiled_fused) vs the generic run_naive
over the reference's own inference DAG, bit-exact."""
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


def run_device(plan, axioms, steps):
    import torch
    ax = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in axioms]
    dt = {8: torch.float64, 4: torch.float32}
    goals = [torch.full(t.extent, float("nan"), dtype=dt[t.elem_bytes], device="cuda") for t in plan.goals]
    plan.run(ax + goals, steps=steps)
    torch.cuda.synchronize()
    return [g.cpu().numpy() for g in goals]


CASES = {
    "biharm_body": lambda: {"g_u": inputs.biharm_input(40, 72, seed=5)},
    "heat3d_body": lambda: {"g_u": inputs.heat3d_input(9, 12, 40, seed=6, sigma=3.0)},
    "box_body": lambda: {"g_img": inputs.box_input(33, 70, seed=7)},
    "multi_body": lambda: {"g_x": np.random.default_rng(1).random((21, 52)), "g_scale": np.array([0.75])},
    "laplace3_body": lambda: {"g_x": np.random.default_rng(2).random(1002)},
    # multi-nest plans: reductions (inner and outer dim) and broadcast splits
    "normalization_body": lambda: {"g_q": np.random.default_rng(3).random((37, 151)),
                                   "g_zero": np.random.default_rng(4).random(37) * 0.1},
    "colsum_body": lambda: {"g_u": np.random.default_rng(5).random((47, 72)), "g_z": np.zeros(70),
                            "g_k": np.array([0.3])},
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("steps", [1, 3])
def test_jit_matches_generic_oracle(name, steps):
    plan = lf.Plan.from_file(SPECS / f"{name}.lf")
    assert plan.executor.startswith("jit_")
    if steps > 1 and name not in ("biharm_body", "heat3d_body"):
        pytest.skip("chain has no iterate pairs")
    ax = CASES[name]()
    got = run_device(plan, [ax[t.name] for t in plan.axioms], steps)
    ref = generic.run_naive(SPECS / f"{name}.lf", ax, steps=steps)
    for g, t in zip(got, plan.goals):
        assert np.array_equal(bits(g), bits(ref[t.name])), t.name


def test_jit_host_path_and_large_grid():
    spec = lf.set_ranges((SPECS / "biharm_body.lf").read_text(), (300, 1000))
    plan = lf.Plan(spec, "big.lf")
    u = inputs.biharm_input(300, 1000, seed=9)
    out = np.zeros_like(u)
    plan.run_host([u, out], steps=2)
    assert np.array_equal(bits(out), bits(oracle.biharm(u, 2)))


def test_jit_slab_parts_compose():
    import torch
    plan = lf.Plan.from_file(SPECS / "heat3d_body.lf")
    u = torch.from_numpy(inputs.heat3d_input(9, 12, 40, seed=6, sigma=3.0)).cuda()
    whole, parts = torch.zeros_like(u), torch.zeros_like(u)
    plan.run_slab([u, whole], 0, 9, 9)
    for part in [(0, 1), (8, 9), (1, 8)]:
        plan.run_slab([u, parts], 0, 9, 9, part=part)
    torch.cuda.synchronize()
    assert torch.equal(whole[1:-1], parts[1:-1])

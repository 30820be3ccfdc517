"""sm_100a fused biharmonic executor vs the CPU oracle, bit-exact (config 1)."""
import numpy as np
import pytest

import oracle
import paper_1710_08774_b200 as lf
from paper_1710_08774_b200 import inputs

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def run_device(plan, u, steps):
    import torch
    du = torch.from_numpy(u).cuda()
    keep = du.clone()
    out = torch.full_like(du, float("nan"))
    plan.run([du, out], steps=steps)
    torch.cuda.synchronize()
    assert torch.equal(du, keep), "axiom buffer must not be written"
    return out.cpu().numpy()


@pytest.mark.parametrize("shape,steps", [((1, 128), 1), ((5, 128), 2), ((16, 128), 1), ((37, 256), 3),
                                         ((64, 384), 4), ((200, 256), 2), ((333, 128), 5)])
def test_device_path_matches_naive(shape, steps):
    plan = lf.Plan.with_ranges("biharmonic2d", shape)
    assert plan.executor == "biharm2d_fused_tma"
    u = inputs.biharm_input(*shape, seed=sum(shape))
    got = run_device(plan, u, steps)
    ref = oracle.biharm(u, steps)
    # whole buffer, ghost ring included (zero Dirichlet, refilled every step)
    assert np.array_equal(bits(got), bits(ref))


# in place (config.aliases: g_unew on g_u's buffer): one strip and several, cuts
# inside strips, fewer rows than the row-band depth
@pytest.mark.parametrize("shape,steps", [((1, 128), 2), ((5, 128), 3), ((37, 256), 3), ((64, 384), 4),
                                         ((200, 256), 2), ((333, 128), 5), ((700, 1024), 3)])
def test_in_place_matches_naive(shape, steps):
    import torch
    plan = lf.Plan.with_ranges("biharmonic2d", shape, inplace=True)
    assert plan.executor == "biharm2d_fused_tma"
    u = inputs.biharm_input(*shape, seed=sum(shape) + 1)
    du = torch.from_numpy(u).cuda()
    plan.run([du, du], steps=steps)
    torch.cuda.synchronize()
    got = du.cpu().numpy()
    ref = oracle.biharm(u, steps)
    assert np.array_equal(bits(got), bits(ref)), int(np.count_nonzero(got != ref))
    # host path: one device buffer
    h = u.copy()
    plan.run_host([h, h], steps=steps)
    assert np.array_equal(bits(h), bits(ref))


def test_in_place_full_size_4096_and_undeclared_alias():
    import torch
    plan = lf.Plan.with_ranges("biharmonic2d", (4096, 4096), inplace=True)
    u = inputs.biharm_input(4096, 4096, seed=0)
    du = torch.from_numpy(u).cuda()
    plan.run([du, du], steps=5)
    torch.cuda.synchronize()
    assert np.array_equal(bits(du.cpu().numpy()), bits(oracle.biharm(u, 5, fused=True)))
    with pytest.raises(lf.LoomfuseError, match="config.aliases does not declare"):
        lf.Plan.bundled("biharmonic2d").run([du, du], steps=1)


def test_host_path_and_reuse():
    shape = (48, 128)
    plan = lf.Plan.with_ranges("biharmonic2d", shape)
    u = inputs.biharm_input(*shape, seed=4)
    for steps in (3, 1, 2):
        out = np.full_like(u, 7.0)
        plan.run_host([u, out], steps=steps)
        assert np.array_equal(bits(out), bits(oracle.biharm(u, steps)))


def test_full_size_4096_matches_fused_cpu():
    plan = lf.Plan.bundled("biharmonic2d")
    u = inputs.biharm_input(4096, 4096, seed=0)
    got = run_device(plan, u, 3)
    ref = oracle.biharm(u, 3, fused=True)
    assert np.array_equal(bits(got), bits(ref))


def test_configs0_all_100_iterations_match_fused_cpu():
    """BASELINE configs[0] as quoted: 4096 x 4096, all 100 iterations."""
    plan = lf.Plan.bundled("biharmonic2d")
    u = inputs.biharm_input(4096, 4096, seed=0)
    got = run_device(plan, u, 100)
    ref = oracle.biharm(u, 100, fused=True)
    assert np.array_equal(bits(got), bits(ref))


def test_slab_rows_leave_internal_ghosts_to_the_exchange():
    import torch
    shape = (24, 128)
    plan = lf.Plan.with_ranges("biharmonic2d", shape)
    u = inputs.biharm_input(*shape, seed=8)
    ref = oracle.biharm(u, 1)
    # middle slab rows [8, 16): buffer holds rows 6..17 (2 ghost rows each side)
    local = torch.from_numpy(np.ascontiguousarray(u[8:8 + 8 + 4])).cuda()
    out = torch.full_like(local, 5.0)
    plan.run_slab([local, out], 8, 16, 24)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert np.array_equal(bits(got[2:-2]), bits(ref[10:18]))
    assert np.all(got[:2, 2:-2] == 5.0) and np.all(got[-2:, 2:-2] == 5.0)


@pytest.mark.parametrize("name,gen,shape", [
    ("biharmonic2d", lambda s: [inputs.biharm_input(*s, seed=2)], (40, 256)),
    ("box2x", lambda s: [inputs.box_input(*s, seed=2)], (40, 256)),
])
def test_row_parts_compose_to_the_whole_slab(name, gen, shape):
    import torch
    plan = lf.Plan.with_ranges(name, shape)
    ax = [torch.from_numpy(a).cuda() for a in gen(shape)]
    g = plan.goals[0]
    dt = torch.float64 if g.elem_bytes == 8 else torch.float32
    whole = torch.zeros(g.extent, dtype=dt, device="cuda")
    parts = torch.zeros(g.extent, dtype=dt, device="cuda")
    plan.run_slab(ax + [whole], 0, shape[0], shape[0])
    for part in [(0, 2), (shape[0] - 2, shape[0]), (2, shape[0] - 2)]:
        plan.run_slab(ax + [parts], 0, shape[0], shape[0], part=part)
    torch.cuda.synchronize()
    assert torch.equal(whole, parts)

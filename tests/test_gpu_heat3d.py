"""sm_100a fused heat3d executor vs the CPU oracle, bit-exact (config 2).

Small grids are compared against run_naive; the full 512^3 grid against the
HFAV fused CPU schedule (itself pinned to run_naive in test_oracle.py) plus
size-independent properties (mass conservation under periodic diffusion, the
maximum principle)."""
import numpy as np
import pytest

import oracle
import paper_1710_08774_b200 as lf
from paper_1710_08774_b200 import inputs

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def interior(a):
    return a[1:-1, 1:-1, 1:-1]


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("shape,steps", [((4, 16, 64), 1), ((8, 16, 64), 3), ((20, 32, 128), 2),
                                         ((64, 64, 64), 4), ((3, 48, 192), 5)])
def test_device_path_matches_naive(shape, steps):
    torch = _torch()
    plan = lf.Plan.with_ranges("heat3d", shape)
    assert plan.executor == "heat3d_fused_tma"
    u = inputs.heat3d_input(*shape, seed=11, sigma=4.0)
    ref = oracle.heat3d(u, steps)
    du = torch.from_numpy(u).cuda()
    keep = du.clone()
    out = torch.full_like(du, float("nan"))
    plan.run([du, out], steps=steps)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    # the whole goal buffer: interior plus every ghost cell (faces, edges and
    # corners are the periodic images the oracle's ghost fill composes)
    assert np.array_equal(bits(got), bits(ref))
    assert torch.equal(du, keep), "axiom buffer must not be written"
    # the periodic ghost faces the next step reads are refilled
    g = got.copy()
    for ax in range(3):
        sl_g = [slice(1, -1)] * 3
        sl_s = [slice(1, -1)] * 3
        sl_g[ax], sl_s[ax] = 0, -2
        assert np.array_equal(bits(g[tuple(sl_g)]), bits(g[tuple(sl_s)]))


def test_host_path_matches_oracle():
    shape, steps = (16, 32, 128), 3
    plan = lf.Plan.with_ranges("heat3d", shape)
    u = inputs.heat3d_input(*shape, seed=5, sigma=5.0)
    out = np.full_like(u, np.nan)
    plan.run_host([u, out], steps=steps)
    ref = oracle.heat3d(u, steps, fused=True)
    # every cell of the caller's goal buffer comes back defined (ghost edges
    # and corners included), equal to the oracle's
    assert np.array_equal(bits(out), bits(ref))
    # a second call reuses the cached device buffers; the single-step host run
    # is pipelined in row parts
    out2 = np.full_like(u, np.nan)
    plan.run_host([u, out2], steps=1)
    assert np.array_equal(bits(out2), bits(oracle.heat3d(u, 1)))
    big = (1024, 16, 64)  # >= 1024 planes: the pipelined row-part path
    ub = inputs.heat3d_input(*big, seed=6, sigma=5.0)
    out3 = np.full_like(ub, np.nan)
    lf.Plan.with_ranges("heat3d", big).run_host([ub, out3], steps=1)
    assert np.array_equal(bits(out3), bits(oracle.heat3d(ub, 1)))


def test_full_size_512_matches_fused_cpu_and_conserves_mass():
    torch = _torch()
    shape, steps = (512, 512, 512), 2
    plan = lf.Plan.bundled("heat3d")
    u = inputs.heat3d_input(*shape, seed=0)
    du = torch.from_numpy(u).cuda()
    out = torch.empty_like(du)
    plan.run([du, out], steps=steps)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    ref = oracle.heat3d(u, steps, fused=True)
    assert np.array_equal(bits(interior(got)), bits(interior(ref)))
    s0 = interior(u).sum(dtype=np.float64)
    assert interior(got).sum(dtype=np.float64) == pytest.approx(s0, rel=1e-12)
    assert interior(got).max() <= interior(u).max() and interior(got).min() >= interior(u).min()


def test_configs1_all_50_steps_match_fused_cpu():
    """BASELINE configs[1] as quoted: 512^3, all 50 steps."""
    torch = _torch()
    plan = lf.Plan.bundled("heat3d")
    u = inputs.heat3d_input(512, 512, 512, seed=0)
    du = torch.from_numpy(u).cuda()
    out = torch.empty_like(du)
    plan.run([du, out], steps=50)
    torch.cuda.synchronize()
    ref = oracle.heat3d(u, 50, fused=True)
    assert np.array_equal(bits(interior(out.cpu().numpy())), bits(interior(ref)))


def test_slab_mode_skips_k_wrap():
    torch = _torch()
    shape = (8, 16, 64)
    plan = lf.Plan.with_ranges("heat3d", shape)
    u = inputs.heat3d_input(*shape, seed=3, sigma=3.0)
    du = torch.from_numpy(u).cuda()
    out = torch.zeros_like(du)
    plan.run_slab([du, out], 0, 8, 8)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    ref = oracle.heat3d(u, 1)
    assert np.array_equal(bits(interior(got)), bits(interior(ref)))
    assert not got[0].any() and not got[-1].any()


def test_slab_parts_compose_to_the_whole_slab():
    """Face rows + interior rows computed by separate lf_run_slab parts (the
    overlapped multi-GPU schedule) equal one whole-slab call, bit for bit."""
    torch = _torch()
    shape = (12, 32, 128)
    plan = lf.Plan.with_ranges("heat3d", shape)
    u = inputs.heat3d_input(*shape, seed=13, sigma=3.0)
    du = torch.from_numpy(u).cuda()
    whole = torch.zeros_like(du)
    parts = torch.zeros_like(du)
    plan.run_slab([du, whole], 0, 12, 12)
    for part in [(0, 1), (11, 12), (1, 11)]:
        plan.run_slab([du, parts], 0, 12, 12, part=part)
    torch.cuda.synchronize()
    assert torch.equal(whole, parts)


def test_overlapped_slab_schedule_single_rank_periodic():
    """The multi-GPU schedule (face planes, exchange on a side stream, interior
    planes) run with one rank: the periodic self-exchange closes the ring and
    the result equals the oracle's multi-step run."""
    torch = _torch()
    from paper_1710_08774_b200 import slabs
    shape, steps = (10, 32, 64), 3
    plan = lf.Plan.with_ranges("heat3d", shape)
    u = inputs.heat3d_input(*shape, seed=17, sigma=3.0)
    cur = [torch.from_numpy(u).cuda()]
    nxt = [torch.zeros_like(cur[0])]

    def launch(src, dst, part):
        plan.run_slab([src[0], dst[0]], 0, shape[0], shape[0], stream=torch.cuda.current_stream(), part=part)

    res = slabs.run_slabs_overlapped(launch, cur, nxt, steps, slabs.Halo(1, 1, True), 0, 1, shape[0])
    torch.cuda.synchronize()
    got = res[0].cpu().numpy()
    ref = oracle.heat3d(u, steps)
    assert np.array_equal(bits(interior(got)), bits(interior(ref)))


@pytest.mark.parametrize("shape,steps", [((8, 16, 64), 2), ((20, 32, 128), 3), ((64, 64, 64), 4), ((3, 48, 192), 5)])
def test_two_step_passes_match_naive(shape, steps, monkeypatch):
    """Opt-in temporal blocking (LF_HEAT3D_TB=1): two time steps per pass over
    the grid, periodic images patched on face tiles -- bit-exact, faces of the
    ghost layer refilled as by the single-step kernel."""
    monkeypatch.setenv("LF_HEAT3D_TB", "1")
    torch = _torch()
    plan = lf.Plan.with_ranges("heat3d", shape)
    assert plan.grid_passes(steps) == (steps + 1) // 2
    u = inputs.heat3d_input(*shape, seed=13, sigma=4.0)
    ref = oracle.heat3d(u, steps)
    du = torch.from_numpy(u).cuda()
    out = torch.full_like(du, float("nan"))
    plan.run([du, out], steps=steps)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert np.array_equal(bits(interior(got)), bits(interior(ref)))
    for ax in range(3):
        sl_g = [slice(1, -1)] * 3
        sl_s = [slice(1, -1)] * 3
        sl_g[ax], sl_s[ax] = 0, -2
        assert np.array_equal(bits(got[tuple(sl_g)]), bits(got[tuple(sl_s)]))

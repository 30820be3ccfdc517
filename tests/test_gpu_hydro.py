"""sm_100a fused Hydro2D executor (x- and y-sweep in one pass) vs the CPU
oracle, bit-exact (configs 3 and 5)."""
import numpy as np
import pytest

import oracle
import paper_1710_08774_b200 as lf
from paper_1710_08774_b200 import inputs

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def run_device(plan, st, dtdx, steps):
    import torch
    ax = [torch.from_numpy(a).cuda() for a in st] + [torch.tensor([dtdx], dtype=torch.float64, device="cuda")]
    keep = [a.clone() for a in ax]
    goals = [torch.full_like(ax[0], float("nan")) for _ in range(4)]
    plan.run(ax + goals, steps=steps)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(ax, keep)), "axiom buffers must not be written"
    return [g.cpu().numpy() for g in goals]


@pytest.mark.parametrize("shape,steps", [((4, 4), 1), ((8, 16), 1), ((12, 20), 3), ((33, 130), 2),
                                         ((64, 256), 3), ((130, 254), 2), ((5, 384), 4)])
def test_device_path_matches_naive(shape, steps):
    plan = lf.Plan.with_ranges("hydro2d", shape)
    assert plan.executor == "hydro2d_fused_tma"
    st, dtdx = inputs.hydro_input(*shape, seed=shape[0] + 7)
    got = run_device(plan, st, dtdx, steps)
    ref = oracle.hydro(st, dtdx, steps)
    # whole buffers: interior and the reflective ghost ring (incl. corners)
    for v in range(4):
        assert np.array_equal(bits(got[v]), bits(ref[v])), v


def test_host_path():
    shape = (40, 200)
    plan = lf.Plan.with_ranges("hydro2d", shape)
    st, dtdx = inputs.hydro_input(*shape, seed=3)
    outs = [np.zeros_like(st[0]) for _ in range(4)]
    plan.run_host(st + [np.array([dtdx])] + outs, steps=2)
    ref = oracle.hydro(st, dtdx, 2, fused=True)
    for v in range(4):
        assert np.array_equal(bits(outs[v]), bits(ref[v]))


def test_full_size_4096_matches_fused_cpu_and_conserves():
    plan = lf.Plan.bundled("hydro2d")
    st, dtdx = inputs.hydro_input(4096, 4096, seed=0)
    got = run_device(plan, st, dtdx, 2)
    ref = oracle.hydro(st, dtdx, 2, fused=True)
    for v in range(4):
        assert np.array_equal(bits(got[v]), bits(ref[v])), v
    # reflective walls conserve mass and energy to rounding
    for v in (0, 3):
        assert got[v][2:-2, 2:-2].sum() == pytest.approx(st[v][2:-2, 2:-2].sum(), rel=1e-12)


def test_configs2_all_20_steps_match_fused_cpu():
    """BASELINE configs[2] as quoted: 4096 x 4096, all 20 steps."""
    plan = lf.Plan.bundled("hydro2d")
    st, dtdx = inputs.hydro_input(4096, 4096, seed=0)
    got = run_device(plan, st, dtdx, 20)
    ref = oracle.hydro(st, dtdx, 20, fused=True)
    for v in range(4):
        assert np.array_equal(bits(got[v]), bits(ref[v])), v


def run_in_place(plan, st, dtdx, steps):
    import torch
    u = [torch.from_numpy(a).cuda() for a in st]
    plan.run(u + [torch.tensor([dtdx], dtype=torch.float64, device="cuda")] + u, steps=steps)
    torch.cuda.synchronize()
    return [a.cpu().numpy() for a in u]


# in place (config.aliases): every goal on its axiom's
# buffer -- half the device footprint; shapes with one and several strips,
# segment cuts inside strips, strips of 2 and 124 cells, fewer rows than the
# row-band depth
@pytest.mark.parametrize("shape,steps", [((4, 4), 2), ((8, 16), 1), ((12, 20), 3), ((33, 130), 2), ((64, 256), 3),
                                         ((130, 254), 2), ((5, 384), 4), ((700, 126), 2), ((257, 1000), 3)])
def test_in_place_matches_naive(shape, steps):
    plan = lf.Plan.with_ranges("hydro2d", shape, inplace=True)
    assert plan.executor == "hydro2d_fused_tma"
    st, dtdx = inputs.hydro_input(*shape, seed=shape[1] + 11)
    got = run_in_place(plan, st, dtdx, steps)
    ref = oracle.hydro(st, dtdx, steps)
    for v in range(4):
        assert np.array_equal(bits(got[v]), bits(ref[v])), (v, int(np.count_nonzero(got[v] != ref[v])))


def test_in_place_full_size_4096_matches_fused_cpu():
    plan = lf.Plan.with_ranges("hydro2d", (4096, 4096), inplace=True)
    st, dtdx = inputs.hydro_input(4096, 4096, seed=0)
    got = run_in_place(plan, st, dtdx, 3)
    ref = oracle.hydro(st, dtdx, 3, fused=True)
    for v in range(4):
        assert np.array_equal(bits(got[v]), bits(ref[v])), v


def test_in_place_host_path_keeps_one_device_buffer():
    shape = (40, 200)
    plan = lf.Plan.with_ranges("hydro2d", shape, inplace=True)
    st, dtdx = inputs.hydro_input(*shape, seed=3)
    u = [a.copy() for a in st]
    plan.run_host(u + [np.array([dtdx])] + u, steps=3)
    ref = oracle.hydro(st, dtdx, 3, fused=True)
    for v in range(4):
        assert np.array_equal(bits(u[v]), bits(ref[v]))


def test_in_place_needs_declared_aliases_and_every_pair():
    import torch
    shape = (16, 128)
    st, dtdx = inputs.hydro_input(*shape, seed=1)
    u = [torch.from_numpy(a).cuda() for a in st]
    d = [torch.tensor([dtdx], dtype=torch.float64, device="cuda")]
    with pytest.raises(lf.LoomfuseError, match="config.aliases does not declare"):
        lf.Plan.with_ranges("hydro2d", shape).run(u + d + u, steps=1)
    plan = lf.Plan.with_ranges("hydro2d", shape, inplace=True)
    with pytest.raises(lf.LoomfuseError, match="every iterated goal"):
        plan.run(u + d + [u[0], u[1], u[2], torch.empty_like(u[3])], steps=1)
    with pytest.raises(lf.LoomfuseError, match="not an iterate pair"):
        plan.run(u + d + [u[1], u[0], u[2], u[3]], steps=1)
    # distinct buffers still ping-pong on an alias-declaring plan
    out = [torch.empty_like(a) for a in u]
    plan.run(u + d + out, steps=2)
    torch.cuda.synchronize()
    ref = oracle.hydro(st, dtdx, 2)
    for v in range(4):
        assert np.array_equal(bits(out[v].cpu().numpy()), bits(ref[v]))


def test_row_parts_compose_to_the_whole_slab():
    import torch
    shape = (40, 300)
    plan = lf.Plan.with_ranges("hydro2d", shape)
    st, dtdx = inputs.hydro_input(*shape, seed=9)
    ax = [torch.from_numpy(a).cuda() for a in st] + [torch.tensor([dtdx], dtype=torch.float64, device="cuda")]
    whole = [torch.zeros_like(ax[0]) for _ in range(4)]
    parts = [torch.zeros_like(ax[0]) for _ in range(4)]
    plan.run_slab(ax + whole, 0, 40, 40)
    for part in [(0, 2), (38, 40), (2, 38)]:
        plan.run_slab(ax + parts, 0, 40, 40, part=part)
    torch.cuda.synchronize()
    for a, b in zip(whole, parts):
        assert torch.equal(a, b)


def test_exact_fallbacks_of_the_fast_paths():
    """Every branch-free division / square root (csrc/exec/fastmath.cuh) has an
    out-of-line exact fallback taken when its operands leave the fast range --
    rare in practice, so force it everywhere (LF_HYDRO_FORCE_SLOW, set
    in-process) and check the result is still the oracle's, bit for bit."""
    import torch
    shape = (33, 130)
    plan = lf.Plan.with_ranges("hydro2d", shape)
    st, dtdx = inputs.hydro_input(*shape, seed=11)
    with lf.option("LF_HYDRO_FORCE_SLOW", 1):
        got = run_device(plan, st, dtdx, 2)
    ref = oracle.hydro(st, dtdx, 2)
    for v in range(4):
        assert np.array_equal(bits(got[v]), bits(ref[v])), v

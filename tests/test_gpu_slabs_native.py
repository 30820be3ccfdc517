"""Native multi-GPU slab runs (lf_run_slabs / lf_run_slabs_local, SURVEY.md
8(e)) against whole-domain lf_run, bit-exact.

lf_run_slabs_local runs every rank of the decomposition on this GPU with the
halo exchange as device copies -- the same slab geometry, face/interior split
and ping-pong as lf_run_slabs -- so the decomposition logic is checked on one
GPU without running mutually-waiting ranks.  lf_run_slabs itself is run on a
one-rank NCCL communicator (the periodic ring sends to itself)."""
import numpy as np
import pytest

import paper_1710_08774_b200 as lf
from paper_1710_08774_b200 import inputs
from pathlib import Path

pytestmark = pytest.mark.gpu

SPECS = Path(__file__).parent / "specs"


def _case(name, shape):
    """plan, axiom arrays (in order), global goal shapes"""
    if name == "heat3d":
        plan = lf.Plan.with_ranges("heat3d", shape)
        ax = [inputs.heat3d_input(*shape, seed=3, sigma=2.0)]
    elif name == "biharm":
        plan = lf.Plan.with_ranges("biharmonic2d", shape)
        ax = [inputs.biharm_input(*shape, seed=4)]
    elif name in ("hydro", "hydro_adaptive"):
        plan = lf.Plan.with_ranges("hydro2d" if name == "hydro" else "hydro2d_adaptive", shape)
        st, dtdx = inputs.hydro_input(*shape, seed=5)
        ax = list(st) + [np.array(dtdx, dtype=np.float64)]
    elif name == "heat3d_jit":
        plan = lf.Plan(lf.set_ranges((SPECS / "heat3d_body.lf").read_text(), shape), "h.lf")
        assert plan.executor.startswith("jit_")
        ax = [inputs.heat3d_input(*shape, seed=6, sigma=2.0)]
    elif name == "biharm_jit":
        plan = lf.Plan(lf.set_ranges((SPECS / "biharm_body.lf").read_text(), shape), "b.lf")
        assert plan.executor.startswith("jit_")
        ax = [inputs.biharm_input(*shape, seed=7)]
    else:
        raise KeyError(name)
    return plan, ax


def _whole(plan, ax, steps):
    import torch
    d_ax = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in ax]
    goals = [torch.zeros(t.extent, dtype=torch.float64, device="cuda") for t in plan.goals]
    plan.run(d_ax + goals, steps=steps)
    torch.cuda.synchronize()
    return [g.cpu().numpy() for g in goals]


def _slab_bufs(plan, ax, n0, lo, hi):
    import torch
    bufs = []
    for t, a in zip(plan.axioms, ax):
        if not t.extent:
            bufs.append(torch.from_numpy(np.ascontiguousarray(a)).cuda())
            continue
        rows = hi - lo + t.extent[0] - n0
        bufs.append(torch.from_numpy(np.ascontiguousarray(a[lo:lo + rows])).cuda())
    for k, t in enumerate(plan.goals):
        idx = len(plan.axioms) + k
        # zeros like _whole's goals: the heat chain never writes the (j, i)
        # ghost edges (the 7-point stencil does not read them)
        bufs.append(torch.zeros(plan.slab_terminal_extent(idx, lo, hi, n0), dtype=torch.float64, device="cuda"))
    return bufs


def _assemble(plan, rank_bufs, ranges, n0):
    """global goal arrays from the ranks' slab goals: interiors, plus rank 0's
    lower and the last rank's upper ghost rows"""
    out = []
    na = len(plan.axioms)
    for k, t in enumerate(plan.goals):
        if not t.extent:  # a rank-0 goal (the adaptive chain's dt/dx): every rank holds the same value
            vals = [bufs[na + k].cpu().numpy() for bufs in rank_bufs]
            assert all(np.array_equal(v, vals[0]) for v in vals)
            out.append(vals[0])
            continue
        below = -t.base[0]
        above = t.extent[0] - n0 - below
        g = np.empty(t.extent)
        for (lo, hi), bufs in zip(ranges, rank_bufs):
            s = bufs[na + k].cpu().numpy()
            g[below + lo:below + hi] = s[below:below + hi - lo]
            if lo == 0:
                g[:below] = s[:below]
            if hi == n0:
                g[below + n0:] = s[below + hi - lo:below + hi - lo + above]
        out.append(g)
    return out


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def _defined(name, a):
    """cells the chain defines: the 7-point heat chain neither reads nor
    writes ghost edges/corners (two or more ghost coordinates), so the whole
    domain leaves them as initialised while an exchanged ghost plane carries
    the neighbour's -- compare everything else"""
    if not name.startswith("heat3d"):
        return a
    ghost = np.zeros(a.shape, dtype=np.int8)
    for d, n in enumerate(a.shape):
        idx = [None] * a.ndim
        idx[d] = slice(None)
        g = np.zeros(n, dtype=np.int8)
        g[0] = g[-1] = 1
        ghost = ghost + g[tuple(idx)]
    return np.where(ghost >= 2, 0.0, a)


CASES = [
    ("heat3d", (12, 32, 128), 3, [2, 3]),   # heat3d_fused_tma
    ("heat3d", (12, 16, 40), 3, [2, 3]),    # sizes the built-in rejects: generic executor
    ("heat3d", (9, 32, 64), 2, [4]),
    ("biharm", (30, 64), 3, [2, 3]),
    ("hydro", (24, 64), 2, [2, 3]),
    ("hydro_adaptive", (24, 64), 3, [2, 3]),  # + one MAX reduction per step across the ranks
    ("heat3d_jit", (10, 12, 40), 3, [2]),
    ("biharm_jit", (26, 70), 2, [3]),
]


@pytest.mark.parametrize("name,shape,steps,worlds", CASES)
def test_local_slab_decomposition_matches_whole_domain(name, shape, steps, worlds):
    import torch
    plan, ax = _case(name, shape)
    if shape == (12, 32, 128):
        assert plan.executor == "heat3d_fused_tma"
    n0 = shape[0]
    ref = _whole(plan, ax, steps)
    for world in worlds:
        ranges = [(n0 * r // world, n0 * (r + 1) // world) for r in range(world)]
        rank_bufs = [_slab_bufs(plan, ax, n0, lo, hi) for lo, hi in ranges]
        lf.run_slabs_local(plan, rank_bufs, steps=steps)
        torch.cuda.synchronize()
        got = _assemble(plan, rank_bufs, ranges, n0)
        for g, r, t in zip(got, ref, plan.goals):
            assert np.array_equal(bits(_defined(name, g)), bits(_defined(name, r))), (name, world, t.name)


@pytest.mark.parametrize("name,shape,steps,worlds", [("hydro", (24, 64), 3, [2, 3]), ("hydro", (40, 300), 2, [4]),
                                                     ("hydro_adaptive", (24, 130), 3, [2, 3])])
def test_local_slabs_in_place(name, shape, steps, worlds):
    """Slab runs IN PLACE (config.aliases; every rank passes its state goals on
    its axioms' slab buffers): whole-slab launches with deferred boundary
    writes, then the exchange -- equal to the whole-domain ping-pong run."""
    import torch
    plan, ax = _case(name, shape)
    spec = "hydro2d" if name == "hydro" else "hydro2d_adaptive"
    ip = lf.Plan.with_ranges(spec, shape, inplace=True)
    n0 = shape[0]
    ref = _whole(plan, ax, steps)
    for world in worlds:
        ranges = [(n0 * r // world, n0 * (r + 1) // world) for r in range(world)]
        rank_bufs = []
        for lo, hi in ranges:
            b = _slab_bufs(ip, ax, n0, lo, hi)
            na = len(ip.axioms)
            for k in range(4):  # the four state goals on their axioms' buffers
                b[na + k] = b[k]
            rank_bufs.append(b)
        lf.run_slabs_local(ip, rank_bufs, steps=steps)
        torch.cuda.synchronize()
        got = _assemble(ip, rank_bufs, ranges, n0)
        for g, r, t in zip(got, ref, ip.goals):
            assert np.array_equal(bits(g), bits(r)), (name, world, t.name)
    # a one-rank NCCL communicator: lf_run_slabs itself, in place
    bufs = _slab_bufs(ip, ax, n0, 0, n0)
    for k in range(4):
        bufs[len(ip.axioms) + k] = bufs[k]
    comm = lf.NcclComm.single()
    try:
        ip.run_slabs(bufs, comm, steps=steps)
        torch.cuda.synchronize()
        got = _assemble(ip, [bufs], [(0, n0)], n0)
        for g, r, t in zip(got, ref, ip.goals):
            assert np.array_equal(bits(g), bits(r)), (name, t.name)
    finally:
        comm.destroy()


@pytest.mark.parametrize("name,shape,steps", [("heat3d", (12, 16, 40), 3), ("biharm", (30, 64), 2),
                                              ("hydro", (16, 48), 3), ("hydro_adaptive", (16, 48), 3),
                                              ("heat3d_jit", (8, 12, 40), 2)])
def test_nccl_one_rank_matches_whole_domain(name, shape, steps):
    import torch
    plan, ax = _case(name, shape)
    n0 = shape[0]
    ref = _whole(plan, ax, steps)
    comm = lf.NcclComm.single()
    try:
        bufs = _slab_bufs(plan, ax, n0, 0, n0)
        keep = [b.clone() for b in bufs[:len(plan.axioms)]]
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            plan.run_slabs(bufs, comm, steps=steps, stream=stream)
        stream.synchronize()
        got = _assemble(plan, [bufs], [(0, n0)], n0)
        for g, r, t in zip(got, ref, plan.goals):
            assert np.array_equal(bits(_defined(name, g)), bits(_defined(name, r))), (name, t.name)
        assert all(torch.equal(a, b) for a, b in zip(bufs, keep)), "axiom buffers must not be written"
    finally:
        comm.destroy()


def test_slab_run_argument_errors():
    plan, ax = _case("heat3d", (4, 8, 32))
    bufs = _slab_bufs(plan, ax, 4, 0, 4)
    with pytest.raises(lf.LoomfuseError) as e:
        lf.run_slabs_local(plan, [bufs] * 5, steps=1)  # more ranks than planes
    assert e.value.code == lf.LF_ERR_SPEC


@pytest.mark.parametrize("schedule", ["serial", "concurrent", "whole", "parallel"])
def test_alternative_slab_schedules_match_whole_domain(schedule):
    """Every selectable slab schedule (LF_SLAB_SCHEDULE, set in-process with
    lf.option; the default picks `whole` for slabs of >= 1024 rows, else
    `parallel`) gives the same bits: the decomposition tests of this file."""
    with lf.option("LF_SLAB_SCHEDULE", schedule):
        for case in CASES:
            test_local_slab_decomposition_matches_whole_domain(*case)
        for name, shape, steps in [("heat3d", (12, 16, 40), 3), ("biharm", (30, 64), 2), ("hydro", (16, 48), 3)]:
            test_nccl_one_rank_matches_whole_domain(name, shape, steps)

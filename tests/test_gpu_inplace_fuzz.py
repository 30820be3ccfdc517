"""Seeded random shapes: the in-place runs of the hand-written executors
(config.aliases) against their own ping-pong runs, bit
for bit over the whole buffers -- device path, pipelined host path (random row
parts, wavefront forced) and local slab decompositions.  The ping-pong runs
are pinned to the CPU oracle elsewhere (tests/test_gpu_hydro.py,
tests/test_gpu_biharm.py); this file needs no oracle, so it can afford many
shapes: strips of every width, segment cuts at every phase of the march."""
import numpy as np
import pytest

import paper_1710_08774_b200 as lf
from paper_1710_08774_b200 import inputs

pytestmark = pytest.mark.gpu


def _hydro_pingpong(shape, st, dtdx, steps):
    import torch
    plan = lf.Plan.with_ranges("hydro2d", shape)
    ax = [torch.from_numpy(a).cuda() for a in st] + [torch.tensor([dtdx], dtype=torch.float64, device="cuda")]
    goals = [torch.full_like(ax[0], float("nan")) for _ in range(4)]
    plan.run(ax + goals, steps=steps)
    torch.cuda.synchronize()
    return goals


@pytest.mark.parametrize("seed", range(32))
def test_hydro_in_place_equals_ping_pong(seed, monkeypatch):
    import torch
    rng = np.random.default_rng(1000 + seed)
    nj = int(rng.integers(4, 400))
    ni = 2 * int(rng.integers(2, 700))
    steps = int(rng.integers(1, 6))
    shape = (nj, ni)
    st, dtdx = inputs.hydro_input(nj, ni, seed=seed)
    ref = _hydro_pingpong(shape, st, dtdx, steps)
    plan = lf.Plan.with_ranges("hydro2d", shape, inplace=True)
    d = torch.tensor([dtdx], dtype=torch.float64, device="cuda")
    u = [torch.from_numpy(a).cuda() for a in st]
    plan.run(u + [d] + u, steps=steps)
    torch.cuda.synchronize()
    for v in range(4):
        assert torch.equal(u[v].view(torch.int64), ref[v].view(torch.int64)), (shape, steps, v)
    # pipelined host path, wavefront forced, random row parts (thin parts fall back to the serial path)
    parts = int(rng.integers(2, max(3, nj // 4 + 1)))
    monkeypatch.setenv("LF_HOST_WAVEFRONT", "1")
    monkeypatch.setenv("LF_HOST_PARTS", str(parts))
    h = [a.copy() for a in st]
    plan.run_host(h + [np.array([dtdx])] + h, steps=steps)
    for v in range(4):
        assert np.array_equal(h[v].view(np.uint64), ref[v].cpu().numpy().view(np.uint64)), (shape, steps, parts, v)
    # local slab decomposition in place (every rank at least two halos of rows)
    world = int(rng.integers(2, 5))
    if nj // world >= 4:
        ranges = [(nj * r // world, nj * (r + 1) // world) for r in range(world)]
        rank_bufs = []
        for lo, hi in ranges:
            s_ax = [torch.from_numpy(np.ascontiguousarray(a[lo:hi + 4])).cuda() for a in st]
            rank_bufs.append(s_ax + [d.clone()] + s_ax)
        lf.run_slabs_local(plan, rank_bufs, steps=steps)
        torch.cuda.synchronize()
        for (lo, hi), bufs in zip(ranges, rank_bufs):
            for v in range(4):
                a, b = bufs[v][2:2 + hi - lo], ref[v][2 + lo:2 + hi]
                assert torch.equal(a.view(torch.int64), b.view(torch.int64)), (shape, steps, world, lo, v)


@pytest.mark.parametrize("seed", range(24))
def test_biharm_in_place_equals_ping_pong(seed):
    import torch
    rng = np.random.default_rng(2000 + seed)
    nj = int(rng.integers(1, 600))
    ni = 128 * int(rng.integers(1, 12))
    steps = int(rng.integers(1, 7))
    u0 = inputs.biharm_input(nj, ni, seed=seed)
    du = torch.from_numpy(u0).cuda()
    out = torch.full_like(du, float("nan"))
    lf.Plan.with_ranges("biharmonic2d", (nj, ni)).run([du, out], steps=steps)
    plan = lf.Plan.with_ranges("biharmonic2d", (nj, ni), inplace=True)
    dv = torch.from_numpy(u0).cuda()
    plan.run([dv, dv], steps=steps)
    torch.cuda.synchronize()
    assert torch.equal(dv.view(torch.int64), out.view(torch.int64)), (nj, ni, steps)


@pytest.mark.parametrize("seed", range(6))
def test_band_stores_stay_inside_their_buffers(seed, monkeypatch):
    """LF_BAND_GUARD=1: canary zones either side of the plan-owned bands, checked
    after every in-place run (stands in for compute-sanitizer memcheck, which the
    GPU pool does not allow): device runs, the host wavefront, the adaptive chain
    and the biharmonic chain on shapes whose last strip / segment is ragged."""
    import torch
    rng = np.random.default_rng(3000 + seed)
    nj, ni, steps = int(rng.integers(4, 300)), 2 * int(rng.integers(2, 600)), int(rng.integers(1, 5))
    st, dtdx = inputs.hydro_input(nj, ni, seed=seed)
    ref = _hydro_pingpong((nj, ni), st, dtdx, steps)
    with lf.option("LF_BAND_GUARD", 1):
        plan = lf.Plan.with_ranges("hydro2d", (nj, ni), inplace=True)
        d = torch.tensor([dtdx], dtype=torch.float64, device="cuda")
        u = [torch.from_numpy(a).cuda() for a in st]
        plan.run(u + [d] + u, steps=steps)
        torch.cuda.synchronize()
        for v in range(4):
            assert torch.equal(u[v].view(torch.int64), ref[v].view(torch.int64)), v
        monkeypatch.setenv("LF_HOST_WAVEFRONT", "1")
        monkeypatch.setenv("LF_HOST_PARTS", str(max(2, nj // 8)))
        h = [a.copy() for a in st]
        plan.run_host(h + [np.array([dtdx])] + h, steps=max(2, steps))
        ad = lf.Plan.with_ranges("hydro2d_adaptive", (nj, ni), inplace=True)
        u = [torch.from_numpy(a).cuda() for a in st]
        ad.run(u + [d.reshape(())] + u + [torch.zeros((), dtype=torch.float64, device="cuda")], steps=steps)
        bj, bi = int(rng.integers(1, 300)), 128 * int(rng.integers(1, 9))
        bu = torch.from_numpy(inputs.biharm_input(bj, bi, seed=seed)).cuda()
        lf.Plan.with_ranges("biharmonic2d", (bj, bi), inplace=True).run([bu, bu], steps=steps)
        torch.cuda.synchronize()


def test_band_guard_catches_a_store_past_the_bands():
    """Fault injection (LF_BAND_GUARD=2 shifts the executor's range 64 bytes into
    the rear guard): the adaptive chain's second dt/dx slot is the last thing in
    the band memory, a two-step run writes it, and the run must fail."""
    import torch
    st, dtdx = inputs.hydro_input(24, 130, seed=1)
    plan = lf.Plan.with_ranges("hydro2d_adaptive", (24, 130), inplace=True)
    u = [torch.from_numpy(a).cuda() for a in st]
    d = torch.tensor(dtdx, dtype=torch.float64, device="cuda")
    out = torch.zeros((), dtype=torch.float64, device="cuda")
    with lf.option("LF_BAND_GUARD", 2):
        with pytest.raises(lf.LoomfuseError, match="outside its buffer"):
            plan.run(u + [d] + u + [out], steps=2)
    with lf.option("LF_BAND_GUARD", 1):
        u = [torch.from_numpy(a).cuda() for a in st]
        plan.run(u + [d] + u + [out], steps=2)

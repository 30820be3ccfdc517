"""Hydro2D with the adaptive CFL time step (specs/hydro2d_adaptive.lf,
SURVEY.md 8(f) row 4): the fused executor reduces max(|u|, |v|) + c over every
cell it stores and the next step takes dt/dx = 0.5 / max -- bit-exact against
the CPU oracle (whose reduction is run_naive's sequential sweep: the maximum is
exact in any order), the final dt/dx goal included."""
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
    ax = [torch.from_numpy(a).cuda() for a in st] + [torch.tensor(dtdx, dtype=torch.float64, device="cuda")]
    goals = [torch.full_like(ax[0], float("nan")) for _ in range(4)] + [torch.zeros((), dtype=torch.float64,
                                                                                    device="cuda")]
    plan.run(ax + goals, steps=steps)
    torch.cuda.synchronize()
    return [g.cpu().numpy() for g in goals]


@pytest.mark.parametrize("shape,steps", [((8, 16), 1), ((12, 20), 3), ((33, 130), 4), ((64, 256), 5),
                                         ((130, 254), 2)])
def test_adaptive_matches_oracle(shape, steps):
    plan = lf.Plan.with_ranges("hydro2d_adaptive", shape)
    assert plan.executor == "hydro2d_adaptive_fused_tma"
    st, dtdx = inputs.hydro_input(*shape, seed=shape[1] + 3)
    got = run_device(plan, st, dtdx, steps)
    ref, dref = oracle.hydro_adaptive(st, dtdx, steps)
    for v in range(4):
        assert np.array_equal(bits(got[v]), bits(ref[v])), v
    assert bits(got[4]).item() == np.float64(dref).view(np.uint64), (float(got[4]), dref)
    # the time step does adapt: the first state's dt/dx is not the last one's
    assert dref != dtdx


def test_adaptive_host_path_and_full_size():
    shape, steps = (40, 200), 3
    plan = lf.Plan.with_ranges("hydro2d_adaptive", shape)
    st, dtdx = inputs.hydro_input(*shape, seed=2)
    outs = [np.zeros_like(st[0]) for _ in range(4)] + [np.zeros(1)]
    plan.run_host(st + [np.array([dtdx])] + outs, steps=steps)
    ref, dref = oracle.hydro_adaptive(st, dtdx, steps, fused=True)
    for v in range(4):
        assert np.array_equal(bits(outs[v]), bits(ref[v]))
    assert outs[4][0] == dref
    # configs[2]'s grid, 2 adaptive steps, against the fused CPU schedule
    big = lf.Plan.with_ranges("hydro2d_adaptive", (4096, 4096))
    st, dtdx = inputs.hydro_input(4096, 4096, seed=0)
    got = run_device(big, st, dtdx, 2)
    ref, dref = oracle.hydro_adaptive(st, dtdx, 2, fused=True)
    for v in range(4):
        assert np.array_equal(bits(got[v]), bits(ref[v])), v
    assert float(got[4]) == dref


@pytest.mark.parametrize("steps", [1, 2, 5])
def test_adaptive_host_path_pipelined(steps, monkeypatch):
    """lf_run_host with the copies overlapping the first and the last step's
    row parts (no wavefront: every step needs the previous one's whole-grid
    maximum); the driver zeroes each step's reduction slot and finalises the
    last."""
    monkeypatch.setenv("LF_HOST_PARTS", "5")
    shape = (60, 300)
    plan = lf.Plan.with_ranges("hydro2d_adaptive", shape)
    st, dtdx = inputs.hydro_input(*shape, seed=steps)
    outs = [np.full_like(st[0], np.nan) for _ in range(4)] + [np.zeros(1)]
    plan.run_host(st + [np.array([dtdx])] + outs, steps=steps)
    ref, dref = oracle.hydro_adaptive(st, dtdx, steps, fused=True)
    for v in range(4):
        assert np.array_equal(bits(outs[v]), bits(ref[v])), v
    assert outs[4][0] == dref


@pytest.mark.parametrize("shape,steps,share_dt", [((12, 20), 3, False), ((64, 256), 4, True), ((130, 254), 2, False),
                                                  ((257, 1000), 3, True)])
def test_adaptive_in_place(shape, steps, share_dt):
    """The adaptive chain in place (config.aliases for every iterate pair): the
    four state arrays on one buffer each; the dt/dx pair on one slot or two."""
    import torch
    plan = lf.Plan.with_ranges("hydro2d_adaptive", shape, inplace=True)
    assert plan.executor == "hydro2d_adaptive_fused_tma"
    st, dtdx = inputs.hydro_input(*shape, seed=shape[1] + 5)
    u = [torch.from_numpy(a).cuda() for a in st]
    d_in = torch.tensor(dtdx, dtype=torch.float64, device="cuda")
    d_out = d_in if share_dt else torch.zeros((), dtype=torch.float64, device="cuda")
    plan.run(u + [d_in] + u + [d_out], steps=steps)
    torch.cuda.synchronize()
    ref, dref = oracle.hydro_adaptive(st, dtdx, steps)
    for v in range(4):
        assert np.array_equal(bits(u[v].cpu().numpy()), bits(ref[v])), v
    assert float(d_out) == dref
    # through host buffers: one device buffer per state array
    h = [a.copy() for a in st]
    dh = np.array([dtdx])
    plan.run_host(h + [dh] + h + [dh if share_dt else np.zeros(1)], steps=steps)
    for v in range(4):
        assert np.array_equal(bits(h[v]), bits(ref[v])), v


def test_caller_driven_slab_steps_are_refused():
    """One step of a slab with the caller's own exchange cannot combine the
    per-step reduction across ranks: lf_run_slab refuses the chain."""
    import torch
    plan = lf.Plan.with_ranges("hydro2d_adaptive", (16, 64))
    bufs = [torch.zeros(t.extent or (), dtype=torch.float64, device="cuda") for t in plan.terminals]
    with pytest.raises(lf.LoomfuseError) as e:
        plan.run_slab(bufs, 0, 16, 16)
    assert e.value.code == lf.LF_ERR_UNSUPPORTED

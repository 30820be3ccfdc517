"""lf_run_host, pipelined (row parts: the first step computes part p while
part p+1 comes up, the last step sends part p down while part p+1 is computed;
one step overlaps both directions; multi-step runs of non-periodic chains as a
wavefront over (step, part)) -- bit-exact against the oracles, ghost rows
included, for single steps and for multi-step runs (2, 3 and 4 steps: the
ping-pong through the plan's scratch ends in the goals either way)."""
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


@pytest.fixture(params=["3", "7"])
def parts(request, monkeypatch):
    monkeypatch.setenv("LF_HOST_PARTS", request.param)
    return int(request.param)


def test_box(parts):
    plan = lf.Plan.with_ranges("box2x", (100, 256))
    img = inputs.box_input(100, 256, seed=1)
    out = np.full((100, 256), np.nan, np.float32)
    plan.run_host([img, out], steps=1)
    assert np.array_equal(bits(out), bits(oracle.box(img)))


def test_biharm(parts):
    plan = lf.Plan.with_ranges("biharmonic2d", (90, 256))
    u = inputs.biharm_input(90, 256, seed=2)
    out = np.full_like(u, np.nan)
    plan.run_host([u, out], steps=1)
    assert np.array_equal(bits(out), bits(oracle.biharm(u, 1)))


def test_heat3d(parts):
    plan = lf.Plan.with_ranges("heat3d", (20, 32, 128))
    u = inputs.heat3d_input(20, 32, 128, seed=3, sigma=4.0)
    out = np.full_like(u, np.nan)
    plan.run_host([u, out], steps=1)
    ref = oracle.heat3d(u, 1)
    assert np.array_equal(bits(out[1:-1, 1:-1, 1:-1]), bits(ref[1:-1, 1:-1, 1:-1]))
    # periodic ghost faces, including the k planes the first / last parts refill
    for ax in range(3):
        sl_g = [slice(1, -1)] * 3
        sl_s = [slice(1, -1)] * 3
        sl_g[ax], sl_s[ax] = 0, -2
        assert np.array_equal(bits(out[tuple(sl_g)]), bits(out[tuple(sl_s)]))


def test_hydro(parts):
    plan = lf.Plan.with_ranges("hydro2d", (64, 256))
    st, dtdx = inputs.hydro_input(64, 256, seed=4)
    outs = [np.full_like(st[0], np.nan) for _ in range(4)]
    plan.run_host(st + [np.array([dtdx])] + outs, steps=1)
    ref = oracle.hydro(st, dtdx, 1)
    for v in range(4):
        assert np.array_equal(bits(outs[v]), bits(ref[v])), v


def test_generic_executor(parts):
    spec = lf.set_ranges((SPECS / "heat3d_body.lf").read_text(), (24, 20, 50))
    path = SPECS / "_pipe_heat3d_body.lf"
    path.write_text(spec)
    try:
        plan = lf.Plan(spec, "p.lf")
        u = inputs.heat3d_input(24, 20, 50, seed=5, sigma=3.0)
        out = np.full_like(u, np.nan)
        plan.run_host([u, out], steps=1)
        ref = generic.run_naive(path, {"g_u": u}, steps=1)["g_unew"]
    finally:
        path.unlink()
    assert np.array_equal(bits(out), bits(ref))


@pytest.mark.parametrize("steps", [2, 3, 4])
def test_multistep_biharm_heat3d_hydro(parts, steps):
    plan = lf.Plan.with_ranges("biharmonic2d", (90, 256))
    u = inputs.biharm_input(90, 256, seed=12)
    out = np.full_like(u, np.nan)
    plan.run_host([u, out], steps=steps)
    assert np.array_equal(bits(out), bits(oracle.biharm(u, steps)))
    plan = lf.Plan.with_ranges("heat3d", (20, 32, 128))
    u = inputs.heat3d_input(20, 32, 128, seed=13, sigma=4.0)
    out = np.full_like(u, np.nan)
    plan.run_host([u, out], steps=steps)
    assert np.array_equal(bits(out), bits(oracle.heat3d(u, steps)))
    plan = lf.Plan.with_ranges("hydro2d", (64, 256))
    st, dtdx = inputs.hydro_input(64, 256, seed=14)
    outs = [np.full_like(st[0], np.nan) for _ in range(4)]
    plan.run_host(st + [np.array([dtdx])] + outs, steps=steps)
    ref = oracle.hydro(st, dtdx, steps)
    for v in range(4):
        assert np.array_equal(bits(outs[v]), bits(ref[v])), v


def test_multistep_generic_executor(parts):
    spec = lf.set_ranges((SPECS / "biharm_body.lf").read_text(), (60, 100))
    plan = lf.Plan(spec, "b.lf")
    assert plan.executor.startswith("jit_")
    u = inputs.biharm_input(60, 100, seed=15)
    out = np.full_like(u, np.nan)
    plan.run_host([u, out], steps=3)
    assert np.array_equal(bits(out), bits(oracle.biharm(u, 3)))


@pytest.mark.parametrize("wave", ["1", "0"])
def test_wavefront_over_steps_and_parts(wave, monkeypatch):
    """Multi-step runs of chains whose outer dimension does not wrap run as a
    wavefront over (step, part) -- part p of step s right after part p+1 of
    step s-1 -- with parts barely wider than the halo (the dependence reaches
    exactly the neighbouring parts) and many steps, so every ping-pong buffer
    is rewritten while neighbouring parts of the step before still read it.
    LF_HOST_WAVEFRONT=0: the first / last step pipelined only."""
    monkeypatch.setenv("LF_HOST_WAVEFRONT", wave)
    monkeypatch.setenv("LF_HOST_PARTS", "10")
    plan = lf.Plan.with_ranges("biharmonic2d", (30, 256))
    u = inputs.biharm_input(30, 256, seed=21)
    out = np.full_like(u, np.nan)
    plan.run_host([u, out], steps=9)
    assert np.array_equal(bits(out), bits(oracle.biharm(u, 9)))
    monkeypatch.setenv("LF_HOST_PARTS", "8")
    plan = lf.Plan.with_ranges("hydro2d", (24, 128))
    st, dtdx = inputs.hydro_input(24, 128, seed=22)
    outs = [np.full_like(st[0], np.nan) for _ in range(4)]
    plan.run_host(st + [np.array([dtdx])] + outs, steps=6)
    ref = oracle.hydro(st, dtdx, 6)
    for v in range(4):
        assert np.array_equal(bits(outs[v]), bits(ref[v])), v
    spec = lf.set_ranges((SPECS / "biharm_body.lf").read_text(), (40, 100))
    plan = lf.Plan(spec, "b.lf")
    u = inputs.biharm_input(40, 100, seed=23)
    out = np.full_like(u, np.nan)
    plan.run_host([u, out], steps=5)
    assert np.array_equal(bits(out), bits(oracle.biharm(u, 5)))


# (40, 300) in 4 parts for 9 steps: the row-band slots of a step are reused by the step 4 ahead
@pytest.mark.parametrize("shape,parts,steps", [((24, 128), 6, 6), ((40, 300), 10, 5), ((64, 1000), 7, 4),
                                               ((33, 254), 8, 3), ((40, 300), 4, 9), ((48, 130), 2, 12)])
def test_in_place_wavefront(shape, parts, steps, monkeypatch):
    """Hydro2D in place through lf_run_host (one device buffer per state array)
    as a wavefront over (step, part): a part's last two rows stay deferred until
    the next part's launch of the same step has read them.  Parts of four rows
    (two halos) up, segment cuts inside parts, several strips."""
    monkeypatch.setenv("LF_HOST_WAVEFRONT", "1")
    monkeypatch.setenv("LF_HOST_PARTS", str(parts))
    plan = lf.Plan.with_ranges("hydro2d", shape, inplace=True)
    assert plan.executor == "hydro2d_fused_tma"
    st, dtdx = inputs.hydro_input(*shape, seed=shape[0] + parts)
    u = [a.copy() for a in st]
    plan.run_host(u + [np.array([dtdx])] + u, steps=steps)
    ref = oracle.hydro(st, dtdx, steps)
    for v in range(4):
        assert np.array_equal(bits(u[v]), bits(ref[v])), (v, int(np.count_nonzero(u[v] != ref[v])))
    # parts thinner than two halos: the serial in-place path, same result
    monkeypatch.setenv("LF_HOST_PARTS", str(shape[0] // 2))
    u = [a.copy() for a in st]
    plan.run_host(u + [np.array([dtdx])] + u, steps=steps)
    for v in range(4):
        assert np.array_equal(bits(u[v]), bits(ref[v])), v

"""CPU oracle self-consistency: run_naive == HFAV fused CPU schedule, bit-exact
(R/SPEC.md:547, 553: run_schedule == run_naive), plus known-answer cases."""
import numpy as np
import pytest

import oracle
from paper_1710_08774_b200 import inputs


def bits_equal(a, b):
    return np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))


@pytest.mark.parametrize("nj,ni,steps,threads", [(8, 8, 1, 1), (16, 24, 3, 3), (33, 17, 2, 4), (64, 64, 5, 8)])
def test_biharm_naive_equals_fused(nj, ni, steps, threads):
    u = inputs.biharm_input(nj, ni, seed=nj * 131 + ni)
    a = oracle.biharm(u, steps)
    b = oracle.biharm(u, steps, fused=True, threads=threads)
    assert bits_equal(a, b)


def test_biharm_known_answer_single_spike():
    # lap(lap(delta)) is the 13-point biharmonic stencil 20,-8,2,1
    u = np.zeros((11 + 4, 11 + 4))
    u[2 + 5, 2 + 5] = 1.0
    out = oracle.biharm(u, 1)[2:-2, 2:-2]
    c = out[5, 5]
    assert c == pytest.approx(1.0 - 0.01 * 20.0, abs=0)
    assert out[5, 6] == pytest.approx(0.01 * 8.0, abs=1e-18)
    assert out[6, 6] == pytest.approx(-0.01 * 2.0, abs=1e-18)
    assert out[5, 7] == pytest.approx(-0.01 * 1.0, abs=1e-18)
    assert out[5, 8] == 0.0


def test_biharm_zero_halo_kept():
    u = inputs.biharm_input(12, 12, seed=3)
    out = oracle.biharm(u, 4)
    ring = out.copy()
    ring[2:-2, 2:-2] = 0
    assert not ring.any()


@pytest.mark.parametrize("shape,steps,threads", [((4, 4, 4), 1, 1), ((8, 16, 12), 3, 3), ((16, 8, 32), 2, 8)])
def test_heat3d_naive_equals_fused(shape, steps, threads):
    u = inputs.heat3d_input(*shape, seed=7, sigma=3.0)
    a = oracle.heat3d(u, steps)
    b = oracle.heat3d(u, steps, fused=True, threads=threads)
    assert bits_equal(a, b)


def test_heat3d_constant_is_fixed_point_and_mass_conserved():
    u = np.full((10, 10, 10), 0.375)
    out = oracle.heat3d(u, 3)
    assert np.all(out == 0.375)
    v = inputs.heat3d_input(8, 8, 8, seed=1, sigma=2.0)
    w = oracle.heat3d(v, 5)
    assert w[1:-1, 1:-1, 1:-1].sum() == pytest.approx(v[1:-1, 1:-1, 1:-1].sum(), rel=1e-13)


def test_heat3d_periodic_ghosts_refilled():
    v = inputs.heat3d_input(6, 6, 6, seed=2, sigma=2.0)
    w = oracle.heat3d(v, 2)
    ref = w.copy()
    inputs.fill_periodic(ref, 1)
    assert bits_equal(w, ref)


@pytest.mark.parametrize("nj,ni,threads", [(4, 4, 1), (16, 20, 3), (37, 64, 8)])
def test_box_naive_equals_fused(nj, ni, threads):
    img = inputs.box_input(nj, ni, seed=5)
    assert bits_equal(oracle.box(img), oracle.box(img, fused=True, threads=threads))


def test_box_known_answer_constant_and_ramp():
    img = np.full((9, 9), 3.0, dtype=np.float32)
    assert np.all(oracle.box(img) == 3.0)
    # separable box filter of a linear ramp is the ramp itself, away from edges
    x = np.arange(20 + 4, dtype=np.float32) * 3.0
    img = np.tile(x, (6 + 4, 1))
    out = oracle.box(img)
    assert np.allclose(out[:, 2:-2], x[4:-4], rtol=0, atol=1e-4)


def test_fault_injection_wrong_window_is_detected():
    # R/SPEC.md:557: a corrupted rolling window must be reported.  Reading the
    # lap1 window one row short is equivalent to feeding lap2 a shifted L.
    u = inputs.biharm_input(16, 16, seed=9)
    good = oracle.biharm(u, 1)
    shifted = np.roll(u, 1, axis=0)
    bad = oracle.biharm(shifted, 1)
    assert not bits_equal(good, bad)


@pytest.mark.parametrize("band", [(0, 10), (50, 70), (97, 128)])
def test_hydro_row_band_cone_equals_the_whole_grid(band):
    """The band check of tests/test_gpu_hydro_large.py: a strip of the band's
    rows plus 2 rows per step each side, cut from the initial state, advanced
    by the fused CPU schedule, reproduces the whole-grid run on the band's rows
    (ghost rows at the global faces included) bit for bit."""
    n, steps = 128, 2
    st, dtdx = inputs.hydro_input(n, 96, seed=5)
    whole = oracle.hydro(st, dtdx, steps, fused=True)
    a, b = band
    A, B = max(0, a - 2 * steps), min(n, b + 2 * steps)
    strip = [np.ascontiguousarray(x[A:B + 4]) for x in st]
    ref = oracle.hydro(strip, dtdx, steps, fused=True)
    lo = a + 2 - (2 if a == 0 else 0)
    hi = b + 2 + (2 if b == n else 0)
    for v in range(4):
        assert np.array_equal(whole[v][lo:hi].view(np.uint64), ref[v][lo - A:hi - A].view(np.uint64))


@pytest.mark.parametrize("nj,ni,steps,threads", [(8, 8, 1, 1), (16, 24, 3, 3), (33, 17, 2, 4)])
def test_hydro_adaptive_naive_equals_fused(nj, ni, steps, threads):
    st, dtdx = inputs.hydro_input(nj, ni, seed=nj + ni)
    a, da = oracle.hydro_adaptive(st, dtdx, steps)
    b, db = oracle.hydro_adaptive(st, dtdx, steps, fused=True, threads=threads)
    assert all(bits_equal(x, y) for x, y in zip(a, b)) and da == db
    # one adaptive step with the initial dt/dx is the fixed-dt step
    f = oracle.hydro(st, dtdx, 1)
    c, _ = oracle.hydro_adaptive(st, dtdx, 1)
    assert all(bits_equal(x, y) for x, y in zip(f, c))

"""Seeded input generator: counter-based splitmix64 and ghost conventions."""
import numpy as np

from paper_1710_08774_b200 import inputs

MASK = (1 << 64) - 1


def splitmix_ref(seed, n):
    z = (seed + (n + 1) * 0x9E3779B97F4A7C15) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    z ^= z >> 31
    return (z >> 11) * 2.0 ** -53


def test_uniform_matches_scalar_reference_and_chunks():
    for seed in (0, 1, 12345):
        u = inputs.uniform(1000, seed, chunk=77)
        assert all(u[n] == splitmix_ref(seed, n) for n in (0, 1, 2, 500, 999))
        assert np.array_equal(u[300:], inputs.uniform(700, seed, offset=300))
    u = inputs.uniform(100000)
    assert 0.0 <= u.min() and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.01


def test_ghost_fills():
    a = np.arange(36, dtype=np.float64).reshape(6, 6)
    inputs.fill_periodic(a, 1)
    assert a[0, 3] == a[4, 3] and a[5, 2] == a[1, 2] and a[3, 0] == a[3, 4]
    b = np.arange(64, dtype=np.float64).reshape(8, 8)
    inputs.fill_reflect(b, 2, odd_axes=(1,))
    assert b[3, 1] == -b[3, 2] and b[3, 0] == -b[3, 3] and b[1, 4] == b[2, 4] and b[0, 4] == b[3, 4]
    c = np.arange(64, dtype=np.float32).reshape(8, 8)
    inputs.fill_clamp(c, 2)
    assert c[0, 0] == c[2, 2] and c[7, 5] == c[5, 5]


def test_hydro_initial_state():
    st, dtdx = inputs.hydro_input(8, 16)
    rho = st[0][2:-2, 2:-2]
    assert np.all(np.abs(rho[:, :8] - 1.0) <= 1e-3) and np.all(np.abs(rho[:, 8:] - 0.125) <= 1e-3)
    assert not st[1].any() and not st[2].any()
    assert 0.0 < dtdx < 0.5

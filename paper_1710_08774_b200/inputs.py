"""Seeded synthetic inputs for the BASELINE.json configs (host side).

Counter-based splitmix64: element n of stream `seed` is
``mix(seed + (n+1) * 0x9E3779B97F4A7C15)`` and ``u = (z >> 11) * 2**-53`` in
[0, 1) -- R/SPEC.md:617 (seed defaults to 0).  Values are generated once on
the host and handed to both the GPU path and the CPU oracle, so the RNG never
needs a device twin.  Every array is laid out exactly as the planner sizes the
terminal (buffer_extents, storage.cpp:403-427): interior plus ghost cells,
ghosts filled by the config's boundary convention.

The public benchmarks of the paper (COSMO, Hydro2D) are not in the image; these
generators stand in with the shapes and value distributions BASELINE.json gives.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
GAMMA = 1.4


def uniform(n: int, seed: int = 0, offset: int = 0, chunk: int = 1 << 24) -> np.ndarray:
    """n doubles in [0,1) from the counter-based splitmix64 stream `seed`."""
    out = np.empty(n, dtype=np.float64)
    s = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        for a in range(0, n, chunk):
            b = min(n, a + chunk)
            z = np.arange(offset + a + 1, offset + b + 1, dtype=np.uint64) * GOLDEN + s
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            z = z ^ (z >> np.uint64(31))
            out[a:b] = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return out


# ---------------------------------------------------------------- ghost fills
def fill_zero(a: np.ndarray, h: int) -> np.ndarray:
    for ax in range(a.ndim):
        sl = [slice(None)] * a.ndim
        sl[ax] = slice(0, h)
        a[tuple(sl)] = 0
        sl[ax] = slice(a.shape[ax] - h, a.shape[ax])
        a[tuple(sl)] = 0
    return a


def fill_periodic(a: np.ndarray, h: int) -> np.ndarray:
    """Wrap ghosts of width h along every axis (innermost first, so edges and
    corners come out as the composition of the per-axis wraps)."""
    for ax in reversed(range(a.ndim)):
        n = a.shape[ax] - 2 * h
        src_lo = [slice(None)] * a.ndim
        dst_lo = [slice(None)] * a.ndim
        src_lo[ax] = slice(n, n + h)
        dst_lo[ax] = slice(0, h)
        a[tuple(dst_lo)] = a[tuple(src_lo)]
        src_hi = [slice(None)] * a.ndim
        dst_hi = [slice(None)] * a.ndim
        src_hi[ax] = slice(h, 2 * h)
        dst_hi[ax] = slice(n + h, n + 2 * h)
        a[tuple(dst_hi)] = a[tuple(src_hi)]
    return a


def fill_reflect(a: np.ndarray, h: int, odd_axes: tuple[int, ...] = ()) -> np.ndarray:
    """Mirror ghosts (cell -1 <- 0, -2 <- 1, ...), negated along odd_axes."""
    for ax in reversed(range(a.ndim)):
        n = a.shape[ax] - 2 * h
        sign = -1.0 if ax in odd_axes else 1.0
        for g in range(h):
            dst = [slice(None)] * a.ndim
            src = [slice(None)] * a.ndim
            dst[ax] = h - 1 - g
            src[ax] = h + g
            a[tuple(dst)] = sign * a[tuple(src)]
            dst[ax] = n + h + g
            src[ax] = n + h - 1 - g
            a[tuple(dst)] = sign * a[tuple(src)]
    return a


def fill_clamp(a: np.ndarray, h: int) -> np.ndarray:
    for ax in reversed(range(a.ndim)):
        n = a.shape[ax] - 2 * h
        for g in range(h):
            dst = [slice(None)] * a.ndim
            src = [slice(None)] * a.ndim
            dst[ax] = g
            src[ax] = h
            a[tuple(dst)] = a[tuple(src)]
            dst[ax] = n + h + g
            src[ax] = n + h - 1
            a[tuple(dst)] = a[tuple(src)]
    return a


# ---------------------------------------------------------------- configs
def biharm_input(nj: int, ni: int, seed: int = 0) -> np.ndarray:
    """configs[0]: u ~ U[0,1) interior, zero halo of 2 -> (nj+4, ni+4) fp64."""
    a = np.zeros((nj + 4, ni + 4), dtype=np.float64)
    a[2:-2, 2:-2] = uniform(nj * ni, seed).reshape(nj, ni)
    return a


def heat3d_input(nk: int, nj: int, ni: int, seed: int = 0, sigma: float = 32.0) -> np.ndarray:
    """configs[1]: u = U[0,1) + exp(-r^2/(2 sigma^2)) about the centre cell,
    periodic halo of 1 -> (nk+2, nj+2, ni+2) fp64.  Bump amplitude 1 is a
    pinned choice (BASELINE.json gives none)."""
    a = np.empty((nk + 2, nj + 2, ni + 2), dtype=np.float64)
    ck, cj, ci = nk // 2, nj // 2, ni // 2
    di2 = (np.arange(ni, dtype=np.float64) - ci) ** 2
    dj2 = (np.arange(nj, dtype=np.float64) - cj) ** 2
    inv = 1.0 / (2.0 * sigma * sigma)
    for k in range(nk):
        u = uniform(nj * ni, seed, offset=k * nj * ni).reshape(nj, ni)
        r2 = (float(k - ck) ** 2 + dj2)[:, None] + di2[None, :]
        a[k + 1, 1:-1, 1:-1] = u + np.exp(-r2 * inv)
    return fill_periodic(a, 1)


def box_input(nj: int, ni: int, seed: int = 0) -> np.ndarray:
    """configs[3]: img = float(255 u), replicate-padded by 2 -> (nj+4, ni+4) fp32."""
    a = np.empty((nj + 4, ni + 4), dtype=np.float32)
    a[2:-2, 2:-2] = (255.0 * uniform(nj * ni, seed)).astype(np.float32).reshape(nj, ni)
    return fill_clamp(a, 2)


def hydro_input(nj: int, ni: int, seed: int = 0):
    """configs[2]/[4]: Sod-like split at x = 0.5 with density perturbations
    U[-1e-3, 1e-3), zero velocity, E = p/(gamma-1); reflective ghosts of 2.
    Returns ([rho, rhou, rhov, E] each (nj+4, ni+4) fp64, dtdx) with dt fixed
    from CFL 0.5 on the initial state: dt/dx = 0.5 / max(|u| + c)."""
    x_left = (np.arange(ni) + 0.5) / ni < 0.5
    delta = (2.0 * uniform(nj * ni, seed) - 1.0).reshape(nj, ni) * 1e-3
    rho0 = np.where(x_left, 1.0, 0.125)[None, :] + delta
    p0 = np.broadcast_to(np.where(x_left, 1.0, 0.1)[None, :], (nj, ni))
    st = [np.zeros((nj + 4, ni + 4), dtype=np.float64) for _ in range(4)]
    st[0][2:-2, 2:-2] = rho0
    st[3][2:-2, 2:-2] = p0 / (GAMMA - 1.0)
    fill_reflect(st[0], 2)
    fill_reflect(st[1], 2, odd_axes=(1,))
    fill_reflect(st[2], 2, odd_axes=(0,))
    fill_reflect(st[3], 2)
    c = np.sqrt(GAMMA * p0 / rho0)
    smax = float(np.max(c))  # |u| = 0 initially
    dtdx = 0.5 / smax
    return st, dtdx


# ---------------------------------------------------------------- slabs
def heat3d_planes(nk: int, nj: int, ni: int, k0: int, k1: int, seed: int = 0, sigma: float = 32.0) -> np.ndarray:
    """Storage planes [k0, k1) of heat3d_input(nk, nj, ni) (logical k0-1 .. k1-2),
    generated without building the whole grid: what one slab rank needs."""
    out = np.empty((k1 - k0, nj + 2, ni + 2), dtype=np.float64)
    ck, cj, ci = nk // 2, nj // 2, ni // 2
    di2 = (np.arange(ni, dtype=np.float64) - ci) ** 2
    dj2 = (np.arange(nj, dtype=np.float64) - cj) ** 2
    inv = 1.0 / (2.0 * sigma * sigma)
    for s in range(k0, k1):
        k = (s - 1) % nk  # periodic: storage plane s holds logical plane s-1
        u = uniform(nj * ni, seed, offset=k * nj * ni).reshape(nj, ni)
        r2 = (float(k - ck) ** 2 + dj2)[:, None] + di2[None, :]
        plane = out[s - k0]
        plane[1:-1, 1:-1] = u + np.exp(-r2 * inv)
        fill_periodic(plane, 1)
    return out


def hydro_rows(nj: int, ni: int, r0: int, r1: int, seed: int = 0):
    """Logical rows [r0, r1) (-2 <= r0 < r1 <= nj+2) of hydro_input's four
    state arrays, each (r1-r0, ni+4), without building the whole grid, plus
    this block's max(|u| + c) for the global dt (combine with a MAX reduce)."""
    lo, hi = max(0, r0), min(nj, r1)
    x_left = (np.arange(ni) + 0.5) / ni < 0.5
    delta = (2.0 * uniform((hi - lo) * ni, seed, offset=lo * ni) - 1.0).reshape(hi - lo, ni) * 1e-3
    rho0 = np.where(x_left, 1.0, 0.125)[None, :] + delta
    p0 = np.broadcast_to(np.where(x_left, 1.0, 0.1)[None, :], (hi - lo, ni))
    smax = float(np.max(np.sqrt(GAMMA * p0 / rho0))) if hi > lo else 0.0
    inner = [np.zeros((hi - lo, ni + 4)) for _ in range(4)]
    inner[0][:, 2:-2] = rho0
    inner[3][:, 2:-2] = p0 / (GAMMA - 1.0)
    for a, odd_i in zip(inner, (False, True, False, False)):
        for g in range(2):  # reflective ghost columns
            s = -1.0 if odd_i else 1.0
            a[:, 1 - g] = s * a[:, 2 + g]
            a[:, ni + 2 + g] = s * a[:, ni + 1 - g]
    out = [np.empty((r1 - r0, ni + 4)) for _ in range(4)]
    for v, odd_j in enumerate((False, False, True, False)):
        for r in range(r0, r1):
            src = r if 0 <= r < nj else (-1 - r if r < 0 else 2 * nj - 1 - r)  # mirrored row
            row = inner[v][src - lo]
            out[v][r - r0] = -row if (odd_j and src != r) else row
    return out, smax

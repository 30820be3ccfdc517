"""CPU ORACLE -- test infrastructure only (see oracle.h).

ctypes wrappers around liblforacle.so (run_naive and the HFAV-style fused CPU
schedule) and around the reference-planner driver oracle/_ref/refplan.
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess
from pathlib import Path

import numpy as np

DIR = Path(__file__).resolve().parent
LIB = DIR / "liblforacle.so"
REFPLAN = DIR / "_ref" / "refplan"
REFERENCE = Path("/root/reference/proj")

_libs: dict = {}
NATIVE_DIR = DIR / "_native"


def build(ref: bool = True) -> None:
    """make the oracle .so (and, where /root/reference exists, _ref/refplan)."""
    subprocess.run(["make", "-s", "-C", str(DIR), "liblforacle.so"], check=True)
    if ref and REFERENCE.exists():
        subprocess.run(["make", "-s", "-C", str(DIR), "ref"], check=True)


def native_build() -> Path:
    """The same sources built with -march=native for THIS host (the CPU
    baseline of bench.py); built on first use on the
    machine that runs it, under oracle/_native/ (git-ignored)."""
    out = NATIVE_DIR / "liblforacle_native.so"
    if not out.exists():
        NATIVE_DIR.mkdir(exist_ok=True)
        srcs = sorted(str(p) for p in DIR.glob("*.c") if p.name != "div3check.c")
        tmp = out.with_suffix(f".{os.getpid()}.tmp")
        subprocess.run(["gcc", "-O3", "-march=native", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
                        "-std=c11", "-shared", "-o", str(tmp), *srcs, "-lm"], check=True, cwd=str(DIR))
        os.replace(tmp, out)
    return out


def lib(native: bool = False) -> ctypes.CDLL:
    """liblforacle.so (x86-64-v3, the parity checker) or, with native=True,
    the -march=native build timed as the CPU baseline."""
    if native not in _libs:
        if native:
            path = native_build()
        else:
            if not LIB.exists():
                build(ref=False)
            path = LIB
        L = ctypes.CDLL(str(path))
        D, F, I, Lg = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_long
        L.lfo_biharm_naive.argtypes = [D, D, Lg, Lg, I]
        L.lfo_biharm_fused.argtypes = [D, D, Lg, Lg, I, I]
        L.lfo_heat3d_naive.argtypes = [D, D, Lg, Lg, Lg, I]
        L.lfo_heat3d_fused.argtypes = [D, D, Lg, Lg, Lg, I, I]
        L.lfo_biharm_fused_step.argtypes = [D, D, Lg, Lg, I]
        L.lfo_heat3d_fused_step.argtypes = [D, D, Lg, Lg, Lg, I]
        L.lfo_box_naive.argtypes = [F, F, Lg, Lg]
        L.lfo_box_fused.argtypes = [F, F, Lg, Lg, I]
        if hasattr(L, "lfo_hydro_naive"):
            PP = ctypes.POINTER(ctypes.c_void_p)
            L.lfo_hydro_naive.argtypes = [PP, PP, Lg, Lg, ctypes.c_double, I]
            L.lfo_hydro_fused.argtypes = [PP, PP, Lg, Lg, ctypes.c_double, I, I]
            L.lfo_hydro_fused_step.argtypes = [PP, PP, Lg, Lg, ctypes.c_double, I]
            L.lfo_hydro_adaptive.argtypes = [PP, PP, Lg, Lg, ctypes.POINTER(ctypes.c_double), I, I, I]
        _libs[native] = L
    return _libs[native]


def max_threads() -> int:
    return lib().lfo_max_threads()


def _p(a: np.ndarray) -> int:
    assert a.flags.c_contiguous
    return a.ctypes.data


def _ok(code: int) -> None:
    if code != 0:
        raise RuntimeError(f"oracle failed with status {code}")


# ---- config 1 -----------------------------------------------------------------
def biharm(u: np.ndarray, steps: int, fused: bool = False, threads: int = 0, native: bool = False) -> np.ndarray:
    nj, ni = u.shape[0] - 4, u.shape[1] - 4
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    if fused:
        _ok(lib(native).lfo_biharm_fused(_p(u), _p(out), nj, ni, steps, threads))
    else:
        _ok(lib(native).lfo_biharm_naive(_p(u), _p(out), nj, ni, steps))
    return out


def biharm_step(u: np.ndarray, out: np.ndarray, threads: int = 0, native: bool = False) -> None:
    """One fused CPU step in -> out with no copies (the CPU-baseline unit)."""
    _ok(lib(native).lfo_biharm_fused_step(_p(u), _p(out), u.shape[0] - 4, u.shape[1] - 4, threads))


# ---- config 2 -----------------------------------------------------------------
def heat3d(u: np.ndarray, steps: int, fused: bool = False, threads: int = 0, native: bool = False) -> np.ndarray:
    nk, nj, ni = (s - 2 for s in u.shape)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    if fused:
        _ok(lib(native).lfo_heat3d_fused(_p(u), _p(out), nk, nj, ni, steps, threads))
    else:
        _ok(lib(native).lfo_heat3d_naive(_p(u), _p(out), nk, nj, ni, steps))
    return out


def heat3d_step(u: np.ndarray, out: np.ndarray, threads: int = 0, native: bool = False) -> None:
    """One fused CPU step in -> out with no copies (the CPU-baseline unit)."""
    nk, nj, ni = (s - 2 for s in u.shape)
    _ok(lib(native).lfo_heat3d_fused_step(_p(u), _p(out), nk, nj, ni, threads))


# ---- config 4 -----------------------------------------------------------------
def box(img: np.ndarray, fused: bool = False, threads: int = 0, native: bool = False) -> np.ndarray:
    nj, ni = img.shape[0] - 4, img.shape[1] - 4
    img = np.ascontiguousarray(img, dtype=np.float32)
    out = np.empty((nj, ni), dtype=np.float32)
    if fused:
        _ok(lib(native).lfo_box_fused(_p(img), _p(out), nj, ni, threads))
    else:
        _ok(lib(native).lfo_box_naive(_p(img), _p(out), nj, ni))
    return out


# ---- configs 3/5 --------------------------------------------------------------
def hydro(state, dtdx: float, steps: int, fused: bool = False, threads: int = 0, native: bool = False):
    nj, ni = state[0].shape[0] - 4, state[0].shape[1] - 4
    ins = [np.ascontiguousarray(a, dtype=np.float64) for a in state]
    outs = [np.empty_like(a) for a in ins]
    PA = ctypes.c_void_p * 4
    pin, pout = PA(*[_p(a) for a in ins]), PA(*[_p(a) for a in outs])
    if fused:
        _ok(lib(native).lfo_hydro_fused(pin, pout, nj, ni, dtdx, steps, threads))
    else:
        _ok(lib(native).lfo_hydro_naive(pin, pout, nj, ni, dtdx, steps))
    return outs


def hydro_adaptive(state, dtdx: float, steps: int, fused: bool = False, threads: int = 0):
    """`steps` steps with the CFL time step (specs/hydro2d_adaptive.lf): returns
    (state after the last step, the dt/dx that state gives)."""
    nj, ni = state[0].shape[0] - 4, state[0].shape[1] - 4
    ins = [np.ascontiguousarray(a, dtype=np.float64) for a in state]
    outs = [np.empty_like(a) for a in ins]
    PA = ctypes.c_void_p * 4
    d = ctypes.c_double(dtdx)
    _ok(lib().lfo_hydro_adaptive(PA(*[_p(a) for a in ins]), PA(*[_p(a) for a in outs]), nj, ni, ctypes.byref(d),
                                 steps, 1 if fused else 0, threads))
    return outs, d.value


def hydro_step(state, outs, dtdx: float, threads: int = 0, native: bool = False) -> None:
    """One fused CPU step in -> out with no copies (the CPU-baseline unit)."""
    nj, ni = state[0].shape[0] - 4, state[0].shape[1] - 4
    PA = ctypes.c_void_p * 4
    _ok(lib(native).lfo_hydro_fused_step(PA(*[_p(a) for a in state]), PA(*[_p(a) for a in outs]), nj, ni, dtdx,
                                   threads))



# ---- reference planner (bookkeeping oracle) -------------------------------------
def ref_plan(spec_path: str | os.PathLike) -> dict:
    """The reference's own planner verdict on a rule file (oracle/_ref/refplan)."""
    if not REFPLAN.exists():
        if REFERENCE.exists():
            build(ref=True)
        else:
            raise FileNotFoundError(f"{REFPLAN} not built and /root/reference is absent")
    r = subprocess.run([str(REFPLAN), str(spec_path)], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"refplan failed ({r.returncode}): {r.stderr}")
    return json.loads(r.stdout)

"""loomfuse-b200: B200-native fused stencil-chain executor.

Python mirror of the C ABI in ``include/loomfuse_b200.h``.  The interface is
the reference's: a `.lf` rule file (kernels / globals / config, R/SPEC.md:88)
planned once (``Plan``), then the emitted per-goal-set function
(R/SPEC.md:500) -- here ``Plan.run`` on device buffers or ``Plan.run_host``
on host arrays, terminals ordered axioms then goals.

The compute path is the sm_100a library ``libloomfuse_b200.so`` built in-tree
by ``paper_1710_08774_b200.build``; there is no CPU fallback -- importing the
package without the library raises.
"""
from __future__ import annotations

import ctypes
import json
import re
from dataclasses import dataclass
from pathlib import Path
from typing import Any, Sequence

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libloomfuse_b200.so"
SPEC_DIR = PKG_DIR / "specs"

LF_OK = 0
LF_ERR_SPEC = 1
LF_ERR_MISMATCH = 2
LF_ERR_INTERNAL = 3
LF_ERR_CUDA = 4
LF_ERR_UNSUPPORTED = 5
LF_MAX_DIMS = 4

#: every symbol the header declares (checked by tests/test_abi.py)
ABI_SYMBOLS = (
    "lf_plan_create", "lf_plan_create_ex", "lf_plan_destroy", "lf_plan_num_terminals", "lf_plan_terminal",
    "lf_plan_report", "lf_plan_executor", "lf_run", "lf_run_host", "lf_run_slab",
    "lf_plan_launches_per_step", "lf_plan_compulsory_bytes_per_cell", "lf_plan_grid_passes", "lf_plan_launches",
    "lf_last_error",
    "lf_version", "lf_spec_print", "lf_plan_source",
    "lf_run_slabs", "lf_run_slabs_local", "lf_nccl_unique_id", "lf_nccl_comm_init_rank",
    "lf_nccl_comm_init_single", "lf_nccl_comm_destroy", "lf_set_option",
)


class LoomfuseError(RuntimeError):
    """A non-zero status from the C ABI; ``code`` is the LF_* status."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[{code}] {message}")
        self.code = code


class _Terminal(ctypes.Structure):
    _fields_ = [
        ("name", ctypes.c_char * 64),
        ("type", ctypes.c_char * 32),
        ("is_goal", ctypes.c_int32),
        ("elem_bytes", ctypes.c_int32),
        ("ndim", ctypes.c_int32),
        ("loop_dim", ctypes.c_int32 * LF_MAX_DIMS),
        ("extent", ctypes.c_int64 * LF_MAX_DIMS),
        ("base", ctypes.c_int64 * LF_MAX_DIMS),
        ("bytes", ctypes.c_int64),
    ]


class _Slab(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_int64), ("hi", ctypes.c_int64), ("global_", ctypes.c_int64),
                ("part_lo", ctypes.c_int64), ("part_hi", ctypes.c_int64)]


_lib: ctypes.CDLL | None = None


def lib() -> ctypes.CDLL:
    """Load the in-tree sm_100a library (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: run `python -m paper_1710_08774_b200.build` "
            "(there is no CPU fallback for the fused executor)")
    L = ctypes.CDLL(str(LIB_PATH))
    P = ctypes.c_void_p
    L.lf_plan_create.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p, ctypes.POINTER(P)]
    L.lf_plan_create_ex.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p, ctypes.c_char_p,
                                    ctypes.c_size_t, ctypes.POINTER(P)]
    L.lf_spec_print.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p, ctypes.c_char_p,
                                ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
    L.lf_set_option.argtypes = [ctypes.c_char_p, ctypes.c_char_p]
    L.lf_plan_destroy.argtypes = [P]
    L.lf_plan_destroy.restype = None
    L.lf_plan_num_terminals.argtypes = [P]
    L.lf_plan_terminal.argtypes = [P, ctypes.c_int, ctypes.POINTER(_Terminal)]
    L.lf_plan_report.argtypes = [P, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
    L.lf_plan_executor.argtypes = [P]
    L.lf_plan_executor.restype = ctypes.c_char_p
    L.lf_plan_source.argtypes = [P]
    L.lf_plan_source.restype = ctypes.c_char_p
    L.lf_run.argtypes = [P, ctypes.POINTER(P), ctypes.c_int, ctypes.c_int, P]
    L.lf_run_host.argtypes = [P, ctypes.POINTER(P), ctypes.c_int, ctypes.c_int]
    L.lf_run_slab.argtypes = [P, ctypes.POINTER(P), ctypes.c_int, ctypes.POINTER(_Slab), P]
    L.lf_run_slabs.argtypes = [P, P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(P), ctypes.c_int, ctypes.c_int, P]
    L.lf_run_slabs_local.argtypes = [P, ctypes.c_int, ctypes.POINTER(P), ctypes.c_int, ctypes.c_int, P]
    L.lf_nccl_unique_id.argtypes = [ctypes.c_char_p]
    L.lf_nccl_comm_init_rank.argtypes = [ctypes.POINTER(P), ctypes.c_int, ctypes.c_char_p, ctypes.c_int]
    L.lf_nccl_comm_init_single.argtypes = [ctypes.POINTER(P)]
    L.lf_nccl_comm_destroy.argtypes = [P]
    L.lf_plan_launches_per_step.argtypes = [P]
    L.lf_plan_compulsory_bytes_per_cell.argtypes = [P]
    L.lf_plan_compulsory_bytes_per_cell.restype = ctypes.c_double
    L.lf_plan_grid_passes.argtypes = [P, ctypes.c_int]
    L.lf_plan_launches.argtypes = [P, ctypes.c_int]
    L.lf_last_error.restype = ctypes.c_char_p
    L.lf_version.restype = ctypes.c_char_p
    _lib = L
    return L


def _check(code: int) -> None:
    if code != LF_OK:
        raise LoomfuseError(code, lib().lf_last_error().decode(errors="replace"))


_NP_DTYPES = {("double", 8): np.float64, ("float", 4): np.float32}


@dataclass(frozen=True)
class Terminal:
    """One terminal buffer as sized by the reference's buffer_extents."""
    name: str
    type: str
    is_goal: bool
    elem_bytes: int
    loop_dims: tuple[int, ...]
    extent: tuple[int, ...]
    base: tuple[int, ...]
    bytes: int

    @property
    def dtype(self) -> np.dtype:
        for (t, b), dt in _NP_DTYPES.items():
            if t in self.type and b == self.elem_bytes:
                return np.dtype(dt)
        raise TypeError(f"no numpy dtype for terminal type {self.type!r}")


def _ptr(x: Any) -> int:
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    if isinstance(x, np.ndarray):
        if not x.flags.c_contiguous:
            raise ValueError("host arrays must be C-contiguous")
        return int(x.ctypes.data)
    raise TypeError(f"cannot take a buffer pointer from {type(x).__name__}")


def spec_path(name: str) -> Path:
    """Path of a bundled rule file (``heat3d``, ``biharmonic2d``, ...)."""
    p = SPEC_DIR / (name if name.endswith(".lf") else name + ".lf")
    if not p.exists():
        raise FileNotFoundError(p)
    return p


class Plan:
    """A planned rule file (lf_plan_create) -- immutable, reusable."""

    def __init__(self, text: str, filename: str = "<input>", kernel_source: str | None = None):
        """`kernel_source`: CUDA C defining the `declaration:` functions of a
        chain that has no built-in executor (lf_plan_create_ex)."""
        L = lib()
        h = ctypes.c_void_p()
        raw = text.encode()
        ks = kernel_source.encode() if kernel_source else None
        _check(L.lf_plan_create_ex(raw, len(raw), filename.encode(), ks, len(ks) if ks else 0, ctypes.byref(h)))
        self._h = h
        self.filename = filename
        self.terminals: list[Terminal] = []
        for i in range(L.lf_plan_num_terminals(h)):
            t = _Terminal()
            _check(L.lf_plan_terminal(h, i, ctypes.byref(t)))
            n = t.ndim
            self.terminals.append(Terminal(
                t.name.decode(), t.type.decode(), bool(t.is_goal), t.elem_bytes,
                tuple(t.loop_dim[:n]), tuple(t.extent[:n]), tuple(t.base[:n]), t.bytes))

    @classmethod
    def from_file(cls, path: str | Path, kernel_source: str | None = None) -> "Plan":
        p = Path(path)
        return cls(p.read_text(), str(p), kernel_source)

    @classmethod
    def bundled(cls, name: str) -> "Plan":
        return cls.from_file(spec_path(name))

    @classmethod
    def with_ranges(cls, name: str, sizes: Sequence[int], inplace: bool = False) -> "Plan":
        """A bundled spec with its `ranges:` replaced by [0, n) per loop dim;
        `inplace` also declares every iterate pair in `config.aliases`."""
        text = set_ranges(spec_path(name).read_text(), sizes)
        return cls(alias_iterates(text) if inplace else text, str(spec_path(name)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.lf_plan_destroy(h)
            self._h = None

    # ---- introspection ---------------------------------------------------
    def report(self) -> dict:
        L = lib()
        need = ctypes.c_size_t()
        _check(L.lf_plan_report(self._h, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        _check(L.lf_plan_report(self._h, buf, need.value, None))
        return json.loads(buf.value.decode())

    @property
    def executor(self) -> str:
        return lib().lf_plan_executor(self._h).decode()

    @property
    def source(self) -> str:
        """CUDA source of the generic executor ("" for hand-written executors)."""
        return lib().lf_plan_source(self._h).decode()

    @property
    def launches_per_step(self) -> int:
        return lib().lf_plan_launches_per_step(self._h)

    @property
    def compulsory_bytes_per_cell(self) -> float:
        return lib().lf_plan_compulsory_bytes_per_cell(self._h)

    def grid_passes(self, steps: int) -> int:
        """passes over the grid lf_run makes for `steps` steps (whole domain)"""
        return lib().lf_plan_grid_passes(self._h, steps)

    def launches(self, steps: int) -> int:
        """kernel launches lf_run issues for `steps` steps (whole domain)"""
        return lib().lf_plan_launches(self._h, steps)

    @property
    def axioms(self) -> list[Terminal]:
        return [t for t in self.terminals if not t.is_goal]

    @property
    def goals(self) -> list[Terminal]:
        return [t for t in self.terminals if t.is_goal]

    # ---- execution -----------------------------------------------------------
    @property
    def outer_trips(self) -> int:
        """Trips of the outermost loop dimension (the one slabs split)."""
        if not hasattr(self, "_outer"):
            lo, hi, stride = self.report()["ranges"][0]
            self._outer = (hi - lo) // stride
        return self._outer

    def _ptrs(self, bufs: Sequence[Any], device: bool = True, rows: tuple[int, int, int] | None = None):
        """Pointer array of the terminal buffers, axioms then goals.  Tensors
        and arrays are checked against the terminal they stand for: C-contiguous,
        its element size, exactly its bytes (a slab's rows (lo, hi) of an n0-row
        outer dimension when `rows` is given), and -- for the device entry
        points -- a CUDA tensor on the current device.  Raw integer pointers
        are passed through unchecked."""
        if len(bufs) != len(self.terminals):
            raise ValueError(f"expected {len(self.terminals)} buffers (axioms then goals), got {len(bufs)}")
        for i, (b, t) in enumerate(zip(bufs, self.terminals)):
            if isinstance(b, int):
                continue
            want = t.bytes
            if rows is not None and t.extent:
                lo, hi, n0 = rows
                want = int(np.prod(self.slab_terminal_extent(i, lo, hi, n0))) * t.elem_bytes
            if hasattr(b, "data_ptr"):  # torch tensor
                if device:
                    import torch
                    if not b.is_cuda:
                        raise ValueError(f"{t.name}: expected a CUDA tensor, got one on {b.device}")
                    if b.device.index != torch.cuda.current_device():
                        raise ValueError(f"{t.name}: expected a CUDA tensor on the current device "
                                         f"{torch.cuda.current_device()}, got one on {b.device}")
                if not b.is_contiguous():
                    raise ValueError(f"{t.name}: tensor must be contiguous")
                size, nbytes = b.element_size(), b.numel() * b.element_size()
            elif isinstance(b, np.ndarray):
                if device:
                    raise ValueError(f"{t.name}: a host array passed to a device entry point (use run_host)")
                if not b.flags.c_contiguous:
                    raise ValueError(f"{t.name}: host arrays must be C-contiguous")
                size, nbytes = b.itemsize, b.nbytes
            else:
                raise TypeError(f"{t.name}: cannot take a buffer pointer from {type(b).__name__}")
            if size != t.elem_bytes:
                raise ValueError(f"{t.name}: element size {size} B, the terminal's type {t.type!r} is {t.elem_bytes} B")
            if nbytes != want:
                raise ValueError(f"{t.name}: expected {want} bytes, got {nbytes}")
        arr = (ctypes.c_void_p * len(bufs))(*[_ptr(b) for b in bufs])
        return arr

    def run(self, bufs: Sequence[Any], steps: int = 1, stream: Any = None) -> None:
        """Device buffers (torch tensors or raw pointers), stream-ordered."""
        s = _stream_handle(stream)
        _check(lib().lf_run(self._h, self._ptrs(bufs), len(bufs), steps, s))

    def run_host(self, arrays: Sequence[np.ndarray], steps: int = 1) -> None:
        """Host arrays in, goals written back (the emitted function's contract)."""
        _check(lib().lf_run_host(self._h, self._ptrs(arrays, device=False), len(arrays), steps))

    def run_slab(self, bufs: Sequence[Any], lo: int, hi: int, global_: int, stream: Any = None,
                 part: tuple[int, int] | None = None) -> None:
        """One step on rows [lo, hi) of the outer dimension (slab-local buffers);
        `part` = slab-local rows to compute (default: all)."""
        p0, p1 = part if part is not None else (0, 0)
        slab = _Slab(lo, hi, global_, p0, p1)
        _check(lib().lf_run_slab(self._h, self._ptrs(bufs, rows=(lo, hi, global_)), len(bufs), ctypes.byref(slab),
                                 _stream_handle(stream)))

    def run_slabs(self, bufs: Sequence[Any], comm: "NcclComm", steps: int = 1, stream: Any = None) -> None:
        """This rank's slab for `steps` steps, NCCL halo exchange inside (see run_slabs)."""
        run_slabs(self, bufs, comm, steps, stream)

    def slab_terminal_extent(self, idx: int, lo: int, hi: int, n0: int) -> tuple[int, ...]:
        """Extent of terminal `idx` for a slab of rows [lo, hi) of an outer
        dimension of n0 rows: the planner's halo with hi-lo rows."""
        t = self.terminals[idx]
        if not t.extent:
            return ()
        return (t.extent[0] - n0 + (hi - lo),) + tuple(t.extent[1:])


class NcclComm:
    """An NCCL communicator for ``Plan.run_slabs`` (one rank per GPU).

    ``NcclComm.single()`` makes a one-rank communicator on the current device;
    ``NcclComm.from_group(rank, world)`` creates one rank of a ``world``-rank
    communicator, the unique id broadcast from rank 0 over the default
    ``torch.distributed`` group (the plumbing only: the exchange itself is
    issued by the library)."""

    def __init__(self, handle: int, rank: int, world: int):
        self.handle, self.rank, self.world = handle, rank, world

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(lib().lf_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def init_rank(cls, world: int, uid: bytes, rank: int) -> "NcclComm":
        h = ctypes.c_void_p()
        _check(lib().lf_nccl_comm_init_rank(ctypes.byref(h), world, uid, rank))
        return cls(h.value, rank, world)

    @classmethod
    def single(cls) -> "NcclComm":
        h = ctypes.c_void_p()
        _check(lib().lf_nccl_comm_init_single(ctypes.byref(h)))
        return cls(h.value, 0, 1)

    @classmethod
    def from_group(cls, rank: int, world: int) -> "NcclComm":
        import torch.distributed as dist
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls.init_rank(world, obj[0], rank)

    def destroy(self) -> None:
        if self.handle:
            _check(lib().lf_nccl_comm_destroy(self.handle))
            self.handle = None


def run_slabs(plan: "Plan", bufs: Sequence[Any], comm: NcclComm, steps: int = 1, stream: Any = None) -> None:
    """``steps`` steps of this rank's slab (lf_run_slabs): rows
    [n*rank/world, n*(rank+1)/world) of the outer dimension, buffers sized for
    the slab, faces exchanged with the neighbours by NCCL overlapped with the
    interior rows, the final state in the goal buffers."""
    n0 = plan.outer_trips
    lo, hi = n0 * comm.rank // comm.world, n0 * (comm.rank + 1) // comm.world
    _check(lib().lf_run_slabs(plan._h, comm.handle, comm.rank, comm.world, plan._ptrs(bufs, rows=(lo, hi, n0)),
                              len(bufs), steps,
                              _stream_handle(stream)))


def run_slabs_local(plan: "Plan", rank_bufs: Sequence[Sequence[Any]], steps: int = 1, stream: Any = None) -> None:
    """All ranks of a slab decomposition on the current GPU, the exchange as
    device copies (lf_run_slabs_local): the same schedule and halo geometry as
    ``run_slabs``, testable on one GPU."""
    nterm = len(plan.terminals)
    if any(len(b) != nterm for b in rank_bufs):
        raise ValueError(f"expected {nterm} buffers per rank (axioms then goals)")
    n0, world = plan.outer_trips, len(rank_bufs)
    if world <= n0:  # (more ranks than rows: the library reports LF_ERR_SPEC)
        for r, bufs in enumerate(rank_bufs):
            plan._ptrs(bufs, rows=(n0 * r // world, n0 * (r + 1) // world, n0))  # validation only
    flat = [_ptr(b) for bufs in rank_bufs for b in bufs]
    arr = (ctypes.c_void_p * len(flat))(*flat)
    _check(lib().lf_run_slabs_local(plan._h, len(rank_bufs), arr, nterm, steps,
                                    _stream_handle(stream)))


def set_option(name: str, value: "str | int | None") -> None:
    """Set a tuning / A-B switch (an LF_* name) in this process,
    overriding the environment variable of that name; None drops the
    override.  Switches take effect where they are read: plan creation or the
    next run.  No switch changes results."""
    _check(lib().lf_set_option(name.encode(), None if value is None else str(value).encode()))


class option:
    """Context manager: `with lf.option("LF_JIT_RM", 0): plan = lf.Plan(...)`."""

    def __init__(self, name: str, value: "str | int | None"):
        self.name, self.value = name, value

    def __enter__(self):
        set_option(self.name, self.value)
        return self

    def __exit__(self, *exc):
        set_option(self.name, None)


def print_spec(text: str, filename: str = "<input>") -> str:
    """Canonical text of a rule file (lf_spec_print; round-trips through parse)."""
    L = lib()
    raw = text.encode()
    need = ctypes.c_size_t()
    _check(L.lf_spec_print(raw, len(raw), filename.encode(), None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(L.lf_spec_print(raw, len(raw), filename.encode(), buf, need.value, None))
    return buf.value.decode()


def _stream_handle(stream: Any):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    if hasattr(stream, "cuda_stream"):
        return int(stream.cuda_stream)
    raise TypeError("stream must be a torch.cuda.Stream, an int handle or None")


def set_ranges(text: str, sizes: Sequence[int]) -> str:
    """Rewrite the `ranges:` block of a rule file to [0, n) per loop-order dim."""
    lines = text.splitlines()
    out, i = [], 0
    order = None
    for ln in lines:
        s = ln.strip()
        if s.startswith("loop-order:"):
            order = [v.strip() for v in s.split(":", 1)[1].strip().strip("[]").split(",")]
    if order is None or len(order) != len(sizes):
        raise ValueError("sizes must match the spec's loop-order")
    while i < len(lines):
        ln = lines[i]
        out.append(ln)
        if ln.strip() == "ranges:":
            ind = len(ln) - len(ln.lstrip()) + 2
            i += 1
            while i < len(lines) and (len(lines[i]) - len(lines[i].lstrip())) >= ind and lines[i].strip():
                i += 1
            for v, n in zip(order, sizes):
                out.append(" " * ind + f"{v}: [0, {int(n)}]")
            continue
        i += 1
    return "\n".join(out) + "\n"


def alias_iterates(text: str) -> str:
    """Declare every `iterate: [[goal, axiom], ...]` pair of a rule file as an
    in-place alias (`aliases: [[axiom, goal], ...]`, the reference's
    config.aliases): goal and axiom may then be passed on one buffer."""
    out = []
    for ln in text.splitlines():
        s = ln.strip()
        if s.startswith("aliases:"):
            raise ValueError("the spec already declares aliases")
        out.append(ln)
        if s.startswith("iterate:"):
            value = s.split(":", 1)[1].strip()
            pairs = re.findall(r"\[\s*([^\[\],\s]+)\s*,\s*([^\[\],\s]+)\s*\]", value)
            if not pairs or re.sub(r"\[\s*[^\[\],\s]+\s*,\s*[^\[\],\s]+\s*\]|[\s,]", "", value) != "[]":
                raise ValueError("iterate: must be a flow sequence of [goal, axiom] pairs on one line")
            ind = ln[:len(ln) - len(ln.lstrip())]
            out.append(ind + "aliases: [" + ", ".join(f"[{a.strip()}, {g.strip()}]" for g, a in pairs) + "]")
    return "\n".join(out) + "\n"


__all__ = ["Plan", "Terminal", "LoomfuseError", "lib", "spec_path", "set_ranges", "alias_iterates", "print_spec", "ABI_SYMBOLS",
           "set_option", "option"]

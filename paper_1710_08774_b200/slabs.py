"""Multi-GPU slab decomposition of a fused chain.

One process per GPU (torchrun), the outermost loop dimension split into
contiguous slabs.  Each step: the fused executor advances the slab
(``Plan.run_slab``: interior plus the ghosts it can refill locally), then the
slab faces are exchanged with the neighbouring ranks by point-to-point
send/recv -- NCCL over NVLink on GPUs, gloo on CPU for the tests.  The halo is
the planner's terminal halo along the slab dimension (``Plan.report()``
halo_lo/halo_hi), e.g. one plane for the 3D heat chain and two rows for the
2D chains.  Periodic boundaries close the ring (rank 0 <-> rank P-1).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import torch
import torch.distributed as dist


def slab_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [lo, hi) of an n-row outer dimension owned by `rank` (balanced)."""
    return n * rank // world, n * (rank + 1) // world


@dataclass
class Halo:
    lo: int        # ghost rows below the slab
    hi: int        # ghost rows above the slab
    periodic: bool


def exchange(bufs: Sequence[torch.Tensor], halo: Halo, rank: int, world: int, group=None) -> None:
    """Fill the slab-dimension ghost rows of every buffer from the neighbours.

    Each buffer is [halo.lo + n_local + halo.hi, ...] along dim 0.  The last
    `halo.lo` interior rows go up to rank+1 (its lower ghosts), the first
    `halo.hi` interior rows go down to rank-1 (its upper ghosts).  With two
    ranks on a periodic ring both faces talk to the same peer; sends and
    receives are issued in one fixed order (send-up, send-down / recv-down,
    recv-up) so they pair off correctly.
    """
    for b in bufs:
        n = b.shape[0] - halo.lo - halo.hi
        if n < max(halo.lo, halo.hi):
            raise ValueError(f"a slab of {n} row(s) is thinner than the {max(halo.lo, halo.hi)}-row halo "
                             "exchanged with each neighbour (use fewer ranks)")
    if world == 1:
        if halo.periodic:
            for b in bufs:
                n = b.shape[0] - halo.lo - halo.hi
                b[:halo.lo].copy_(b[n:n + halo.lo])
                b[halo.lo + n:].copy_(b[halo.lo:halo.lo + halo.hi])
        return
    up = rank + 1 if rank + 1 < world else (0 if halo.periodic else None)
    down = rank - 1 if rank > 0 else (world - 1 if halo.periodic else None)
    # dim-0 row blocks of a contiguous buffer are contiguous: send from and
    # receive into the buffers directly (no staging copies)
    ops = []
    for b in bufs:
        n = b.shape[0] - halo.lo - halo.hi
        if up is not None and halo.lo:
            ops.append(dist.P2POp(dist.isend, b[n:n + halo.lo], up, group))
        if down is not None and halo.hi:
            ops.append(dist.P2POp(dist.isend, b[halo.lo:halo.lo + halo.hi], down, group))
    for b in bufs:
        n = b.shape[0] - halo.lo - halo.hi
        if down is not None and halo.lo:
            ops.append(dist.P2POp(dist.irecv, b[:halo.lo], down, group))
        if up is not None and halo.hi:
            ops.append(dist.P2POp(dist.irecv, b[halo.lo + n:], up, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()


def run_slabs(step: Callable[[Sequence[torch.Tensor], Sequence[torch.Tensor]], None],
              state: Sequence[torch.Tensor], scratch: Sequence[torch.Tensor], steps: int,
              halo: Halo, rank: int, world: int, group=None) -> Sequence[torch.Tensor]:
    """Advance `steps` steps: step(src, dst) on the local slab, then exchange
    dst's faces; src/dst ping-pong.  Returns the buffers holding the result."""
    src, dst = list(state), list(scratch)
    for _ in range(steps):
        step(src, dst)
        exchange(dst, halo, rank, world, group)
        src, dst = dst, src
    return src


def run_slabs_overlapped(launch: Callable[[Sequence[torch.Tensor], Sequence[torch.Tensor], tuple[int, int]], None],
                         state: Sequence[torch.Tensor], scratch: Sequence[torch.Tensor], steps: int, halo: Halo,
                         rank: int, world: int, rows: int, group=None,
                         comm_stream: "torch.cuda.Stream | None" = None) -> Sequence[torch.Tensor]:
    """Like run_slabs, with the face exchange overlapped with the interior.

    Each step: launch(src, dst, part) computes the slab-local output rows the
    neighbours need first -- [0, halo.hi) and [rows-halo.lo, rows) -- then the
    exchange of those rows runs on `comm_stream` while the interior rows
    [halo.hi, rows-halo.lo) are computed on the current stream; the next step
    starts once both are done.  Falls back to the sequential schedule on CPU
    tensors or when the slab is too thin to have an interior."""
    src, dst = list(state), list(scratch)
    cuda = src[0].is_cuda
    inner_lo, inner_hi = halo.hi, rows - halo.lo
    if not cuda or inner_hi - inner_lo < 1:
        return run_slabs(lambda s, d: launch(s, d, (0, rows)), state, scratch, steps, halo, rank, world, group)
    main = torch.cuda.current_stream()
    comm = comm_stream or torch.cuda.Stream(device=src[0].device, priority=-1)
    for _ in range(steps):
        if halo.hi:
            launch(src, dst, (0, halo.hi))
        if halo.lo:
            launch(src, dst, (rows - halo.lo, rows))
        comm.wait_stream(main)
        with torch.cuda.stream(comm):
            exchange(dst, halo, rank, world, group)
        launch(src, dst, (inner_lo, inner_hi))
        main.wait_stream(comm)
        src, dst = dst, src
    return src

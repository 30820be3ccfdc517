"""Tuning probe (not part of the bench contract): per-step cost of the
multi-GPU slab schedule (lf_run_slabs: face launches, NCCL exchange on a side
stream, interior) against the plain single-domain run, on one GPU with a
one-rank communicator.  Run it on a grid 1/N of the bench grid along the
outer dimension to see the per-step overhead one rank of an N-GPU run pays.
usage: python tools/slab_probe.py <spec> <steps> <n0> <n1> [n2]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1710_08774_b200 as lf  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    spec, steps, sizes = sys.argv[1], int(sys.argv[2]), tuple(int(x) for x in sys.argv[3:])
    plan = lf.Plan.with_ranges(spec, sizes)
    bufs = []
    for t in plan.axioms + plan.goals:
        shape = tuple(int(e) for e in t.extent) or (1,)
        bufs.append(torch.rand(shape, dtype=torch.float64 if t.elem_bytes == 8 else torch.float32, device="cuda"))
    if spec == "hydro2d":
        for b in bufs[:4]:
            b.add_(1.0)
        bufs[1].mul_(0.01)
        bufs[2].mul_(0.01)
        bufs[4].fill_(0.01)
    comm = lf.NcclComm.single()
    stream = torch.cuda.current_stream()
    plain = timed(lambda: plan.run(bufs, steps=steps))
    slabs = timed(lambda: lf.run_slabs(plan, bufs, comm, steps=steps, stream=stream))
    print(f"{spec} {sizes} x{steps} [{plan.executor}]: plain {plain / steps * 1e3:.1f} us/step, "
          f"slab schedule {slabs / steps * 1e3:.1f} us/step (+{(slabs - plain) / steps * 1e3:.1f} us, "
          f"efficiency {plain / slabs:.3f})")
    comm.destroy()


if __name__ == "__main__":
    main()

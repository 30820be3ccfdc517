"""Tuning probe (not part of the bench contract): the same aliased chain run
out of place (two buffers) and in place (one buffer), CUDA events.
usage: python tools/inplace_probe.py <examples spec> <steps> <n0> [n1 [n2]]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1710_08774_b200 as lf  # noqa: E402


def rate(plan, bufs, steps, cells):
    for _ in range(2):
        plan.run(bufs, steps=steps)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        plan.run(bufs, steps=steps)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 3
    return ms / steps * 1e3, cells * steps / ms * 1e-6


def main():
    spec, steps, sizes = sys.argv[1], int(sys.argv[2]), tuple(int(x) for x in sys.argv[3:])
    plan = lf.Plan(lf.set_ranges((lf.SPEC_DIR / "examples" / f"{spec}.lf").read_text(), sizes), f"{spec}.lf")
    (ax,), (goal,) = plan.axioms, plan.goals
    u = torch.rand(tuple(ax.extent), dtype=torch.float64, device="cuda")
    v = torch.rand(tuple(goal.extent), dtype=torch.float64, device="cuda")
    cells = float(np.prod(sizes))
    for name, bufs in (("out of place", [u, v]), ("in place", [u, u])):
        us, g = rate(plan, bufs, steps, cells)
        print(f"{spec} {sizes} x{steps} {name}: {us:.1f} us/step, {g:.1f} G/s")


if __name__ == "__main__":
    main()

"""Tuning probe (not part of the bench contract): device rate of a bundled
chain at arbitrary sizes / step counts, CUDA events on the launching stream.
usage: python tools/rate_probe.py <spec> <steps> <n0> [n1 [n2]]  (env vars select variants)"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1710_08774_b200 as lf  # noqa: E402


def main():
    spec, steps, sizes = sys.argv[1], int(sys.argv[2]), tuple(int(x) for x in sys.argv[3:])
    plan = lf.Plan.with_ranges(spec, sizes)
    bufs = []
    for t in plan.axioms + plan.goals:
        shape = tuple(int(e) for e in t.extent) or (1,)
        bufs.append(torch.rand(shape, dtype=torch.float64 if t.elem_bytes == 8 else torch.float32, device="cuda"))
    if spec == "hydro2d":  # positive density / energy, small dt
        for b in bufs[:4]:
            b.add_(1.0)
        bufs[1].mul_(0.01)
        bufs[2].mul_(0.01)
        bufs[4].fill_(0.01)
    for _ in range(2):
        plan.run(bufs, steps=steps)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    s.record()
    for _ in range(reps):
        plan.run(bufs, steps=steps)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    cells = float(np.prod(sizes)) * steps
    print(f"{spec} {sizes} x{steps} [{plan.executor}]: {ms / steps * 1e3:.1f} us/step, {cells / ms * 1e-6:.1f} G/s")


if __name__ == "__main__":
    main()

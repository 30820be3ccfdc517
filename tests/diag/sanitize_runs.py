"""One small run of every mbarrier / TMA pipeline, for compute-sanitizer
(racecheck, synccheck, memcheck): the four hand-written executors and the
generic executor's register march (2D, out of place and in place), its
warp-specialised march (3D) and its plain march.  Each run is compared with
the CPU oracle, so a tool that perturbs timing cannot hide a wrong result.

    compute-sanitizer --tool racecheck python tests/diag/sanitize_runs.py
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import oracle  # noqa: E402  (the checker)
import paper_1710_08774_b200 as lf  # noqa: E402
from paper_1710_08774_b200 import inputs  # noqa: E402


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def check(name, got, ref):
    ok = np.array_equal(bits(got), bits(ref))
    print(f"{name}: {'bit-exact' if ok else 'MISMATCH'}", flush=True)
    return ok


def main():
    ok = True
    dev = torch.device("cuda", 0)
    # heat3d_fused_tma
    shape, steps = (8, 16, 64), 2
    plan = lf.Plan.with_ranges("heat3d", shape)
    u = inputs.heat3d_input(*shape, seed=1, sigma=3.0)
    d, o = torch.from_numpy(u).to(dev), torch.empty(u.shape, dtype=torch.float64, device=dev)
    plan.run([d, o], steps=steps)
    ok &= check(plan.executor, o.cpu().numpy()[1:-1, 1:-1, 1:-1], oracle.heat3d(u, steps)[1:-1, 1:-1, 1:-1])
    # biharm2d_fused_tma
    shape = (24, 128)
    plan = lf.Plan.with_ranges("biharmonic2d", shape)
    u = inputs.biharm_input(*shape, seed=2)
    d, o = torch.from_numpy(u).to(dev), torch.empty(u.shape, dtype=torch.float64, device=dev)
    plan.run([d, o], steps=2)
    ok &= check(plan.executor, o.cpu().numpy(), oracle.biharm(u, 2))
    # box2x_fused_tma
    shape = (16, 256)
    plan = lf.Plan.with_ranges("box2x", shape)
    img = inputs.box_input(*shape, seed=3)
    d = torch.from_numpy(img).to(dev)
    o = torch.empty(tuple(plan.terminals[1].extent), dtype=torch.float32, device=dev)
    plan.run([d, o])
    ok &= check(plan.executor, o.cpu().numpy(), oracle.box(img))
    # hydro2d_fused_tma
    shape = (12, 128)
    plan = lf.Plan.with_ranges("hydro2d", shape)
    st, dtdx = inputs.hydro_input(*shape, seed=4)
    ax = [torch.from_numpy(a).to(dev) for a in st] + [torch.tensor([dtdx], dtype=torch.float64, device=dev)]
    goals = [torch.empty_like(ax[0]) for _ in range(4)]
    plan.run(ax + goals, steps=1)
    ref = oracle.hydro(st, dtdx, 1)
    ok &= all([check(f"{plan.executor}[{v}]", goals[v].cpu().numpy(), ref[v]) for v in range(4)])
    # generic executor: register march (2D), in place, warp-specialised (3D)
    for name, shape, steps, inplace in (("biharm_body", (40, 600), 2, False), ("box_body", (20, 1100), 1, False),
                                        ("biharm_inplace", (70, 1000), 2, True), ("heat3d_body", (6, 20, 70), 2, False)):
        spec = lf.set_ranges((lf.SPEC_DIR / "examples" / f"{name}.lf").read_text(), shape)
        plan = lf.Plan(spec, f"{name}.lf")
        src = plan.source
        kind = "rm" if "lf_jit_step_rm(" in src else ("ws" if "lf_jit_step_ws(" in src else "plain")
        if name.startswith("box"):
            x = inputs.box_input(*shape, seed=5)
            ref = oracle.box(x)
        elif len(shape) == 3:
            x = inputs.heat3d_input(*shape, seed=5, sigma=3.0)
            ref = oracle.heat3d(x, steps)
        else:
            x = inputs.biharm_input(*shape, seed=5)
            ref = oracle.biharm(x, steps)
        d = torch.from_numpy(x).to(dev)
        if inplace:
            plan.run([d, d], steps=steps)
            got = d
        else:
            got = torch.empty(tuple(plan.goals[0].extent), dtype=d.dtype, device=dev)
            plan.run([d, got], steps=steps)
        g = got.cpu().numpy()
        if len(shape) == 3:
            g, ref = g[1:-1, 1:-1, 1:-1], ref[1:-1, 1:-1, 1:-1]
        ok &= check(f"{plan.executor}/{kind} {name}{' in place' if inplace else ''}", g, ref)
    torch.cuda.synchronize()
    print("all bit-exact" if ok else "MISMATCHES", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

"""Fuzz-chain diagnostics on the GPU: for each seed, the generic executor's
result vs the generic run_naive; prints the mismatching rows/columns."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from test_gpu_jit_fuzz import random_chain  # noqa: E402
from oracle import generic  # noqa: E402
import paper_1710_08774_b200 as lf  # noqa: E402

seeds = [int(s) for s in sys.argv[1:]] or range(48)
for seed in seeds:
    text = random_chain(seed)
    path = Path(f"/tmp/fuzz{seed}.lf")
    path.write_text(text)
    plan = lf.Plan(text, path.name)
    (ax,) = plan.axioms
    x = np.random.default_rng(seed).random(ax.extent).astype(ax.dtype)
    dx = torch.from_numpy(x).cuda()
    (goal,) = plan.goals
    dz = torch.full(goal.extent, float("nan"), dtype=dx.dtype, device="cuda")
    plan.run([dx, dz], steps=1)
    torch.cuda.synchronize()
    ref = generic.run_naive(path, {ax.name: x}, steps=1)[goal.name]
    got = dz.cpu().numpy()
    view = np.uint64 if got.dtype == np.float64 else np.uint32
    bad = got.view(view) != np.ascontiguousarray(ref).view(view)
    rm = "lf_jit_step_rm(" in plan.source
    if bad.any():
        idx = np.argwhere(bad)
        print(f"seed {seed} rm={rm} shape={got.shape} dtype={got.dtype}: {bad.sum()} bad; rows {sorted(set(idx[:, 0].tolist()))[:40]} "
              f"cols {sorted(set(idx[:, -1].tolist()))[:40]} nan={np.isnan(got[bad]).sum()}")
    else:
        print(f"seed {seed} rm={rm} ok")

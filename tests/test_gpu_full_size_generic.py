"""The generic executor at the BASELINE sizes: the `body:` forms of the chains
(register march in 2D, warp-specialised march in 3D), out of place and in
place, against the hand-written executors on the same inputs, bit for bit.
The hand-written executors are pinned to the CPU oracle at these sizes by
their own tests (test_gpu_{biharm,box,heat3d}.py), so equality here carries
the oracle's verdict over to the generic kernels -- including the deferred
in-place writes, whose bands and commit only engage on grids of many units."""
import numpy as np
import pytest

import paper_1710_08774_b200 as lf
from paper_1710_08774_b200 import inputs

pytestmark = pytest.mark.gpu


def bits(t):
    a = t.cpu().numpy()
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def _body_plan(name, sizes):
    return lf.Plan(lf.set_ranges((lf.SPEC_DIR / "examples" / f"{name}.lf").read_text(), sizes), f"{name}.lf")


def _run(plan, x, steps, inplace=False):
    import torch
    d = torch.from_numpy(x).cuda()
    if inplace:
        plan.run([d, d], steps=steps)
        torch.cuda.synchronize()
        return d
    out = torch.empty(tuple(plan.goals[0].extent), dtype=d.dtype, device="cuda")
    plan.run([d, out], steps=steps)
    torch.cuda.synchronize()
    return out


def test_biharm_4096_register_march_and_in_place_match_hand_written():
    sizes, steps = (4096, 4096), 3
    u = inputs.biharm_input(*sizes, seed=31)
    ref = _run(lf.Plan.with_ranges("biharmonic2d", sizes), u, steps)
    gen = _body_plan("biharm_body", sizes)
    assert "lf_jit_step_rm(" in gen.source
    assert np.array_equal(bits(_run(gen, u, steps)), bits(ref))
    ip = _body_plan("biharm_inplace", sizes)
    assert "lf_jit_commit_rm(" in ip.source
    assert np.array_equal(bits(_run(ip, u, steps, inplace=True)), bits(ref))


def test_box_16384_register_march_matches_hand_written():
    sizes = (16384, 16384)
    img = inputs.box_input(*sizes, seed=32)
    ref = _run(lf.Plan.with_ranges("box2x", sizes), img, 1)
    gen = _body_plan("box_body", sizes)
    assert "lf_jit_step_rm(" in gen.source
    assert np.array_equal(bits(_run(gen, img, 1)), bits(ref))


def test_heat3d_512_warp_specialised_and_in_place_match_hand_written():
    sizes, steps = (512, 512, 512), 2
    u = inputs.heat3d_input(*sizes, seed=33)
    inner = (slice(1, -1),) * 3
    ref = _run(lf.Plan.with_ranges("heat3d", sizes), u, steps)[inner]
    gen = _body_plan("heat3d_body", sizes)
    assert np.array_equal(bits(_run(gen, u, steps)[inner]), bits(ref))
    ip = _body_plan("heat3d_inplace", sizes)
    assert "lf_jit_commit_ws(" in ip.source
    assert np.array_equal(bits(_run(ip, u, steps, inplace=True)[inner]), bits(ref))

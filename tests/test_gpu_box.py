"""sm_100a fused box-filter executor vs the CPU oracle, bit-exact (config 4)."""
import numpy as np
import pytest

import oracle
import paper_1710_08774_b200 as lf
from paper_1710_08774_b200 import inputs

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def run_device(plan, img):
    import torch
    d = torch.from_numpy(img).cuda()
    out = torch.full(plan.terminals[1].extent, float("nan"), dtype=torch.float32, device="cuda")
    plan.run([d, out])
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("shape", [(1, 128), (4, 128), (16, 128), (37, 256), (100, 384), (257, 640)])
def test_device_path_matches_naive(shape):
    plan = lf.Plan.with_ranges("box2x", shape)
    assert plan.executor == "box2x_fused_tma"
    img = inputs.box_input(*shape, seed=shape[0])
    assert np.array_equal(bits(run_device(plan, img)), bits(oracle.box(img)))


def test_host_path():
    shape = (64, 256)
    plan = lf.Plan.with_ranges("box2x", shape)
    img = inputs.box_input(*shape, seed=2)
    out = np.zeros(shape, np.float32)
    plan.run_host([img, out])
    assert np.array_equal(bits(out), bits(oracle.box(img)))


def test_full_size_16384_matches_fused_cpu():
    plan = lf.Plan.bundled("box2x")
    img = inputs.box_input(16384, 16384, seed=0)
    got = run_device(plan, img)
    ref = oracle.box(img, fused=True)
    assert np.array_equal(bits(got), bits(ref))
    # a box filter never leaves the input's value range
    assert got.min() >= img.min() and got.max() <= img.max()

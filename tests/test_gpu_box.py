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


@pytest.mark.parametrize("kind", ["negative", "special", "patches"])
def test_special_values_take_the_exact_path(kind):
    """The executor's packed fast path runs only on rows of non-negative
    floats below 2^126; negative values, -0, +inf, denormals and huge values
    must still come out bit-identical to the user kernel's x / 3.0f."""
    shape = (96, 384)
    rng = np.random.default_rng(11)
    img = inputs.box_input(*shape, seed=3)
    if kind == "negative":
        img -= 128.0
    elif kind == "special":
        cells = rng.integers(0, img.size, 400)
        vals = np.array([-0.0, np.inf, 1e-45, -1e-45, 3e38, 1.2e-38, -7.5], np.float32)
        img.reshape(-1)[cells] = vals[rng.integers(0, len(vals), cells.size)]
    else:  # isolated bad rows among good ones: fast/exact switching mid-strip
        for j in (0, 5, 6, 40, 41, 42, 43, 90):
            img[j, rng.integers(0, img.shape[1], 3)] = -0.0
        img[60, 7] = np.float32(2.0 ** 126)
    plan = lf.Plan.with_ranges("box2x", shape)
    assert np.array_equal(bits(run_device(plan, img)), bits(oracle.box(img)))

"""Generic NVRTC-compiled executor (jit_tiled_fused) vs the generic run_naive
over the reference's own inference DAG, bit-exact."""
import numpy as np
import pytest

import oracle
from oracle import generic
import paper_1710_08774_b200 as lf
from paper_1710_08774_b200 import inputs

pytestmark = pytest.mark.gpu
SPECS = lf.PKG_DIR.parent / "tests" / "specs"


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def run_device(plan, axioms, steps):
    import torch
    ax = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in axioms]
    dt = {8: torch.float64, 4: torch.float32}
    goals = [torch.full(t.extent, float("nan"), dtype=dt[t.elem_bytes], device="cuda") for t in plan.goals]
    plan.run(ax + goals, steps=steps)
    torch.cuda.synchronize()
    return [g.cpu().numpy() for g in goals]


def _div_operands(shape, seed):
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal(shape) * 10.0 ** rng.uniform(-44, 37, size=shape)).astype(np.float32)
    x.flat[::7] = 0.0
    x.flat[3::11] = -0.0
    return x


CASES = {
    "biharm_body": lambda: {"g_u": inputs.biharm_input(40, 72, seed=5)},
    "heat3d_body": lambda: {"g_u": inputs.heat3d_input(9, 12, 40, seed=6, sigma=3.0)},
    "box_body": lambda: {"g_img": inputs.box_input(33, 70, seed=7)},
    "multi_body": lambda: {"g_x": np.random.default_rng(1).random((21, 52)), "g_scale": np.array([0.75])},
    "laplace3_body": lambda: {"g_x": np.random.default_rng(2).random(1002)},
    # divisions by literals, strength-reduced (powers of two, fp32 / 3): magnitudes
    # across the float range incl. zeros, signed zeros and subnormal results
    "divs_body": lambda: {"g_x": _div_operands((31, 85), seed=8)},
    # multi-nest plans: reductions (inner and outer dim) and broadcast splits
    "normalization_body": lambda: {"g_q": np.random.default_rng(3).random((37, 151)),
                                   "g_zero": np.random.default_rng(4).random(37) * 0.1},
    "colsum_body": lambda: {"g_u": np.random.default_rng(5).random((47, 72)), "g_z": np.zeros(70),
                            "g_k": np.array([0.3])},
    # a full reduction to a scalar (both loop dims, loop order) and its broadcast
    "meansub_body": lambda: {"g_u": np.random.default_rng(7).random((23, 57)), "g_z": np.array([0.0]),
                             "g_inv": np.array([1.0 / (23 * 57)])},
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("steps", [1, 3])
def test_jit_matches_generic_oracle(name, steps):
    plan = lf.Plan.from_file(SPECS / f"{name}.lf")
    assert plan.executor.startswith("jit_")
    if steps > 1 and name not in ("biharm_body", "heat3d_body"):
        pytest.skip("chain has no iterate pairs")
    ax = CASES[name]()
    got = run_device(plan, [ax[t.name] for t in plan.axioms], steps)
    ref = generic.run_naive(SPECS / f"{name}.lf", ax, steps=steps)
    for g, t in zip(got, plan.goals):
        assert np.array_equal(bits(g), bits(ref[t.name])), t.name


def test_jit_host_path_and_large_grid():
    spec = lf.set_ranges((SPECS / "biharm_body.lf").read_text(), (300, 1000))
    plan = lf.Plan(spec, "big.lf")
    u = inputs.biharm_input(300, 1000, seed=9)
    out = np.zeros_like(u)
    plan.run_host([u, out], steps=2)
    assert np.array_equal(bits(out), bits(oracle.biharm(u, 2)))


def test_jit_slab_parts_compose():
    import torch
    plan = lf.Plan.from_file(SPECS / "heat3d_body.lf")
    u = torch.from_numpy(inputs.heat3d_input(9, 12, 40, seed=6, sigma=3.0)).cuda()
    whole, parts = torch.zeros_like(u), torch.zeros_like(u)
    plan.run_slab([u, whole], 0, 9, 9)
    for part in [(0, 1), (8, 9), (1, 8)]:
        plan.run_slab([u, parts], 0, 9, 9, part=part)
    torch.cuda.synchronize()
    assert torch.equal(whole[1:-1], parts[1:-1])


@pytest.mark.parametrize("name,shape,steps,chunk,knob", [
    ("biharm_inplace", (300, 1000), 3, None, ""),
    ("biharm_inplace", (300, 1000), 2, "24", ""),
    ("biharm_inplace", (130, 2100), 2, "16", ""),
    ("biharm_inplace", (300, 1000), 2, "24", "LF_JIT_RM=0"),
    ("heat3d_inplace", (20, 40, 130), 3, None, ""),
    ("heat3d_inplace", (20, 40, 130), 2, "5", ""),
    ("heat3d_inplace", (23, 70, 200), 2, "4", ""),
    ("heat3d_inplace", (20, 40, 130), 2, "5", "LF_JIT_WS=0"),
])
def test_inplace_matches_out_of_place_oracle(name, shape, steps, chunk, knob, monkeypatch):
    """config.aliases + one buffer for axiom and goal: the generic executor
    runs in place and must equal the out-of-place run_naive bit for bit, ghost
    ring included.  2D chains run on the register march and 3D chains on the
    warp-specialised march, both deferring the boundary writes other units
    still read to bands committed after the step; LF_JIT_RM=0 / LF_JIT_WS=0
    keep the plain march's band loader (bands captured before the step)."""
    import torch
    if knob:
        monkeypatch.setenv(*knob.split("="))
    if chunk:
        monkeypatch.setenv("LF_JIT_CHUNK", chunk)  # many row chunks -> many row bands
    spec = lf.set_ranges((SPECS / f"{name}.lf").read_text(), shape)
    plan = lf.Plan(spec, f"{name}.lf")
    assert plan.executor == "jit_window_fused"
    deferred = "lf_jit_commit_rm(" if len(shape) == 2 else "lf_jit_commit_ws("
    assert (deferred in plan.source) == (not knob)
    if len(shape) == 2:
        u0 = inputs.biharm_input(*shape, seed=8)
    else:
        u0 = inputs.heat3d_input(*shape, seed=8, sigma=4.0)
    u = torch.from_numpy(u0.copy()).cuda()
    plan.run([u, u], steps=steps)
    torch.cuda.synchronize()
    path = SPECS / f"_tmp_{name}_{'x'.join(map(str, shape))}.lf"
    path.write_text(spec)
    try:
        ref = generic.run_naive(path, {"g_u": u0}, steps=steps)["g_unew"]
    finally:
        path.unlink()
    assert np.array_equal(bits(u.cpu().numpy()), bits(ref))


def test_shared_buffers_need_declared_aliases_and_the_generic_executor():
    import torch
    # generic executor, aliases not declared
    p = lf.Plan.from_file(SPECS / "biharm_body.lf")
    u = torch.from_numpy(inputs.biharm_input(40, 72, seed=1)).cuda()
    with pytest.raises(lf.LoomfuseError) as e:
        p.run([u, u])
    assert e.value.code == lf.LF_ERR_UNSUPPORTED and "aliases" in str(e.value)
    # built-in executor: ping-pong only
    b = lf.Plan.with_ranges("biharmonic2d", (64, 128))
    v = torch.from_numpy(inputs.biharm_input(64, 128, seed=1)).cuda()
    with pytest.raises(lf.LoomfuseError) as e:
        b.run([v, v])
    assert e.value.code == lf.LF_ERR_UNSUPPORTED


def test_inplace_host_path():
    """lf_run_host with one host buffer for the aliased axiom and goal keeps
    one device buffer and runs in place."""
    spec = lf.set_ranges((SPECS / "biharm_inplace.lf").read_text(), (200, 600))
    plan = lf.Plan(spec, "b.lf")
    u0 = inputs.biharm_input(200, 600, seed=12)
    u = u0.copy()
    plan.run_host([u, u], steps=3)
    assert np.array_equal(bits(u), bits(oracle.biharm(u0, 3)))


@pytest.mark.parametrize("name,shift", [("biharm_body", (3, 5)), ("heat3d_body", (2, 1, 7)),
                                        ("normalization_body", (4, 9))])
def test_ranges_not_starting_at_zero(name, shift, tmp_path):
    """Loop ranges [lo, hi) with lo != 0: terminal bases move with lo
    (buffer_extents, storage.cpp:403-427); results equal the oracle's."""
    import re
    text = (SPECS / f"{name}.lf").read_text()
    dims = re.findall(r"^    (\w+): \[0, (\d+)\]$", text, flags=re.M)
    for (d, hi), s in zip(dims, shift):
        text = text.replace(f"    {d}: [0, {hi}]", f"    {d}: [{s}, {int(hi) + s}]")
    path = tmp_path / f"{name}_lo.lf"
    path.write_text(text)
    plan = lf.Plan.from_file(path)
    assert plan.executor.startswith("jit_")
    ax = CASES[name]()
    steps = 2 if name != "normalization_body" else 1
    got = run_device(plan, [ax[t.name] for t in plan.axioms], steps)
    ref = generic.run_naive(path, ax, steps=steps)
    for g, t in zip(got, plan.goals):
        assert np.array_equal(bits(g), bits(ref[t.name])), t.name


@pytest.mark.parametrize("name", ["biharm_body", "heat3d_body"])
def test_register_window_rotation_is_exact(name, monkeypatch):
    """LF_JIT_ROT=1 (opt-in): window rows rotate through registers across trips."""
    monkeypatch.setenv("LF_JIT_ROT", "1")
    plan = lf.Plan.from_file(SPECS / f"{name}.lf")
    assert "rw0_" in plan.source or "rw1_" in plan.source
    ax = CASES[name]()
    got = run_device(plan, [ax[t.name] for t in plan.axioms], 3)
    ref = generic.run_naive(SPECS / f"{name}.lf", ax, steps=3)
    for g, t in zip(got, plan.goals):
        assert np.array_equal(bits(g), bits(ref[t.name])), t.name


def test_fault_injection_corrupted_span_is_caught(monkeypatch):
    """R/SPEC.md:557 fault injection: the same chain emitted with one rolling
    window a row short (LF_JIT_FAULT=span:L, the corrupted rotation span the
    SPEC names) no longer matches run_naive, and the first mismatching trip is
    the witness; the uncorrupted plan stays bit-exact."""
    shape = (48, 160)
    text = lf.set_ranges((lf.SPEC_DIR / "examples" / "biharm_body.lf").read_text(), shape)
    u = inputs.biharm_input(*shape, seed=9)
    ref = oracle.biharm(u, 1)
    monkeypatch.setenv("LF_JIT_WS", "0")  # plain march: windows are exactly the contraction span
    good = lf.Plan(text, "biharm_body.lf")
    assert np.array_equal(bits(run_device(good, [u], 1)[0]), bits(ref))
    monkeypatch.setenv("LF_JIT_FAULT", "span:L")
    bad = lf.Plan(text, "biharm_body_fault.lf")
    L = lf.lib()
    src_good, src_bad = L.lf_plan_source(good._h).decode(), L.lf_plan_source(bad._h).decode()
    assert src_good != src_bad  # the window is emitted one row shorter
    got = run_device(bad, [u], 1)[0]
    diff = np.argwhere(bits(got) != bits(ref))
    assert diff.size > 0, "a corrupted rotation span went unnoticed"
    witness = tuple(int(x) for x in diff[0])
    assert 2 <= witness[0] < shape[0] + 2  # a trip (row) of the interior


@pytest.mark.parametrize("name", ["normalization_body", "colsum_body"])
def test_transposed_reduction_nests(name):
    """LF_JIT_RED_TILED=1 (opt-in): reduction nests with one ordered chain per
    lane (32 parallel cells per CTA, element operands evaluated by the whole
    CTA into a double-buffered tile) -- bit-exact as the warp-per-cell kernel."""
    with lf.option("LF_JIT_RED_TILED", 1):
        plan = lf.Plan.from_file(SPECS / f"{name}.lf")
    assert "lf_t[buf]" in plan.source
    ax = CASES[name]()
    got = run_device(plan, [ax[t.name] for t in plan.axioms], 1)
    ref = generic.run_naive(SPECS / f"{name}.lf", ax, steps=1)
    for g, t in zip(got, plan.goals):
        assert np.array_equal(bits(g), bits(ref[t.name])), t.name

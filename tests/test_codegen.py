"""Generated-source checks of the generic executor (no GPU: plans compile with
NVRTC here): the warp-specialised march is emitted where every streamed axiom
can be fetched by TMA, single-read producers are evaluated inside their
consumer (scalar contraction), and divisions by literals are strength-reduced
only where the result is provably the IEEE quotient.  Numerics are checked on
the GPU (tests/test_gpu_jit.py)."""
import re

import paper_1710_08774_b200 as lf

SPECS = lf.PKG_DIR.parent / "tests" / "specs"


def _kernel(src, name):
    if name + "(" not in src:
        return ""
    body = src[src.index(name + "("):]
    nxt = body.find('extern "C" __global__', 1)
    return body if nxt < 0 else body[:nxt]


def kernels(plan):
    src = plan.source
    return _kernel(src, "lf_jit_step"), _kernel(src, "lf_jit_step_ws")


def test_register_march_for_2d_chains():
    """2D chains get lf_jit_step_rm: warp strips with intermediates in
    register windows, neighbours by shuffles, no CTA barrier in the march."""
    for name in ("biharm_body", "multi_body"):
        rm = _kernel(lf.Plan.from_file(SPECS / f"{name}.lf").source, "lf_jit_step_rm")
        assert rm, name
        assert "lf_tma2(" in rm and "lf_mbar_wait(&lf_full" in rm
        assert rm.count("__syncthreads") == 1 and "bar.sync" not in rm
    rm = _kernel(lf.Plan.from_file(SPECS / "biharm_body.lf").source, "lf_jit_step_rm")
    assert "__shfl_down_sync" in rm and "__shfl_up_sync" in rm
    assert "T R" in rm and "double2" in rm  # register windows, 16-B vector loads
    # 3D chains keep the shared-memory window marches
    assert "lf_jit_step_rm(" not in lf.Plan.from_file(SPECS / "heat3d_body.lf").source


def test_warp_specialised_variant_for_streamed_axioms():
    for name in ("heat3d_body", "biharm_body"):
        plain, ws = kernels(lf.Plan.from_file(SPECS / f"{name}.lf"))
        assert ws, name
        assert ("lf_tma2(" in ws or "lf_tma3(" in ws) and "lf_mbar_wait(&lf_full" in ws
        assert "__syncthreads();\n  const bool producer" in ws  # the only CTA-wide barrier: after mbarrier init
        assert ws.count("__syncthreads") == 1


def test_unaligned_row_pitch_keeps_the_plain_kernel():
    # g_img of box_body.lf: 74 floats per row = 296 B, not a 16-B multiple (TMA strides)
    plain, ws = kernels(lf.Plan.from_file(SPECS / "box_body.lf"))
    assert plain and not ws


def test_single_level_chain_has_no_consumer_barrier():
    _, ws = kernels(lf.Plan.from_file(SPECS / "heat3d_body.lf"))
    assert "bar.sync" not in ws  # fluxes inlined: one group, one level


def test_in_place_chains_defer_their_boundary_writes():
    """3D in place: the warp-specialised march with deferred boundary writes
    (band stores + lf_jit_commit_ws); the plain march keeps the band loader
    (LF_JIT_WS=0 or untileable buffers)."""
    src = lf.Plan.from_file(SPECS / "heat3d_inplace.lf").source
    plain, ws = kernels(lf.Plan.from_file(SPECS / "heat3d_inplace.lf"))
    assert ws and "lf_jit_commit_ws(" in src and "cbo0_" in ws
    assert "cp.async.ca.shared.global" in plain and "lf_jit_capture(" in src


def test_single_read_producer_is_evaluated_in_its_consumer():
    plain, ws = kernels(lf.Plan.from_file(SPECS / "biharm_body.lf"))
    groups = re.findall(r"// group \d+: kernel '(\w+)'", ws)
    assert groups == ["lap1", "upd"]  # lap2 (read once, at offset 0) runs inside upd
    assert "'L2'" not in ws and "inlined 'lap2'" in ws
    assert ws.count("bar.sync") == 1


def test_division_by_literal_strength_reduction():
    plain, _ = kernels(lf.Plan.from_file(SPECS / "divs_body.lf"))
    assert "lf_div3f(" in plain                      # fp32 / 3 (oracle/div3check: exhaustive)
    assert "* 0x1p-2f" in plain and "* 0x1p1f" in plain  # / 4, / 0.5: exact reciprocals
    assert "/ static_cast<float>(7.0)" in plain       # not provable: stays a division
    assert "/ static_cast<float>(1.0e-30)" in plain   # not a power of two
    plain64, _ = kernels(lf.Plan.from_file(SPECS / "biharm_body.lf"))
    assert "lf_div3f" not in plain64


def test_switches_set_in_process_override_the_environment(monkeypatch):
    """lf_set_option: a tuning switch set in-process wins over the environment
    and takes effect at the next plan creation; dropping it restores the
    environment's value; names outside LF_* are refused."""
    spec = SPECS / "biharm_body.lf"
    assert "lf_jit_step_rm(" in lf.Plan.from_file(spec).source
    monkeypatch.setenv("LF_JIT_RM", "0")
    assert "lf_jit_step_rm(" not in lf.Plan.from_file(spec).source
    with lf.option("LF_JIT_RM", "1"):
        assert "lf_jit_step_rm(" in lf.Plan.from_file(spec).source
    assert "lf_jit_step_rm(" not in lf.Plan.from_file(spec).source  # the environment again
    import pytest
    with pytest.raises(lf.LoomfuseError):
        lf.set_option("PATH", "x")


def test_every_generated_kernel_waits_for_the_previous_grid():
    """Launched with programmatic stream serialization, every generated kernel
    must start with griddepcontrol.wait (lf_pdl / lf_pdl_wait) before touching
    memory -- the ghost fill, the in-place commit kernels and the nest kernels
    included."""
    import re
    for name in ("heat3d_body", "biharm_body", "biharm_inplace", "heat3d_inplace", "normalization_body",
                 "colsum_body", "box_body", "multi_body"):
        path = SPECS / f"{name}.lf"
        if not path.exists():
            path = lf.SPEC_DIR / "examples" / f"{name}.lf"
        src = lf.Plan.from_file(path).source
        kernels = re.findall(r'__global__ void[^\n]*\) \{\n([^\n]*)\n', src)
        assert kernels and len(kernels) == src.count("__global__ void"), name
        assert all(k.strip() in ("lf_pdl();", "lf_pdl_wait();") for k in kernels), (name, kernels)

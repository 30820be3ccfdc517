"""The C ABI from a C program (examples/run_chain.c): compiles and links
against libloomfuse_b200.so with the public header only; plans here, runs on
the GPU in the gpu-marked test (bit-exact against the oracle)."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_1710_08774_b200 as lf

ROOT = Path(__file__).resolve().parents[1]


def build_exe(tmp_path):
    lf.lib()
    exe = tmp_path / "run_chain"
    pkg = ROOT / "paper_1710_08774_b200"
    subprocess.run(["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", str(ROOT / "include"),
                    str(ROOT / "examples" / "run_chain.c"), "-L", str(pkg), "-lloomfuse_b200",
                    f"-Wl,-rpath,{pkg}", "-o", str(exe)], check=True)
    return exe


def test_c_program_plans(tmp_path):
    exe = build_exe(tmp_path)
    out = subprocess.run([str(exe), str(lf.spec_path("biharmonic2d")), "0"], capture_output=True, text=True,
                         check=True).stdout
    assert "executor biharm2d_fused_tma" in out
    assert "axiom double g_u bytes 134480000 extent 4100 4100" in out
    # a rule-file error comes back as a status with a positioned diagnostic
    bad = tmp_path / "bad.lf"
    bad.write_text(lf.spec_path("heat3d").read_text().replace("loop-order:", "loop-ordr:"))
    r = subprocess.run([str(exe), str(bad), "0"], capture_output=True, text=True)
    assert r.returncode == 1 and "bad.lf" in r.stderr


@pytest.mark.gpu
def test_c_program_runs_bit_exact(tmp_path):
    import oracle
    from paper_1710_08774_b200 import inputs
    exe = build_exe(tmp_path)
    spec = tmp_path / "heat3d_small.lf"
    spec.write_text(lf.set_ranges(lf.spec_path("heat3d").read_text(), (8, 16, 64)))
    u = inputs.heat3d_input(8, 16, 64, seed=21, sigma=2.0)
    fin, fout = tmp_path / "u.bin", tmp_path / "unew.bin"
    u.tofile(fin)
    out = subprocess.run([str(exe), str(spec), "3", str(fin), str(fout)], capture_output=True, text=True,
                         check=True).stdout
    assert "ran 3 steps" in out
    got = np.fromfile(fout, dtype=np.float64).reshape(u.shape)
    ref = oracle.heat3d(u, 3)
    assert np.array_equal(got[1:-1, 1:-1, 1:-1].view(np.uint64), ref[1:-1, 1:-1, 1:-1].view(np.uint64))


@pytest.mark.gpu
def test_c_program_runs_hydro_in_place(tmp_path):
    """The C ABI in place from a C host program: goals given the axioms' files
    share the axioms' host buffers; lf_run_host keeps one device buffer per pair."""
    import oracle
    from paper_1710_08774_b200 import inputs
    exe = build_exe(tmp_path)
    shape = (40, 200)
    spec = tmp_path / "hydro_inplace.lf"
    spec.write_text(lf.alias_iterates(lf.set_ranges(lf.spec_path("hydro2d").read_text(), shape)))
    st, dtdx = inputs.hydro_input(*shape, seed=8)
    files = []
    for name, a in zip(("rho", "mx", "my", "E"), st):
        f = tmp_path / f"{name}.bin"
        a.tofile(f)
        files.append(str(f))
    fd = tmp_path / "dtdx.bin"
    np.array([dtdx]).tofile(fd)
    out = subprocess.run([str(exe), str(spec), "3"] + files + [str(fd)] + files, capture_output=True, text=True,
                         check=True).stdout
    assert "executor hydro2d_fused_tma" in out and out.count("in place on terminal") == 4 and "ran 3 steps" in out
    ref = oracle.hydro(st, dtdx, 3)
    for v, f in enumerate(files):
        got = np.fromfile(f, dtype=np.float64).reshape(st[v].shape)
        assert np.array_equal(got.view(np.uint64), ref[v].view(np.uint64)), v

"""The C-ABI library loads on a CPU-only host and exports every symbol the
header declares; argument errors come back as status codes, never crashes."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1710_08774_b200 as lf
from paper_1710_08774_b200 import inputs

HEADER = Path(lf.PKG_DIR).parent / "include" / "loomfuse_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(lf_\w+)\s*\(", text, re.M)))


def test_header_symbols_all_exported():
    syms = declared_symbols()
    assert len(syms) >= 13
    L = lf.lib()
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(lf.ABI_SYMBOLS)


def test_version_and_last_error():
    L = lf.lib()
    assert b"sm_100a" in L.lf_version()
    with pytest.raises(lf.LoomfuseError):
        lf.Plan("not: [a valid", "x.lf")
    assert L.lf_last_error().decode()


def test_run_argument_errors_are_status_codes():
    p = lf.Plan.with_ranges("heat3d", (4, 16, 64))
    with pytest.raises(ValueError):
        p.run([0])
    L = lf.lib()
    one = (ctypes.c_void_p * 1)(1)
    assert L.lf_run(p._h, one, 1, 1, None) == lf.LF_ERR_SPEC  # wrong terminal count
    arr = (ctypes.c_void_p * 2)(0, 0)
    assert L.lf_run(p._h, arr, 2, 1, None) == lf.LF_ERR_SPEC  # NULL buffers
    arr = (ctypes.c_void_p * 2)(1, 1)
    assert L.lf_run(p._h, arr, 2, 0, None) == lf.LF_ERR_SPEC  # steps < 1
    box = lf.Plan.with_ranges("box2x", (16, 16))
    a = np.zeros(box.terminals[0].bytes // 4, np.float32)
    b = np.zeros(box.terminals[1].bytes // 4, np.float32)
    with pytest.raises(lf.LoomfuseError):
        box.run_host([a, b], steps=2)  # no iterate: pairs


def test_terminal_layout_matches_inputs():
    p = lf.Plan.with_ranges("heat3d", (4, 16, 64))
    u = inputs.heat3d_input(4, 16, 64)
    assert u.shape == p.terminals[0].extent and u.nbytes == p.terminals[0].bytes
    q = lf.Plan.with_ranges("biharmonic2d", (32, 32))
    assert inputs.biharm_input(32, 32).shape == q.terminals[0].extent == q.terminals[1].extent
    r = lf.Plan.with_ranges("box2x", (8, 12))
    assert inputs.box_input(8, 12).shape == r.terminals[0].extent
    assert r.terminals[0].dtype == np.float32


def test_slabs_thinner_than_the_halo_are_rejected():
    """A rank must own at least as many rows as the ghost band it sends its
    neighbours (Hydro2D / biharmonic halo: 2 rows): 3 ranks over 5 rows is
    refused before any device work, natively and in slabs.py."""
    p = lf.Plan.with_ranges("hydro2d", (5, 16))
    n = len(p.terminals)
    ptrs = (ctypes.c_void_p * (3 * n))(*range(16, 16 * (3 * n + 1), 16))  # distinct, never dereferenced
    assert lf.lib().lf_run_slabs_local(p._h, 3, ptrs, n, 2, None) == lf.LF_ERR_SPEC
    assert "halo" in lf.lib().lf_last_error().decode()
    import torch
    from paper_1710_08774_b200 import slabs
    with pytest.raises(ValueError, match="halo"):
        slabs.exchange([torch.zeros(5, 4)], slabs.Halo(2, 2, False), 0, 1)


def test_buffer_arguments_are_checked_against_the_terminals():
    """Plan.run / run_host / run_slab refuse buffers that do not match the
    terminal they stand for (wrong dtype, size, layout or device
    would otherwise read or write out of bounds)."""
    import torch
    p = lf.Plan.with_ranges("biharmonic2d", (16, 32))
    t = p.terminals[0]
    good = np.zeros(t.extent, np.float64)
    with pytest.raises(ValueError, match="expected"):
        p.run_host([good, np.zeros((4, 4))], steps=1)  # wrong size
    with pytest.raises(ValueError, match="element size"):
        p.run_host([good, np.zeros(t.extent, np.float32)], steps=1)
    with pytest.raises(ValueError, match="contiguous"):
        p.run_host([good, np.zeros((t.extent[1], t.extent[0])).T], steps=1)
    with pytest.raises(ValueError, match="host array"):
        p.run([good, good.copy()])
    with pytest.raises(ValueError, match="CUDA tensor"):
        p.run([torch.zeros(t.extent, dtype=torch.float64)] * 2)


def test_alias_iterates_declares_every_pair_and_the_plan_keeps_its_executor():
    """Plan.with_ranges(..., inplace=True): every iterate pair becomes a
    config.aliases entry (input then output, the reference's order); the chain
    signature -- and so the hand-written executor -- does not depend on it."""
    import paper_1710_08774_b200 as lf
    text = lf.set_ranges(lf.spec_path("hydro2d").read_text(), (64, 256))
    aliased = lf.alias_iterates(text)
    line = [ln.strip() for ln in aliased.splitlines() if ln.strip().startswith("aliases:")]
    assert line == ["aliases: [[g_rho, g_rho_n], [g_mx, g_mx_n], [g_my, g_my_n], [g_E, g_E_n]]"]
    assert lf.alias_iterates("config:\n  iterate: [[a_n,a],[ b_n , b ]]\n").count("aliases: [[a, a_n], [b, b_n]]") == 1
    import pytest
    with pytest.raises(ValueError):
        lf.alias_iterates(aliased)  # already declared
    with pytest.raises(ValueError):
        lf.alias_iterates("config:\n  iterate: [[a_n, a], b]\n")
    plain, inplace = lf.Plan(text, "h.lf"), lf.Plan(aliased, "h.lf")
    assert plain.executor == inplace.executor == "hydro2d_fused_tma"
    assert plain.report()["signature"] == inplace.report()["signature"]

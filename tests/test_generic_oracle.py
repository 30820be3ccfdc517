"""The generic run_naive (oracle/generic.py) evaluates `body:` chains over the
DAG the REFERENCE's own inference derives (oracle/_ref/refplan --dag).  Pin it
against the hand-written C restatements of the BASELINE chains (same chains
written as bodies) and against direct numpy formulas."""
import numpy as np
import pytest

import oracle
from oracle import generic
from paper_1710_08774_b200 import inputs
import paper_1710_08774_b200 as lf

SPECS = lf.PKG_DIR.parent / "tests" / "specs"


def need_ref():
    if not oracle.REFPLAN.exists() and not oracle.REFERENCE.exists():
        pytest.skip("reference planner not available")


def test_dsl_parse_and_precedence():
    e = generic.parse_body("a - b * c / d + -e")
    env = {k: np.float64(v) for k, v in dict(a=1.5, b=2.0, c=3.0, d=4.0, e=0.25).items()}
    assert generic.eval_body(e, env, np.float64) == 1.5 - 2.0 * 3.0 / 4.0 + -0.25
    m = generic.eval_body(generic.parse_body("min(a, b) + max(a, b) * sqrt(abs(a - b))"), env, np.float64)
    assert m == 1.5 + 2.0 * np.sqrt(0.5)


def test_generic_matches_c_oracle_biharm_multistep():
    need_ref()
    u = inputs.biharm_input(40, 72, seed=3)
    g = generic.run_naive(SPECS / "biharm_body.lf", {"g_u": u}, steps=3)["g_unew"]
    assert np.array_equal(g.view(np.uint64), oracle.biharm(u, 3).view(np.uint64))


def test_generic_matches_c_oracle_heat3d_incl_ghosts():
    need_ref()
    h = inputs.heat3d_input(9, 12, 40, seed=2, sigma=3.0)
    g = generic.run_naive(SPECS / "heat3d_body.lf", {"g_u": h}, steps=2)["g_unew"]
    assert np.array_equal(g.view(np.uint64), oracle.heat3d(h, 2).view(np.uint64))


def test_generic_matches_c_oracle_box_fp32():
    need_ref()
    b = inputs.box_input(33, 70, seed=1)
    g = generic.run_naive(SPECS / "box_body.lf", {"g_img": b})["g_out"]
    assert np.array_equal(g.view(np.uint32), oracle.box(b).view(np.uint32))


def multi_reference(x, s):
    a, b = x[:, 0:50], x[:, 2:52]
    p = np.where(a < b, a, b) * s
    q = np.where(a > b, a, b) + np.sqrt(np.abs(a - b))
    return (p[:20] - -p[1:21]) / (1.0 + q[:20] * q[:20])


def test_generic_multi_output_scalar_and_asymmetric_halo():
    need_ref()
    x = np.random.default_rng(0).random((21, 52))
    y = generic.run_naive(SPECS / "multi_body.lf", {"g_x": x, "g_scale": np.array([0.5])})["g_y"]
    assert np.array_equal(y.view(np.uint64), multi_reference(x, np.float64(0.5)).view(np.uint64))


def test_jit_plans_for_body_chains_and_reports_source():
    for s in ["biharm_body", "heat3d_body", "box_body", "multi_body", "laplace3_body"]:
        p = lf.Plan.from_file(SPECS / f"{s}.lf")
        assert p.executor.startswith("jit_"), s
        assert "lf_jit_step" in p.source
    # a chain without bodies and without a matching built-in stays unsupported
    q = lf.Plan.from_file(SPECS / "cosmo.lf")
    assert q.executor == ""


def normalization_reference(q, z):
    fl = (q[:, 1:] - q[:, :-1]) * (q[:, 1:] - q[:, :-1])
    acc = z.copy()
    for i in range(fl.shape[1]):  # run_naive's sequential sweep of the associative group
        acc = acc + fl[:, i]
    return fl / np.sqrt(acc)[:, None]


def colsum_reference(u, z, k):
    L = u[1:-1, :-2] + u[1:-1, 2:] + u[:-2, 1:-1] + u[2:, 1:-1] - 4.0 * u[1:-1, 1:-1]
    acc = z.copy()
    for j in range(L.shape[0]):
        acc = np.where(acc > np.abs(L[j]), acc, np.abs(L[j]))
    cs = acc + 1.0
    return u[1:-1, 1:-1] + k * L / cs[None, :], cs


def test_generic_reductions_match_numpy():
    """Associative kernels reduce sequentially in loop order (inner dim and
    outer dim), then broadcast across a split."""
    need_ref()
    rng = np.random.default_rng(3)
    q, z = rng.random((37, 151)), rng.random(37) * 0.1
    got = generic.run_naive(SPECS / "normalization_body.lf", {"g_q": q, "g_zero": z})["g_out"]
    assert np.array_equal(got, normalization_reference(q, z))
    u = rng.random((47, 72))
    got = generic.run_naive(SPECS / "colsum_body.lf", {"g_u": u, "g_z": np.zeros(70), "g_k": np.array([0.3])})
    out, cs = colsum_reference(u, np.zeros(70), np.float64(0.3))
    assert np.array_equal(got["g_out"], out) and np.array_equal(got["g_cs"], cs)


def test_multi_nest_body_chains_plan_to_the_nest_executor():
    for s, nests in [("normalization_body", 2), ("colsum_body", 3)]:
        p = lf.Plan.from_file(SPECS / f"{s}.lf")
        assert p.report()["nests"] == nests and p.report()["splits"] == 1
        assert p.executor == "jit_nests_fused", s
        assert "lf_nest0" in p.source and "lf_red" in p.source


@pytest.mark.parametrize("shape,steps", [((9, 14), 3), ((16, 6), 1)])
def test_generic_named_hydro_matches_c_oracle(shape, steps, tmp_path):
    """Hydro2D has no `body:` form: its 12 rules name the user-kernel functions.
    run_naive over the reference's inference DAG calls those functions element
    by element (oracle/kernels_ffi.c) and must reproduce the C restatement of
    the chain bit for bit, reflective ghost ring included."""
    need_ref()
    spec = tmp_path / "hydro2d.lf"
    spec.write_text(lf.set_ranges(lf.spec_path("hydro2d").read_text(), shape))
    st, dtdx = inputs.hydro_input(*shape, seed=shape[0] * 7 + 1)
    ax = {"g_rho": st[0], "g_mx": st[1], "g_my": st[2], "g_E": st[3], "g_dtdx": np.array([dtdx])}
    g = generic.run_naive(spec, ax, steps=steps)
    ref = oracle.hydro(st, dtdx, steps)
    for v, name in enumerate(("g_rho_n", "g_mx_n", "g_my_n", "g_E_n")):
        assert np.array_equal(g[name].view(np.uint64), ref[v].view(np.uint64)), name


@pytest.mark.parametrize("shape,steps", [((12, 20), 3), ((9, 14), 2)])
def test_generic_adaptive_hydro_matches_c_oracle(shape, steps, tmp_path):
    """The adaptive-dt chain (specs/hydro2d_adaptive.lf): the CFL speed, an
    associative MAX reduction seeded by a kernel with no inputs, and the dt/dx
    broadcast through an iterate pair -- run_naive over the reference's DAG
    equals the C oracle's fused step + sequential reduction, dt/dx included."""
    need_ref()
    spec = tmp_path / "hydro2d_adaptive.lf"
    spec.write_text(lf.set_ranges(lf.spec_path("hydro2d_adaptive").read_text(), shape))
    st, dtdx = inputs.hydro_input(*shape, seed=shape[0])
    ax = {"g_rho": st[0], "g_mx": st[1], "g_my": st[2], "g_E": st[3], "g_dtdx": np.array([dtdx])}
    g = generic.run_naive(spec, ax, steps=steps)
    ref, dref = oracle.hydro_adaptive(st, dtdx, steps)
    for v, name in enumerate(("g_rho_n", "g_mx_n", "g_my_n", "g_E_n")):
        assert np.array_equal(g[name].view(np.uint64), ref[v].view(np.uint64)), name
    assert float(g["g_dtdx_n"].reshape(-1)[0]) == dref

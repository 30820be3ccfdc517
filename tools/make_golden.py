"""Regenerate tests/golden/ -- committed fixtures that pin the product
without needing /root/reference at test time.

  refplan/<spec>.json   the reference planner's own verdict (oracle/_ref/refplan,
                        compiled from /root/reference/proj/src) on every bundled
                        and test spec: counts, nests/splits, footprint, storage,
                        buffer_extents, alias plan
  numeric/<case>.npz    seeded small cases, inputs and outputs.  The stencil
                        chains' outputs come from the generic run_naive over the
                        dataflow DAG the REFERENCE's inference derives
                        (oracle/generic.py + refplan --dag) on their `body:`
                        forms; Hydro2D from the same run_naive with its named
                        user kernels (hydro_kernels.h, element-wise through
                        oracle/kernels_ffi.c) over the reference's DAG.

Run in the CPU container (needs /root/reference):  python tools/make_golden.py
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from oracle import generic  # noqa: E402
import paper_1710_08774_b200 as lf  # noqa: E402
from paper_1710_08774_b200 import inputs  # noqa: E402

GOLD = ROOT / "tests" / "golden"
SPECS = ROOT / "tests" / "specs"


def refplans():
    out = GOLD / "refplan"
    out.mkdir(parents=True, exist_ok=True)
    paths = sorted(lf.SPEC_DIR.glob("*.lf")) + sorted(SPECS.glob("*.lf"))
    for p in paths:
        if p.name.startswith("_"):
            continue
        (out / f"{p.stem}.json").write_text(json.dumps(oracle.ref_plan(p), indent=1, sort_keys=True) + "\n")


# (case, body spec, sizes, steps, input generator)
CASES = [
    ("biharm", "biharm_body", (40, 128), 3, lambda s: {"g_u": inputs.biharm_input(*s, seed=5)}),
    ("heat3d", "heat3d_body", (8, 16, 64), 3, lambda s: {"g_u": inputs.heat3d_input(*s, seed=6, sigma=3.0)}),
    ("box", "box_body", (33, 128), 1, lambda s: {"g_img": inputs.box_input(*s, seed=7)}),
    ("normalization", "normalization_body", (20, 70), 1,
     lambda s: {"g_q": np.random.default_rng(3).random((s[0], s[1] + 1)), "g_zero": np.zeros(s[0])}),
    ("multi", "multi_body", (20, 50), 1,
     lambda s: {"g_x": np.random.default_rng(1).random((21, 52)), "g_scale": np.array([0.75])}),
]


def numerics():
    out = GOLD / "numeric"
    out.mkdir(parents=True, exist_ok=True)
    for case, spec, sizes, steps, gen in CASES:
        text = lf.set_ranges((SPECS / f"{spec}.lf").read_text(), sizes)
        tmp = SPECS / f"_golden_{spec}.lf"
        tmp.write_text(text)
        try:
            ax = gen(sizes)
            goals = generic.run_naive(tmp, ax, steps=steps)
        finally:
            tmp.unlink()
        arrays = {f"in_{k}": v for k, v in ax.items()}
        arrays.update({f"out_{k}": v for k, v in goals.items()})
        np.savez_compressed(out / f"{case}.npz", sizes=np.array(sizes), steps=np.array(steps), **arrays)
    # Hydro2D: the 12 named kernels evaluated over the reference's inference DAG
    sizes = (12, 20)
    st, dtdx = inputs.hydro_input(*sizes, seed=8)
    tmp = SPECS / "_golden_hydro2d.lf"
    tmp.write_text(lf.set_ranges(lf.spec_path("hydro2d").read_text(), sizes))
    try:
        g = generic.run_naive(tmp, {"g_rho": st[0], "g_mx": st[1], "g_my": st[2], "g_E": st[3],
                                    "g_dtdx": np.array([dtdx])}, steps=2)
    finally:
        tmp.unlink()
    ref = [g[n] for n in ("g_rho_n", "g_mx_n", "g_my_n", "g_E_n")]
    # ... and the adaptive-dt chain (CFL reduction, rank-0 dt/dx goal), 3 steps
    tmp.write_text(lf.set_ranges(lf.spec_path("hydro2d_adaptive").read_text(), sizes))
    try:
        ga = generic.run_naive(tmp, {"g_rho": st[0], "g_mx": st[1], "g_my": st[2], "g_E": st[3],
                                     "g_dtdx": np.array([dtdx])}, steps=3)
    finally:
        tmp.unlink()
    np.savez_compressed(out / "hydro_adaptive.npz", sizes=np.array(sizes), steps=np.array(3), dtdx=np.array([dtdx]),
                        **{f"in_{v}": st[v] for v in range(4)},
                        **{f"out_{v}": ga[n] for v, n in enumerate(("g_rho_n", "g_mx_n", "g_my_n", "g_E_n"))},
                        out_dtdx=np.asarray(ga["g_dtdx_n"]).reshape(1))
    np.savez_compressed(out / "hydro.npz", sizes=np.array((12, 20)), steps=np.array(2), dtdx=np.array([dtdx]),
                        **{f"in_{v}": st[v] for v in range(4)}, **{f"out_{v}": ref[v] for v in range(4)})


if __name__ == "__main__":
    refplans()
    numerics()
    print("wrote", sorted(str(p.relative_to(ROOT)) for p in GOLD.rglob("*.*")))

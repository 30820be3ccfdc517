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
                        forms; Hydro2D (no body form) from the C oracle.

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
    # Hydro2D: the C oracle (the chain has no body form)
    st, dtdx = inputs.hydro_input(12, 20, seed=8)
    ref = oracle.hydro(st, dtdx, 2)
    np.savez_compressed(out / "hydro.npz", sizes=np.array((12, 20)), steps=np.array(2), dtdx=np.array([dtdx]),
                        **{f"in_{v}": st[v] for v in range(4)}, **{f"out_{v}": ref[v] for v in range(4)})


if __name__ == "__main__":
    refplans()
    numerics()
    print("wrote", sorted(str(p.relative_to(ROOT)) for p in GOLD.rglob("*.*")))

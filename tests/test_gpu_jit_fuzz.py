"""Seeded random `body:` chains through the generic executor, bit-exact against
the generic run_naive over the reference's own inference DAG.

Each chain is 2-5 kernels over a 2D or 3D grid (fp64 or fp32): kernel t reads
its predecessor's output at a random offset plus up to three more (variable,
offset) pairs from anything produced before it (the axiom included), and
combines them with + - *, min / max / abs, square roots of positive values and
divisions by literals (some of them strength-reduced by the code generator).
Random offsets in [-2, 2] exercise the pipeline shifts, window depths,
dependency levels, producer inlining, both march kernels (warp-specialised and
plain) and tile edges against grids that are not tile multiples."""
import random

import numpy as np
import pytest

from oracle import generic
import paper_1710_08774_b200 as lf

DIMS = {2: ["j", "i"], 3: ["k", "j", "i"]}


def _subscript(names, off):
    return "".join(f"[{n}?{'' if o == 0 else f'{o:+d}'}]" for n, o in zip(names, off))


def _expr(rng, params):
    consts = ["0.5", "0.25", "2.0", "1.5", "0.125", "3.0"]

    def leaf():
        return rng.choice(params) if rng.random() < 0.75 else rng.choice(consts)

    def node(depth):
        if depth == 0:
            return leaf()
        r = rng.random()
        if r < 0.45:
            return f"({node(depth - 1)} {rng.choice(['+', '-', '*'])} {node(depth - 1)})"
        if r < 0.6:
            return f"{rng.choice(['min', 'max'])}({node(depth - 1)}, {node(depth - 1)})"
        if r < 0.7:
            return f"sqrt(abs({node(depth - 1)}) + 1.0)"
        if r < 0.8:
            return f"({node(depth - 1)} / {rng.choice(['3.0', '4.0', '0.5', '7.0', '1.0e-2'])})"
        return leaf()

    # every parameter appears at least once: sum them, then mix in a random tree
    return "(" + " + ".join(params) + f") * 0.25 + {node(2)} * 0.125"


def random_chain(seed):
    rng = random.Random(seed)
    nd = rng.choice([2, 2, 3])
    names = DIMS[nd]
    ty = rng.choice(["double", "double", "float"])
    nk = rng.randint(2, 5)
    sizes = [rng.randint(5, 11), rng.randint(9, 23), rng.randint(20, 70)] if nd == 3 else \
        [rng.randint(12, 40), rng.randint(30, 300)]
    produced = ["x"]
    kernels = []
    for t in range(1, nk + 1):
        out = "z" if t == nk else f"a{t}"
        reads = [(produced[-1], tuple(rng.randint(-2, 2) if rng.random() < 0.5 else 0 for _ in names))]
        for _ in range(rng.randint(0, 3)):
            r = (rng.choice(produced), tuple(rng.randint(-2, 2) if rng.random() < 0.5 else 0 for _ in names))
            if r not in reads:
                reads.append(r)
        params = [f"p{q}" for q in range(len(reads))]
        decl = f"void f{t}(" + ", ".join(f"{ty} {p}" for p in params) + f", {ty}* o)"
        ins = "\n".join(f"      {p} : {v}{_subscript(names, off)}" for p, (v, off) in zip(params, reads))
        kernels.append(f"""  k{t}:
    declaration: "{decl}"
    inputs: |
{ins}
    outputs: |
      o : {out}{_subscript(names, [0] * nd)}
    body: |
      o = {_expr(rng, params)}""")
        produced.append(out)
    sub_free = "".join(f"[{n}?]" for n in names)
    sub = "".join(f"[{n}]" for n in names)
    ranges = "\n".join(f"    {n}: [0, {s}]" for n, s in zip(names, sizes))
    return f"""# random chain, seed {seed}
kernels:
{chr(10).join(kernels)}
globals:
  inputs: |
    {ty} g_x{sub_free} => x{sub_free}
  outputs: |
    z{sub} => {ty} g_z{sub}
config:
  loop-order: [{", ".join(names)}]
  ranges:
{ranges}
"""


def test_random_chains_plan_on_cpu():
    for seed in range(4):
        plan = lf.Plan(random_chain(seed), f"fuzz{seed}.lf")
        assert plan.executor.startswith("jit_"), (seed, plan.executor)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(48))
def test_random_chain_matches_generic_oracle(seed, tmp_path):
    import torch
    text = random_chain(seed)
    path = tmp_path / f"fuzz{seed}.lf"
    path.write_text(text)
    plan = lf.Plan(text, path.name)
    (ax,) = plan.axioms
    x = np.random.default_rng(seed).random(ax.extent).astype(ax.dtype)
    dx = torch.from_numpy(x).cuda()
    (goal,) = plan.goals
    dz = torch.full(goal.extent, float("nan"), dtype=dx.dtype, device="cuda")
    plan.run([dx, dz], steps=1)
    torch.cuda.synchronize()
    ref = generic.run_naive(path, {ax.name: x}, steps=1)[goal.name]
    got = dz.cpu().numpy()
    view = np.uint64 if got.dtype == np.float64 else np.uint32
    bad = np.count_nonzero(got.view(view) != np.ascontiguousarray(ref).view(view))
    assert bad == 0, f"seed {seed}: {bad} cells differ\n{text}"


@pytest.mark.gpu
@pytest.mark.parametrize("knob", ["LF_JIT_VEC=2", "LF_JIT_RM_PACK=1", "LF_JIT_RM_UNROLL=0", "LF_JIT_RM=0", "LF_JIT_WS=0",
                                  "LF_JIT_RM_V=8", "LF_JIT_RM_WARPS=3"])
def test_random_chains_with_opt_in_variants(knob, tmp_path):
    """Opt-in / comparison variants on the same random chains (the knobs are
    read at plan creation; set in-process with lf.option): LF_JIT_VEC=2 (plain
    march, two adjacent columns per thread sharing window loads),
    LF_JIT_RM_PACK=1 (register march, fp32 cells in fp32x2 pairs),
    LF_JIT_RM_UNROLL=0 (register windows shifted by moves instead of renamed),
    LF_JIT_RM=0 / LF_JIT_WS=0 (the warp-specialised / plain smem-window
    marches where the register march / TMA would run), LF_JIT_RM_V=8 /
    LF_JIT_RM_WARPS=3 (register march: 8 cells per lane, 3 consumer warps --
    other lane spans, margins and strip widths)."""
    k, v = knob.split("=")
    with lf.option(k, v):
        for seed in range(48):
            test_random_chain_matches_generic_oracle(seed, tmp_path)

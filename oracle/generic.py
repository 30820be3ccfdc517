"""GENERIC run_naive -- test infrastructure only.

Evaluates any rule file whose kernels carry `body:` expressions (R/SPEC.md:82)
with the naive semantics of R/SPEC.md:532-540, over the dataflow DAG that the
REFERENCE's own inference derives (oracle/_ref/refplan --dag, built from
/root/reference/proj/src/inference.cpp).  Each concrete term -- a variable at
an offset from the canonical cell -- is evaluated as a full array over the
trip space, rule application by rule application in the DAG's topological
order: the value every cell of every intermediate would have in the naive
schedule's full-size arrays.  Bodies are parsed here independently of the
product's DSL and evaluated with numpy in the chain's element type
(correctly rounded + - * / sqrt, min/max as a<b?a:b, a>b?a:b).

Only tests/ use this; it is the parity oracle of the generic JIT executor.
"""
from __future__ import annotations

import json
import re
import subprocess
from pathlib import Path

import numpy as np

from . import REFPLAN, build, REFERENCE

_TOK = re.compile(r"\s*(?:(\d+\.\d*(?:[eE][-+]?\d+)?|\.\d+(?:[eE][-+]?\d+)?|\d+(?:[eE][-+]?\d+)?)|([A-Za-z_]\w*)|(.))")


def _tokens(s):
    out = []
    for m in _TOK.finditer(s):
        num, name, op = m.groups()
        if num is not None:
            out.append(("num", num))
        elif name is not None:
            out.append(("name", name))
        elif op is not None and not op.isspace():
            out.append(("op", op))
    return out


def parse_body(text):
    """-> expression tree of tuples: ('num', s) ('var', n) ('neg', e) (op, a, b) ('call', f, [args])."""
    toks = _tokens(text)
    pos = [0]

    def peek():
        return toks[pos[0]] if pos[0] < len(toks) else (None, None)

    def take():
        t = peek()
        pos[0] += 1
        return t

    def primary():
        k, v = take()
        if k == "num":
            return ("num", v)
        if k == "op" and v == "(":
            e = expr()
            assert take() == ("op", ")"), text
            return e
        if k == "op" and v == "-":
            return ("neg", primary())
        if k == "name":
            if peek() == ("op", "("):
                take()
                args = []
                if peek() != ("op", ")"):
                    while True:
                        args.append(expr())
                        if peek() == ("op", ","):
                            take()
                            continue
                        break
                assert take() == ("op", ")"), text
                return ("call", v, args)
            return ("var", v)
        raise ValueError(f"bad body expression {text!r}")

    def term():
        e = primary()
        while peek() in (("op", "*"), ("op", "/")):
            op = take()[1]
            e = (op, e, primary())
        return e

    def expr():
        e = term()
        while peek() in (("op", "+"), ("op", "-")):
            op = take()[1]
            e = (op, e, term())
        return e

    e = expr()
    assert pos[0] == len(toks), text
    return e


def eval_body(e, env, dt):
    k = e[0]
    if k == "num":
        return dt(float(e[1]))
    if k == "var":
        return env[e[1]]
    if k == "neg":
        return -eval_body(e[1], env, dt)
    if k == "call":
        a = [eval_body(x, env, dt) for x in e[2]]
        if e[1] == "sqrt":
            return np.sqrt(a[0])
        if e[1] == "abs":
            return np.abs(a[0])
        if e[1] == "min":
            return np.where(a[0] < a[1], a[0], a[1]).astype(dt)
        if e[1] == "max":
            return np.where(a[0] > a[1], a[0], a[1]).astype(dt)
        raise ValueError(e[1])
    a, b = eval_body(e[1], env, dt), eval_body(e[2], env, dt)
    return {"+": np.add, "-": np.subtract, "*": np.multiply, "/": np.divide}[k](a, b)


def ref_dag(spec_path) -> dict:
    if not REFPLAN.exists():
        if not REFERENCE.exists():
            raise FileNotFoundError("oracle/_ref/refplan not built and /root/reference absent")
        build(ref=True)
    r = subprocess.run([str(REFPLAN), "--dag", str(spec_path)], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    return json.loads(r.stdout)


def _fill(a, modes, n, base):
    """ghost refill, innermost dim first (edges/corners = composed maps)."""
    nd = a.ndim
    for d in reversed(range(nd)):
        h_lo = -base[d]
        h_hi = a.shape[d] - n[d] - h_lo
        m = modes[min(d, len(modes) - 1)]
        if m == "none":
            continue
        for g in range(max(h_lo, h_hi)):
            for side in (0, 1):
                if (side == 0 and g >= h_lo) or (side == 1 and g >= h_hi):
                    continue
                dst = [slice(None)] * nd
                src = [slice(None)] * nd
                if side == 0:
                    y = -1 - g
                    dst[d] = h_lo + y
                else:
                    y = n[d] + g
                    dst[d] = h_lo + y
                if m == "zero":
                    a[tuple(dst)] = 0
                    continue
                if m == "periodic":
                    z = y % n[d]
                elif m == "clamp":
                    z = 0 if y < 0 else n[d] - 1
                else:
                    z = -1 - y if y < 0 else 2 * n[d] - 1 - y
                src[d] = h_lo + z
                a[tuple(dst)] = -a[tuple(src)] if m == "odd" else a[tuple(src)]


def run_naive(spec_path, axioms: dict, steps: int = 1) -> dict:
    """Goal buffers after `steps` applications of the chain (axioms untouched).
    Iterated goals take their paired axiom's layout and ghost refill."""
    d = ref_dag(spec_path)
    n = [hi - lo for lo, hi in d["ranges"]]
    nd = len(n)
    raps, terms, kern = d["raps"], d["terms"], d["kernels"]
    pair = {g: a for g, a in d["iterate"]}
    bodies = {k: {o: parse_body(b) for o, b in v["bodies"].items()} for k, v in kern.items()}
    cur = {k: np.array(v) for k, v in axioms.items()}
    goals = {}
    for _ in range(steps):
        vals = {}
        goals = {}
        for g in d["goals"]:
            like = cur[pair[g]] if g in pair else None
            ext = d["externals"][g]
            dt = np.float32 if "float" in ext["type"] else np.float64
            goals[g] = np.zeros(like.shape if like is not None else [e for e, _ in ext["extents"]], dtype=dt)
        for r in d["topo"]:
            rap = raps[r]
            if rap["kind"] == "load":
                a = cur[rap["external"]]
                if not rap["slots"]:
                    vals[rap["out"][0]] = a.reshape(-1)[0]
                    continue
                ext = d["externals"][rap["external"]]["extents"]
                sl = []
                for k, (dim, shift) in enumerate(rap["slots"]):
                    start = shift - ext[k][1]
                    sl.append(slice(start, start + n[dim]))
                vals[rap["out"][0]] = a[tuple(sl)]
            elif rap["kind"] == "kernel":
                k = kern[rap["kernel"]]
                env = dict(zip(k["inputs"], (vals[t] for t in rap["in"])))
                dt = None
                for v in env.values():
                    dt = np.asarray(v).dtype.type
                for o, t in zip(k["outputs"], rap["out"]):
                    vals[t] = np.asarray(eval_body(bodies[rap["kernel"]][o], env, dt), dtype=dt)
            else:
                g = rap["external"]
                a = goals[g]
                base = [b for _, b in (d["externals"][pair[g]] if g in pair else d["externals"][g])["extents"]]
                sl = tuple(slice(-base[k], -base[k] + n[k]) for k in range(nd))
                a[sl] = np.broadcast_to(vals[rap["in"][0]], [n[k] for k in range(nd)])
        for g, a_name in pair.items():
            modes = d["boundary"].get(g) or d["boundary"].get("*") or ["none"]
            base = [b for _, b in d["externals"][a_name]["extents"]]
            _fill(goals[g], modes, n, base)
            cur[a_name] = goals[g]
    return goals

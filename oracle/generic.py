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


_DECL = re.compile(r"^\s*\w[\w\s\*&]*?\b(\w+)\s*\((.*)\)\s*$")


def call_named(kernel, ins):
    """Outputs of a kernel given by its `declaration:` only: the user-kernel
    function of userkernels/*.h (oracle/kernels_ffi.c) applied element by
    element to the broadcast inputs, parameters passed in declaration order."""
    import ctypes
    from . import lib
    m = _DECL.match(kernel["declaration"])
    if not m:
        raise ValueError(f"cannot read declaration {kernel['declaration']!r}")
    fn = getattr(lib(), "lfk_" + m.group(1), None)
    if fn is None:
        raise KeyError(f"no element-wise wrapper for user kernel {m.group(1)!r} (oracle/kernels_ffi.c)")
    params = []
    for piece in m.group(2).split(","):
        words = re.findall(r"\w+", piece)
        params.append((words[-1], np.float32 if "float" in words[:-1] else np.float64))
    arrays = np.broadcast_arrays(*[np.asarray(v) for v in ins])
    shape = arrays[0].shape if arrays else ()
    by_name = dict(zip(kernel["inputs"], arrays))
    outs = {o: None for o in kernel["outputs"]}
    args = []
    for name, dt in params:
        if name in by_name:
            a = np.ascontiguousarray(by_name[name], dtype=dt)
            by_name[name] = a
        else:
            a = outs[name] = np.empty(shape, dtype=dt)
        args.append(a)
    ptrs = (ctypes.c_void_p * len(args))(*[a.ctypes.data for a in args])
    fn.argtypes = [ctypes.c_long, ctypes.POINTER(ctypes.c_void_p)]
    if fn(int(np.prod(shape, dtype=np.int64)), ptrs) != 0:
        raise RuntimeError(f"lfk_{m.group(1)} failed")
    return [outs[o] for o in kernel["outputs"]]


def _term_axes(term, nd):
    """loop dims a term spans (others are broadcast axes of length 1)"""
    return {dim for dim, _ in term["dims"]}


def run_naive(spec_path, axioms: dict, steps: int = 1) -> dict:
    """Goal buffers after `steps` applications of the chain (axioms untouched).
    Iterated goals take their paired axiom's layout and ghost refill.

    Every term value is an array over all loop dims (length 1 along the dims
    the term does not span).  An associative kernel (a reduction: its element
    inputs span loop dims its output does not) runs sequentially over those
    dims in loop order, starting from its carry input -- the order in which
    run_naive's sweep of the group over its space visits them
    (R/SPEC.md:532-540)."""
    d = ref_dag(spec_path)
    n = [hi - lo for lo, hi in d["ranges"]]
    lo = [r[0] for r in d["ranges"]]
    nd = len(n)
    raps, terms, kern = d["raps"], d["terms"], d["kernels"]
    pair = {g: a for g, a in d["iterate"]}
    bodies = {k: {o: parse_body(b) for o, b in v["bodies"].items()} for k, v in kern.items()}
    cur = {k: np.array(v) for k, v in axioms.items()}
    goals = {}

    def shape_of(axes):
        return [n[k] if k in axes else 1 for k in range(nd)]

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
                sl, axes = [], []
                for k, (dim, shift) in enumerate(rap["slots"]):
                    start = (lo[dim] if dim >= 0 else 0) + shift - ext[k][1]
                    if dim < 0:
                        sl.append(start)  # constant subscript
                    else:
                        sl.append(slice(start, start + n[dim]))
                        axes.append(dim)
                v = a[tuple(sl)]
                # slot order follows the loop order: place the sliced axes, pad the rest
                vals[rap["out"][0]] = v.reshape(shape_of(set(axes)))
            elif rap["kind"] == "kernel":
                k = kern[rap["kernel"]]
                ins = [vals[t] for t in rap["in"]]
                dt = None
                for v in ins:
                    dt = np.asarray(v).dtype.type
                if k.get("associative"):
                    (o_name,) = k["outputs"]
                    out_t = terms[rap["out"][0]]
                    out_axes = _term_axes(out_t, nd)
                    space = set(out_axes)
                    carry = None
                    for i, t in enumerate(rap["in"]):
                        tt = terms[t]
                        space |= _term_axes(tt, nd)
                        if tt["ident"] == out_t["ident"] and tt["dims"] == out_t["dims"] and tt["tag"] != out_t["tag"]:
                            carry = i
                    red = sorted(space - out_axes)
                    acc = np.broadcast_to(np.asarray(ins[carry], dtype=dt), shape_of(out_axes)).copy()
                    for pos in np.ndindex(*[n[a] for a in red]):
                        env = {}
                        for i, (pname, v) in enumerate(zip(k["inputs"], ins)):
                            if i == carry:
                                env[pname] = acc
                                continue
                            v = np.asarray(v)
                            ix = [slice(None)] * nd
                            for a, p in zip(red, pos):
                                if v.ndim == nd and v.shape[a] > 1:
                                    ix[a] = slice(p, p + 1)
                            env[pname] = v[tuple(ix)] if v.ndim == nd else v
                        if bodies[rap["kernel"]]:
                            acc = np.asarray(eval_body(bodies[rap["kernel"]][o_name], env, dt), dtype=dt)
                        else:  # a named kernel: the user-kernel function, element-wise
                            acc = call_named(k, [env[pn] for pn in k["inputs"]])[0]
                    vals[rap["out"][0]] = acc
                    continue
                if not bodies[rap["kernel"]]:
                    # a named kernel: the shipped user-kernel function itself, element-wise
                    for t, v in zip(rap["out"], call_named(k, ins)):
                        vals[t] = v
                    continue
                env = dict(zip(k["inputs"], ins))
                for o, t in zip(k["outputs"], rap["out"]):
                    vals[t] = np.asarray(eval_body(bodies[rap["kernel"]][o], env, dt), dtype=dt)
            else:
                g = rap["external"]
                a = goals[g]
                ext = (d["externals"][pair[g]] if g in pair else d["externals"][g])["extents"]
                sl, axes = [], []
                for k, (dim, shift) in enumerate(rap["slots"]):
                    start = lo[dim] + shift - ext[k][1]
                    sl.append(slice(start, start + n[dim]))
                    axes.append(dim)
                v = np.broadcast_to(vals[rap["in"][0]], shape_of(set(axes)))
                a[tuple(sl)] = v.reshape([n[dim] for dim in axes])
        for g, a_name in pair.items():
            if not d["externals"][a_name]["extents"]:  # a rank-0 terminal: no ghosts
                cur[a_name] = goals[g]
                continue
            modes = d["boundary"].get(g) or d["boundary"].get("*") or ["none"]
            base = [b - l for (_, b), l in zip(d["externals"][a_name]["extents"], lo)]  # relative to the range start
            _fill(goals[g], modes, n, base)
            cur[a_name] = goals[g]
    return goals

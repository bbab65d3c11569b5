"""Benchmark µGraph fixtures (RMSNorm→MatMul, GatedMLP, GQA decode, LoRA).

The reference's ``fixtures.cpp`` is absent (``proj/core/CMakeLists.txt:24``);
these constructions follow SURVEY §8d, which authored them with the
reference builder API and checked each one with the reference's
``validate`` and ``random_test_equivalence`` against its flat program.  Every
builder takes shapes and (grid, forloop) so the same code yields the
BASELINE configurations and the reduced "verification shapes" candidate
pools ("Pool recipe").

Each family function returns ``(program, mugraph)`` as wire-format dicts.
``mutant=True`` yields the deliberately non-equivalent variant used in the
verifier pools.
"""
from __future__ import annotations

from typing import Dict, List, Tuple

from .graph import PHI, BlockBuilder, GraphBuilder, OpType as O

X_, Y_, Z_ = 0, 1, 2  # data dims


# ---- RMSNorm -> MatMul ------------------------------------------------------

def rmsnorm_program(b: int, h: int, n: int) -> dict:
    """Z = Matmul(EwDiv(EwMul(X,G), Sqrt(EwMul(Sum(Sqr X, dim1, h), D))), W)."""
    gb = GraphBuilder()
    X, G, W, D = gb.input([b, h]), gb.input([1, h]), gb.input([h, n]), gb.input([1, 1])
    ss = gb.op(O.Sum, [gb.op(O.Sqr, [X])], {"dim": 1, "group": h})
    r = gb.op(O.Sqrt, [gb.op(O.EwMul, [ss, D])])
    y = gb.op(O.EwDiv, [gb.op(O.EwMul, [X, G]), r])
    return gb.finish([gb.op(O.Matmul, [y, W])])


def rmsnorm_mugraph(b: int, h: int, n: int, grid: int, forloop: int, mutant: bool = False) -> dict:
    """One GraphDef: grid (gx,1,1), loop f; B=Accum(Matmul(X̄·Ḡ, W̄)), A=Accum(Sum(X̄²)·D̄);
    post EwDiv(B, Sqrt(A)); omap x<->1."""
    gb = GraphBuilder()
    X, G, W, D = gb.input([b, h]), gb.input([1, h]), gb.input([h, n]), gb.input([1, 1])
    bb = BlockBuilder([grid, 1, 1], forloop, [[b, h], [1, h], [h, n], [1, 1]])
    xb = bb.initer(0, [PHI], [1])
    gbar = bb.initer(1, [PHI], [1])
    wb = bb.initer(2, [1], [0])
    db = bb.initer(3, [PHI], [PHI])
    xg = bb.op(O.EwMul, [xb, xb if mutant else gbar])
    B = bb.op(O.Accum, [bb.op(O.Matmul, [xg, wb])], {"fmap": [PHI]})
    ssq = bb.op(O.Sum, [bb.op(O.Sqr, [xb])], {"dim": 1, "group": h // forloop})
    A = bb.op(O.Accum, [bb.op(O.EwMul, [ssq, db])], {"fmap": [PHI]})
    out = bb.op(O.EwDiv, [B, bb.op(O.Sqrt, [A])])
    bb.outsaver(out, [1])
    out_t = gb.graphdef([X, G, W, D], bb)
    return gb.finish([out_t])


# ---- GatedMLP ----------------------------------------------------------------

def gatedmlp_program(b: int, h: int, n: int) -> dict:
    """EwMul(SiLU(Matmul(X,W1)), Matmul(X,W3))"""
    gb = GraphBuilder()
    X, W1, W3 = gb.input([b, h]), gb.input([h, n]), gb.input([h, n])
    a1 = gb.op(O.SiLU, [gb.op(O.Matmul, [X, W1])])
    return gb.finish([gb.op(O.EwMul, [a1, gb.op(O.Matmul, [X, W3])])])


def gatedmlp_mugraph(b: int, h: int, n: int, grid: int, forloop: int, mutant: bool = False) -> dict:
    """Two φ-Accum matmuls sharing X̄; post EwMul(SiLU(A1), A3); omap x<->1."""
    gb = GraphBuilder()
    X, W1, W3 = gb.input([b, h]), gb.input([h, n]), gb.input([h, n])
    bb = BlockBuilder([grid, 1, 1], forloop, [[b, h], [h, n], [h, n]])
    xb = bb.initer(0, [PHI], [1])
    w1 = bb.initer(1, [1], [0])
    w3 = bb.initer(2, [1], [0])
    A1 = bb.op(O.Accum, [bb.op(O.Matmul, [xb, w1])], {"fmap": [PHI]})
    A3 = bb.op(O.Accum, [bb.op(O.Matmul, [xb, w3])], {"fmap": [PHI]})
    if mutant:
        out = bb.op(O.EwMul, [A1, bb.op(O.SiLU, [A3])])
    else:
        out = bb.op(O.EwMul, [bb.op(O.SiLU, [A1]), A3])
    bb.outsaver(out, [1])
    out_t = gb.graphdef([X, W1, W3], bb)
    return gb.finish([out_t])


# ---- GQA decode ---------------------------------------------------------------

def gqa_program(g: int, qh: int, hd: int, L: int) -> dict:
    """EwDiv(Matmul(EwExp(Matmul(Q,K)),V), Sum(EwExp(Matmul(Q,K)), dim2, L)); K stored [g,hd,L]."""
    gb = GraphBuilder()
    Q, K, V = gb.input([g, qh, hd]), gb.input([g, hd, L]), gb.input([g, L, hd])
    e = gb.op(O.EwExp, [gb.op(O.Matmul, [Q, K])])
    num = gb.op(O.Matmul, [e, V])
    den = gb.op(O.Sum, [e], {"dim": 2, "group": L})
    return gb.finish([gb.op(O.EwDiv, [num, den])])


def gqa_mugraph(g: int, qh: int, hd: int, L: int, grid: int, forloop: int,
                mutant: bool = False) -> dict:
    """grid (gx,1,1) over groups (imap x<->0), loop over kv (K fmap i<->2, V fmap i<->1);
    Accums N=Σ exp(QK̄)V̄, D=Σ rowsum exp(QK̄); post N/D; omap x<->0 (no max-subtraction: Lax)."""
    gb = GraphBuilder()
    Q, K, V = gb.input([g, qh, hd]), gb.input([g, hd, L]), gb.input([g, L, hd])
    bb = BlockBuilder([grid, 1, 1], forloop, [[g, qh, hd], [g, hd, L], [g, L, hd]])
    qb = bb.initer(0, [0], [PHI])
    kb = bb.initer(1, [0], [2])
    vb = bb.initer(2, [0], [1])
    s = bb.op(O.Matmul, [qb, kb])
    e = bb.op(O.EwExp, [s])
    N = bb.op(O.Accum, [bb.op(O.Matmul, [e, vb])], {"fmap": [PHI]})
    D = bb.op(O.Accum, [bb.op(O.Sum, [s if mutant else e], {"dim": 2, "group": L // forloop})],
              {"fmap": [PHI]})
    bb.outsaver(bb.op(O.EwDiv, [N, D]), [0])
    out_t = gb.graphdef([Q, K, V], bb)
    return gb.finish([out_t])


# ---- LoRA ---------------------------------------------------------------------

def lora_program(b: int, h: int, n: int, r: int) -> dict:
    """EwAdd(Matmul(X,W), Matmul(Matmul(X,A),B))"""
    gb = GraphBuilder()
    X, W, A, B = gb.input([b, h]), gb.input([h, n]), gb.input([h, r]), gb.input([r, n])
    xa = gb.op(O.Matmul, [X, A])
    return gb.finish([gb.op(O.EwAdd, [gb.op(O.Matmul, [X, W]), gb.op(O.Matmul, [xa, B])])])


def lora_mugraph(b: int, h: int, n: int, r: int, grid: int, forloop: int,
                 mutant: bool = False) -> dict:
    """Single-kernel LoRA: Accums XW (φ), XA (φ, A imap φ), B̄ (concat fmap i<->0);
    post EwAdd(XW, Matmul(XA, B̄)); omap x<->1."""
    gb = GraphBuilder()
    X, W, A, B = gb.input([b, h]), gb.input([h, n]), gb.input([h, r]), gb.input([r, n])
    bb = BlockBuilder([grid, 1, 1], forloop, [[b, h], [h, n], [h, r], [r, n]])
    xb = bb.initer(0, [PHI], [1])
    wb = bb.initer(1, [1], [0])
    ab = bb.initer(2, [PHI], [0])
    bbar = bb.initer(3, [1], [0])
    XW = bb.op(O.Accum, [bb.op(O.Matmul, [xb, wb])], {"fmap": [PHI]})
    XA = bb.op(O.Accum, [bb.op(O.Matmul, [xb, ab])], {"fmap": [PHI]})
    Bc = bb.op(O.Accum, [bbar], {"fmap": [0]})
    t = bb.op(O.Matmul, [XA, Bc])
    out = t if mutant else bb.op(O.EwAdd, [XW, t])
    bb.outsaver(out, [1])
    out_t = gb.graphdef([X, W, A, B], bb)
    return gb.finish([out_t])


# ---- BASELINE configurations --------------------------------------------------

BENCH = {
    # name: (program builder args, mugraph builder args) at BASELINE.json configs
    "rmsnorm": dict(args=(8, 4096, 4096), grid=128, forloop=16),
    "gatedmlp": dict(args=(8, 4096, 14336), grid=112, forloop=16),
    "gqa": dict(args=(64, 8, 128, 4096), grid=64, forloop=16),
    "lora": dict(args=(16, 4096, 4096, 16), grid=128, forloop=16),
}

_PROG = {"rmsnorm": rmsnorm_program, "gatedmlp": gatedmlp_program, "gqa": gqa_program,
         "lora": lora_program}
_MU = {"rmsnorm": rmsnorm_mugraph, "gatedmlp": gatedmlp_mugraph, "gqa": gqa_mugraph,
       "lora": lora_mugraph}


def family_program(name: str, *args) -> dict:
    return _PROG[name](*args)


def family_mugraph(name: str, *args, grid: int, forloop: int, mutant: bool = False) -> dict:
    return _MU[name](*args, grid, forloop, mutant)


def bench_pair(name: str) -> Tuple[dict, dict]:
    c = BENCH[name]
    return _PROG[name](*c["args"]), _MU[name](*c["args"], c["grid"], c["forloop"])


# ---- verification-shape candidate pools (SURVEY §8d "Pool recipe") -------------

VERIFY_SHAPES = {
    "rmsnorm": (1, 64, 64),
    "gatedmlp": (8, 64, 64),
    "gqa": (4, 8, 16, 64),
    "lora": (16, 64, 64, 16),
}
_GRIDS = (1, 2, 4, 8, 16)
_LOOPS = (1, 2, 4, 8, 16)


def family_pool(name: str, shapes=None) -> List[Tuple[str, dict]]:
    """All valid (grid, loop) variants, each equivalent and mutant: [(tag, graph)]."""
    args = shapes or VERIFY_SHAPES[name]
    out = []
    for gx in _GRIDS:
        for fl in _LOOPS:
            for mut in (False, True):
                try:
                    g = _MU[name](*args, gx, fl, mut)
                except Exception:
                    continue
                out.append((f"{name}/g{gx}/f{fl}/{'mut' if mut else 'eq'}", g))
    return out


def verify_families() -> Dict[str, Tuple[dict, List[Tuple[str, dict]]]]:
    """family -> (program, pool) at verification shapes."""
    return {f: (_PROG[f](*VERIFY_SHAPES[f]), family_pool(f)) for f in VERIFY_SHAPES}


# ---- search-loop candidate streams ----------------------------------------------

_BIN = ("ewadd", "ewmul", "ewdiv")
_UN = ("sqr", "sqrt", "silu", "ewexp")


def search_stream(bases: List[dict], n: int, seed: int = 0) -> List[dict]:
    """Up to ``n`` DISTINCT candidate graphs for a search-loop stream: the
    ``bases`` (e.g. a family pool plus the generator's candidates), then
    mutants of them — up to two elementwise ops rewritten to another op of
    the same arity (EwAdd/EwMul/EwDiv, Sqr/Sqrt/SiLU/EwExp) and a chain of
    up to two unary ops inserted before the first OutSaver.  Shapes and
    Definition-1 validity are unchanged; equivalence mostly is not, as for
    the bulk of what a search proposes.  Distinct by canonical JSON;
    deterministic in ``seed``; fewer than ``n`` when the mutation space of
    the bases is exhausted."""
    import itertools
    import json
    import random

    rnd = random.Random(seed)
    seen, out = set(), []

    def add(g):
        key = json.dumps(g, sort_keys=True)
        if key not in seen:
            seen.add(key)
            out.append(g)

    for g in bases:
        if len(out) >= n:
            return out
        add(g)

    def recipes(g):
        sites = []
        for oi, op in enumerate(g["ops"]):
            for bi, bop in enumerate(op.get("blockGraph", {}).get("ops", [])):
                if bop["type"] in _BIN or bop["type"] in _UN:
                    cls = _BIN if bop["type"] in _BIN else _UN
                    sites.append([(oi, bi, t) for t in cls if t != bop["type"]])
        edits = [()]
        for a in range(len(sites)):
            edits += [(e,) for e in sites[a]]
            for b in range(a + 1, len(sites)):
                edits += list(itertools.product(sites[a], sites[b]))
        chains = [()] + [(u,) for u in _UN] + list(itertools.product(_UN, _UN))
        rs = [(e, c) for e in edits for c in chains if e or c]
        rnd.shuffle(rs)
        return rs

    def apply(text, edit, chain):
        g = json.loads(text)
        for oi, bi, t in edit:
            g["ops"][oi]["blockGraph"]["ops"][bi]["type"] = t
        if chain:
            gd = next(op for op in g["ops"] if "blockGraph" in op)
            bg = gd["blockGraph"]
            j = next(i for i, op in enumerate(bg["ops"]) if op["type"] == "outsaver")
            t = bg["ops"][j]["inputs"][0]
            shape = next(x["shape"] for x in bg["tensors"] if x["id"] == t)
            nid = max(x["id"] for x in bg["tensors"]) + 1
            new = []
            for u in chain:
                bg["tensors"].append({"id": nid, "shape": list(shape), "scope": "shared"})
                new.append({"id": -1, "type": u, "attrs": {}, "inputs": [t], "outputs": [nid]})
                t, nid = nid, nid + 1
            bg["ops"][j]["inputs"] = [t]
            bg["ops"][j:j] = new
            for i, op in enumerate(bg["ops"]):
                op["id"] = i
        return g

    texts = [json.dumps(g) for g in bases]
    queues = [iter(recipes(g)) for g in bases]
    live = list(range(len(bases)))
    while len(out) < n and live:
        nxt = []
        for i in live:
            r = next(queues[i], None)
            if r is None:
                continue
            nxt.append(i)
            add(apply(texts[i], *r))
            if len(out) >= n:
                break
        live = nxt
    return out


def attribute_mutants(bases: List[dict], n: int, seed: int = 0) -> List[dict]:
    """``n`` graphs with one block-graph attribute of a base redrawn — grid
    x extent, for-loop trip count, an InIter imap / fmap, an OutSaver omap,
    an Accum fmap or a Sum dim / group — most of them invalid (Definition 1,
    shapes, divisibility), the valid ones re-partitioned µGraphs.  For
    validate / verifier parity against the reference; deterministic."""
    import copy
    import random

    rnd = random.Random(seed)
    out = []
    while len(out) < n:
        g = copy.deepcopy(rnd.choice(bases))
        gds = [op for op in g["ops"] if "blockGraph" in op]
        if not gds:
            continue
        bg = rnd.choice(gds)["blockGraph"]
        k = rnd.randint(0, 5)
        if k == 0:
            bg["grid"][0] = rnd.choice([1, 2, 3, 4, 8, 16, 32])
        elif k == 1:
            bg["forloop"] = rnd.choice([1, 2, 3, 4, 8, 16, 64])
        else:
            o = rnd.choice([o for o in bg["ops"] if o["type"] in ("initer", "outsaver", "accum", "sum")])
            at = o["attrs"]
            if o["type"] == "initer":
                key = rnd.choice(["imap", "fmap"])
                at[key] = {("x" if key == "imap" else "i"): rnd.choice(["phi", 0, 1, 2])}
            elif o["type"] == "outsaver":
                at["omap"] = {"x": rnd.choice(["phi", 0, 1, 2])}
            elif o["type"] == "accum":
                at["fmap"] = {"i": rnd.choice(["phi", 0, 1, 2])}
            else:
                at["dim"] = rnd.choice([0, 1, 2])
                at["group"] = rnd.choice([1, 2, 4, 8, 16, 64])
        out.append(g)
    return out

#!/usr/bin/env python
"""Generates the committed golden vectors in tests/golden/ by running the
REFERENCE ITSELF (oracle/_ref/libtpo_ref.so, compiled from the unmodified
sources under /root/reference by oracle/Makefile) in this container.

The reference ships no tests, fixtures or known-answer vectors for this path
(SURVEY §4), so these files are what pins the CPU restatement
(oracle/restate.py) and, through it, the GPU path — on boxes where the
reference sources do not exist.  Re-run with

    make -C oracle && python tests/golden/make_golden.py

Outputs (all small):
  graphs.json   the µGraphs the vectors refer to (wire format, serialize.hpp schema)
  golden.npz    arrays (RNG draws, field tables, FF attempts, verdicts, fp outputs)
  golden.json   scalars (known answers, madds, validate counts, canonical keys)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2405_05751_b200 import fixtures as F  # noqa: E402
from paper_2405_05751_b200.graph import PHI, BlockBuilder, GraphBuilder, OpType as O  # noqa: E402

FIELDS = [(227, 113, 4), (103, 17, 8)]
RNG_CASES = [(0, None), (7, 0), (1, 5), (0xDEADBEEF, 131071), (2**63 + 11, 3)]
VERDICT_N = 240          # candidates per family (seeds 0..N-1) with full verdicts
FP_SHAPES = {            # small fp cases (args, grid, forloop)
    "rmsnorm": ((4, 64, 32), 2, 4),
    "gatedmlp": ((8, 64, 32), 2, 4),
    "gqa": ((4, 8, 16, 64), 2, 4),
    "lora": ((16, 64, 32, 16), 2, 4),
}


FUSED_SHAPES = {
    "rmsnorm": ((8, 512, 256), 2, 4),
    "gatedmlp": ((8, 512, 256), 2, 4),
    "gqa": ((4, 8, 128, 512), 2, 4),
    "lora": ((16, 512, 256, 16), 2, 4),
}


def edge_graphs():
    """Small graphs exercising broadcasting, Repeat/Reshape, grouped Sum,
    Sqrt/Div resampling, Exp + SiLU, concat Accum, partial omap and
    ConcatMatmul (the same constructions as tests/test_verify_gpu.py)."""
    gs = {}
    gb = GraphBuilder()
    x = gb.input([4, 8])
    gs["identity"] = gb.finish([x])
    gb = GraphBuilder()
    x, y = gb.input([2, 4, 8]), gb.input([1, 8])
    a = gb.op(O.EwMul, [x, y])
    r = gb.op(O.Repeat, [y], {"target": [2, 4, 8]})
    s = gb.op(O.Sum, [gb.op(O.EwAdd, [a, r])], {"dim": 2, "group": 4})
    q = gb.op(O.Sqrt, [gb.op(O.Sqr, [s])])
    d = gb.op(O.EwDiv, [s, q])
    e = gb.op(O.SiLU, [gb.op(O.EwExp, [gb.op(O.Reshape, [d], {"target": [4, 4]})])])
    gs["mixed_kernel"] = gb.finish([e, d])
    gb = GraphBuilder()
    x, w = gb.input([4, 16]), gb.input([16, 8])
    bb = BlockBuilder([2, 3, 1], 4, [[4, 16], [16, 8]])
    xb = bb.initer(0, [PHI, PHI], [1])
    wb = bb.initer(1, [1, PHI], [0])
    m = bb.op(O.Accum, [bb.op(O.Matmul, [xb, wb])], {"fmap": [PHI]})
    cc = bb.op(O.Accum, [xb], {"fmap": [1]})
    bb.outsaver(m, [1])
    bb.outsaver(bb.op(O.EwAdd, [cc, cc]), [0])
    gd = gb.graphdef([x, w], bb)
    gs["omap_partial"] = gb.finish([gd, gd + 1])
    gb = GraphBuilder()
    X, T, W, B = gb.input([4, 8]), gb.input([4, 2]), gb.input([8, 6]), gb.input([2, 6])
    bb = BlockBuilder([2, 3, 1], 2, [[4, 8], [4, 2], [8, 6], [2, 6]])
    xb = bb.initer(0, [0, PHI], [1])
    tb = bb.initer(1, [0, PHI], [PHI])
    wb = bb.initer(2, [PHI, 1], [0])
    bbar = bb.initer(3, [PHI, 1], [PHI])
    acc = bb.op(O.Accum, [bb.op(O.ConcatMatmul, [xb, tb, wb, bbar])], {"fmap": [PHI]})
    bb.outsaver(acc, [0, 1])
    gs["concatmatmul"] = gb.finish([gb.graphdef([X, T, W, B], bb)])
    return gs


def main():
    assert ref.available(), "build the reference first: make -C oracle"
    graphs = {}
    arrays = {}
    scal = {"source": "oracle/_ref/libtpo_ref.so (reference proj/core compiled unmodified)"}

    # ---- RNG (rng.hpp:25-63)
    scal["rng"] = []
    for i, (seed, stream) in enumerate(RNG_CASES):
        arrays[f"rng_{i}"] = ref.rng_draws(seed, 256, stream)
        scal["rng"].append({"seed": seed, "stream": stream, "key": f"rng_{i}"})
    arrays["normals_17_0"] = ref.rng_normals(17, 0, 64)
    arrays["normals_17_3"] = ref.rng_normals(17, 3, 64)

    # ---- field tables + op table (field.cpp:43-127)
    scal["fields"] = []
    rs = np.random.default_rng(0)
    for p, q, w in FIELDS:
        ip, iq, sp, sq = ref.field_tables(p, q, w)
        k = f"f{p}_{q}"
        arrays[k + "_inv_p"], arrays[k + "_inv_q"] = ip, iq
        arrays[k + "_sqrt_p"], arrays[k + "_sqrt_q"] = sp, sq
        n = 600
        a = np.stack([rs.integers(0, p, n), rs.integers(0, q, n), rs.integers(0, 2, n)], 1)
        b = np.stack([rs.integers(0, p, n), rs.integers(0, q, n), rs.integers(0, 2, n)], 1)
        a[::7, 0] = 0
        b[::5, 0] = 0
        b[::11, 1] = 0
        a[1::3, 2] = 1
        a[:, 1] *= a[:, 2]  # canonical: undefined => xq = 0
        b[:, 1] *= b[:, 2]
        res = np.zeros((6, n, 4), np.int32)  # (rc, xp, xq, qd)
        omega = pow(w, 5, p)
        for op in range(6):
            for j in range(n):
                rc, r = ref.field_op(op, a[j], b[j], omega=omega, p=p, q=q, wbase=w)
                res[op, j] = (rc,) + r
        arrays[k + "_opa"], arrays[k + "_opb"], arrays[k + "_opres"] = a, b, res
        scal["fields"].append({"p": p, "q": q, "wbase": w, "key": k, "omega": omega})

    # ---- known answers
    kat = {}
    kat["add_10_5__220_110"] = ref.field_op(0, (10, 5, 1), (220, 110, 1))[1]
    kat["div_10_3"] = ref.field_op(3, (10, 0, 0), (3, 0, 0))[1]
    kat["sqrt_4_4"] = ref.field_op(5, (4, 4, 1))[1]
    kat["exp_5_1_omega4"] = ref.field_op(4, (5, 1, 1), omega=4)[1]
    kat["rng0_first3"] = [f"{int(x):016x}" for x in ref.rng_draws(0, 3)]
    kat["derive7_0_first"] = f"{int(ref.rng_draws(7, 1, 0)[0]):016x}"
    scal["kat"] = kat

    # ---- graphs: programs, a slice of each pool, edge graphs
    fams = F.verify_families()
    for f, (prog, pool) in fams.items():
        graphs[f"{f}/program"] = prog
        for tag, g in pool:
            graphs[tag] = g
    for name, g in edge_graphs().items():
        graphs[f"edge/{name}"] = g
    for f, (args, gx, fl) in FP_SHAPES.items():
        graphs[f"fp/{f}/program"] = F.family_program(f, *args)
        graphs[f"fp/{f}/mugraph"] = F.family_mugraph(f, *args, grid=gx, forloop=fl)
    for f, (args, gx, fl) in FUSED_SHAPES.items():  # shapes inside the fused kernels' limits
        graphs[f"fused/{f}"] = F.family_mugraph(f, *args, grid=gx, forloop=fl)

    # ---- per-graph host facts: op_madds, validate, canonical key
    scal["graph_facts"] = {}
    for tag, g in graphs.items():
        scal["graph_facts"][tag] = {
            "madds": int(ref.op_madds(g)), "validate_48k": int(ref.validate(g, 48 * 1024)),
            "validate_b200": int(ref.validate(g)), "canonical_key_sha": hashlib.sha256(
                ref.canonical_key(g).encode()).hexdigest()[:16]}

    # ---- single FF attempts (equiv.cpp:57-68): programs, 1/6 of each pool, edges
    att_tags = [t for t in graphs if t.endswith("/program") and not t.startswith("fp/")]
    for f, (prog, pool) in fams.items():
        att_tags += [tag for tag, _ in pool[::6]]
    att_tags += [t for t in graphs if t.startswith("edge/")]
    scal["attempts"] = []
    for i, tag in enumerate(att_tags):
        for seed, stream in ((0, 0), (12345, 1), (3, 131071)):
            a = ref.ff_attempt(graphs[tag], seed, stream)
            k = f"att_{len(scal['attempts'])}"
            rec = {"tag": tag, "seed": seed, "stream": stream, "rc": int(a["rc"]),
                   "omega": int(a["omega"]), "key": k,
                   "in_sha": hashlib.sha256(a["in_xp"].tobytes() + a["in_xq"].tobytes()).hexdigest()}
            arrays[k + "_in_xp"] = a["in_xp"][:64]
            arrays[k + "_in_xq"] = a["in_xq"][:64]
            if a["rc"] == 0:
                arrays[k + "_xp"] = np.concatenate([o[0].reshape(-1) for o in a["out"]])
                arrays[k + "_xq"] = np.concatenate(
                    [np.where(o[2], o[1], 0).reshape(-1) for o in a["out"]]).astype(np.uint16)
                arrays[k + "_qd"] = np.concatenate([o[2].reshape(-1) for o in a["out"]])
            scal["attempts"].append(rec)

    # ---- verdicts of the sharded pool form (candidate i = pool[i % n], seed i)
    for f, (prog, pool) in fams.items():
        v, _ = ref.verify_batch(prog, [g for _, g in pool], 0, VERDICT_N, threads=8)
        arrays[f"verdicts_{f}"] = v
    # explicit multi-round configs on a few pairs
    scal["rte"] = []
    for f, (prog, pool) in fams.items():
        for j in (0, 1, 7):
            tag, g = pool[j]
            for nt, mr, seed in ((1, 16, 5), (4, 16, 11), (2, 0, 2), (3, 3, 99)):
                scal["rte"].append({"program": f"{f}/program", "cand": tag, "num_tests": nt,
                                    "max_resamples": mr, "seed": seed,
                                    "verdict": ref.random_test_equivalence(prog, g, nt, seed, mr)})

    # ---- fp eval_mugraph / eval_program (double) on seeded inputs
    scal["fp"] = []
    for f, (args, gx, fl) in FP_SHAPES.items():
        mu = graphs[f"fp/{f}/mugraph"]
        prog = graphs[f"fp/{f}/program"]
        rs = np.random.default_rng(42)
        ins = []
        for t in mu["inputs"]:
            shp = mu["tensors"][t]["shape"]
            x = rs.standard_normal(shp) * (1.0 / np.sqrt(shp[-1]) if f != "rmsnorm" else 1.0)
            ins.append(x.astype(np.float32).astype(np.float64))
        if f == "rmsnorm":
            ins[3] = np.full((1, 1), 1.0 / args[1])
        for i, x in enumerate(ins):
            arrays[f"fp_{f}_in{i}"] = x
        arrays[f"fp_{f}_mugraph"] = ref.eval_mugraph(mu, ins, mode=0)[0]
        arrays[f"fp_{f}_program"] = ref.eval_mugraph(prog, ins, mode=1)[0]
        arrays[f"fp_{f}_f32"] = ref.eval_mugraph(mu, ins, mode=2)[0]
        scal["fp"].append({"family": f, "n_inputs": len(ins)})
    # SPEC.md:613 RMSNorm known answer
    kg = F.family_mugraph("rmsnorm", 1, 2, 2, grid=1, forloop=1)
    kat["rmsnorm_3_4"] = [float(v) for v in ref.eval_mugraph(
        kg, [np.array([[3.0, 4.0]]), np.array([[1.0, 1.0]]), np.eye(2), np.array([[0.5]])])[0][0]]
    graphs["kat/rmsnorm_1x2"] = kg
    # stability filter verdicts (stability.cpp:25-50)
    scal["stability"] = []
    for f in ("gatedmlp", "lora"):
        prog, pool = fams[f]
        for tag, g in pool[:4]:
            scal["stability"].append({"program": f"{f}/program", "cand": tag,
                                      "ok": ref.float_stability_filter(g, prog, trials=2)})

    with open(os.path.join(HERE, "graphs.json"), "w") as fh:
        json.dump(graphs, fh, separators=(",", ":"))
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(scal, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    sz = sum(os.path.getsize(os.path.join(HERE, n)) for n in ("graphs.json", "golden.json", "golden.npz"))
    print(f"wrote {len(graphs)} graphs, {len(arrays)} arrays, {sz / 1e6:.2f} MB")


if __name__ == "__main__":
    main()

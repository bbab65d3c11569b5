"""Thread-graph construction (the reference's absent
fusion.cpp): groups, fan-out rule, and — against the compiled reference —
validity, shared-memory accounting with register-resident edges
(validate.cpp:115-140), serialization round trip and unchanged semantics
(random_test_equivalence of the unfused and fused graphs)."""
import json
import os

import pytest

from oracle import ref
from paper_2405_05751_b200 import api
from paper_2405_05751_b200 import fixtures as F
from paper_2405_05751_b200.graph import PHI, BlockBuilder, GraphBuilder, OpType as O

HERE = os.path.dirname(os.path.abspath(__file__))
GRAPHS = json.load(open(os.path.join(HERE, "golden", "graphs.json")))
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def _groups(g):
    out = []
    for op in g["ops"]:
        for tg in op.get("blockGraph", {}).get("threadGroups", []):
            types = [op["blockGraph"]["ops"][i]["type"] for i in tg["ops"]]
            out.append((types, tg["forloop"]))
    return out


def test_rmsnorm_post_chain_is_one_group():
    g = api.construct_thread_graphs(F.family_mugraph("rmsnorm", 1, 64, 64, grid=4, forloop=4))
    assert _groups(g) == [(["sqrt", "ewdiv"], 1)]


def _paper_rmsnorm():
    """Fig. 2(b): post-loop Mul -> Sqrt -> Div chain (§4.2)."""
    gb = GraphBuilder()
    X, G, W, D = gb.input([1, 64]), gb.input([1, 64]), gb.input([64, 64]), gb.input([1, 1])
    bb = BlockBuilder([4, 1, 1], 4, [[1, 64], [1, 64], [64, 64], [1, 1]])
    xb, gbar = bb.initer(0, [PHI], [1]), bb.initer(1, [PHI], [1])
    wb, db = bb.initer(2, [1], [0]), bb.initer(3, [PHI], [PHI])
    B = bb.op(O.Accum, [bb.op(O.Matmul, [bb.op(O.EwMul, [xb, gbar]), wb])], {"fmap": [PHI]})
    A = bb.op(O.Accum, [bb.op(O.Sum, [bb.op(O.Sqr, [xb])], {"dim": 1, "group": 16})], {"fmap": [PHI]})
    r = bb.op(O.Sqrt, [bb.op(O.EwMul, [A, db])])
    bb.outsaver(bb.op(O.EwDiv, [B, r]), [1])
    return gb.finish([gb.graphdef([X, G, W, D], bb)])


def test_paper_mul_sqrt_div_chain():
    g = api.construct_thread_graphs(_paper_rmsnorm())
    assert _groups(g) == [(["ewmul", "sqrt", "ewdiv"], 1)]


def test_no_fusion_past_fanout():
    gb = GraphBuilder()
    x, y = gb.input([4, 8]), gb.input([4, 8])
    bb = BlockBuilder([2, 1, 1], 2, [[4, 8], [4, 8]])
    xb, yb = bb.initer(0, [0], [1]), bb.initer(1, [0], [1])
    e = bb.op(O.EwExp, [xb])                       # fan-out: two consumers
    m = bb.op(O.EwMul, [e, yb])
    a = bb.op(O.EwAdd, [e, yb])
    s = bb.op(O.Sqr, [bb.op(O.EwAdd, [m, a])])     # add -> sqr chain
    acc = bb.op(O.Accum, [s], {"fmap": [PHI]})
    bb.outsaver(acc, [0])
    g = api.construct_thread_graphs(gb.finish([gb.graphdef([x, y], bb)]))
    groups = _groups(g)
    assert (["ewexp"] not in [t for t, _ in groups])
    flat = [t for ts, _ in groups for t in ts]
    assert flat.count("ewexp") == 0  # the exp stays alone
    assert any(ts == ["ewmul", "ewadd", "ewadd", "sqr"] and fl == 2 for ts, fl in groups)


@needs_ref
@pytest.mark.parametrize("tag", [t for t in GRAPHS if "/g" in t or t.startswith(("fp/", "fused/", "edge/"))][::4])
def test_fused_graphs_against_reference(tag):
    g = GRAPHS[tag]
    f = api.construct_thread_graphs(g)
    assert ref.validate(f) == ref.validate(g) == 0 or ref.validate(f) <= ref.validate(g)
    assert api.validate(f)[0] == ref.validate(f)
    assert api.validate(f, smem_bytes=48 * 1024)[0] == ref.validate(f, smem_bytes=48 * 1024)
    for k, op in enumerate(f["ops"]):
        if op["type"] == "graphdef":
            assert ref.block_shared_bytes(f, k) <= ref.block_shared_bytes(g, k)
    assert ref.roundtrip_json(f) == ref.roundtrip_json(ref.roundtrip_json(f))
    v = ref.random_test_equivalence(g, f, num_tests=2, seed=3)
    assert v["kind"] in (0, 2) and v["kind"] != 1

"""Block-graph scheduling and shared-memory planning (the reference's absent
schedule.cpp / memplan.cpp; SPEC.md:527-545 — schedule_ops, plan_memory),
checked against the SPEC's examples and independently coded brute forces:
all topological orders for the minimal number of sync points, all placement
orders for the minimal peak."""
import itertools
import random

import pytest

from paper_2405_05751_b200 import api
from paper_2405_05751_b200 import _native as N
from paper_2405_05751_b200 import fixtures as F
from paper_2405_05751_b200.graph import PHI, BlockBuilder, ErrCode, GraphBuilder, OpType as O


def _plan(g, **kw):
    return api.plan_block_graphs(g, **kw)["graphdefs"]


def _block(g, k=0):
    return [op for op in g["ops"] if "blockGraph" in op][k]["blockGraph"]


# ------------------------------------------------------------ schedule_ops
def _chain():
    """InIter -> Exp -> Sqr -> Accum -> OutSaver: a linear chain."""
    gb = GraphBuilder()
    x = gb.input([4, 8])
    bb = BlockBuilder([2, 1, 1], 2, [[4, 8]])
    xb = bb.initer(0, [0], [1])
    a = bb.op(O.Accum, [bb.op(O.Sqr, [bb.op(O.EwExp, [xb])])], {"fmap": [PHI]})
    bb.outsaver(a, [0])
    return gb.finish([gb.graphdef([x], bb)])


def test_linear_chain_depths_and_syncs():
    p = _plan(_chain())[0]
    d = p["depth"]
    # SPEC example: a chain of 3 ops -> depths 1, 2, 3 and 2 sync points among them
    assert d[:3] == [1, 2, 3]
    assert p["order"][:3] == [0, 1, 2]
    assert [s for s in p["sync_after"] if s < 2] == [0, 1]
    assert d == [1, 2, 3, 4, 5]


def _paper_rmsnorm():
    """Fig. 2(b) topology: two parallel Accum chains (no D input)."""
    gb = GraphBuilder()
    X, G, W = gb.input([1, 64]), gb.input([1, 64]), gb.input([64, 64])
    bb = BlockBuilder([4, 1, 1], 4, [[1, 64], [1, 64], [64, 64]])
    xb, gbar = bb.initer(0, [PHI], [1]), bb.initer(1, [PHI], [1])
    wb = bb.initer(2, [1], [0])
    B = bb.op(O.Accum, [bb.op(O.Matmul, [bb.op(O.EwMul, [xb, gbar]), wb])], {"fmap": [PHI]})
    A = bb.op(O.Accum, [bb.op(O.Sum, [bb.op(O.Sqr, [xb])], {"dim": 1, "group": 16})], {"fmap": [PHI]})
    bb.outsaver(bb.op(O.EwDiv, [B, bb.op(O.Sqrt, [A])]), [1])
    return gb.finish([gb.graphdef([X, G, W], bb)])


def test_paper_accums_share_a_depth():
    g = _paper_rmsnorm()
    bg = _block(g)
    p = _plan(g)[0]
    accs = [i for i, op in enumerate(bg["ops"]) if op["type"] == "accum"]
    assert len(accs) == 2
    assert p["depth"][accs[0]] == p["depth"][accs[1]]
    # adjacent in the order, no sync point between them
    pos = [p["order"].index(a) for a in accs]
    assert abs(pos[0] - pos[1]) == 1 and min(pos) not in p["sync_after"]


def _diamond():
    gb = GraphBuilder()
    x = gb.input([4, 8])
    bb = BlockBuilder([2, 1, 1], 2, [[4, 8]])
    xb = bb.initer(0, [0], [1])
    s = bb.op(O.EwAdd, [bb.op(O.EwExp, [xb]), bb.op(O.Sqr, [xb])])
    bb.outsaver(bb.op(O.Accum, [s], {"fmap": [PHI]}), [0])
    return gb.finish([gb.graphdef([x], bb)])


def _min_phases(ops, pre):
    """Brute force: every topological order of `ops` (pre[k] = producers),
    greedily cut into barrier phases (a new phase when an op reads a value
    produced in the current one); the minimum over all orders."""
    best = None
    for perm in itertools.permutations(ops):
        seen, ok = set(), True
        for k in perm:
            if any(p in ops and p not in seen for p in pre[k]):
                ok = False
                break
            seen.add(k)
        if not ok:
            continue
        phases, cur = 1, set()
        for k in perm:
            if any(p in cur for p in pre[k]):
                phases, cur = phases + 1, set()
            cur.add(k)
        best = phases if best is None else min(best, phases)
    return best


@pytest.mark.parametrize("make", [_diamond, _paper_rmsnorm, _chain])
def test_sync_count_is_minimal(make):
    g = make()
    bg = _block(g)
    p = _plan(g)[0]
    prod = {}
    for i, op in enumerate(bg["ops"]):
        for t in op["outputs"]:
            prod[t] = i
    pre = {i: [prod[t] for t in op["inputs"] if t in prod] for i, op in enumerate(bg["ops"])}
    loop = [i for i in range(len(bg["ops"])) if not p["post"][i] and bg["ops"][i]["type"] != "outsaver"]
    syncs_in_loop = sum(1 for s in p["sync_after"] if s + 1 < len(loop))
    assert syncs_in_loop + 1 == _min_phases(loop, pre)
    assert syncs_in_loop + 1 == len({p["depth"][i] for i in loop})


def test_order_is_topological_and_phased():
    for fam in ("rmsnorm", "gatedmlp", "gqa", "lora"):
        g = F.family_mugraph(fam, *F.VERIFY_SHAPES[fam], grid=4, forloop=4) \
            if hasattr(F, "VERIFY_SHAPES") else F.verify_families()[fam][1][0][1]
        bg = _block(g)
        p = _plan(g)[0]
        pos = {k: i for i, k in enumerate(p["order"])}
        assert sorted(p["order"]) == list(range(len(bg["ops"])))
        prod = {t: i for i, op in enumerate(bg["ops"]) for t in op["outputs"]}
        for i, op in enumerate(bg["ops"]):
            for t in op["inputs"]:
                if t in prod:
                    assert pos[prod[t]] < pos[i]
        posts = [p["post"][k] for k in p["order"] if bg["ops"][k]["type"] != "outsaver"]
        assert posts == sorted(posts)  # loop body first, then post-loop


# ------------------------------------------------------------ plan_memory
def test_disjoint_lifetimes_share_space():
    off, peak, ex = api.plan_intervals([100, 80], [0, 2], [1, 3])
    assert peak == 100 and ex and off == [0, 0]


def test_overlapping_lifetimes_sum():
    off, peak, ex = api.plan_intervals([100, 80], [0, 1], [2, 3])
    assert peak == 180 and sorted(off) == [0, 100]


def _conflict(a, b):
    return a[1] <= b[2] and b[1] <= a[2]


def _brute_peak(bufs):
    """Independent brute force: every placement order, lowest-offset first fit."""
    best = None
    for perm in itertools.permutations(range(len(bufs))):
        off = {}
        peak = 0
        for v in perm:
            taken = sorted((off[u], off[u] + bufs[u][0]) for u in off if _conflict(bufs[u], bufs[v]))
            at = 0
            for lo, hi in taken:
                if at + bufs[v][0] <= lo:
                    break
                at = max(at, hi)
            off[v] = at
            peak = max(peak, at + bufs[v][0])
        best = peak if best is None else min(best, peak)
    return best


def _check_plan(bufs, off, peak):
    for i, j in itertools.combinations(range(len(bufs)), 2):
        if _conflict(bufs[i], bufs[j]):
            assert off[i] + bufs[i][0] <= off[j] or off[j] + bufs[j][0] <= off[i]
    assert peak == max(o + b[0] for o, b in zip(off, bufs))


@pytest.mark.parametrize("seed", range(12))
def test_exhaustive_matches_brute_force(seed):
    rnd = random.Random(seed)
    n = rnd.randint(3, 6)
    bufs = []
    for _ in range(n):
        s = rnd.randint(0, 8)
        bufs.append((rnd.choice([16, 48, 64, 80, 100, 128]), s, s + rnd.randint(0, 5)))
    off, peak, ex = api.plan_intervals(*zip(*bufs))
    assert ex
    _check_plan(bufs, off, peak)
    assert peak == _brute_peak(bufs)
    # the first-fit-decreasing path is valid and never below the optimum
    off2, peak2, ex2 = api.plan_intervals(*zip(*bufs), exhaustive_max=0)
    assert not ex2
    _check_plan(bufs, off2, peak2)
    assert peak2 >= peak


def test_block_plan_within_reference_accounting():
    for fam in ("rmsnorm", "gatedmlp", "gqa", "lora"):
        g = F.verify_families()[fam][1][0][1]
        p = _plan(g)[0]
        bg = _block(g)
        nbytes = sum(2 * _numel(t["shape"]) for t in bg["tensors"])
        assert 0 < p["peak"] <= nbytes  # lifetime reuse never costs more than no reuse
        assert all(o >= 0 for o in p["offset"])


def _numel(shape):
    n = 1
    for d in shape:
        n *= d
    return n


def test_does_not_fit():
    g = F.verify_families()["gatedmlp"][1][0][1]
    with pytest.raises(N.NativeError) as e:
        api.plan_block_graphs(g, smem_bytes=64)
    assert e.value.status == 1000 + int(ErrCode.DoesNotFit)


def test_plan_respects_barrier_phases():
    """Ops of one depth run without a sync between them: buffers whose
    lifetimes meet in a phase never share bytes."""
    for fam in ("rmsnorm", "gatedmlp", "gqa", "lora"):
        for _, g in F.verify_families()[fam][1][:12]:
            bg = _block(g)
            p = _plan(g)[0]
            phase, ph, k = {}, 0, 0
            for pos, op in enumerate(p["order"]):
                phase[op] = ph
                if k < len(p["sync_after"]) and p["sync_after"][k] == pos:
                    ph, k = ph + 1, k + 1
            loop_end = max((phase[o] for o in p["order"] if not p["post"][o]
                            and bg["ops"][o]["type"] != "outsaver"), default=0)
            span = {}
            for o, op in enumerate(bg["ops"]):
                for t in op["outputs"]:
                    s0 = 0 if op["type"] == "accum" else phase[o]
                    e0 = loop_end if op["type"] == "accum" else phase[o]
                    lo, hi = span.get(t, (s0, e0))
                    span[t] = (min(lo, s0), max(hi, e0))
                for t in op["inputs"]:
                    lo, hi = span.get(t, (phase[o], phase[o]))
                    span[t] = (lo, max(hi, phase[o]))
            sizes = {t["id"]: 2 * _numel(t["shape"]) for t in bg["tensors"]}
            live = [t for t in span if p["offset"][t] >= 0]
            for i, a in enumerate(live):
                for b in live[i + 1:]:
                    if span[a][0] <= span[b][1] and span[b][0] <= span[a][1]:
                        oa, ob = p["offset"][a], p["offset"][b]
                        assert oa + sizes[a] <= ob or ob + sizes[b] <= oa, (fam, a, b)

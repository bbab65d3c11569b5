"""GPU parity of the Z_p x Z_q path against the compiled reference (oracle/_ref).

Bit-exact: sampled inputs, omega, FF output tensors (xp, xq, q_defined) of
single attempts, and every EquivVerdict field (kind, rounds_run, resamples,
witness) of batched verification.
"""
import numpy as np
import pytest

from oracle import ref
from paper_2405_05751_b200 import _native as N
from paper_2405_05751_b200 import api
from paper_2405_05751_b200 import fixtures as F
from paper_2405_05751_b200.graph import PHI, BlockBuilder, GraphBuilder, OpType as O

pytestmark = pytest.mark.gpu

FAMS = F.verify_families()


def _graphs():
    out = []
    for f, (prog, pool) in FAMS.items():
        out.append((f + "/program", prog))
        out += pool
    return out


ALL = _graphs()


def _same_attempt(a, b, tag):
    assert (a["rc"] != 0) == (b["rc"] != 0), (tag, a["rc"], b["rc"])
    assert a["omega"] == b["omega"], tag
    assert np.array_equal(a["in_xp"], b["in_xp"]) and np.array_equal(a["in_xq"], b["in_xq"]), tag
    if a["rc"] == 0:
        for (xp, xq, qd), (yp, yq, yd) in zip(a["out"], b["out"]):
            assert np.array_equal(xp, yp), tag
            assert np.array_equal(qd.astype(bool), yd.astype(bool)), tag
            assert np.array_equal(np.where(qd, xq, 0), np.where(yd, yq, 0)), tag


@pytest.mark.parametrize("stream", [0, 5, 131071])
def test_ff_attempt_bit_exact_all_pool_graphs(ctx, stream):
    for tag, g in ALL:
        for seed in (0, 12345):
            a = ref.ff_attempt(g, seed, stream)
            b = ctx.ff_eval(g, seed, stream)
            _same_attempt(a, b, (tag, seed, stream))


VCOLS = ["kind", "rounds_run", "resamples", "has_witness", "w_seed", "w_round", "w_omega",
         "w_tensor", "w_index"]


def _cmp_verdicts(a, b, ctxmsg=""):
    for c in VCOLS:
        bad = np.nonzero(a[c] != b[c])[0]
        assert bad.size == 0, f"{ctxmsg} field {c}: {bad.size} mismatches, first {bad[:5]}"


@pytest.mark.parametrize("fam", list(FAMS))
def test_verify_pool_matches_reference(ctx, fam):
    prog, pool = FAMS[fam]
    graphs = [g for _, g in pool]
    n = 2500
    want, _ = ref.verify_batch(prog, graphs, first=0, n=n, threads=8)
    got, att = ctx.verify_pool(prog, graphs, first=0, n=n, want_verdicts=True)
    _cmp_verdicts(want, got, fam)
    assert att == int((want["resamples"] + want["rounds_run"]).sum())


def test_verify_batch_explicit_seeds_and_rounds(ctx):
    prog, pool = FAMS["rmsnorm"]
    rng = np.random.default_rng(1)
    idx = rng.integers(0, len(pool), 400)
    seeds = rng.integers(0, 2**63, 400, dtype=np.uint64)
    cands = [pool[i][1] for i in idx]
    for num_tests, maxr in ((1, 16), (4, 16), (2, 0), (3, 3)):
        got, acc = ctx.verify_batch(prog, cands, seeds, num_tests=num_tests, max_resamples=maxr)
        for k in range(0, 400, 7):
            w = ref.random_test_equivalence(prog, cands[k], num_tests=num_tests, seed=int(seeds[k]),
                                            max_resamples=maxr)
            for c in VCOLS:
                assert got[c][k] == w[c], (num_tests, maxr, k, c, got[k], w)
        assert np.array_equal(acc, got["kind"] == 0)


def test_random_test_equivalence_pair(ctx):
    prog, pool = FAMS["gatedmlp"]
    for tag, g in pool[:6]:
        for seed in (0, 7, 99):
            w = ref.random_test_equivalence(prog, g, num_tests=2, seed=seed)
            v = ctx.random_test_equivalence(prog, g, num_tests=2, seed=seed)
            for c in VCOLS:
                assert v[c] == w[c], (tag, seed, c)


# ---- edge-case graphs -------------------------------------------------------

def _edge_graphs():
    gs = {}
    # identity: output is an input
    gb = GraphBuilder()
    x = gb.input([4, 8])
    gs["identity"] = gb.finish([x])
    # broadcasting, repeat, reshape, sum groups, sqrt/div resampling, exp + silu
    gb = GraphBuilder()
    x, y = gb.input([2, 4, 8]), gb.input([1, 8])
    a = gb.op(O.EwMul, [x, y])
    r = gb.op(O.Repeat, [y], {"target": [2, 4, 8]})
    s = gb.op(O.Sum, [gb.op(O.EwAdd, [a, r])], {"dim": 2, "group": 4})
    q = gb.op(O.Sqrt, [gb.op(O.Sqr, [s])])
    d = gb.op(O.EwDiv, [s, q])
    e = gb.op(O.SiLU, [gb.op(O.EwExp, [gb.op(O.Reshape, [d], {"target": [4, 4]})])])
    gs["mixed_kernel"] = gb.finish([e, d])
    # grid axis absent from omap (last block wins), concat accum, 2-D grid
    gb = GraphBuilder()
    x, w = gb.input([4, 16]), gb.input([16, 8])
    bb = BlockBuilder([2, 3, 1], 4, [[4, 16], [16, 8]])
    xb = bb.initer(0, [PHI, PHI], [1])
    wb = bb.initer(1, [1, PHI], [0])
    m = bb.op(O.Accum, [bb.op(O.Matmul, [xb, wb])], {"fmap": [PHI]})
    cc = bb.op(O.Accum, [xb], {"fmap": [1]})
    bb.outsaver(m, [1])
    bb.outsaver(bb.op(O.EwAdd, [cc, cc]), [0])
    outs = gb.g  # noqa
    gd = gb.graphdef([x, w], bb)
    gs["omap_partial"] = gb.finish([gd, gd + 1])
    # ConcatMatmul inside a block, imap on two axes
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


EDGE = _edge_graphs()


@pytest.mark.parametrize("name", list(EDGE))
def test_edge_graph_attempts(ctx, name):
    g = EDGE[name]
    for seed in range(6):
        for stream in (0, 1, 2):
            a = ref.ff_attempt(g, seed, stream)
            b = ctx.ff_eval(g, seed, stream)
            _same_attempt(a, b, (name, seed, stream))


def test_edge_self_equivalence_and_resamples(ctx):
    for name, g in EDGE.items():
        for seed in range(20):
            w = ref.random_test_equivalence(g, g, num_tests=2, seed=seed)
            v = ctx.random_test_equivalence(g, g, num_tests=2, seed=seed)
            for c in VCOLS:
                assert v[c] == w[c], (name, seed, c, v, w)


def test_other_field_params(ctx):
    # p = 103, q = 17 (17 | 102); 8^17 = 1 mod 103 with 8 != 1
    p, q = 103, 17
    wb = next(b for b in range(2, p) if pow(b, q, p) == 1)
    prog, pool = FAMS["lora"]
    for tag, g in pool[:10]:
        for seed in range(3):
            w = ref.random_test_equivalence(prog, g, seed=seed, p=p, q=q, wbase=wb)
            v = ctx.random_test_equivalence(prog, g, seed=seed, p=p, q=q, wbase=wb)
            for c in VCOLS:
                assert v[c] == w[c], (tag, seed, c)


def test_shape_mismatch_is_error_verdict(ctx):
    prog, _ = FAMS["rmsnorm"]
    other, _ = FAMS["gatedmlp"]
    got, acc = ctx.verify_batch(prog, [other], [0])
    assert got["kind"][0] == 3 and got["err_code"][0] == 1000  # ShapeMismatch
    assert not acc[0]


def test_distinct_candidate_stream_matches_reference(ctx):
    """The search-loop path: every candidate a distinct handle compiled from
    JSON text on all host cores (tpo_gpu_compile_many) and verified in one
    batch (parallel lowering + bytecode assembly) — verdicts bit-exact."""
    import json
    rng = np.random.default_rng(7)
    for fam in ("rmsnorm", "gqa", "lora", "gatedmlp"):
        prog, pool = FAMS[fam]
        # the pool, the generator's candidates and their mutants
        bases = [g for _, g in pool] + api.generate(prog, grids=[1, 2, 4, 8, 16], loops=[1, 2, 4, 8, 16])
        stream = F.search_stream(bases, 3000, seed=5)
        idx = rng.integers(0, len(stream), 300)
        cands = [stream[i] for i in idx]
        texts = [json.dumps(g) for g in cands]
        gs, st = ctx.compile_many(texts)
        assert all(s == 0 for s in st)
        assert len({g.h.value for g in gs}) == len(gs)  # no dedup: 300 distinct handles
        seeds = rng.integers(0, 2**62, 300, dtype=np.uint64)
        got, acc = ctx.verify_batch(prog, gs, seeds)
        for k in range(0, 300, 3):
            w = ref.random_test_equivalence(prog, cands[k], num_tests=1, seed=int(seeds[k]))
            for c in VCOLS:
                assert got[c][k] == w[c], (fam, k, c)
        assert np.array_equal(acc, got["kind"] == 0)
        # the handle-array fast path (compile_many(batch=True)): same verdicts
        gb, st2 = ctx.compile_many(texts, batch=True)
        assert len(gb) == 300 and all(s == 0 for s in st2)
        got2, acc2 = ctx.verify_batch(prog, gb, seeds)
        assert np.array_equal(got2, got) and np.array_equal(acc2, acc)


@pytest.mark.parametrize("fam", ["rmsnorm", "lora", "gqa"])
def test_same_seed_batch_matches_reference(ctx, fam):
    """A search loop verifies every candidate with the VerifyConfig seed:
    the batch's first attempt (inputs, tables, program outputs) is computed
    once and shared.  Verdicts stay bit-exact, including seeds whose first
    attempt the program itself must resample (RMSNorm's sqrt)."""
    prog, pool = FAMS[fam]
    graphs = [g for _, g in pool]
    cands = [graphs[i % len(graphs)] for i in range(96)]
    for seed in range(6):
        seeds = np.full(len(cands), seed, dtype=np.uint64)
        for num_tests in (1, 2):
            got, acc = ctx.verify_batch(prog, cands, seeds, num_tests=num_tests)
            for k in range(0, len(cands), 5):
                w = ref.random_test_equivalence(prog, cands[k], num_tests=num_tests, seed=seed)
                for c in VCOLS:
                    assert got[c][k] == w[c], (fam, seed, num_tests, k, c)
            assert np.array_equal(acc, got["kind"] == 0)


def test_generated_candidates_verify_on_gpu(ctx):
    """The search-loop caller end to end: candidates from the fused-kernel
    generator (tpo_gpu_generate) verified on the GPU with the VerifyConfig
    seed; verdicts bit-exact with the reference, all Equivalent."""
    from paper_2405_05751_b200 import api
    for fam in ("rmsnorm", "gatedmlp", "gqa", "lora"):
        prog, _ = FAMS[fam]
        cands = api.generate(prog, grids=[1, 2, 4, 8, 16], loops=[1, 2, 4, 8, 16])
        gs, st = ctx.compile_many(cands)
        assert all(s == 0 for s in st)
        seeds = np.zeros(len(gs), dtype=np.uint64)
        got, acc = ctx.verify_batch(prog, gs, seeds, num_tests=2)
        for k in range(len(cands)):
            w = ref.random_test_equivalence(prog, cands[k], num_tests=2, seed=0)
            for c in VCOLS:
                assert got[c][k] == w[c], (fam, k, c)
        assert (got["kind"] != 1).all()


def test_optimize_pipeline(ctx):
    """generate -> verify -> stability -> select (SPEC Fig. 1 flow) on the
    GPU: stage counts non-increasing, the winner is one fused kernel that the
    reference verifies Equivalent."""
    from paper_2405_05751_b200 import pipeline
    prog, _ = FAMS["gatedmlp"]
    rep = pipeline.optimize(ctx, prog, grids=[1, 2, 4, 8, 16], loops=[1, 2, 4, 8, 16])
    assert rep["generated"] >= rep["compiled"] >= rep["verified"] >= rep["stable"] > 0
    best = rep["best"]
    assert [op["type"] for op in best["ops"]] == ["graphdef"]
    assert ref.random_test_equivalence(prog, best, num_tests=4, seed=5)["kind"] == 0
    assert "forloop" in rep["describe"]
    # with the kernel level: more candidates survive, the single fused
    # kernel still ranks first (fewer launches and device bytes)
    rep3 = pipeline.optimize(ctx, prog, grids=[1, 2, 4, 8, 16], loops=[1, 2, 4, 8, 16], max_kernels=3)
    assert rep3["generated"] > rep["generated"] and rep3["stable"] > rep["stable"]
    assert [op["type"] for op in rep3["best"]["ops"]] == ["graphdef"]


def test_rejection_rate_and_no_false_negatives(ctx):
    """SPEC acceptance: over 1000 seeds, >= 99% rejection
    of non-equivalent pairs at num_tests=4 (20 mutant pairs, 5 per family;
    Inconclusive verdicts — exhausted sqrt resampling, ~1% for RMSNorm,
    identical in the reference — are excluded) and no false negatives for
    the equivalent variants.""" 
    for fam in ("rmsnorm", "gatedmlp", "gqa", "lora"):
        prog, pool = FAMS[fam]
        muts = [g for tag, g in pool if tag.endswith("/mut")][:5]
        eqs = [g for tag, g in pool if tag.endswith("/eq")][:5]
        seeds = np.arange(1000, dtype=np.uint64)
        for g in muts:
            got, acc = ctx.verify_batch(prog, [g] * 1000, seeds, num_tests=4)
            assert not acc.any(), fam  # never accepted
            decided = got["kind"] != 2  # Inconclusive: sqrt resampling exhausted (~1% for RMSNorm)
            assert (got["kind"][decided] == 1).mean() >= 0.99 and decided.mean() >= 0.97, fam
        for g in eqs:
            got, acc = ctx.verify_batch(prog, [g] * 1000, seeds, num_tests=4)
            assert not (got["kind"] == 1).any(), fam  # Equivalent or (sqrt) Inconclusive, never rejected


@pytest.mark.parametrize("name", ["rmsnorm", "lora"])
def test_full_shape_verification_matches_reference(ctx, name):
    """random_test_equivalence at BASELINE shapes, beyond shared memory: the
    global-memory field executor (VM words in HBM, one launch per
    instruction) returns the reference's verdict field for field, for the
    benchmark µGraph against its program and for a mutant (witness)."""
    prog, mu = F.bench_pair(name)
    b = F.BENCH[name]
    mut = F.family_mugraph(name, *b["args"], grid=b["grid"], forloop=b["forloop"], mutant=True)
    wants = []
    for cand in (mu, mut):
        got = ctx.random_test_equivalence(prog, cand, num_tests=1, seed=3)
        want = ref.random_test_equivalence(prog, cand, num_tests=1, seed=3)
        wants.append(want)
        for c in VCOLS:
            assert got[c] == want[c], (name, c, got, want)
    # the batched entry point falls back to the same executor
    got, acc = ctx.verify_batch(prog, [mu, mut], np.array([3, 3], dtype=np.uint64))
    for k in range(2):
        for c in VCOLS:
            assert got[c][k] == wants[k][c], (name, k, c)
    assert list(acc) == [w["kind"] == 0 for w in wants]


def _exp_heavy(fam, n, seed):
    """Search-stream mutants with two or more EwExp ops: most exponentiate a
    q-undefined value (PoisonedExponent unless a resample comes first)."""
    prog, pool = FAMS[fam]
    bases = [g for _, g in pool] + api.generate(prog, grids=[1, 2, 4, 8, 16], loops=[1, 2, 4, 8, 16])
    out = []
    for g in F.search_stream(bases, 6000, seed=seed):
        ops = [o["type"] for op in g["ops"] for o in op.get("blockGraph", {}).get("ops", [])]
        if ops.count("ewexp") >= 2:
            out.append(g)
    return prog, out[:n]


@pytest.mark.parametrize("fam", ["rmsnorm", "gqa", "lora", "gatedmlp"])
def test_poisoned_exponent_ordering_matches_reference(ctx, fam):
    """Error(PoisonedExponent) is raised where the reference evaluates the
    offending EwExp: a DivByZero / NonResidue evaluated before it (the
    program, earlier ops, grid block 0 of its GraphDef) turns the attempt
    into a resample (Inconclusive after 17), any later one does not."""
    prog, cands = _exp_heavy(fam, 120, seed=11)
    assert len(cands) >= 40
    rng = np.random.default_rng(3)
    seeds = rng.integers(0, 2**62, len(cands), dtype=np.uint64)
    got, acc = ctx.verify_batch(prog, cands, seeds)
    kinds = set()
    for k, g in enumerate(cands):
        w = ref.random_test_equivalence(prog, g, num_tests=1, seed=int(seeds[k]))
        kinds.add((w["kind"], w["err_code"]))
        for c in VCOLS:
            assert got[c][k] == w[c], (fam, k, c, w)
    assert (3, 1006) in kinds


def test_poisoned_ff_eval_status_matches_reference(ctx):
    """tpo_gpu_ff_eval: ResampleNeeded (2000 + code) or Error(PoisonedExponent)
    by evaluation order, as ff_eval throws."""
    _, cands = _exp_heavy("rmsnorm", 30, seed=13)
    for g in cands:
        for stream in range(3):
            w = ref.ff_attempt(g, 5, stream)
            try:
                rc = ctx.ff_eval(g, 5, stream)["rc"]
            except N.NativeError as e:
                rc = e.status
            assert rc == w["rc"], (stream, rc, w["rc"])


def test_poisoned_exponent_global_executor(ctx, monkeypatch):
    """The global-memory field executor (graphs beyond shared memory) stops
    at the same VM_RAISE with the same event rule."""
    prog, cands = _exp_heavy("gqa", 36, seed=17)
    seeds = np.arange(len(cands), dtype=np.uint64) * 7 + 1
    monkeypatch.setenv("TPO_VM_GLOBAL", "1")
    got, _ = ctx.verify_batch(prog, cands, seeds)
    monkeypatch.delenv("TPO_VM_GLOBAL")
    for k, g in enumerate(cands):
        w = ref.random_test_equivalence(prog, g, num_tests=1, seed=int(seeds[k]))
        for c in VCOLS:
            assert got[c][k] == w[c], (k, c, w)


@pytest.mark.parametrize("fam", ["rmsnorm", "gatedmlp", "gqa", "lora"])
def test_ff_attempt_bit_exact_on_mutants(ctx, fam):
    """One verifier attempt (inputs, ω, outputs, resample status) on
    search-stream mutants: bit-exact with the reference."""
    prog, pool = FAMS[fam]
    bases = [g for _, g in pool] + api.generate(prog, grids=[1, 2, 4, 8, 16], loops=[1, 2, 4, 8, 16])
    s = F.search_stream(bases, 3000, seed=29)[len(bases):]
    for g in s[::max(1, len(s) // 30)][:30]:
        w = ref.ff_attempt(g, 19, 0)
        try:
            got = ctx.ff_eval(g, 19, 0)
        except N.NativeError as e:
            assert e.status == w["rc"]
            continue
        assert got["rc"] == w["rc"] and got["omega"] == w["omega"]
        if got["rc"] == 0:
            for (a, b, c), (x, y, z) in zip(got["out"], w["out"]):
                assert np.array_equal(a, x) and np.array_equal(c, z)
                assert np.array_equal(b[c == 1], y[z == 1])


@pytest.mark.parametrize("fam", ["rmsnorm", "gatedmlp", "gqa", "lora"])
def test_multi_kernel_candidates_verified_like_reference(ctx, fam):
    """Generator µGraphs of 2-4 kernels (kernel-level ops + GraphDefs) through
    the batched verifier: every verdict field equals the reference's."""
    prog, _ = FAMS[fam]
    cands = api.generate(prog, grids=[1, 2, 4], loops=[1, 2, 4], max_kernels=4)
    cands = [g for g in cands if len(g["ops"]) > 1][::5][:80]
    seeds = np.arange(len(cands), dtype=np.uint64) * 977 + 3
    got, acc = ctx.verify_batch(prog, cands, seeds)
    for k, g in enumerate(cands):
        w = ref.random_test_equivalence(prog, g, num_tests=1, seed=int(seeds[k]))
        for c in VCOLS:
            assert got[c][k] == w[c], (fam, k, c)
    assert acc.sum() >= len(cands) * 3 // 4


def test_concurrent_contexts_match_sequential(ctx):
    """SURVEY §8b threading: the reference is re-entrant; here a context is
    single-stream and concurrency is one context per thread.  Four threads,
    each with its own context, verify and evaluate at once: identical to the
    sequential results."""
    import threading
    from paper_2405_05751_b200.api import Context
    jobs = []
    for fam in ("rmsnorm", "gatedmlp", "gqa", "lora"):
        prog, pool = FAMS[fam]
        cands = [g for _, g in pool] * 4
        seeds = np.arange(len(cands), dtype=np.uint64) * 13 + 1
        jobs.append((prog, cands, seeds))
    want = []
    for prog, cands, seeds in jobs:
        v, a = ctx.verify_batch(prog, cands, seeds)
        want.append((v, a, ctx.ff_eval(cands[1], 9, 0)))
    got, errs = [None] * len(jobs), []

    def work(i):
        try:
            c = Context(0)
            prog, cands, seeds = jobs[i]
            out = []
            for _ in range(3):
                v, a = c.verify_batch(prog, cands, seeds)
                out.append((v, a, c.ff_eval(cands[1], 9, 0)))
            got[i] = out
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i, (v, a, fe) in enumerate(want):
        for gv, ga, gfe in got[i]:
            for c in VCOLS:
                assert np.array_equal(gv[c], v[c]), (i, c)
            assert np.array_equal(ga, a)
            assert gfe["rc"] == fe["rc"] and gfe["omega"] == fe["omega"]
            for x, y in zip(gfe["out"], fe["out"]):
                assert all(np.array_equal(p, q) for p, q in zip(x, y))


@pytest.mark.parametrize("fam", ["rmsnorm", "gatedmlp", "gqa", "lora"])
def test_attribute_mutants_verified_like_reference(ctx, fam):
    """Re-partitioned / re-mapped µGraphs that still pass validate (grid,
    for-loop, imap / fmap / omap, Accum fmap, Sum dim / group redrawn): every
    verdict field equals the reference's, and so does fp64 evaluation."""
    prog, pool = FAMS[fam]
    bases = [g for _, g in pool] + api.generate(prog, grids=[1, 2, 4], loops=[1, 2, 4], max_kernels=3)
    cands = [g for g in F.attribute_mutants(bases, 600, seed=9) if ref.validate(g) == 0][:60]
    assert len(cands) >= 30
    seeds = np.arange(len(cands), dtype=np.uint64) * 7 + 11
    got, _ = ctx.verify_batch(prog, cands, seeds)
    for k, g in enumerate(cands):
        w = ref.random_test_equivalence(prog, g, num_tests=1, seed=int(seeds[k]))
        for c in VCOLS:
            assert got[c][k] == w[c], (fam, k, c, w)
    rs = np.random.default_rng(2)
    for g in cands[::6]:
        ins = [rs.standard_normal(g["tensors"][t]["shape"]) for t in g["inputs"]]
        a = ctx.eval_vm(g, ins, mode=0)
        b = ref.eval_mugraph(g, ins, mode=0)
        for x, y in zip(a, b):
            assert np.allclose(x, y, rtol=1e-12, atol=1e-12, equal_nan=True)


@pytest.mark.parametrize("fam", list(FAMS))
def test_lazy_input_sampling_matches_eager(ctx, fam):
    """Lazy input sampling (each input drawn right before the program's
    first reader, TpoVmGraph::gen_*) gives the verdicts of drawing every
    input up front (TPO_VM_EAGER=1, a fresh process) field for field, and
    the kernel's draw counter accounts for exactly the skipped draws: eager
    = attempts x (2 x input elements + omega [+ SiLU tables])."""
    import json
    import os
    import subprocess
    import sys
    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prog, pool = FAMS[fam]
    graphs = [g for _, g in pool]
    n = 3000
    lazy, att = ctx.verify_pool(prog, graphs, first=0, n=n, want_verdicts=True)
    lazy_draws = ctx.last_verify_draws()
    code = (
        "import json, sys; sys.path.insert(0, %r); import numpy as np\n"
        "from paper_2405_05751_b200 import fixtures as F\n"
        "from paper_2405_05751_b200.api import Context\n"
        "prog, pool = F.verify_families()[%r]\n"
        "ctx = Context(0)\n"
        "v, att = ctx.verify_pool(prog, [g for _, g in pool], first=0, n=%d, want_verdicts=True)\n"
        "print(json.dumps({'att': att, 'draws': ctx.last_verify_draws(),"
        " 'v': {c: v[c].tolist() for c in %r}}))\n" % (ROOT, fam, n, VCOLS))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True,
                       env=dict(os.environ, TPO_VM_EAGER="1"))
    eager = json.loads(r.stdout.strip().splitlines()[-1])
    assert eager["att"] == att
    for c in VCOLS:
        assert np.array_equal(np.asarray(eager["v"][c]), lazy[c]), (fam, c)
    from paper_2405_05751_b200.graph import has_silu
    idx = np.arange(n) % len(graphs)
    silu = np.array([has_silu(g) or has_silu(prog) for g in graphs])[idx]
    a = (lazy["resamples"] + lazy["rounds_run"]).astype(np.int64)
    n_in = ctx.compile(prog).info.input_elems
    want_eager = int(np.sum(a * (2 * n_in + 1 + (227 + 113) * silu)))
    assert eager["draws"] == want_eager
    assert lazy_draws <= want_eager
    if fam == "rmsnorm":  # its program resamples at the Sqrt before the Matmul reads W
        assert lazy_draws < 0.6 * want_eager

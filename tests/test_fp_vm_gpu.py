"""GPU parity of the generic floating-point µGraph VM (kernels/fp_vm.cu)
against the compiled reference: eval_mugraph / eval_program /
eval_mugraph_f32 on any graph (bit-exact where the graph uses only
add/mul/div/sqrt, within 1e-13 relative where exp/SiLU enter), and the
float stability filter verdicts (stability.cpp:25-50), single and batched."""
import json
import os

import numpy as np
import pytest

from oracle import ref
from paper_2405_05751_b200 import fixtures as F
from paper_2405_05751_b200.graph import has_silu

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GRAPHS = json.load(open(os.path.join(HERE, "golden", "graphs.json")))


def _has_exp(g):
    types = [op["type"] for op in g["ops"]]
    for op in g["ops"]:
        types += [b["type"] for b in op.get("blockGraph", {}).get("ops", [])]
    return "ewexp" in types or "silu" in types


def _inputs(g, seed):
    """N(0,1) inputs; 1x1 inputs (the RMSNorm D = 1/d scale) positive so
    sqrt stays real."""
    rs = np.random.default_rng(seed)
    out = []
    for t in g["inputs"]:
        shp = g["tensors"][t]["shape"]
        x = rs.standard_normal(shp)
        out.append(np.abs(x) + 0.01 if int(np.prod(shp)) == 1 else x)
    return out


def _close(got, want, g):
    for a, b in zip(got, want):
        assert np.array_equal(np.isnan(a), np.isnan(b))
        if _has_exp(g):
            fa, fb = a[np.isfinite(b)], b[np.isfinite(b)]
            scale = max(np.max(np.abs(fb)), 1e-300) if fb.size else 1.0
            assert np.max(np.abs(fa - fb), initial=0.0) <= 1e-13 * scale
        else:
            assert np.array_equal(a, b, equal_nan=True), np.nanmax(np.abs(a - b))


@pytest.mark.parametrize("tag", [t for t in GRAPHS if not t.startswith(("fused/",))][::3])
def test_eval_mugraph_vm_matches_reference(ctx, tag):
    g = GRAPHS[tag]
    ins = _inputs(g, 3)
    _close(ctx.eval_vm(g, ins, mode=0), ref.eval_mugraph(g, ins, mode=0), g)


def test_eval_program_and_f32_modes(ctx):
    for f in ("rmsnorm", "gatedmlp", "gqa", "lora"):
        prog = GRAPHS[f"fp/{f}/program"]
        mu = GRAPHS[f"fp/{f}/mugraph"]
        ins = _inputs(prog, 11)
        _close(ctx.eval_vm(prog, ins, mode=1), ref.eval_mugraph(prog, ins, mode=1), prog)
        got = ctx.eval_vm(mu, ins, mode=2)
        want = ref.eval_mugraph(mu, ins, mode=2)
        for a, b in zip(got, want):
            a = a.astype(np.float64)
            assert np.array_equal(np.isnan(a), np.isnan(b))
            if _has_exp(mu):
                m = np.isfinite(b)
                assert np.max(np.abs(a[m] - b[m]), initial=0.0) <= 1e-5 * np.max(np.abs(b[m]), initial=1.0)
            else:
                assert np.array_equal(a, b, equal_nan=True), f
        with pytest.raises(Exception):
            ctx.eval_vm(mu, ins, mode=1)  # eval_program rejects GraphDefs


def test_stability_filter_single_matches_reference(ctx):
    for f in ("rmsnorm", "gatedmlp", "gqa", "lora"):
        prog, pool = F.verify_families()[f]
        for tag, g in pool[::7]:
            for trials, seed, scale in ((1, 17, 1.0), (3, 5, 2.0)):
                want = ref.float_stability_filter(g, prog, trials=trials, seed=seed, scale=scale)
                got = ctx.float_stability_filter(g, prog, trials=trials, seed=seed, scale=scale)
                assert got == want, (tag, trials, seed)


def test_stability_batch_matches_reference(ctx):
    for f in ("gatedmlp", "lora", "rmsnorm"):
        prog, pool = F.verify_families()[f]
        graphs = [g for _, g in pool]
        cands = [graphs[i % len(graphs)] for i in range(300)]
        seeds = np.arange(300, dtype=np.uint64) * 7919
        ok = ctx.stability_batch(prog, cands, seeds=seeds, trials=2)
        for k in range(0, 300, 11):
            want = ref.float_stability_filter(cands[k], prog, trials=2, seed=int(seeds[k]))
            assert ok[k] == int(want), (f, k)
        # equivalent candidates pass, mutants fail (SURVEY §8f rank 2 semantics)
        tags = [t for t, _ in pool]
        for k in range(300):
            if tags[k % len(tags)].endswith("/mut"):
                assert ok[k] == 0
    other, _ = F.verify_families()["gatedmlp"]
    prog, _ = F.verify_families()["rmsnorm"]
    assert ctx.stability_batch(prog, [other])[0] == -1


def test_global_memory_executor_matches(ctx, monkeypatch):
    """The global-memory executor (one grid-wide launch per VM instruction)
    computes exactly what the shared-memory VM does."""
    for tag in ("fp/gatedmlp/mugraph", "fp/lora/mugraph", "fp/rmsnorm/program", "edge/omap_partial",
                "edge/concatmatmul", "gqa/g4/f4/eq"):
        g = GRAPHS[tag]
        ins = _inputs(g, 5)
        smem = ctx.eval_vm(g, ins)
        monkeypatch.setenv("TPO_VM_GLOBAL", "1")
        glob = ctx.eval_vm(g, ins)
        monkeypatch.delenv("TPO_VM_GLOBAL")
        for a, b in zip(smem, glob):
            assert np.array_equal(a, b, equal_nan=True), tag


@pytest.mark.parametrize("name", ["rmsnorm", "lora"])
def test_baseline_shape_eval_bit_exact(ctx, name):
    """eval_mugraph of the BASELINE µGraph and eval_program of its flat
    program at full size on the GPU (global-memory executor, fp64) are
    bit-identical to the compiled reference (no exp in these graphs)."""
    prog, mu = F.bench_pair(name)
    rs = np.random.default_rng(9)
    ins = []
    for t in mu["inputs"]:
        shp = mu["tensors"][t]["shape"]
        x = rs.standard_normal(shp) / np.sqrt(shp[-1])
        ins.append(np.abs(x) + 1e-3 if int(np.prod(shp)) == 1 else x)
    got = ctx.eval_vm(mu, ins, mode=0)[0]
    want = ref.eval_mugraph(mu, ins, mode=0)[0]
    assert np.array_equal(got, want)
    got_p = ctx.eval_vm(prog, ins, mode=1)[0]
    want_p = ref.eval_mugraph(prog, ins, mode=1)[0]
    assert np.array_equal(got_p, want_p)


def test_stability_filter_full_shape(ctx):
    """float_stability_filter at BASELINE shapes, beyond shared memory:
    normals in HBM, program and candidate on the global-memory fp64
    executor; the verdict equals the reference's (stable µGraph: pass;
    mutant: fail)."""
    prog, mu = F.bench_pair("rmsnorm")
    args = F.BENCH["rmsnorm"]["args"]
    mut = F.family_mugraph("rmsnorm", *args, grid=F.BENCH["rmsnorm"]["grid"],
                           forloop=F.BENCH["rmsnorm"]["forloop"], mutant=True)
    for cand in (mu, mut):
        got = ctx.float_stability_filter(cand, prog, trials=1, seed=17)
        want = ref.float_stability_filter(cand, prog, trials=1, seed=17)
        assert got == want
    assert ctx.float_stability_filter(mu, prog, trials=1, seed=17)


def _mutants(fam, n, seed):
    """Generator candidates and op-rewrite mutants (fixtures.search_stream)."""
    from paper_2405_05751_b200 import api
    prog, pool = F.verify_families()[fam]
    bases = [g for _, g in pool] + api.generate(prog, grids=[1, 2, 4, 8, 16], loops=[1, 2, 4, 8, 16])
    s = F.search_stream(bases, 4000, seed=seed)
    return prog, s[len(bases):][::max(1, (len(s) - len(bases)) // n)][:n]


@pytest.mark.parametrize("fam", ["rmsnorm", "gatedmlp", "gqa", "lora"])
def test_eval_vm_on_mutants_matches_reference(ctx, fam):
    """fp64 eval_mugraph of search-stream mutants (NaN / inf from sqrt of
    negatives and division included) equals the reference."""
    _, cands = _mutants(fam, 40, seed=21)
    for g in cands:
        ins = _inputs(g, 9)
        _close(ctx.eval_vm(g, ins, mode=0), ref.eval_mugraph(g, ins, mode=0), g)


def test_stability_batch_on_mutants_matches_reference(ctx):
    for fam in ("rmsnorm", "gqa", "lora"):
        prog, cands = _mutants(fam, 60, seed=23)
        seeds = np.arange(len(cands), dtype=np.uint64) * 104729 + 5
        ok = ctx.stability_batch(prog, cands, seeds=seeds, trials=2)
        for k in range(len(cands)):
            want = ref.float_stability_filter(cands[k], prog, trials=2, seed=int(seeds[k]))
            assert ok[k] == int(want), (fam, k)


def test_multi_kernel_candidates_fp_and_stability(ctx):
    """The generator's multi-kernel µGraphs on the fp64 VM (eval_mugraph) and
    through the batched stability filter: identical to the reference."""
    from paper_2405_05751_b200 import api
    for fam in ("rmsnorm", "gatedmlp", "gqa", "lora"):
        prog, _ = F.verify_families()[fam]
        cands = [g for g in api.generate(prog, grids=[1, 2, 4], loops=[1, 2, 4], max_kernels=4)
                 if len(g["ops"]) > 1][::9][:30]
        for g in cands[::3]:
            ins = _inputs(g, 4)
            _close(ctx.eval_vm(g, ins, mode=0), ref.eval_mugraph(g, ins, mode=0), g)
        seeds = np.arange(len(cands), dtype=np.uint64) * 31 + 2
        ok = ctx.stability_batch(prog, cands, seeds=seeds, trials=2)
        for k in range(len(cands)):
            assert ok[k] == int(ref.float_stability_filter(cands[k], prog, trials=2, seed=int(seeds[k]))), (fam, k)

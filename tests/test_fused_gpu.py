"""GPU numerics of the fused benchmark µGraph kernels against the compiled
reference's eval_mugraph (double precision) on identical bf16-rounded inputs.

Tolerance: per element |o - r| <= 1e-3 * max(|r|, rms(r)) — the
fp32-accumulation criterion — plus a normwise ||o - r||_inf / ||r||_inf bound.
A plain torch fp32 reference of the same op is checked as well.
"""
import numpy as np
import pytest
import torch

from oracle import ref
from paper_2405_05751_b200 import fixtures as F

pytestmark = pytest.mark.gpu

TOL = 1e-3


def make_inputs(name, args, seed=0):
    """bf16 synthetic inputs, scaled so outputs are O(1)."""
    g = torch.Generator().manual_seed(seed)
    if name == "rmsnorm":
        b, h, n = args
        x = torch.randn(b, h, generator=g)
        gg = 1.0 + 0.1 * torch.randn(1, h, generator=g)
        w = torch.randn(h, n, generator=g) / h ** 0.5
        d = torch.full((1, 1), 1.0 / h)
        ins = [x, gg, w, d]
    elif name == "gatedmlp":
        b, h, n = args
        ins = [torch.randn(b, h, generator=g), torch.randn(h, n, generator=g) / h ** 0.5,
               torch.randn(h, n, generator=g) / h ** 0.5]
    elif name == "gqa":
        G, qh, hd, L = args
        ins = [torch.randn(G, qh, hd, generator=g) / hd ** 0.5, torch.randn(G, hd, L, generator=g),
               torch.randn(G, L, hd, generator=g)]
    else:
        b, h, n, r = args
        ins = [torch.randn(b, h, generator=g), torch.randn(h, n, generator=g) / h ** 0.5,
               torch.randn(h, r, generator=g) / h ** 0.5, torch.randn(r, n, generator=g) / r ** 0.5]
    return [x.to(torch.bfloat16) for x in ins]


def torch_ref(name, ins):
    x = [t.float() for t in ins]
    if name == "rmsnorm":
        X, G, W, D = x
        return (X * G / torch.sqrt((X * X).sum(1, keepdim=True) * D)) @ W
    if name == "gatedmlp":
        X, W1, W3 = x
        return torch.nn.functional.silu(X @ W1) * (X @ W3)
    if name == "gqa":
        Q, K, V = x
        e = torch.exp(Q @ K)
        return (e @ V) / e.sum(2, keepdim=True)
    X, W, A, B = x
    return X @ W + (X @ A) @ B


def check(out, r):
    r = np.asarray(r, np.float64)
    o = np.asarray(out, np.float64)
    assert np.all(np.isfinite(o))
    rms = np.sqrt(np.mean(r * r))
    err = np.abs(o - r)
    bound = TOL * np.maximum(np.abs(r), rms)
    worst = float(np.max(err / np.maximum(np.abs(r), rms)))
    assert np.all(err <= bound), f"max scaled err {worst:.3e}"
    assert np.max(err) / np.max(np.abs(r)) < 1e-4
    return worst


SMALL = {
    "gatedmlp": [((8, 512, 256), 2, 4), ((8, 1024, 512), 4, 16), ((3, 256, 128), 1, 1)],
    "rmsnorm": [((8, 512, 256), 2, 4), ((8, 1024, 512), 4, 16), ((5, 256, 384), 1, 2)],
    "lora": [((16, 512, 256, 16), 2, 4), ((16, 1024, 512, 16), 4, 16), ((7, 256, 128, 16), 1, 1)],
    "gqa": [((4, 8, 128, 512), 2, 4), ((8, 8, 128, 1024), 4, 8), ((2, 5, 128, 256), 1, 2),
            ((3, 8, 128, 2048), 3, 16)],
}


@pytest.mark.parametrize("name", list(SMALL))
def test_fused_small_shapes_vs_reference(ctx, name):
    for args, grid, fl in SMALL[name]:
        mu = F.family_mugraph(name, *args, grid=grid, forloop=fl)
        g = ctx.compile(mu)
        assert g.fused == name, (name, args)
        ins = make_inputs(name, args)
        out = ctx.eval_mugraph(g, [x.cuda() for x in ins])[0].cpu().numpy()
        want = ref.eval_mugraph(mu, [x.float().numpy() for x in ins])[0]
        check(out, want)
        check(out, torch_ref(name, ins).numpy())


@pytest.mark.parametrize("name", ["gatedmlp", "rmsnorm", "lora", "gqa"])
def test_fused_bench_shape_vs_reference(ctx, name):
    prog, mu = F.bench_pair(name)
    args = F.BENCH[name]["args"]
    g = ctx.compile(mu)
    assert g.fused == name
    ins = make_inputs(name, args, seed=1)
    out = ctx.eval_mugraph(g, [x.cuda() for x in ins])[0].cpu().numpy()
    want = ref.eval_mugraph(mu, [x.float().numpy() for x in ins])[0]
    check(out, want)
    # the flat program (reference eval_program) agrees too
    check(out, ref.eval_mugraph(prog, [x.float().numpy() for x in ins], mode=1)[0])


@pytest.mark.parametrize("name", ["gatedmlp", "rmsnorm", "lora", "gqa"])
def test_eval_mugraph_host_buffers(ctx, name):
    """tpo_gpu_eval_mugraph_host: host bf16 inputs (pinned and pageable) and
    host fp32 inputs (rounded to bf16 on the device) give exactly the
    device-buffer result."""
    args, grid, fl = SMALL[name][1]
    mu = F.family_mugraph(name, *args, grid=grid, forloop=fl)
    g = ctx.compile(mu)
    ins = make_inputs(name, args, seed=5)
    dev = ctx.eval_mugraph(g, [x.cuda() for x in ins])[0].cpu()
    pinned = ctx.eval_mugraph_host(g, [x.pin_memory() for x in ins])[0]
    pageable = ctx.eval_mugraph_host(g, ins)[0]
    f32 = ctx.eval_mugraph_host(g, [x.float() for x in ins])[0]
    assert torch.equal(dev, pinned) and torch.equal(dev, pageable) and torch.equal(dev, f32)


def test_unfused_mugraphs_run_on_the_generic_vm(ctx):
    """eval_mugraph is total: a µGraph with no hand-written kernel (pool
    variants at verification shapes, a GatedMLP outside the kernel's limits)
    runs on the generic GPU VM in the reference's fp32 semantics."""
    for fam in ("rmsnorm", "gqa", "lora"):
        prog, pool = F.verify_families()[fam]
        for tag, g in pool[:6]:
            cg = ctx.compile(g)
            assert not cg.fused
            shapes = cg.shapes(False)
            gen = torch.Generator().manual_seed(1)
            ins = [(torch.rand(s, generator=gen) + 0.5).to(torch.bfloat16) for s in shapes]
            out = ctx.eval_mugraph(cg, [x.cuda() for x in ins])[0].cpu().numpy()
            want = ref.eval_mugraph(g, [x.float().numpy() for x in ins], mode=2)[0]
            assert np.allclose(out, want, rtol=1e-5, atol=1e-6), tag
            host = ctx.eval_mugraph_host(cg, [x.float() for x in ins])[0].numpy()
            assert np.allclose(host, want, rtol=1e-5, atol=1e-6), tag
    args = (16, 256, 192)  # 16 tokens, 192 columns: outside the skinny kernel's limits
    mu = F.family_mugraph("gatedmlp", *args, grid=2, forloop=4)
    g = ctx.compile(mu)
    assert not g.fused
    ins = make_inputs("gatedmlp", args)
    out = ctx.eval_mugraph(g, [x.cuda() for x in ins])[0].cpu().numpy()
    check(out, ref.eval_mugraph(mu, [x.float().numpy() for x in ins])[0])


@pytest.mark.parametrize("name", ["gatedmlp", "rmsnorm", "lora", "gqa"])
def test_generated_candidates_run_fused(ctx, name):
    """The fusion generator's candidates at BASELINE shapes lower to the
    hand-written kernels (structural match, independent of op order) and
    agree with the reference."""
    from paper_2405_05751_b200 import api
    prog, _ = F.bench_pair(name)
    b = F.BENCH[name]
    cands = api.generate(prog, grids=[b["grid"]], loops=[b["forloop"]])
    assert cands
    ins = make_inputs(name, b["args"])
    want = ref.eval_mugraph(prog, [x.float().numpy() for x in ins])[0]
    for g in cands:
        cg = ctx.compile(g)
        assert cg.fused == name
        out = ctx.eval_mugraph(cg, [x.cuda() for x in ins])[0].cpu().numpy()
        check(out, want)


def test_fused_concurrent_contexts(ctx):
    """One context per thread, each on its own stream: the four fused
    kernels at small shapes evaluate concurrently and reproduce the
    sequential (bitwise deterministic) outputs."""
    import threading
    from paper_2405_05751_b200.api import Context
    names = ["gatedmlp", "rmsnorm", "lora", "gqa"]
    inputs, want = {}, {}
    for n in names:
        args, grid, fl = SMALL[n][1]
        mu = F.family_mugraph(n, *args, grid=grid, forloop=fl)
        inputs[n] = (mu, make_inputs(n, args, seed=21))
        want[n] = ctx.eval_mugraph(ctx.compile(mu), [x.cuda() for x in inputs[n][1]])[0].cpu()
    got, errs = {}, []

    def work(n):
        try:
            c = Context(0)
            mu, ins = inputs[n]
            g = c.compile(mu)
            dev = [x.cuda() for x in ins]
            got[n] = [c.eval_mugraph(g, dev)[0].cpu() for _ in range(5)]
        except Exception as e:
            errs.append(e)

    th = [threading.Thread(target=work, args=(n,)) for n in names]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for n in names:
        for o in got[n]:
            assert torch.equal(o, want[n]), n


@pytest.mark.parametrize("name", list(SMALL))
def test_attribute_mutants_take_the_right_path(ctx, name):
    """Valid attribute mutants of a fusable µGraph (grid, for-loop, maps,
    Sum attrs redrawn): whichever path the backend picks — a fused kernel
    when the mutant still matches one structurally, the generic VM otherwise —
    its output equals the reference's eval_mugraph of that mutant."""
    args, grid, fl = SMALL[name][0]
    mu = F.family_mugraph(name, *args, grid=grid, forloop=fl)
    ins = make_inputs(name, args, seed=4)
    fused = 0
    muts = [g for g in F.attribute_mutants([mu], 400, seed=13) if ref.validate(g) == 0][:12]
    assert len(muts) >= 6
    for g in muts:
        h = ctx.compile(g)
        fused += h.fused == name
        out = ctx.eval_mugraph(h, [x.cuda() for x in ins])[0].cpu().numpy()
        want = ref.eval_mugraph(g, [x.float().numpy() for x in ins])[0]
        r = np.asarray(want, np.float64)
        o = np.asarray(out, np.float64)
        fin = np.isfinite(r)
        assert np.array_equal(np.isfinite(o), fin)
        scale = max(np.sqrt(np.mean(r[fin] ** 2)), 1e-30) if fin.any() else 1.0
        assert np.max(np.abs(o[fin] - r[fin]), initial=0.0) <= 1e-3 * scale + 1e-3 * np.max(np.abs(r[fin]), initial=0.0)


@pytest.mark.parametrize("args", [(16, 512, 256, 16), (9, 1024, 512, 16)])
def test_paper_lora_concat_form_runs_fused(ctx, args):
    """The paper's LoRA µGraph — kernel T = Matmul(X, A),
    then one GraphDef running ConcatMatmul(X̄, T̄, W̄, B̄) into a φ-Accum —
    as Algorithm 1 emits it from the flat program, dispatches to the fused
    LoRA kernel and meets the tolerance against the reference's
    eval_mugraph of that same µGraph."""
    from paper_2405_05751_b200 import api
    b, h, n, r = args
    prog = F.family_program("lora", b, h, n, r)
    cands = api.enumerate_mugraphs(prog, grids=[n // 128], loops=[4], max_kernel_ops=1, max_block_ops=4)
    paper = [g for g in cands if [op["type"] for op in g["ops"]] == ["matmul", "graphdef"]
             and g["ops"][0]["inputs"] == [0, 2]
             and any(o["type"] == "concatmatmul" for o in g["ops"][1]["blockGraph"]["ops"])]
    assert paper
    g = ctx.compile(paper[0])
    assert g.fused == "lora", g.fused
    ins = make_inputs("lora", args, seed=5)
    out = ctx.eval_mugraph(g, [x.cuda() for x in ins])[0]
    torch.cuda.synchronize()
    want = ref.eval_mugraph(paper[0], [x.float().numpy() for x in ins])[0]
    check(out.cpu().numpy(), want)


@pytest.mark.parametrize("name,args", [("gatedmlp", (20, 512, 256)), ("rmsnorm", (19, 512, 256)),
                                       ("lora", (40, 512, 256, 16))])
def test_more_tokens_than_a_tile_run_fused_in_chunks(ctx, name, args):
    """Token counts beyond one kernel tile (8, LoRA 16) run the fused kernel
    once per token chunk (ragged last chunk included), bf16 and fp64 (SPLIT)
    inputs alike, within the tolerance against the reference."""
    mu = F.family_mugraph(name, *args, grid=2, forloop=4)
    g = ctx.compile(mu)
    assert g.fused == name
    ins = make_inputs(name, args, seed=7)
    want = ref.eval_mugraph(mu, [x.float().numpy() for x in ins])[0]
    out = ctx.eval_mugraph(g, [x.cuda() for x in ins])[0].cpu().numpy()
    check(out, want)
    rng = np.random.default_rng(3)
    d = [rng.standard_normal(tuple(x.shape)) * (float(x.float().std()) if x.numel() > 1 else 1.0) for x in ins]
    if name == "rmsnorm":
        d[3] = np.full((1, 1), 1.0 / args[1])
    check(ctx.eval_mugraph_f64(g, d)[0], ref.eval_mugraph(mu, d)[0])

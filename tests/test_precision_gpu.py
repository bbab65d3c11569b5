"""The drop-in eval_mugraph contract on ARBITRARY fp64 inputs.

The reference's eval_mugraph takes doubles (proj/core/include/tpo/interp/
interp.hpp:47-48) and its in-tree caller feeds N(0,1)·scale doubles
(proj/core/src/stability.cpp:30-38) — not bf16-representable values.  The
fused kernels' precision policy (include/tpo_gpu.h TPO_PREC_*):

* TPO_PREC_AUTO with fp32 / fp64 inputs runs the SPLIT kernels (every
  operand as bf16 hi + lo, fp32 accumulation) and must meet, per element,
  |o - r| <= 1e-3 * max(|r|, rms(r)) and ||o - r||_inf / ||r||_inf < 1e-4;
* TPO_PREC_VM and µGraphs without a fused kernel run the fp64 VM in the
  reference's operation order: within 1e-12 relative;
* TPO_PREC_BF16 (explicit opt-in) rounds the inputs to bf16 — shown here to
  miss the bound on such inputs, which is why it is not the default.

All at the four BASELINE shapes, against the compiled reference.
"""
import numpy as np
import pytest
import torch

from oracle import ref
from paper_2405_05751_b200 import fixtures as F

pytestmark = pytest.mark.gpu

TOL = 1e-3
NAMES = ["gatedmlp", "rmsnorm", "lora", "gqa"]


def doubles(name, args, seed=0):
    """N(0,1)·scale fp64 inputs (scales as SURVEY §8d, so outputs are O(1))."""
    rng = np.random.default_rng(seed)
    if name == "rmsnorm":
        b, h, n = args
        return [rng.standard_normal((b, h)), 1.0 + 0.1 * rng.standard_normal((1, h)),
                rng.standard_normal((h, n)) / h ** 0.5, np.full((1, 1), 1.0 / h)]
    if name == "gatedmlp":
        b, h, n = args
        return [rng.standard_normal((b, h)), rng.standard_normal((h, n)) / h ** 0.5,
                rng.standard_normal((h, n)) / h ** 0.5]
    if name == "gqa":
        G, qh, hd, L = args
        return [rng.standard_normal((G, qh, hd)) / hd ** 0.5, rng.standard_normal((G, hd, L)),
                rng.standard_normal((G, L, hd))]
    b, h, n, r = args
    return [rng.standard_normal((b, h)), rng.standard_normal((h, n)) / h ** 0.5,
            rng.standard_normal((h, r)) / h ** 0.5, rng.standard_normal((r, n)) / r ** 0.5]


def scaled_err(out, want):
    o, r = np.asarray(out, np.float64), np.asarray(want, np.float64)
    assert np.all(np.isfinite(o))
    rms = np.sqrt(np.mean(r * r))
    return float(np.max(np.abs(o - r) / np.maximum(np.abs(r), rms))), \
        float(np.max(np.abs(o - r)) / np.max(np.abs(r)))


_REF = {}


def reference(name):
    """(µGraph, fp64 inputs, reference eval_mugraph output) at the BASELINE shape."""
    if name not in _REF:
        _, mu = F.bench_pair(name)
        ins = doubles(name, F.BENCH[name]["args"], seed=3)
        _REF[name] = (mu, ins, ref.eval_mugraph(mu, ins)[0])
    return _REF[name]


@pytest.mark.parametrize("name", NAMES)
def test_eval_mugraph_f64_arbitrary_doubles(ctx, name):
    """tpo_gpu_eval_mugraph_f64 (the reference's own types) on N(0,1) doubles:
    the split kernel meets the tolerance at the BASELINE shape."""
    mu, ins, want = reference(name)
    g = ctx.compile(mu)
    assert g.fused == name
    out = ctx.eval_mugraph_f64(g, ins)[0]
    worst, norm = scaled_err(out, want)
    assert worst <= TOL, f"{name}: max scaled err {worst:.3e}"
    assert norm < 1e-4, f"{name}: normwise err {norm:.3e}"


@pytest.mark.parametrize("name", NAMES)
def test_fp32_and_fp64_buffers_take_the_split_kernel(ctx, name):
    """fp32 CUDA tensors (device entry point) and fp64 host tensors
    (eval_mugraph_host) select the split kernel; both meet the tolerance
    against the reference on the same values."""
    mu, ins, want = reference(name)
    g = ctx.compile(mu)
    f32 = [torch.from_numpy(x).float() for x in ins]
    want32 = ref.eval_mugraph(mu, [x.double().numpy() for x in f32])[0]
    dev = ctx.eval_mugraph(g, [x.cuda() for x in f32])[0].cpu().numpy()
    assert scaled_err(dev, want32)[0] <= TOL
    host64 = ctx.eval_mugraph_host(g, [torch.from_numpy(x) for x in ins])[0].numpy()
    assert scaled_err(host64, want)[0] <= TOL
    # mixed dtypes: bf16 activations, fp64 weights
    mixed = [torch.from_numpy(x) for x in ins]
    mixed[0] = mixed[0].to(torch.bfloat16)
    want_m = ref.eval_mugraph(mu, [mixed[0].double().numpy()] + ins[1:])[0]
    out_m = ctx.eval_mugraph_host(g, mixed)[0].numpy()
    assert scaled_err(out_m, want_m)[0] <= TOL


@pytest.mark.parametrize("name", NAMES)
def test_precision_policies(ctx, name):
    """TPO_PREC_VM: fp64 VM, reference arithmetic (<= 1e-12 relative);
    TPO_PREC_BF16: rounding the inputs costs accuracy on arbitrary doubles
    (its error exceeds the split kernel's by orders of magnitude)."""
    mu, ins, want = reference(name)
    g_vm = ctx.compile(mu).set_precision("vm")
    vm = ctx.eval_mugraph_f64(g_vm, ins)[0]
    r = np.asarray(want)
    assert np.max(np.abs(vm - r)) <= 1e-12 * np.max(np.abs(r))
    g_auto = ctx.compile(mu)
    g_bf = ctx.compile(mu).set_precision("bf16")
    e_auto = scaled_err(ctx.eval_mugraph_f64(g_auto, ins)[0], want)[0]
    e_bf = scaled_err(ctx.eval_mugraph_f64(g_bf, ins)[0], want)[0]
    assert e_bf > 10 * e_auto, (e_bf, e_auto)


def test_unfused_graph_f64_is_reference_arithmetic(ctx):
    """A flat program (no fused kernel) through eval_mugraph_f64 runs the fp64
    VM: within 1e-12 of the reference's eval_mugraph."""
    for name in ("gatedmlp", "lora"):
        prog, _ = F.bench_pair(name)
        ins = doubles(name, F.BENCH[name]["args"], seed=8)
        g = ctx.compile(prog)
        assert not g.fused
        out = ctx.eval_mugraph_f64(g, ins)[0]
        want = np.asarray(ref.eval_mugraph(prog, ins)[0])
        assert np.max(np.abs(out - want)) <= 1e-12 * np.max(np.abs(want))


def test_bf16_representable_f32_is_bit_identical_to_bf16_path(ctx):
    """On bf16-representable values the split kernel's lo planes are zero:
    its output equals the bf16 kernel's bit for bit (all four families)."""
    from test_fused_gpu import SMALL, make_inputs
    for name in NAMES:
        args, grid, fl = SMALL[name][1]
        mu = F.family_mugraph(name, *args, grid=grid, forloop=fl)
        g = ctx.compile(mu)
        ins = make_inputs(name, args, seed=6)
        a = ctx.eval_mugraph(g, [x.cuda() for x in ins])[0]
        b = ctx.eval_mugraph(g, [x.float().cuda() for x in ins])[0]
        assert torch.equal(a, b), name


def test_rejects_unsupported_dtypes(ctx):
    mu = F.family_mugraph("gatedmlp", 8, 512, 256, grid=2, forloop=4)
    g = ctx.compile(mu)
    ins = [torch.zeros(s, dtype=torch.float16, device="cuda") for s in g.shapes(False)]
    with pytest.raises(ValueError):
        ctx.eval_mugraph(g, ins)
    with pytest.raises(ValueError):
        ctx.eval_mugraph_host(g, [x.cpu() for x in ins])

#!/usr/bin/env python
"""Kernel-configuration sweep for the fused µGraph kernels (GPU box only).

  python scripts/sweep.py rmsnorm "TPO_KSPLIT=4,TPO_STAGES=4" "TPO_KSPLIT=4,TPO_STAGES=8" ...

For each configuration (env overrides read by csrc/host/fused.cpp at every
launch): checks the output against a torch fp32 reference at the BASELINE
shape, then times 100 evaluations replayed as one CUDA graph over rotating
input copies (> L2), CUDA events on the launching stream.  Prints one line
per configuration: µs/eval and fraction of the measured HBM copy bandwidth.
An empty config string means the library's own choice.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from paper_2405_05751_b200 import fixtures as F  # noqa: E402
from paper_2405_05751_b200.api import Context  # noqa: E402
from test_fused_gpu import make_inputs, torch_ref  # noqa: E402

L2 = 126 * 2**20
WEIGHTS = {"gatedmlp": [1, 2], "rmsnorm": [1, 2, 3], "lora": [1, 2, 3], "gqa": []}


def main():
    name = sys.argv[1]
    cfgs = sys.argv[2:] or [""]
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    ctx = Context(0)
    _, mu = F.bench_pair(name)
    args = F.BENCH[name]["args"]
    host = make_inputs(name, args, seed=3)
    want = torch_ref(name, [x.cuda() for x in host]).float()
    in_b = sum(x.numel() * 2 for x in host)
    alg = in_b + want.numel() * 4
    copies = max(1, -(-3 * L2 // in_b))
    sets = [[x.cuda() for x in host] for _ in range(copies)]
    outs = [torch.empty_like(want) for _ in range(copies)]
    st = torch.cuda.Stream()
    for cfg in cfgs:
        for k in ("TPO_KSPLIT", "TPO_STAGES", "TPO_MINB", "TPO_NO_PDL", "TPO_DBG_FLAGS", "TPO_EPI_ATOMIC", "TPO_TRIG_EARLY", "TPO_PRE_CUT", "TPO_L2_AHEAD", "TPO_GQA_SLOTS", "TPO_GQA_ORDER", "TPO_GQA_L2", "TPO_X_L2", "TPO_TMA_OUT"):
            os.environ.pop(k, None)
        static = False
        for kv in filter(None, cfg.split(",")):
            k, v = kv.split("=")
            if k == "STATIC":
                static = v == "1"
            else:
                os.environ[k] = v
        g = ctx.compile(mu)
        if static:
            g.set_static_inputs(WEIGHTS[name])
        try:
            with torch.cuda.stream(st):
                o = ctx.eval_mugraph(g, sets[0], outputs=[outs[0]], stream=st.cuda_stream)[0]
            st.synchronize()
            err = float(((o - want).abs() / torch.maximum(want.abs(), want.pow(2).mean().sqrt())).max())
            for i in range(5):
                ctx.eval_mugraph(g, sets[i % copies], outputs=[outs[i % copies]], stream=st.cuda_stream)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=st):
                for i in range(100):
                    ctx.eval_mugraph(g, sets[i % copies], outputs=[outs[i % copies]],
                                     stream=torch.cuda.current_stream().cuda_stream)
            graph.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            best = 1e9
            for _ in range(5):
                with torch.cuda.stream(st):
                    e0.record(st)
                    graph.replay()
                    e1.record(st)
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1) * 10.0)  # µs per eval
            print(f"{name:9s} {cfg or 'default':32s} {best:8.2f} us  frac {alg / best / 1e3 / peak:.3f}"
                  f"  maxerr {err:.2e}", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"{name:9s} {cfg or 'default':32s} FAILED {e}", flush=True)


if __name__ == "__main__":
    main()

"""The optimize flow the reference's absent pipeline describes (SPEC.md:
664-668, Fig. 1: generate -> verify -> stability filter -> select), composed
over the C-ABI: candidates from the fusion generator (tpo_gpu_generate),
compiled on all host cores (tpo_gpu_compile_many), verified in one GPU
batch with the VerifyConfig seed (tpo_gpu_verify_batch), survivors through
the GPU float stability filter (tpo_gpu_stability_batch), ranked by the
SPEC's analytic cost (weights wDevice 1.0 per byte,
wShared 0.02, wKernelLaunch 4096, wCompute 0.002 per multiply-add).
"""
from __future__ import annotations

from typing import Dict, List, Optional

import numpy as np

from . import api


def _numel(shape) -> int:
    n = 1
    for d in shape:
        n *= d
    return n


def cost(g: dict, elem_size: int = 2, w_device: float = 1.0, w_shared: float = 0.02,
         w_launch: float = 4096.0, w_compute: float = 0.002, madds: Optional[int] = None) -> float:
    """SPEC cost: device bytes moved by kernel-level edges
    and InIter / OutSaver tiles (per block and iteration), shared-memory
    traffic of block ops, kernel launches, and multiply-adds."""
    device = shared = 0.0
    launches = 0
    for op in g["ops"]:
        launches += 1
        if op["type"] != "graphdef":
            device += sum(_numel(g["tensors"][t]["shape"]) for t in op["inputs"] + op["outputs"]) * elem_size
            continue
        bg = op["blockGraph"]
        blocks = bg["grid"][0] * bg["grid"][1] * bg["grid"][2]
        post = set()
        for b in bg["ops"]:  # post-loop set (eval_core.hpp:277-294)
            if b["type"] == "accum":
                post.add(b["outputs"][0])
            elif b["type"] not in ("initer", "outsaver") and any(t in post for t in b["inputs"]):
                post.update(b["outputs"])
        for b in bg["ops"]:
            if b["type"] == "initer":
                trips = bg["forloop"]
            elif b["type"] == "outsaver":
                trips = 1
            else:
                trips = 1 if b["outputs"] and b["outputs"][0] in post else bg["forloop"]
            ts = (b["outputs"] if b["type"] == "initer" else b["inputs"])
            nbytes = sum(_numel(bg["tensors"][t]["shape"]) for t in ts) * elem_size * blocks * trips
            if b["type"] in ("initer", "outsaver"):
                device += nbytes
            else:
                shared += sum(_numel(bg["tensors"][t]["shape"]) for t in b["inputs"] + b["outputs"]) \
                    * elem_size * blocks * trips
    return w_device * device + w_shared * shared + w_launch * launches + w_compute * (madds or 0)


def optimize(ctx: "api.Context", program: dict, grids=(1, 2, 4, 8, 16, 32, 64, 128),
             loops=(1, 2, 4, 8, 16, 32, 64), num_tests: int = 2, seed: int = 0,
             stability: bool = True, prefer_fused: bool = True, max_resamples: int = 16,
             max_kernels: int = 1) -> Dict:
    """generate -> verify -> stability -> select.  Returns the best candidate,
    its cost and describe() listing, the ranked survivors and stage counts
    (non-increasing, SPEC.md PipelineReport).  Works at any shape: graphs
    beyond shared memory are verified and filtered on the global-memory
    executors.  ``prefer_fused``: candidates that lower to a hand-written
    sm_100a kernel rank first (the SPEC cost does not model parallelism).
    ``max_kernels`` > 1 adds the generator's multi-kernel µGraphs."""
    cands = api.generate(program, grids=grids, loops=loops, max_kernels=max_kernels)
    graphs, status = ctx.compile_many(cands)
    ok = [i for i, s in enumerate(status) if s == 0]
    report = {"generated": len(cands), "compiled": len(ok)}
    if not ok:
        return {**report, "verified": 0, "stable": 0, "best": None, "ranked": []}
    verdicts, _ = ctx.verify_batch(program, [graphs[i] for i in ok],
                                   np.full(len(ok), seed, dtype=np.uint64), num_tests=num_tests,
                                   max_resamples=max_resamples)
    eq = [ok[k] for k in range(len(ok)) if verdicts["kind"][k] == 0]
    report["verified"] = len(eq)
    report["inconclusive"] = int((verdicts["kind"] == 2).sum())
    if stability and eq:
        st = ctx.stability_batch(program, [graphs[i] for i in eq])
        eq = [eq[k] for k in range(len(eq)) if st[k] == 1]
    report["stable"] = len(eq)
    def key(i):
        return (0 if (prefer_fused and graphs[i].fused) else 1, cost(cands[i], madds=graphs[i].info.madds), i)
    ranked: List = [(key(i)[1], i) for i in sorted(eq, key=key)]
    best = cands[ranked[0][1]] if ranked else None
    report.update({"best": best, "best_cost": ranked[0][0] if ranked else None,
                   "best_fused": graphs[ranked[0][1]].fused if ranked else None,
                   "describe": api.describe(best) if best else "",
                   "ranked": [(c, cands[i]) for c, i in ranked]})
    return report

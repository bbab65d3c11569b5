#!/usr/bin/env python
"""Per-CTA phase timestamps of the skinny kernels (TPO_DEBUG_TIMES=1): the
host prints min/mean/max of each phase over all CTAs, µs since the first
CTA started.  GPU box only:  TPO_DEBUG_TIMES=1 python scripts/timeline.py rmsnorm lora"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2405_05751_b200 import fixtures as F  # noqa: E402
from paper_2405_05751_b200.api import Context  # noqa: E402
from test_fused_gpu import make_inputs  # noqa: E402

ctx = Context(0)
for name in sys.argv[1:]:
    _, mu = F.bench_pair(name)
    g = ctx.compile(mu)
    if os.environ.get("STATIC"):
        g.set_static_inputs({"gatedmlp": [1, 2], "rmsnorm": [1, 2, 3], "lora": [1, 2, 3], "gqa": []}[name])
    host = make_inputs(name, F.BENCH[name]["args"])
    # cold runs: a fresh input copy per launch (12 x 34 MB > L2)
    sets = [[x.cuda() for x in host] for _ in range({"gatedmlp": 6, "gqa": 6}.get(name, 12))]
    for i in range(len(sets)):
        print(f"--- {name} launch {i} (inputs copy {i}, cold)", file=sys.stderr, flush=True)
        ctx.eval_mugraph(g, sets[i])

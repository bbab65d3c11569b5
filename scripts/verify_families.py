#!/usr/bin/env python
"""Per-family verifier throughput (GPU box): candidates/s and attempts for
each SURVEY §8d pool, timed with CUDA events around Context.verify_pool.
  python scripts/verify_families.py [n_per_family]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_05751_b200 import fixtures as F  # noqa: E402
from paper_2405_05751_b200.api import Context  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 250000
ctx = Context(0)
for fam, (prog, pool) in F.verify_families().items():
    gs = [g for _, g in pool]
    ctx.verify_pool(prog, gs, first=0, n=20000)  # warm-up (compile + upload)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.verify_pool(prog, gs, first=0, n=n)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{fam:9s} n={n} {ms:8.2f} ms  {n / ms * 1e3:12.0f} cand/s", flush=True)

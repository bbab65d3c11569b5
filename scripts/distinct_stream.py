#!/usr/bin/env python
"""Search-loop candidate stream (GPU box): the pool, the generator's
candidates and their mutants (fixtures.search_stream, distinct graphs)
handed over as JSON (the reference's wire format), compiled on all host
cores (tpo_gpu_compile_many) and verified in one batch (tpo_gpu_verify_batch,
seed i).  Prints wall-clock candidates/s per stage.
  python scripts/distinct_stream.py [n_per_family]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2405_05751_b200 import api  # noqa: E402
from paper_2405_05751_b200 import fixtures as F  # noqa: E402
from paper_2405_05751_b200.api import Context  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 25000
ctx = Context(0)
tot_c = tot_v = 0.0
cnt = 0
for fam, (prog, pool) in F.verify_families().items():
    bases = [g for _, g in pool] + api.generate(prog, grids=[1, 2, 4, 8, 16, 32, 64, 128],
                                                loops=[1, 2, 4, 8, 16, 32, 64], max_kernels=3,
                                                max_candidates=2000)
    cands = F.search_stream(bases, n, seed=1)
    js = [json.dumps(cands[i % len(cands)]) for i in range(n)]
    gp = ctx.compile(prog)
    ctx.verify_batch(gp, ctx.compile_many(js[:64])[0], np.arange(64, dtype=np.uint64), want_verdicts=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gs, st = ctx.compile_many(js)
    t1 = time.perf_counter()
    seeds = np.zeros(n, dtype=np.uint64) if os.environ.get("SAME_SEED", "1") == "1" else np.arange(n, dtype=np.uint64)
    _, acc = ctx.verify_batch(gp, gs, seeds, want_verdicts=False)
    t2 = time.perf_counter()
    assert all(s == 0 for s in st)
    tot_c += t1 - t0
    tot_v += t2 - t1
    cnt += n
    print(f"{fam:9s} n={n} compile {n / (t1 - t0):10.0f}/s  verify {n / (t2 - t1):10.0f}/s  "
          f"end-to-end {n / (t2 - t0):10.0f} cand/s  accepted {int(acc.sum())}  distinct {len(cands)}", flush=True)
print(f"all      n={cnt} compile {cnt / tot_c:10.0f}/s  verify {cnt / tot_v:10.0f}/s  "
      f"end-to-end {cnt / (tot_c + tot_v):10.0f} cand/s  host threads {os.cpu_count()}")

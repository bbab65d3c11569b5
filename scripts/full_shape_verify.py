#!/usr/bin/env python
"""random_test_equivalence at BASELINE shapes (GPU box): the global-memory
field executor against the compiled reference, wall clock per call."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2405_05751_b200 import fixtures as F  # noqa: E402
from paper_2405_05751_b200.api import Context  # noqa: E402

ctx = Context(0)
for name in sys.argv[1:] or ["rmsnorm", "lora", "gqa", "gatedmlp"]:
    prog, mu = F.bench_pair(name)
    ctx.random_test_equivalence(prog, mu, seed=1)  # warm (lowering, arena)
    t0 = time.perf_counter()
    g = ctx.random_test_equivalence(prog, mu, seed=2)
    t1 = time.perf_counter()
    r = ref.random_test_equivalence(prog, mu, seed=2)
    t2 = time.perf_counter()
    same = all(g[k] == r[k] for k in r)
    print(f"{name:9s} gpu {1e3 * (t1 - t0):9.1f} ms  cpu {1e3 * (t2 - t1):10.1f} ms  "
          f"speedup {(t2 - t1) / (t1 - t0):7.1f}x  attempts {g['resamples'] + g['rounds_run']}  same {same}",
          flush=True)

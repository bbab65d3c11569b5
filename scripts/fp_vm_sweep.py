#!/usr/bin/env python
"""Generic fp VM (global-memory executor) on the four BASELINE µGraphs:
device ms per evaluation (fp64 mode 0, fp32 mode 2; inputs already in one
flat device buffer) and the HBM fraction of the unique input + output bytes.
  python scripts/fp_vm_sweep.py      (GPU box)"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2405_05751_b200 import _native as N  # noqa: E402
from paper_2405_05751_b200 import fixtures as F  # noqa: E402
from paper_2405_05751_b200.api import Context  # noqa: E402
from test_fused_gpu import make_inputs  # noqa: E402

ctx = Context(0)
peak = 6560.6
for name in ("gatedmlp", "rmsnorm", "lora", "gqa"):
    _, mu = F.bench_pair(name)
    host = make_inputs(name, F.BENCH[name]["args"], seed=0)
    g = ctx.compile(mu)
    for mode, dt in ((0, torch.float64), (2, torch.float32)):
        flat = torch.cat([x.reshape(-1).to(dt) for x in host]).cuda()
        n_out = sum(int(np.prod(s)) for s in g.shapes(True))
        out = torch.empty(n_out, dtype=dt, device="cuda")
        st = torch.cuda.current_stream()

        def run():
            N.check(N.lib().tpo_gpu_eval_vm_dev(ctx.h, g.h, mode, C.c_void_p(flat.data_ptr()),
                                                C.c_void_p(out.data_ptr()), C.c_void_p(st.cuda_stream)))
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        nb = flat.numel() * flat.element_size() + n_out * out.element_size()
        print(f"{name:9s} {'f64' if mode == 0 else 'f32'} {ms:8.3f} ms  {nb / ms / 1e6:8.1f} GB/s  "
              f"frac {nb / ms / 1e6 / peak:.3f}", flush=True)

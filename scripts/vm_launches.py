#!/usr/bin/env python
"""One generic-VM evaluation (fp64, device buffers) of a BASELINE µGraph or
its flat program, for an ncu launch list (GPU box):
  ncu --metrics gpu__time_duration.sum python scripts/vm_launches.py rmsnorm [mode]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from paper_2405_05751_b200 import fixtures as F  # noqa: E402
from paper_2405_05751_b200.api import Context  # noqa: E402
from test_fused_gpu import make_inputs  # noqa: E402

name = sys.argv[1]
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
prog, mu = F.bench_pair(name)
ctx = Context(0)
g = ctx.compile(mu if mode == 0 else prog)
ins = [x.double().cuda() for x in make_inputs(name, F.BENCH[name]["args"])]
ctx.eval_vm_dev(g, ins, mode=mode)
torch.cuda.synchronize()

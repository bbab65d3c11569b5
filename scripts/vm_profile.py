#!/usr/bin/env python
"""Per-opcode cycle breakdown of the batched verifier (GPU box):
TPO_VM_PROFILE=1 python scripts/vm_profile.py [n_per_family]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_05751_b200 import fixtures as F  # noqa: E402
from paper_2405_05751_b200.api import Context  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
ctx = Context(0)
for fam, (prog, pool) in F.verify_families().items():
    print(f"=== {fam}", file=sys.stderr, flush=True)
    ctx.verify_pool(prog, [g for _, g in pool], first=0, n=n)

"""Debug: ff_eval over every pool graph (first failure under memcheck)."""
import sys
sys.path.insert(0, '.')
from paper_2405_05751_b200 import fixtures as F
from paper_2405_05751_b200.api import Context
ctx = Context(0)
for f, (prog, pool) in F.verify_families().items():
    for tag, g in [(f + "/program", prog)] + pool:
        print(tag, flush=True)
        ctx.ff_eval(g, 0, 0)
print("all ok")

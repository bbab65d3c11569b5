# compute-sanitizer over the kernels (GPU box): racecheck + synccheck on
# shared memory for the verifier VM (barrier phases), the fp VM and the
# stability kernel; memcheck on the fused kernels.  Small shapes.
CS=/usr/local/cuda/bin/compute-sanitizer
OUT=gpurun_out/sanitize; mkdir -p $OUT
cat > /tmp/san_verify.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2405_05751_b200 import fixtures as F
from paper_2405_05751_b200.api import Context
ctx = Context(0)
for fam, (prog, pool) in F.verify_families().items():
    gs = [g for _, g in pool]
    ctx.verify_pool(prog, gs, first=0, n=64, want_verdicts=True)
    ctx.verify_batch(prog, gs[:40], np.zeros(40, dtype=np.uint64))     # same-seed shared attempt
    ctx.stability_batch(prog, gs[:8])
    # search-stream mutants, incl. raising (PoisonedExponent) graphs: VM_RAISE barriers
    ms = F.search_stream(gs, 400, seed=3)[len(gs):]
    ms = [g for g in ms if sum(o["type"] == "ewexp" for op in g["ops"]
                               for o in op.get("blockGraph", {}).get("ops", [])) >= 2][:24] + ms[:24]
    ctx.verify_batch(prog, ms, np.arange(len(ms), dtype=np.uint64))
    # single attempts (eval_kernel): fused thread-graph chains, every pool graph
    for _, g in [(fam, prog)] + pool[:24]:
        ctx.ff_eval(g, 0, 0)
print("ok")
PY
cat > /tmp/san_fused.py <<'PY'
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
from paper_2405_05751_b200 import fixtures as F
from paper_2405_05751_b200.api import Context
from test_fused_gpu import make_inputs
ctx = Context(0)
for name, args, grid, fl in [("gatedmlp", (8, 512, 256), 2, 4), ("rmsnorm", (8, 512, 256), 2, 4),
                             ("lora", (16, 512, 256, 16), 2, 4), ("gqa", (4, 8, 128, 512), 2, 4)]:
    mu = F.family_mugraph(name, *args, grid=grid, forloop=fl)
    g = ctx.compile(mu)
    ins = [x.cuda() for x in make_inputs(name, args)]
    ctx.eval_mugraph(g, ins); torch.cuda.synchronize()
    g.set_static_inputs({"gatedmlp": [1, 2], "rmsnorm": [1, 2, 3], "lora": [1, 2, 3], "gqa": []}[name])
    for _ in range(3): ctx.eval_mugraph(g, ins)
    torch.cuda.synchronize()
# token chunks (ragged) and the paper's ConcatMatmul LoRA form
for name, args in [("gatedmlp", (20, 512, 256)), ("lora", (40, 512, 256, 16))]:
    g = ctx.compile(F.family_mugraph(name, *args, grid=2, forloop=4))
    ctx.eval_mugraph(g, [x.cuda() for x in make_inputs(name, args)])
from paper_2405_05751_b200 import api
prog = F.family_program("lora", 16, 512, 256, 16)
for c in api.enumerate_mugraphs(prog, grids=[2], loops=[4], max_kernel_ops=1, max_block_ops=4):
    if [op["type"] for op in c["ops"]] == ["matmul", "graphdef"] and c["ops"][0]["inputs"] == [0, 2]:
        g = ctx.compile(c)
        ctx.eval_mugraph(g, [x.cuda() for x in make_inputs("lora", (16, 512, 256, 16))])
torch.cuda.synchronize()
print("ok")
PY
timeout 1200 $CS --tool racecheck --racecheck-report hazard python /tmp/san_verify.py > $OUT/racecheck_verify.txt 2>&1
timeout 1200 $CS --tool synccheck python /tmp/san_verify.py > $OUT/synccheck_verify.txt 2>&1
timeout 1200 $CS --tool memcheck python /tmp/san_verify.py > $OUT/memcheck_verify.txt 2>&1
timeout 1200 $CS --tool memcheck python /tmp/san_fused.py > $OUT/memcheck_fused.txt 2>&1
timeout 1200 $CS --tool racecheck --racecheck-report hazard python /tmp/san_fused.py > $OUT/racecheck_fused.txt 2>&1

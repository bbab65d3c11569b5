#!/usr/bin/env bash
# One GPU session (run under gpurun from the repo root): parity tests, smoke,
# the bench lines for every workload, the ncu launch lists and one
# `ncu --set full` capture per fused kernel.  Everything lands in gpurun_out/.
#   gpurun --timeout 3000 -- 'bash scripts/gpu_round.sh [stage ...]'
# Stages: tests smoke bench multirank launches full  (default: all but multirank)
set -u
OUT=gpurun_out
mkdir -p "$OUT"
STAGES=${*:-tests smoke bench launches full}
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
nproc > "$OUT/host_cpu.txt"; grep -m1 "model name" /proc/cpuinfo >> "$OUT/host_cpu.txt"

has() { [[ " $STAGES " == *" $1 "* ]]; }

if has tests; then
  timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
fi
if has smoke; then
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "smoke rc=$?" >> "$OUT/smoke.log"
fi
if has bench; then
  timeout 900 python bench.py > "$OUT/bench_gatedmlp.json" 2> "$OUT/bench_gatedmlp.err"
  for w in rmsnorm lora gqa; do
    timeout 600 python bench.py --workload $w --no-verifier > "$OUT/bench_$w.json" 2> "$OUT/bench_$w.err"
  done
  timeout 900 python bench.py --workload verify > "$OUT/bench_verify.json" 2> "$OUT/bench_verify.err"
  timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"
fi
if has multirank; then
  # N=2 logic check on a 1-GPU box (both ranks on cuda:0 over gloo; not a bench number)
  TPO_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 \
    --verify-candidates 40000 > "$OUT/n2.json" 2> "$OUT/n2.err"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29513 bench.py --gpus 2 --impl reference --steps 1 --warmup 1 > "$OUT/n2r.json" 2> "$OUT/n2r.err"
fi
NCU=/usr/local/cuda/bin/ncu
if has launches; then
  for w in gatedmlp rmsnorm lora gqa; do
    timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
      --log-file "$OUT/launches_$w.csv" python bench.py --workload $w --profile --steps 20 --warmup 3 \
      > "$OUT/launches_$w.log" 2>&1
  done
fi
if has full; then
  for w in gatedmlp rmsnorm lora; do
    timeout 900 $NCU --set full --clock-control none --import-source on -k regex:skinny -s 5 -c 1 \
      -o "$OUT/prof_$w" -f python bench.py --workload $w --profile --steps 8 --warmup 3 \
      > "$OUT/prof_$w.log" 2>&1
  done
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:gqa -s 5 -c 1 \
    -o "$OUT/prof_gqa" -f python bench.py --workload gqa --profile --steps 8 --warmup 3 \
    > "$OUT/prof_gqa.log" 2>&1
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:verify -s 2 -c 1 \
    -o "$OUT/prof_verify" -f python -c "
import sys; sys.path.insert(0, '.')
from paper_2405_05751_b200 import fixtures as F
from paper_2405_05751_b200.api import Context
ctx = Context(0)
prog, pool = F.verify_families()['gatedmlp']
gs = [g for _, g in pool]
for i in range(4):
    ctx.verify_pool(prog, gs, first=i * 20000, n=20000)
" > "$OUT/prof_verify.log" 2>&1
fi
echo done > "$OUT/round_done.txt"

#!/usr/bin/env bash
# Round-2 investigation (GPU box): verifier A/B (register cap, thread-graph
# chains), steady-state rings of the 34 MB kernels, ncu captures.
OUT=gpurun_out; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 600 python -m pytest tests/test_search_gpu.py -x -q > $OUT/pt_search.log 2>&1; echo "rc=$?" >> $OUT/pt_search.log
for rep in 1 2; do
  for L in libtpo_b200.so libtpo_b200_rc0.so libtpo_b200_rc96.so; do
    echo "== $L" >> $OUT/vf_ab.txt
    TPO_NATIVE_LIB=$L timeout 300 python scripts/verify_families.py >> $OUT/vf_ab.txt 2>&1
  done
  echo "== chains off" >> $OUT/vf_ab.txt
  TPO_VM_CHAINS=0 timeout 300 python scripts/verify_families.py >> $OUT/vf_ab.txt 2>&1
done
for w in rmsnorm lora; do
  timeout 300 python scripts/ring_timeline.py $w STATIC=1 > $OUT/ring_$w.txt 2>&1
done
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
for w in rmsnorm lora; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:skinny -s 5 -c 1 \
      -o "$OUT/prof_$w" -f python bench.py --workload $w --profile --steps 8 --warmup 3 \
      > "$OUT/prof_$w.log" 2>&1
done

NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
for fam in gqa lora; do
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:verify -s 1 -c 1 \
  -o gpurun_out/prof_verify_$fam -f python -c "
import sys; sys.path.insert(0, '.')
from paper_2405_05751_b200 import fixtures as F
from paper_2405_05751_b200.api import Context
ctx = Context(0)
prog, pool = F.verify_families()['$fam']
gs = [g for _, g in pool]
for i in range(2):
    ctx.verify_pool(prog, gs, first=i * 50000, n=50000)
" > gpurun_out/prof_verify_$fam.log 2>&1
done

# fused skinny kernels: parity + sweeps + steady-state timelines (GPU box)
timeout 600 python -m pytest tests/test_fused_gpu.py -x -q > gpurun_out/pt_fused.txt 2>&1
python scripts/sweep.py lora "STATIC=1" "STATIC=1,TPO_MINB=2,TPO_STAGES=4" "STATIC=1,TPO_MINB=1" "STATIC=1,TPO_MINB=1,TPO_STAGES=8" "STATIC=1,TPO_MINB=1,TPO_STAGES=10" "STATIC=0" > gpurun_out/sweep_lora.txt 2>&1
python scripts/ring_timeline.py lora STATIC=1 | grep -v launch > gpurun_out/ring_lora.txt 2>&1

timeout 600 python -m pytest tests/test_fused_gpu.py -x -q > gpurun_out/pt_fused.txt 2>&1
python scripts/sweep.py lora "STATIC=1" "STATIC=1,TPO_MINB=2,TPO_STAGES=5" "STATIC=1,TPO_MINB=2,TPO_STAGES=5,TPO_TRIG_EARLY=2" "STATIC=1,TPO_MINB=2,TPO_STAGES=5,TPO_TRIG_EARLY=3" "STATIC=1,TPO_MINB=2,TPO_STAGES=5,TPO_TRIG_EARLY=5" "STATIC=1,TPO_MINB=2,TPO_STAGES=5,TPO_TRIG_EARLY=7" > gpurun_out/sweep_lora.txt 2>&1
python scripts/sweep.py rmsnorm "STATIC=1" "STATIC=1,TPO_KSPLIT=2" > gpurun_out/sweep_rms.txt 2>&1

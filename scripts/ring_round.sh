# fused skinny kernels: sweeps + steady-state timelines (GPU box)
python scripts/sweep.py rmsnorm "STATIC=1" "STATIC=1,TPO_L2PF=2" "STATIC=1,TPO_L2PF=4" "STATIC=1,TPO_L2PF=8" "STATIC=1,TPO_L2PF=16" > gpurun_out/sweep_rms.txt 2>&1
python scripts/sweep.py lora "STATIC=1" "STATIC=1,TPO_L2PF=2" "STATIC=1,TPO_L2PF=4" "STATIC=1,TPO_L2PF=8" > gpurun_out/sweep_lora.txt 2>&1
python scripts/sweep.py gatedmlp "STATIC=1" "STATIC=1,TPO_L2PF=4" > gpurun_out/sweep_g.txt 2>&1

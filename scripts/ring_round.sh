timeout 600 python -m pytest tests/test_fused_gpu.py -x -q > gpurun_out/pt_fused.txt 2>&1
python scripts/sweep.py rmsnorm "STATIC=1" "STATIC=1,TPO_TRIG_EARLY=4" "STATIC=1,TPO_TRIG_EARLY=6" "STATIC=1" > gpurun_out/sweep_rms.txt 2>&1
python bench.py --workload rmsnorm --no-verifier > gpurun_out/bench_rmsnorm.json 2> gpurun_out/bench_rmsnorm.err

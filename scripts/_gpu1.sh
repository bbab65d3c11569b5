cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_precision_gpu.py tests/test_fused_gpu.py tests/test_integration.py -x -q -m gpu > gpurun_out/pt1.log 2>&1
echo "rc=$?" >> gpurun_out/pt1.log

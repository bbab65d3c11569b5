OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_fused_gpu.py tests/test_precision_gpu.py tests/test_integration.py -x -q > $OUT/pt_aa.log 2>&1; echo "rc=$?" >> $OUT/pt_aa.log

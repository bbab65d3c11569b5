OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_fused_gpu.py tests/test_verify_gpu.py -x -q -k "paper_lora or lazy_input or test_fused" > $OUT/pt_z.log 2>&1; echo "rc=$?" >> $OUT/pt_z.log

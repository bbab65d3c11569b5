OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_fp_vm_gpu.py tests/test_precision_gpu.py -x -q > $OUT/pt_ee.log 2>&1; echo "rc=$?" >> $OUT/pt_ee.log
timeout 300 python scripts/fp_vm_sweep.py > $OUT/fp_vm_ee.txt 2>&1

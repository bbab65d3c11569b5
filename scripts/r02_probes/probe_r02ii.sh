OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_fp_vm_gpu.py tests/test_precision_gpu.py tests/test_verify_gpu.py -x -q -k "fp or stability or precision or unfused or optimize or full_shape" > $OUT/pt_ii.log 2>&1; echo "rc=$?" >> $OUT/pt_ii.log
timeout 300 python scripts/fp_vm_sweep.py > $OUT/fp_vm_cols.txt 2>&1
TPO_FP_MM_COLS=0 timeout 300 python scripts/fp_vm_sweep.py > $OUT/fp_vm_nocols.txt 2>&1

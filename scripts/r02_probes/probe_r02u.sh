OUT=gpurun_out; mkdir -p $OUT
for c in 0 1 2 3; do TPO_FP_MM=$c timeout 300 python scripts/fp_vm_sweep.py >> $OUT/fp_vm_sweep.txt 2>&1; done
timeout 600 python -m pytest tests/test_fp_vm_gpu.py -x -q > $OUT/pt_fpvm.log 2>&1; echo "rc=$?" >> $OUT/pt_fpvm.log

OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_fp_vm_gpu.py tests/test_precision_gpu.py -x -q > $OUT/pt_fpvm2.log 2>&1; echo "rc=$?" >> $OUT/pt_fpvm2.log
timeout 300 python scripts/fp_vm_sweep.py > $OUT/fp_vm_pdl.txt 2>&1
TPO_FP_NO_PDL=1 timeout 300 python scripts/fp_vm_sweep.py > $OUT/fp_vm_nopdl.txt 2>&1

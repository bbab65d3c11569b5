OUT=gpurun_out; mkdir -p $OUT
for rep in 1 2; do
timeout 300 python scripts/fp_vm_sweep.py >> $OUT/fp_vm_x.txt 2>&1
TPO_FP_PDL=1 timeout 300 python scripts/fp_vm_sweep.py | sed 's/cfg 0/pdl/' >> $OUT/fp_vm_x.txt 2>&1
done

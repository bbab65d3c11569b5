OUT=gpurun_out; mkdir -p $OUT
TPO_VM_DEBUG=1 timeout 300 python scripts/verify_families.py 50000 > $OUT/vf_dbg.txt 2>&1
for t in 64 128 256; do echo "== threads $t" >> $OUT/vf_thr.txt; TPO_VM_THREADS=$t timeout 300 python scripts/verify_families.py >> $OUT/vf_thr.txt 2>&1; done
echo "== default" >> $OUT/vf_thr.txt; timeout 300 python scripts/verify_families.py >> $OUT/vf_thr.txt 2>&1
TPO_VM_PROFILE=1 timeout 600 python scripts/vm_profile.py 50000 > $OUT/vm_profile2.txt 2>&1

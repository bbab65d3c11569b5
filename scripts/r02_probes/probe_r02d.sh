OUT=gpurun_out; mkdir -p $OUT
TPO_VM_CHAINS=0 timeout 300 python scripts/repro_ffeval.py > $OUT/repro_nochains.txt 2>&1; echo "rc=$?" >> $OUT/repro_nochains.txt
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 5 python scripts/repro_ffeval.py > $OUT/repro_memcheck.txt 2>&1; echo "rc=$?" >> $OUT/repro_memcheck.txt

OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_verify_gpu.py tests/test_search_gpu.py tests/test_chains.py -x -q > $OUT/pt_verify2.log 2>&1; echo "rc=$?" >> $OUT/pt_verify2.log
for rep in 1 2; do timeout 300 python scripts/verify_families.py >> $OUT/vf_sum.txt 2>&1; done
for w in rmsnorm lora; do timeout 300 python scripts/ring_timeline.py $w STATIC=1 > $OUT/ring3_$w.txt 2>&1; done

OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_verify_gpu.py tests/test_search_gpu.py -x -q > $OUT/pt_gg.log 2>&1; echo "rc=$?" >> $OUT/pt_gg.log
for rep in 1 2; do timeout 300 python scripts/verify_families.py >> $OUT/vf_gg.txt 2>&1; done

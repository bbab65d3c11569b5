OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_verify_gpu.py tests/test_search_gpu.py tests/test_chains.py -x -q > $OUT/pt_verify5.log 2>&1; echo "rc=$?" >> $OUT/pt_verify5.log
timeout 900 python bench.py --workload verify --steps 3 --warmup 3 > $OUT/bench_verify2.json 2> $OUT/bench_verify2.err
for rep in 1 2; do timeout 300 python scripts/verify_families.py >> $OUT/vf_t.txt 2>&1; done

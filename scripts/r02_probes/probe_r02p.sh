OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_verify_gpu.py tests/test_search_gpu.py tests/test_chains.py tests/test_shard.py -x -q > $OUT/pt_verify3.log 2>&1; echo "rc=$?" >> $OUT/pt_verify3.log
for rep in 1 2; do
  echo "== lazy" >> $OUT/vf_lazy.txt; timeout 300 python scripts/verify_families.py >> $OUT/vf_lazy.txt 2>&1
  echo "== eager" >> $OUT/vf_lazy.txt; TPO_VM_EAGER=1 timeout 300 python scripts/verify_families.py >> $OUT/vf_lazy.txt 2>&1
done

OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_verify_gpu.py tests/test_search_gpu.py -x -q > $OUT/pt_verify4.log 2>&1; echo "rc=$?" >> $OUT/pt_verify4.log
for rep in 1 2 3; do
  echo "== new" >> $OUT/vf_r.txt; timeout 300 python scripts/verify_families.py >> $OUT/vf_r.txt 2>&1
  echo "== base" >> $OUT/vf_r.txt; TPO_NATIVE_LIB=libtpo_b200_base.so timeout 300 python scripts/verify_families.py >> $OUT/vf_r.txt 2>&1
done

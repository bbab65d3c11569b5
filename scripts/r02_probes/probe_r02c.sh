#!/usr/bin/env bash
OUT=gpurun_out; mkdir -p $OUT
timeout 300 scripts/micro/read_floor_pdl > $OUT/read_floor_pdl.txt 2>&1; echo "rc=$?" >> $OUT/read_floor_pdl.txt
timeout 900 python -m pytest tests/test_verify_gpu.py tests/test_search_gpu.py -x -q > $OUT/pt_verify.log 2>&1; echo "rc=$?" >> $OUT/pt_verify.log
for rep in 1 2; do
  for L in libtpo_b200_new.so libtpo_b200_rc0.so; do
    echo "== $L" >> $OUT/vf_ab3.txt
    TPO_NATIVE_LIB=$L timeout 300 python scripts/verify_families.py >> $OUT/vf_ab3.txt 2>&1
  done
done

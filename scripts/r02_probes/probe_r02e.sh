OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python scripts/verify_families.py > $OUT/vf_new.txt 2>&1
timeout 600 scripts/micro/read_floor_pdl > $OUT/read_floor_pdl2.txt 2>&1; echo "rc=$?" >> $OUT/read_floor_pdl2.txt

OUT=gpurun_out; mkdir -p $OUT
for rep in 1 2 3; do
  echo "== mulc" >> $OUT/vf_q.txt; timeout 300 python scripts/verify_families.py >> $OUT/vf_q.txt 2>&1
  echo "== plain" >> $OUT/vf_q.txt; TPO_NATIVE_LIB=libtpo_b200_plain.so timeout 300 python scripts/verify_families.py >> $OUT/vf_q.txt 2>&1
  echo "== mulc nogroup" >> $OUT/vf_q.txt; TPO_VM_LAZY_GROUP=0 timeout 300 python scripts/verify_families.py >> $OUT/vf_q.txt 2>&1
done

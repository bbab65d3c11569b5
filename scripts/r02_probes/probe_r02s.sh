OUT=gpurun_out; mkdir -p $OUT
for rep in 1 2; do
  for L in libtpo_b200.so libtpo_b200_base.so libtpo_b200_idx0.so libtpo_b200_idx1.so libtpo_b200_idx2.so; do
    echo "== $L" >> $OUT/vf_s.txt; TPO_NATIVE_LIB=$L timeout 300 python scripts/verify_families.py >> $OUT/vf_s.txt 2>&1
  done
done

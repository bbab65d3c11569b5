cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for L in libtpo_b200.so libtpo_b200_rc0.so libtpo_b200_rc88.so; do
echo "== $L" >> gpurun_out/vf_ab.txt
TPO_NATIVE_LIB=$L python scripts/verify_families.py >> gpurun_out/vf_ab.txt 2>&1
done; done

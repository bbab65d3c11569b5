# Verifier at a 64-register cap (8 x 128-thread CTAs per SM, small spills) vs the default 72 (7 CTAs)
mkdir -p gpurun_out
TPO_NATIVE_LIB=libtpo_b200_rc64.so timeout 900 python -m pytest tests/test_verify_gpu.py -x -q -k "pool or distinct" > gpurun_out/rc_pt.txt 2>&1; echo rc=$? >> gpurun_out/rc_pt.txt
for r in 1 2; do
  echo "== default $r" >> gpurun_out/rc_fam.txt; python scripts/verify_families.py >> gpurun_out/rc_fam.txt 2>&1
  echo "== regcap64 $r" >> gpurun_out/rc_fam.txt; TPO_NATIVE_LIB=libtpo_b200_rc64.so python scripts/verify_families.py >> gpurun_out/rc_fam.txt 2>&1
done
TPO_NATIVE_LIB=libtpo_b200_rc64.so TPO_VM_DEBUG=1 python scripts/verify_families.py 20000 2>&1 | grep "tpo vm\]" | sort | uniq >> gpurun_out/rc_fam.txt

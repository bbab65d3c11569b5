# Stability filter: bytecode read in place (new) vs staged in shared memory (old build), plus parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fp_vm_gpu.py -x -q > gpurun_out/st_pt.txt 2>&1; echo rc=$? >> gpurun_out/st_pt.txt
for r in 1 2; do
  python bench.py --workload verify > gpurun_out/st_new_$r.json 2>/dev/null
  TPO_NATIVE_LIB=libtpo_b200_old.so python bench.py --workload verify > gpurun_out/st_old_$r.json 2>/dev/null
done

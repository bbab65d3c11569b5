# Verifier bytecode from global memory (L1) vs staged in shared memory: parity with it forced on, then A/B
mkdir -p gpurun_out
TPO_VM_CODE_GLOBAL=1 timeout 900 python -m pytest tests/test_verify_gpu.py tests/test_search_gpu.py tests/test_chains.py -x -q > gpurun_out/cg_pt.txt 2>&1; echo rc=$? >> gpurun_out/cg_pt.txt
for r in 1 2; do
  echo "== auto $r" >> gpurun_out/cg_fam.txt; python scripts/verify_families.py >> gpurun_out/cg_fam.txt 2>&1
  echo "== smem (0) $r" >> gpurun_out/cg_fam.txt; TPO_VM_CODE_GLOBAL=0 python scripts/verify_families.py >> gpurun_out/cg_fam.txt 2>&1
  echo "== global (1) $r" >> gpurun_out/cg_fam.txt; TPO_VM_CODE_GLOBAL=1 python scripts/verify_families.py >> gpurun_out/cg_fam.txt 2>&1
done
TPO_VM_DEBUG=1 python scripts/verify_families.py 20000 2>&1 | grep "tpo vm\]" | sort | uniq >> gpurun_out/cg_fam.txt

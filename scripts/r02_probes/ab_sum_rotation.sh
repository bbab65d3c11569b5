# Grouped-Sum per-lane start rotation (new) vs none (old build): parity, per-pool A/B, conflict counts on the GQA pool
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_verify_gpu.py tests/test_search_gpu.py tests/test_chains.py -x -q > gpurun_out/sr_pt.txt 2>&1; echo rc=$? >> gpurun_out/sr_pt.txt
for r in 1 2; do
  echo "== new $r" >> gpurun_out/sr_fam.txt; python scripts/verify_families.py >> gpurun_out/sr_fam.txt 2>&1
  echo "== old $r" >> gpurun_out/sr_fam.txt; TPO_NATIVE_LIB=libtpo_b200_old.so python scripts/verify_families.py >> gpurun_out/sr_fam.txt 2>&1
done
bash scripts/ncu_verify_src.sh

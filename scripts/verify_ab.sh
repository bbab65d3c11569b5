timeout 900 python -m pytest tests/test_verify_gpu.py -x -q -k "not full_shape" > gpurun_out/pt.txt 2>&1
TPO_VM_DEBUG=1 python scripts/verify_families.py 20000 2>&1 | grep "tpo vm\]" | sort | uniq > gpurun_out/dbg.txt
python scripts/verify_families.py > gpurun_out/fam.txt 2>&1
python scripts/verify_families.py > gpurun_out/fam2.txt 2>&1

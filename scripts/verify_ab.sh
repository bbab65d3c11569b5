timeout 900 python -m pytest tests/test_verify_gpu.py tests/test_fp_vm_gpu.py -x -q > gpurun_out/pt.txt 2>&1
python scripts/verify_families.py > gpurun_out/fam.txt 2>&1
TPO_VM_NOSYNC=0 python scripts/verify_families.py > gpurun_out/fam_sync.txt 2>&1
TPO_VM_PROFILE=1 python scripts/vm_profile.py 50000 > gpurun_out/vmprof.txt 2>&1

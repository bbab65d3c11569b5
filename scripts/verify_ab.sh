# verifier A/B (GPU box): per-family throughput under lowering toggles
python scripts/verify_families.py > gpurun_out/fam.txt 2>&1
TPO_VM_FFD=0 python scripts/verify_families.py > gpurun_out/fam_noffd.txt 2>&1
python scripts/verify_families.py > gpurun_out/fam2.txt 2>&1
TPO_VM_FFD=0 python scripts/verify_families.py > gpurun_out/fam_noffd2.txt 2>&1

for i in 1 2; do
python scripts/verify_families.py > gpurun_out/fam_a$i.txt 2>&1
TPO_VM_DBG=1 python scripts/verify_families.py > gpurun_out/fam_b$i.txt 2>&1
done

cd $GRAFT_REPO_ROOT
python scripts/verify_families.py > gpurun_out/vf.txt 2>&1
timeout 900 python -m pytest tests/test_verify_gpu.py -x -q > gpurun_out/pt_verify.log 2>&1; echo "rc=$?" >> gpurun_out/pt_verify.log
bash scripts/ncu_verify.sh
/usr/local/cuda/bin/ncu -i gpurun_out/prof_verify_gatedmlp.ncu-rep --page source --csv --print-source sass > gpurun_out/src_verify_gatedmlp.csv 2>&1
/usr/local/cuda/bin/ncu -i gpurun_out/prof_verify_rmsnorm.ncu-rep --page raw --csv > gpurun_out/raw_verify_rmsnorm.csv 2>&1
/usr/local/cuda/bin/ncu -i gpurun_out/prof_verify_gatedmlp.ncu-rep --page raw --csv > gpurun_out/raw_verify_gatedmlp.csv 2>&1

cd $GRAFT_REPO_ROOT
python scripts/verify_families.py > gpurun_out/vf.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pt_all.log 2>&1; echo "rc=$?" >> gpurun_out/pt_all.log
bash scripts/ncu_verify.sh
for f in gatedmlp rmsnorm; do
/usr/local/cuda/bin/ncu -i gpurun_out/prof_verify_$f.ncu-rep --page source --csv --print-source sass > gpurun_out/src_verify_$f.csv 2>&1
/usr/local/cuda/bin/ncu -i gpurun_out/prof_verify_$f.ncu-rep --page raw --csv > gpurun_out/raw_verify_$f.csv 2>&1
done

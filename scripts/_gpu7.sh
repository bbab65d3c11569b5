cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pt7.log 2>&1; echo "rc=$?" >> gpurun_out/pt7.log
python scripts/verify_families.py > gpurun_out/vf7.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo "rc=$?" >> gpurun_out/bench7.err

cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_search_gpu.py tests/test_verify_gpu.py tests/test_precision_gpu.py -x -q > gpurun_out/pt6.log 2>&1; echo "rc=$?" >> gpurun_out/pt6.log
timeout 900 python bench.py > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo "rc=$?" >> gpurun_out/bench6.err

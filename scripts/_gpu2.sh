cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "rc=$?" >> gpurun_out/bench.err

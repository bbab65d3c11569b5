OUT=gpurun_out; mkdir -p $OUT
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on -k regex:matmul_kernel -c 1 -o $OUT/prof_fpmm -f python scripts/vm_launches.py gatedmlp 0 > $OUT/prof_fpmm.log 2>&1

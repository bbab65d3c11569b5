OUT=gpurun_out; mkdir -p $OUT
timeout 300 python scripts/ring_timeline.py rmsnorm STATIC=1 > $OUT/ring7_rmsnorm.txt 2>&1
timeout 300 python scripts/ring_timeline.py rmsnorm STATIC=1 TPO_DBG_FLAGS=1 > $OUT/ring7_rmsnorm_f1.txt 2>&1

OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_fused_gpu.py tests/test_precision_gpu.py -x -q > $OUT/pt_fused.log 2>&1; echo "rc=$?" >> $OUT/pt_fused.log
for w in rmsnorm lora; do
timeout 300 python scripts/sweep.py $w "STATIC=1" "STATIC=1,TPO_DBG_FLAGS=32" "STATIC=1" "STATIC=1,TPO_DBG_FLAGS=32" > $OUT/sweep_st_$w.txt 2>&1
timeout 300 python scripts/ring_timeline.py $w STATIC=1 > $OUT/ring6_$w.txt 2>&1
done
timeout 300 python scripts/sweep.py gatedmlp "STATIC=1" "STATIC=1,TPO_DBG_FLAGS=32" > $OUT/sweep_st_gatedmlp.txt 2>&1

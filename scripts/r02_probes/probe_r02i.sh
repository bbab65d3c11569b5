OUT=gpurun_out; mkdir -p $OUT
for w in rmsnorm lora; do
timeout 300 python scripts/ring_timeline.py $w STATIC=1 > $OUT/ring2_$w.txt 2>&1
done

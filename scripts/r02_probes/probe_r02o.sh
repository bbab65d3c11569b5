OUT=gpurun_out; mkdir -p $OUT
for w in rmsnorm lora; do
timeout 600 python scripts/sweep.py $w "STATIC=1" "STATIC=1,TPO_EPI_ATOMIC=1" "STATIC=1,TPO_PRE_CUT=1" "STATIC=1,TPO_PRE_CUT=2" \
  "STATIC=1,TPO_TRIG_EARLY=3" "STATIC=1,TPO_TRIG_EARLY=4" "STATIC=1,TPO_TRIG_EARLY=6" "STATIC=1,TPO_L2_AHEAD=1" "STATIC=1,TPO_L2_AHEAD=3" "STATIC=1" > $OUT/sweep_misc_$w.txt 2>&1
done

OUT=gpurun_out; mkdir -p $OUT
for w in rmsnorm lora; do
timeout 900 python scripts/sweep.py $w "STATIC=1" "STATIC=1,TPO_DBG_FLAGS=1" "STATIC=1,TPO_DBG_FLAGS=2" "STATIC=1,TPO_DBG_FLAGS=3" \
  "STATIC=1,TPO_DBG_FLAGS=4" "STATIC=1,TPO_DBG_FLAGS=7" "STATIC=1,TPO_NO_PDL=1" "STATIC=0" > $OUT/sweep_dbg_$w.txt 2>&1
done
timeout 300 python scripts/ring_timeline.py rmsnorm STATIC=1 TPO_MINB=1 TPO_L2_AHEAD=0 TPO_STAGES=10 TPO_TRIG_EARLY=4 > $OUT/ring_rms_m1s10.txt 2>&1
TPO_VM_PROFILE=1 timeout 600 python scripts/vm_profile.py 50000 > $OUT/vm_profile.txt 2>&1
timeout 300 python scripts/verify_families.py > $OUT/vf_minb.txt 2>&1

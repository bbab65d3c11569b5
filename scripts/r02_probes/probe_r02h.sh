OUT=gpurun_out; mkdir -p $OUT
timeout 600 python scripts/sweep.py rmsnorm "STATIC=1" "STATIC=1,TPO_DBG_FLAGS=32" "STATIC=1,TPO_DBG_FLAGS=36" "STATIC=1,TPO_DBG_FLAGS=39" "STATIC=1,TPO_DBG_FLAGS=35" > $OUT/sweep_dbg2_rmsnorm.txt 2>&1
timeout 600 python scripts/sweep.py lora "STATIC=1" "STATIC=1,TPO_DBG_FLAGS=16" "STATIC=1,TPO_DBG_FLAGS=20" "STATIC=1,TPO_DBG_FLAGS=23" "STATIC=1,TPO_DBG_FLAGS=19" > $OUT/sweep_dbg2_lora.txt 2>&1
timeout 300 python scripts/ring_timeline.py lora STATIC=1 TPO_DBG_FLAGS=16 > $OUT/ring_lora_f16.txt 2>&1

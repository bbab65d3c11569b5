# LoRA / RMSNorm: PDL release point x L2 run-ahead, re-swept after the final LoRA changes (two passes, interleaved)
mkdir -p gpurun_out
for pass in 1 2; do
python scripts/sweep.py lora "STATIC=1" "STATIC=1,TPO_TRIG_EARLY=5" "STATIC=1,TPO_TRIG_EARLY=6" "STATIC=1,TPO_TRIG_EARLY=7" "STATIC=1,TPO_TRIG_EARLY=3" \
  "STATIC=1,TPO_L2_AHEAD=0" "STATIC=1,TPO_L2_AHEAD=2" "STATIC=1,TPO_TRIG_EARLY=6,TPO_L2_AHEAD=0" "STATIC=1,TPO_TRIG_EARLY=6,TPO_L2_AHEAD=2" \
  "STATIC=1,TPO_PRE_CUT=1" "STATIC=1,TPO_PRE_CUT=2" >> gpurun_out/sweep_trig_lora.txt 2>&1
python scripts/sweep.py rmsnorm "STATIC=1" "STATIC=1,TPO_TRIG_EARLY=4" "STATIC=1,TPO_TRIG_EARLY=6" "STATIC=1,TPO_TRIG_EARLY=7" \
  "STATIC=1,TPO_L2_AHEAD=1" "STATIC=1,TPO_L2_AHEAD=3" "STATIC=1,TPO_TRIG_EARLY=6,TPO_L2_AHEAD=1" "STATIC=1,TPO_PRE_CUT=1" >> gpurun_out/sweep_trig_rms.txt 2>&1
done

# GQA: steady-state timelines + sweep (GPU box)
for cfg in "" "TPO_STAGES=2" "TPO_KSPLIT=4 TPO_STAGES=3" "TPO_KSPLIT=4 TPO_STAGES=2"; do
python scripts/ring_timeline.py gqa $cfg | grep -v "launch  [0-9]:\|launch 1[0-2]"
done > gpurun_out/ring_gqa.txt 2>&1
python scripts/sweep.py gqa "" "TPO_STAGES=2" "TPO_KSPLIT=4" "TPO_KSPLIT=4,TPO_STAGES=2" "TPO_KSPLIT=1" "TPO_NO_PDL=1" > gpurun_out/sweep_gqa.txt 2>&1

OUT=gpurun_out; mkdir -p $OUT
timeout 300 python scripts/sweep.py lora "STATIC=1" "STATIC=1,TPO_TRIG_EARLY=2" "STATIC=1,TPO_L2_AHEAD=0" "STATIC=1,TPO_STAGES=4" > $OUT/sweep_xamma.txt 2>&1
TPO_NATIVE_LIB=libtpo_b200_xaring.so timeout 300 python scripts/sweep.py lora "STATIC=1" >> $OUT/sweep_xamma.txt 2>&1
timeout 900 python -m pytest tests/test_fused_gpu.py tests/test_precision_gpu.py tests/test_integration.py -x -q > $OUT/pt_fused.log 2>&1; echo "rc=$?" >> $OUT/pt_fused.log
timeout 300 python scripts/ring_timeline.py lora STATIC=1 > $OUT/ring5_lora.txt 2>&1

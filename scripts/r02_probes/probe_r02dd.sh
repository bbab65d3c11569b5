OUT=gpurun_out; mkdir -p $OUT
for w in lora gatedmlp; do
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,dram__bytes_read.sum --csv python scripts/vm_launches.py $w 0 > $OUT/vm_launch2_$w.csv 2>&1
done

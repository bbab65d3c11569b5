OUT=gpurun_out; mkdir -p $OUT
/usr/local/cuda/bin/ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:reduce --csv python scripts/r02_probes/l2_writeback.py > $OUT/l2_writeback_cc_all.csv 2>&1
/usr/local/cuda/bin/ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:reduce --csv python scripts/r02_probes/l2_writeback.py > $OUT/l2_writeback_cc_none.csv 2>&1

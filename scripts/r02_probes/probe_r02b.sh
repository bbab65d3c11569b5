#!/usr/bin/env bash
# Round-2 investigation (GPU box): PDL read floor, verifier A/B, shared-GPU
# multi-rank logic check of the verifier's single gather.
OUT=gpurun_out; mkdir -p $OUT
timeout 300 scripts/micro/read_floor_pdl > $OUT/read_floor_pdl.txt 2>&1
for rep in 1 2; do
  for L in libtpo_b200.so libtpo_b200_rc0.so libtpo_b200_rc0r.so libtpo_b200_r.so; do
    echo "== $L" >> $OUT/vf_ab2.txt
    TPO_NATIVE_LIB=$L timeout 300 python scripts/verify_families.py >> $OUT/vf_ab2.txt 2>&1
  done
done
timeout 600 python bench.py --workload verify --steps 3 --warmup 3 --no-cpu-baseline > $OUT/v1.json 2> $OUT/v1.err
for n in 2 4; do
  TPO_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --workload verify --steps 3 --warmup 3 \
    > $OUT/v$n.json 2> $OUT/v$n.err
done

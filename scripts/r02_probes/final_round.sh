#!/usr/bin/env bash
# Round-2 final evidence: the standard GPU round plus the shared-GPU
# multi-rank logic check of the verifier (N = 2, 4; bit-identical gather).
OUT=gpurun_out; mkdir -p $OUT
bash scripts/gpu_round.sh tests smoke bench launches full
timeout 600 python bench.py --workload verify --steps 3 --warmup 3 --no-cpu-baseline > $OUT/v1.json 2> $OUT/v1.err
for n in 2 4; do
  TPO_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n --workload verify --steps 3 --warmup 3 \
    > $OUT/v$n.json 2> $OUT/v$n.err
done

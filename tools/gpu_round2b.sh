#!/bin/bash
# Multi-GPU check (gpurun --gpus N): GPU tests incl. the multi-device ones,
# 1-GPU and N-GPU weak-scaling bench lines, strong scaling of one batch.
OUT=${1:-gpurun_out/r2b}
NG=${2:-2}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/gputest.txt 2>&1
echo "pytest rc=$?" >> $OUT/gputest.txt
timeout 600 python bench.py --no-cpu-baseline --no-api --steps 5 > $OUT/bench_n1.json 2> $OUT/bench_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus $NG --steps 5 --warmup 3 > $OUT/bench_n$NG.json 2> $OUT/bench_n$NG.err
echo "torchrun rc=$?" >> $OUT/bench_n$NG.err
timeout 600 python tools/bench_strong.py > $OUT/strong.jsonl 2> $OUT/strong.err
ls -la $OUT

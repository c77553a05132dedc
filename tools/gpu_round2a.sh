#!/bin/bash
# Round-2 check on one GPU: GPU test suite, default bench (config 3), then the
# launch list of the same bench.  usage: tools/gpu_round2a.sh OUT
OUT=${1:-gpurun_out/r2a}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/gputest.txt 2>&1
echo "pytest rc=$?" >> $OUT/gputest.txt
timeout 900 python bench.py > $OUT/bench_config3.json 2> $OUT/bench_config3.err
echo "bench rc=$?" >> $OUT/bench_config3.err
timeout 600 python bench.py --no-cpu-baseline --no-api --steps 2 --warmup 3 > $OUT/plain_for_ncu.json 2>&1 && \
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_config3.csv \
    python bench.py --no-cpu-baseline --no-api --steps 2 --warmup 3 > $OUT/ncu_launch.log 2>&1
ls -la $OUT

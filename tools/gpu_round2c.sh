#!/bin/bash
# Round-2 regression + headline refresh on one GPU: GPU tests, default bench
# (config 3), config-4 pipeline with the CPU alignment baseline.
OUT=${1:-gpurun_out/r2e}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/gputest.txt 2>&1
echo "pytest rc=$?" >> $OUT/gputest.txt
timeout 900 python bench.py > $OUT/bench_config3.json 2> $OUT/bench_config3.err
timeout 900 python tools/bench_pipeline.py 100000 4 --cpu-baseline > $OUT/config4_pipeline.json 2> $OUT/config4_pipeline.err
timeout 300 python tools/bench_pipeline.py 1000 0 --cpu-baseline > $OUT/config1_pipeline.json 2> $OUT/config1_pipeline.err
ls -la $OUT

#!/bin/bash
# Round-2 profile recipe (one GPU, under gpurun).  Plain runs first (the bench
# lines), then ncu on the same command lines: the launch list of config 3 and
# --set full captures of the dominant kernels (K1p and K5 of class R = 9, the
# largest share of config 3; a later call's launch, after the pool has grown).
# usage: tools/prof_r02.sh OUT
OUT=${1:-gpurun_out/prof_r02}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/gpu.txt
timeout 900 python bench.py > $OUT/bench_config3.json 2> $OUT/bench_config3.err || exit 1
timeout 600 python bench.py --workload config2 --no-api > $OUT/bench_config2.json 2> $OUT/bench_config2.err
timeout 900 python bench.py --workload config5 --steps 3 --no-api > $OUT/bench_config5.json 2> $OUT/bench_config5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
CMD="python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-api"
timeout 600 $CMD > $OUT/plain.json 2>&1 || exit 2
N="ncu --clock-control none"
timeout 900 $N --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_config3.csv \
    $CMD > $OUT/ncu_launches.log 2>&1
timeout 900 $N --set full --import-source on --kernel-name-base mangled \
    -k "regex:k_score_packedILi9E" -s 1 -c 1 -o $OUT/prof_k1p9 $CMD > $OUT/ncu_k1p.log 2>&1
timeout 900 $N --set full --import-source on --kernel-name-base mangled \
    -k "regex:k_tbILi9E" -s 1 -c 1 -o $OUT/prof_k5_9 $CMD > $OUT/ncu_k5.log 2>&1
CMD5="python bench.py --workload config5 --pairs 600 --steps 1 --warmup 1 --no-cpu-baseline --no-api"
timeout 600 $CMD5 > $OUT/plain5.json 2>&1 && \
timeout 900 $N --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_config5.csv \
    $CMD5 > $OUT/ncu_launches5.log 2>&1
ls -la $OUT

#!/bin/bash
# Round profile recipe (run under gpurun, one GPU).  Plain runs first (these are
# the bench numbers), then ncu: the launch list of the default bench command and
# one --set full capture of the dominant kernels.  usage: tools/prof_round.sh <outdir>
OUT=${1:-gpurun_out/round}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/gpu.txt
timeout 600 python bench.py > $OUT/bench_config2.json 2> $OUT/bench_config2.err || exit 1
timeout 600 python bench.py --workload config3 --no-cpu-baseline > $OUT/bench_config3.json 2> $OUT/bench_config3.err
timeout 900 python bench.py --workload config5 --steps 3 --no-cpu-baseline > $OUT/bench_config5.json 2> $OUT/bench_config5.err
N="ncu --clock-control none"
timeout 600 $N --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_config2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 $N --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_config3.csv \
    python bench.py --workload config3 --pairs 100000 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 $N --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_config5.csv \
    python bench.py --workload config5 --pairs 500 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 $N --set full --import-source on --kernel-name-base mangled \
    -k "regex:k_score_packedILi10E|k_tbILi10E" -s 2 -c 2 -o $OUT/prof_config2 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_config2.log 2>&1
timeout 900 $N --set full --import-source on --kernel-name-base mangled \
    -k "regex:k_score_ctaILi16ELi0E" -s 1 -c 1 -o $OUT/prof_config5 \
    python bench.py --workload config5 --pairs 300 --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_config5.log 2>&1
ls -la $OUT

#!/bin/bash
# Round profile refresh (one GPU): benches (plain runs first), reference arm,
# config-4 pipeline, launch lists, --set full captures of K1p / K5 (config 2)
# and the packed long-pair forward (config 5).  usage: tools/prof_round3.sh OUT
OUT=${1:-gpurun_out/round3}
mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_config2.json 2> $OUT/bench_config2.err || exit 1
timeout 600 python bench.py --workload config3 --steps 10 --no-cpu-baseline > $OUT/bench_config3.json 2> $OUT/bench_config3.err
timeout 900 python bench.py --workload config5 --steps 3 --no-cpu-baseline > $OUT/bench_config5.json 2> $OUT/bench_config5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 600 python tools/bench_pipeline.py > $OUT/config4_pipeline.json 2> $OUT/config4_pipeline.err
N="ncu --clock-control none"
timeout 600 $N --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_config2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 $N --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_config3.csv \
    python bench.py --workload config3 --pairs 200000 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 $N --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_config5.csv \
    python bench.py --workload config5 --pairs 1000 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 $N --set full --import-source on --kernel-name-base mangled \
    -k "regex:k_score_packedILi10E|k_tbILi10E" -s 2 -c 2 -o $OUT/prof_config2 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_config2.log 2>&1
timeout 900 $N --set full --import-source on --kernel-name-base mangled \
    -k "regex:k_score_cta_packed" -s 1 -c 1 -o $OUT/prof_ctap \
    python bench.py --workload config5 --pairs 600 --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_ctap.log 2>&1
ls $OUT

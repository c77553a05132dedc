#!/bin/bash
# Profile recipe (run under gpurun): plain run first, then ncu captures.
# usage: tools/prof.sh <tag> [extra bench args]
set -e
TAG=${1:-r1}; shift || true
CMD="python bench.py --pairs 20000 --steps 1 --warmup 3 --no-cpu-baseline $@"
$CMD > gpurun_out/plain_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_score<10, 0|k_box<10>|k_walk' -s 3 -c 3 -o gpurun_out/prof_$TAG $CMD \
    > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log

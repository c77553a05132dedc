#!/bin/bash
# Profile recipe (run under gpurun): plain run first, then ncu captures.
# usage: tools/prof.sh <tag> <mangled-name-regex> [extra bench args]
set -e
TAG=${1:-r1}; shift || true
RX=${1:-k_scoreILi10ELi0ELb0ELb1|k_tbILi10}; shift || true
CMD="python bench.py --pairs 20000 --steps 1 --warmup 3 --no-cpu-baseline $@"
$CMD > gpurun_out/plain_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:$RX" -s 2 -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log

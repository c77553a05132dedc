#!/bin/bash
# config-5 profile of the scalar forward (long pairs)
CMD="python bench.py --workload config5 --pairs 300 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:k_scoreILi16ELi0ELb0" -s 1 -c 1 -o gpurun_out/prof_c5 $CMD > gpurun_out/ncu_c5.log 2>&1
tail -2 gpurun_out/ncu_c5.log

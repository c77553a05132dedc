#!/bin/bash
# ncu --set full capture of one K1p launch (class R = 9, config 3) with source
# correlation, after a plain run of the same command exits 0.
# usage (under gpurun): tools/prof_k1p.sh OUT [lib.so]
OUT=${1:-gpurun_out/k1p}
mkdir -p $OUT
[ -n "$2" ] && export PASTIS_SW_LIB=$2
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-api"
timeout 600 $CMD > $OUT/plain.json 2>&1 || exit 2
timeout 900 ncu --clock-control none --set full --import-source on --kernel-name-base mangled \
    -k "regex:${K:-k_score_packedILi9E}" -s 1 -c 1 -o $OUT/prof $CMD > $OUT/ncu.log 2>&1
ls -la $OUT

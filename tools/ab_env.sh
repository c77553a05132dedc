#!/bin/bash
# A/B environment settings of one build on one GPU (under gpurun):
# tools/ab_env.sh OUTDIR "NAME:VAR=V VAR2=V2" ... [-- extra bench args]
OUT=$1; shift
mkdir -p $OUT
cfgs=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do cfgs+=("$1"); shift; done
[ "$1" == "--" ] && shift
for rep in 1 2; do
for c in "${cfgs[@]}"; do
  name=${c%%:*}; envs=${c#*:}
  env $envs timeout 300 python bench.py --steps 10 --no-cpu-baseline "$@" > $OUT/$name.$rep.json 2> $OUT/$name.$rep.err
  python - "$OUT/$name.$rep.json" "$name" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:>8} fwd {d['forward_gcups']:8.1f} total {d['value']:8.1f} e2e {d['e2e']['value']:8.1f} ok {d.get('results_ok')}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
done | tee $OUT/summary.txt

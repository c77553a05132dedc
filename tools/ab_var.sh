#!/bin/bash
# A/B the var/*.so builds on one GPU: forward GCUPS + total GCUPS per variant.
# usage (under gpurun): tools/ab_var.sh OUTDIR v0 v1 ... [-- extra bench args]
OUT=$1; shift
mkdir -p $OUT
vars=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do vars+=("$1"); shift; done
[ "$1" == "--" ] && shift
for rep in 1 2; do
for v in "${vars[@]}"; do
  PASTIS_SW_LIB=var/$v.so timeout 300 python bench.py --steps 10 --no-cpu-baseline "$@" > $OUT/$v.$rep.json 2> $OUT/$v.$rep.err
  python - "$OUT/$v.$rep.json" "$v" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:>6} fwd {d['forward_gcups']:8.1f} total {d['value']:8.1f} e2e {d['e2e']['value']:8.1f} ok {d.get('results_ok')} mhz {d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
done | tee $OUT/summary.txt

#!/bin/bash
# A/B of env-selected K3 variants on the default library: VARS="NAME=VAL NAME=VAL ..." ("-" = no env)
cd "$(dirname "$0")/.."
for c in ${CFGS:-c2}; do
  for v in ${VARS:--}; do
    if [ "$v" = "-" ]; then e=""; else e="$v"; fi
    env $e timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps ${STEPS:-20} 2>/dev/null | python3 -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c [$v]', round(d['ms_per_step'],3), 'K3', round(d['kernels_ms']['k3_attention'],3), 'K1', round(d['kernels_ms']['k1_reorder_quantize'],4), 'frac', round(d['roofline']['frac'],4))" 2>/dev/null || echo "$c [$v] FAILED"
  done
done

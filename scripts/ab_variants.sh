#!/bin/bash
# K3 d=64 variants: every paro_b200/_lib_*/libparo_b200.so build vs the default library (c2 unless CFGS)
cd "$(dirname "$0")/.."
for c in ${CFGS:-c2}; do
  for lib in paro_b200/_lib/libparo_b200.so paro_b200/_lib_*/libparo_b200.so; do
    tag=$(basename $(dirname $lib))
    PARO_B200_LIB=$PWD/$lib timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps ${STEPS:-20} 2>/dev/null | python3 -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $tag', round(d['ms_per_step'],3), 'K3', round(d['kernels_ms']['k3_attention'],3), 'frac', round(d['roofline']['frac'],4))" 2>/dev/null || echo "$c $tag FAILED"
  done
done

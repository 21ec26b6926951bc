#!/bin/bash
# K3 ms per config for each library variant (default lib first)
cd "$(dirname "$0")/.."
for c in ${CFGS:-c2 c5}; do
  for v in default ${VARIANTS}; do
    if [ "$v" = default ]; then L=$PWD/paro_b200/_lib/libparo_b200.so; else L=$PWD/paro_b200/_lib_$v/libparo_b200.so; fi
    PARO_B200_LIB=$L timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps ${STEPS:-10} 2>&1 | python3 -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', '$v', round(d['kernels_ms']['k3_attention'],3))"
  done
done

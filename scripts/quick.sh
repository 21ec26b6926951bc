#!/bin/bash
# quick GPU check: parity tests (-x) + K3 bench lines for the given configs + phase profile
cd "$(dirname "$0")/.."
CFGS=${CFGS:-"c2 c3 c4 c5"}
timeout 600 python -m pytest tests -m gpu -q -x ${TESTS:-} 2>&1 | tail -4
for c in $CFGS; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps ${STEPS:-20} 2>&1 | python3 -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['kernels_ms'].items()}, 'frac', round(d['roofline']['frac'],4))"
done
if [ -n "$PROF" ]; then
  for c in $PROF; do
    PARO_B200_LIB=$PWD/paro_b200/_lib_prof/libparo_b200.so PARO_K3_PROF_PRINT=1 timeout 300 python bench.py --config $c --profile --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep "k3 prof" | tail -3
  done
fi

#!/bin/bash
# K4 (dense text-prefix rows) A/B: tcgen05 k4_dense_tc vs the mma.sync k4_dense (PARO_K4_LEGACY=1)
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -m gpu -q -x -k "prefix or dense or fuzz" 2>&1 | tail -2
for c in ${CFGS:-c2 c5}; do
  for lg in 1 0; do
    PARO_K4_LEGACY=$lg timeout 300 python bench.py --config $c --dense-prefix 226 --no-cpu-baseline --no-e2e --steps ${STEPS:-10} 2>&1 | python3 -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c legacy=$lg', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['kernels_ms'].items()})"
  done
done
if [ -n "$NCU" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k4 -c 4 --csv python bench.py --config c2 --dense-prefix 226 --profile --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E "k4" | cut -c1-400
fi

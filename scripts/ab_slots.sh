#!/bin/bash
# the d=64 multi-slot kernel (PARO_K3_SLOTS=1) vs the default layout, plus phase timers
cd "$(dirname "$0")/.."
timeout 300 env PARO_K3_SLOTS=1 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for c in ${CFGS:-c2 c3}; do
  for v in 0 1; do
    for lib in paro_b200/_lib paro_b200/_lib_s2n4; do
      [ $v = 0 ] && [ $lib != paro_b200/_lib ] && continue
      PARO_K3_SLOTS=$v PARO_B200_LIB=$PWD/$lib/libparo_b200.so timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python3 -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c slots=$v $lib K3', round(d['kernels_ms']['k3_attention'],3))" || echo "$c slots=$v $lib FAILED"
    done
  done
done
PARO_K3_SLOTS=1 PARO_B200_LIB=$PWD/paro_b200/_lib_prof/libparo_b200.so PARO_K3_PROF_PRINT=1 timeout 300 python bench.py --profile --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep "prof\]" | tail -2

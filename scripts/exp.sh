#!/bin/bash
# K3 time + phase profile for each experiment library variant on config $CFG
cd "$(dirname "$0")/.."
CFG=${CFG:-c2}
for v in ${VARIANTS:-prof NOQUANT NOEXP ONECTA NOEPI}; do
  echo "== $v"
  PARO_B200_LIB=$PWD/paro_b200/_lib_$v/libparo_b200.so timeout 300 python bench.py --config $CFG --no-cpu-baseline --no-e2e --steps 10 2>&1 | python3 -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('k3', round(d['kernels_ms']['k3_attention'],3))"
  PARO_B200_LIB=$PWD/paro_b200/_lib_$v/libparo_b200.so PARO_K3_PROF_PRINT=1 timeout 300 python bench.py --config $CFG --profile --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep "k3 prof" | tail -3
done

#!/bin/bash
# A/B of the d=64 K3 kernels on c2/c3: the multi-slot kernel, PARO_K3_LEGACY=1 (the
# two-CTA layout), and the legacy layout built with passive waits (_lib_passive)
cd "$(dirname "$0")/.."
run() { # label, env...
  local label=$1; shift
  env "$@" timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps ${STEPS:-20} 2>&1 | python3 -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $label', round(d['ms_per_step'],3), 'K3', round(d['kernels_ms']['k3_attention'],3), 'frac', round(d['roofline']['frac'],4))" || echo "$c $label FAILED"
}
for c in ${CFGS:-c2 c3}; do
  run slots PARO_K3_LEGACY=0
  run legacy PARO_K3_LEGACY=1
  [ -f paro_b200/_lib_passive/libparo_b200.so ] && run legacy-passive PARO_K3_LEGACY=1 PARO_B200_LIB=$PWD/paro_b200/_lib_passive/libparo_b200.so
done
# the session-start build (round-1 head) when present, for regression checks
for c in ${CFGS:-c2 c3}; do
  [ -f paro_b200/_lib_old/libparo_b200.so ] && run round1-lib PARO_K3_LEGACY=1 PARO_B200_LIB=$PWD/paro_b200/_lib_old/libparo_b200.so
done

#!/bin/bash
# K3 time and DRAM traffic with the L2-grouped LPT order (default) vs one global LPT order
cd "$(dirname "$0")/.."
for c in ${CFGS:-c2 c5}; do
  for g in default 0; do
    if [ $g = default ]; then unset PARO_L2_GROUP_HEADS; else export PARO_L2_GROUP_HEADS=$g; fi
    timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python3 -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c group=$g K3', round(d['kernels_ms']['k3_attention'],3), 'ms')"
    PARO_WATCHDOG_S=0 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k3_attention -s 1 -c 1 --csv python bench.py --config $c --profile --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' '{print "   ", $(NF-2), $(NF-1), $NF}'
  done
done
unset PARO_L2_GROUP_HEADS

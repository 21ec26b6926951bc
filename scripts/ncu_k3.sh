#!/bin/bash
# one ncu --set full capture of K3 (second launch) for config $1 -> gpurun_out/$2.ncu-rep
cd "$(dirname "$0")/.."
export PARO_WATCHDOG_S=0
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k3_attention -s 1 -c 1 -o gpurun_out/$2 python bench.py --config $1 --profile --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/$2.log 2>&1
grep -E "ERROR|passes" gpurun_out/$2.log

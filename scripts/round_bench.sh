#!/bin/bash
# full evidence run: gpu tests, smoke, bench lines for every config, the reference arm,
# the launch list, ncu captures of K1/K3 (c2) and K3 (c5), sanitizers over smoke
cd "$(dirname "$0")/.."
TAG=${TAG:-r02}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rA 2>&1 | grep -E "PASS|FAIL|ERROR|SKIP|passed|failed" | tail -400 > gpurun_out/${TAG}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
timeout 300 python bench.py --mask-family banded --no-cpu-baseline > gpurun_out/${TAG}_bench_c2_banded.json 2>/dev/null
for c in c3 c4 c4i4 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2>/dev/null; done
for c in c3 c5; do timeout 900 python bench.py --config $c --v-packed --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_${c}_vpacked.json 2>/dev/null; done
timeout 300 python bench.py --schedule 50 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c2_schedule.json 2>/dev/null
timeout 300 python bench.py --schedule 50 --schedule-prefetch --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c2_schedule_prefetch.json 2>/dev/null
timeout 300 python bench.py --config maskgen > gpurun_out/${TAG}_bench_maskgen.json 2>/dev/null
timeout 300 python bench.py --config permsel > gpurun_out/${TAG}_bench_permsel.json 2>/dev/null
for c in c2 c5; do timeout 900 python bench.py --config $c --dense-prefix 226 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_${c}_prefix226.json 2>/dev/null; done
timeout 300 python bench.py --rope --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c2_rope.json 2>/dev/null
PARO_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c2_gpus2_gloo_1gpu.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_ref_c2.json 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --profile --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
PARO_WATCHDOG_S=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k3_attention -s 1 -c 1 -o gpurun_out/${TAG}_k3_c2 python bench.py --profile --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
PARO_WATCHDOG_S=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1_reorder -s 1 -c 1 -o gpurun_out/${TAG}_k1_c2 python bench.py --profile --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
PARO_WATCHDOG_S=0 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k3_attention -s 1 -c 1 -o gpurun_out/${TAG}_k3_c5 python bench.py --config c5 --profile --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
PARO_WATCHDOG_S=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k3_attention -s 1 -c 1 -o gpurun_out/${TAG}_k3_c4 python bench.py --config c4 --profile --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
PARO_WATCHDOG_S=0 timeout 900 compute-sanitizer --tool memcheck --leak-check full python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_memcheck_smoke.log 2>&1
PARO_WATCHDOG_S=0 timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_racecheck_smoke.log 2>&1
PARO_WATCHDOG_S=0 timeout 900 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_synccheck_smoke.log 2>&1
ls -la gpurun_out | grep $TAG

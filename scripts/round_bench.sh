#!/bin/bash
# full evidence run: gpu tests, smoke, bench lines for every config, reference arm, launch list + ncu of K1/K3 (c2)
cd "$(dirname "$0")/.."
TAG=${TAG:-r01b}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rA 2>&1 | grep -E "PASS|FAIL|ERROR|passed|failed|adapter" | tail -200 > gpurun_out/${TAG}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
timeout 300 python bench.py --mask-family banded --no-cpu-baseline > gpurun_out/${TAG}_bench_c2_banded.json 2>/dev/null
for c in c3 c4 c4i4 c5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2>/dev/null; done
timeout 300 python bench.py --config maskgen > gpurun_out/${TAG}_bench_maskgen.json 2>/dev/null
timeout 300 python bench.py --config permsel > gpurun_out/${TAG}_bench_permsel.json 2>/dev/null
for c in c2 c5; do timeout 600 python bench.py --config $c --dense-prefix 226 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_${c}_prefix226.json 2>/dev/null; done
timeout 300 python bench.py --rope --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c2_rope.json 2>/dev/null
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref_c2.json 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --profile --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
PARO_WATCHDOG_S=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k3_attention -s 1 -c 1 -o gpurun_out/${TAG}_k3_c2 python bench.py --profile --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
PARO_WATCHDOG_S=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_reorder -s 1 -c 1 -o gpurun_out/${TAG}_k1_c2 python bench.py --profile --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out | grep $TAG

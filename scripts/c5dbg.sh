cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --config c4i4 --no-cpu-baseline --no-e2e --steps 5 2>&1 | tail -2 | cut -c1-300
for W in 4 30; do
  START=$(date +%s.%N)
  PARO_WATCHDOG_S=$W timeout 300 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-300
  echo "watchdog $W: elapsed $(echo "$(date +%s.%N) - $START" | bc)"
done
timeout 300 python -m pytest tests/test_gpu_fullscale.py -q -x 2>&1 | grep -E "^E |passed|failed" | head -5

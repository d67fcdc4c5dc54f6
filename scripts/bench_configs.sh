#!/bin/bash
# 1-GPU bench of the other BASELINE configs (c1: reference CPU case, c3:
# Reddit-shaped, D = 602 input features) without the e2e / CPU legs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in ${CONFIGS:-c1 c3}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline ${EXTRA:-} > gpurun_out/bench_$c.log 2>&1
  echo "$c rc=$?"
  grep -o '"value": [0-9.]*, "unit": "ms"' gpurun_out/bench_$c.log | head -1
  grep -o '"phases_ms": {[^}]*}' gpurun_out/bench_$c.log | head -1
  grep -o '"spmm_ms_per_epoch": [0-9.]*' gpurun_out/bench_$c.log
  tail -n 3 gpurun_out/bench_$c.log | cut -c 1-300
done

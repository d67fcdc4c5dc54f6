#!/bin/bash
# A/B of runtime env variants on one box: ENVS is a "|"-separated list of
# "VAR=val VAR2=val" strings ("-" = none), run in order (repeat for noise).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
IFS='|' read -ra LIST <<< "${ENVS:--}"
i=0
for v in "${LIST[@]}"; do
  e="$v"; [ "$e" = "-" ] && e=""
  env $e timeout 600 python bench.py --steps ${STEPS:-8} --warmup 3 --no-e2e --no-cpu-baseline ${EXTRA:-} > gpurun_out/abenv_$i.log 2>&1
  echo "[$v] $(grep -o '"value": [0-9.]*' gpurun_out/abenv_$i.log | head -1) $(grep -o '"backward_s": [0-9.]*' gpurun_out/abenv_$i.log) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/abenv_$i.log)"
  i=$((i+1))
done

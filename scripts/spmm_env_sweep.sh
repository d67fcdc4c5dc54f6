#!/bin/bash
# SpMM probe (C2, FAST plans) under env variants: ENVS "|"-separated.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
IFS='|' read -ra LIST <<< "${ENVS:--}"
for v in "${LIST[@]}"; do
  e="$v"; [ "$e" = "-" ] && e=""
  echo "== [$v]"
  env $e timeout 300 python scripts/spmm_probe.py --widths ${WIDTHS:-100,256} --thresholds 4096 --fast 2>&1 | grep '"d"' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if 'd' in d: print('  d', d['d'], 'ms', round(d['plan_ms'][1], 3))"
done

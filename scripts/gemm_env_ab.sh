#!/bin/bash
# GEMM shapes of one C2 epoch (scripts/gemm_bench.py, FAST) under env variants.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
IFS='|' read -ra LIST <<< "${ENVS:--}"
for v in "${LIST[@]}"; do
  e="$v"; [ "$e" = "-" ] && e=""
  echo "== [$v]"
  env $e timeout 600 python scripts/gemm_bench.py fast 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    if 'form' in d: print('  %s m=%d n=%d k=%d  %.3f ms' % (d['form'], d['m'], d['n'], d['k'], d['fast_ms']))
    else: print('  total', d)"
done

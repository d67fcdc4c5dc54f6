#!/bin/bash
# Rebuilds the library with list-kernel tuning macros on the GPU box and
# times the SpMM probe (D=100 and D=256, FAST plans) for each combination.
# COMBOS: "|"-separated "U1 U2 UNROLL HALF32" tuples.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
IFS='|' read -ra LIST <<< "${COMBOS:-4 4 16 0|8 4 16 0|4 4 1 0}"
for combo in "${LIST[@]}"; do
  set -- $combo
  make -s -C paper_2505_04083_b200/csrc clean > /dev/null
  make -s -j16 -C paper_2505_04083_b200/csrc NVFLAGS_EXTRA="-DPK_LIST_U1=$1 -DPK_LIST_U2=$2 -DPK_LIST_UNROLL=$3 -DPK_LIST_HALF32=${4:-0}" > /dev/null 2>&1
  echo "U1=$1 U2=$2 UNROLL=$3 HALF32=${4:-0}"
  timeout 300 python scripts/spmm_probe.py --widths 100,256 --thresholds 4096 --fast 2>&1 | grep '"d"' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if 'd' in d: print('  d', d['d'], 'ms', round(d['plan_ms'][1], 3))"
done

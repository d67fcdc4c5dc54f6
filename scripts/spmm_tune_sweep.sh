#!/bin/bash
# Rebuilds the library with list-kernel tuning macros on the GPU box and
# times the SpMM probe (D=100 and D=256, FAST plans) for each combination.
# COMBOS: "|"-separated "U1 MINB1 U8 MINB8" tuples (VEC<=4 one-vector form,
# VEC=8 form; D=100 runs the first, D=256 the second).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
IFS='|' read -ra LIST <<< "${COMBOS:-4 4 2 4}"
for combo in "${LIST[@]}"; do
  set -- $combo
  rm -f paper_2505_04083_b200/csrc/_obj/spmm.o  # only the SpMM unit sees the macros
  make -s -j16 -C paper_2505_04083_b200/csrc NVFLAGS_EXTRA="-DPK_LIST_U1=$1 -DPK_LIST_MINB1=$2 -DPK_LIST_U8=$3 -DPK_LIST_MINB8=$4" > /dev/null 2>&1
  echo "U1=$1 MINB1=$2 U8=$3 MINB8=$4"
  timeout 300 python scripts/spmm_probe.py --widths ${WIDTHS:-100,256} --thresholds 4096 --fast 2>&1 | grep '"d"' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if 'd' in d: print('  d', d['d'], 'ms', round(d['plan_ms'][1], 3))"
done

#!/bin/bash
# L2 eviction hints on/off and hot-column factor for the 256-bit gathers.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for h in 0 1; do
  make -s -C paper_2505_04083_b200/csrc clean > /dev/null
  make -s -j16 -C paper_2505_04083_b200/csrc NVFLAGS_EXTRA="-DPK_LIST_HINTS=$h" > /dev/null 2>&1
  for f in ${FACTORS:-2}; do
    echo "HINTS=$h HOT_FACTOR=$f"
    PK_HOT_FACTOR=$f timeout 300 python scripts/spmm_probe.py --widths 256 --thresholds 4096 --fast 2>&1 | grep '"d"' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if 'd' in d: print('  d', d['d'], 'ms', round(d['plan_ms'][1], 3))"
  done
done

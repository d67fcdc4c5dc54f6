#!/bin/bash
# Gathers in flight for the narrow 2-vector-per-lane list form (D = 33..64
# at 4-B vectors: C2's transform-first 47-wide SpMMs): rebuilds spmm.o with
# PK_LIST_U2 = each value and times the probe at widths 47 and 41.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for u in ${US:-4 8 12}; do
  rm -f paper_2505_04083_b200/csrc/_obj/spmm.o
  make -s -j16 -C paper_2505_04083_b200/csrc NVFLAGS_EXTRA="-DPK_LIST_U2=$u" > /dev/null 2>&1
  echo "U2=$u"
  timeout 300 python scripts/spmm_probe.py --widths ${WIDTHS:-47,41} --thresholds 4096 --fast 2>&1 | grep '"d"' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if 'd' in d: print('  d', d['d'], 'ms', round(d['plan_ms'][1], 3))"
done

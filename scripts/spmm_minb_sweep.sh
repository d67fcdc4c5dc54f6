#!/bin/bash
# Rebuilds spmm.cu with different PK_LIST_MINB values on the GPU box and
# runs the SpMM probe for each (experiment; the committed build uses the
# default in spmm.cu).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for mb in ${MINBS:-2 3}; do
  make -s -C paper_2505_04083_b200/csrc clean > /dev/null
  make -s -j16 -C paper_2505_04083_b200/csrc NVFLAGS_EXTRA="-DPK_LIST_MINB=$mb" > /dev/null 2>&1
  echo "MINB=$mb"
  timeout 300 python scripts/spmm_probe.py --widths 100,256 --thresholds 4096 2>&1 | grep '"d"'
done

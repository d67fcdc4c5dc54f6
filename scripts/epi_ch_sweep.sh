#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for ch in 8 16 32; do
  rm -f paper_2505_04083_b200/csrc/_obj/gemm_tc.o
  make -s -j16 -C paper_2505_04083_b200/csrc NVFLAGS_EXTRA="-DPK_EPI_CH=$ch" > /dev/null 2>&1 || echo "build failed"
  echo "== PK_EPI_CH=$ch"
  timeout 300 python scripts/gemm_bench.py fast 2>&1 | grep -E '"TN"|total'
done

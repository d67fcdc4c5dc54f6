#!/bin/bash
# Rebuild gemm_tc with -DPK_TC_PROF, print the per-role wait breakdown, restore.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
rm -f paper_2505_04083_b200/csrc/_obj/gemm_tc.o
make -s -j16 -C paper_2505_04083_b200/csrc NVFLAGS_EXTRA="-DPK_TC_PROF ${EXTRA_FLAGS:-}" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 python scripts/tc_prof.py

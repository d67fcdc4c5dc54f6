#!/bin/bash
# Diagnostics: per-role tcgen05 GEMM wait breakdown (PK_TC_PROF build) and
# the per-rank solo compute of the 4-GPU C2 grid on one B200.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python scripts/solo_ranks.py --config c2 --grid 2,1,2 > gpurun_out/solo_c2_212.log 2>&1; echo "solo rc=$?"; grep SOLO gpurun_out/solo_c2_212.log
timeout 600 python scripts/solo_ranks.py --config c2 --grid 2,1,1 > gpurun_out/solo_c2_211.log 2>&1; echo "solo2 rc=$?"; grep SOLO gpurun_out/solo_c2_211.log
bash scripts/tc_prof.sh > gpurun_out/tc_prof.log 2>&1; echo "tc_prof rc=$?"; cat gpurun_out/tc_prof.log

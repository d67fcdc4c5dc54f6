#!/bin/bash
# FAST warp-per-row loss kernel (PK_CE_WARP): FAST tests incl. C2, epoch
# A/B, and the loss launch time in the epoch launch list.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_engine_gpu.py tests/test_switches_gpu.py tests/test_cluster_gpu.py -k "fast or engine or switch or forward" > gpurun_out/cew_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/cew_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest -q -x tests/test_c2_parity_gpu.py -k fast -s > gpurun_out/cew_c2.log 2>&1; echo "c2 fast rc=$?"; grep -a "FAST vs\|passed\|failed" gpurun_out/cew_c2.log | tail -2
ENVS="PK_CE_WARP=0|-|PK_CE_WARP=0|-" bash scripts/ab_env.sh
PK_COMMIT=ce-warp bash scripts/ncu_list_only.sh c2 | grep -E "ce_|serialised"

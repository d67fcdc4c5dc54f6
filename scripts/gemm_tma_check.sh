#!/bin/bash
# TMA-fed tcgen05 GEMM: correctness (tests/test_gemm_tc_gpu.py) then the
# epoch's GEMM shapes with and without it.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_tc_gpu.py -x -q > gpurun_out/pytest_tc_tma.log 2>&1; echo "pytest tma rc=$?"; tail -n 15 gpurun_out/pytest_tc_tma.log
ENVS="${ENVS:--|PK_TC_TMA=0}" bash scripts/gemm_env_ab.sh

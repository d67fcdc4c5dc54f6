#!/bin/bash
# Fused multiply-add chains in FAST SpMM plans (PK_SPMM_FMA_FAST): the
# affected tests, the C2 FAST parity test, and the epoch A/B on C2.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_switches_gpu.py tests/test_cluster_gpu.py -k "spmm or fast or engine or switch" > gpurun_out/fma_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fma_pytest.log
timeout 900 python -m pytest -q -x tests/test_c2_parity_gpu.py -k fast -s > gpurun_out/fma_c2.log 2>&1; echo "c2 fast rc=$?"; grep -a "FAST vs\|passed\|failed" gpurun_out/fma_c2.log | tail -3
ENVS="${ENVS:-PK_SPMM_FMA_FAST=0|-|PK_SPMM_FMA_FAST=0|-}" bash scripts/ab_env.sh

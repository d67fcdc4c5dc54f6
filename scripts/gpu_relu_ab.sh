#!/bin/bash
# ReLU' in the transform-first backward GEMM epilogue (PK_GEMM_RELU_BWD):
# engine / GEMM / C2-FAST tests and an epoch A/B on C2.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x tests/test_engine_gpu.py tests/test_gemm_tc_gpu.py tests/test_cluster_gpu.py -k "fast or gemm or engine" > gpurun_out/relu_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/relu_pytest.log
timeout 900 python -m pytest -q -x tests/test_c2_parity_gpu.py -k fast > gpurun_out/relu_c2.log 2>&1; echo "c2 fast rc=$?"; grep -a "FAST vs\|passed\|failed" gpurun_out/relu_c2.log | tail -2
ENVS="${ENVS:-PK_GEMM_RELU_BWD=0|PK_GEMM_RELU_BWD=1|PK_GEMM_RELU_BWD=0|PK_GEMM_RELU_BWD=1}" bash scripts/ab_env.sh

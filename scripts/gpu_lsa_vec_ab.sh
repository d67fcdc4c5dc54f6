#!/bin/bash
# 256-bit ordered reductions (PK_LSA_VEC=8) on 2 GPUs: multi-GPU parity
# tests with it, then the C2 epoch A/B (gpurun --gpus 2).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
PK_LSA_VEC=8 timeout 1200 python -m pytest -q -x tests/test_multigpu_gpu.py > gpurun_out/lsavec_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/lsavec_pytest.log
REPS="1 2" CFGS="- PK_LSA_VEC=8" bash scripts/overlap_sweep.sh

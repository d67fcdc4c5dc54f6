#!/bin/bash
# TMA bulk-copy two-member reduction (PK_LSA_BULK=1), gpurun --gpus 2: the
# multi-GPU parity tests with it, then the C2 epoch A/B at 2x1x1.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
PK_LSA_BULK=1 timeout 900 python -m pytest -q -x tests/test_multigpu_gpu.py -k "two_gpu or every_grid" > gpurun_out/bulk_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bulk_pytest.log
REPS="1 2" CFGS="- PK_LSA_BULK=1" bash scripts/overlap_sweep.sh

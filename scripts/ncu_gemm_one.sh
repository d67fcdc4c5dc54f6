#!/bin/bash
# Full ncu sections (with source) for one GEMM shape: SHAPE="NN,2097152,47,256"
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
S=${SHAPE:-NN,2097152,47,256}
timeout 300 python scripts/gemm_bench.py fast --only=$S > gpurun_out/gemm_one_plain.log 2>&1 || { echo "plain failed"; cat gpurun_out/gemm_one_plain.log; exit 1; }
cat gpurun_out/gemm_one_plain.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 2 -c 1 -o gpurun_out/prof_gemm_one -f python scripts/gemm_bench.py fast --only=$S > gpurun_out/ncu_gemm_one.log 2>&1; echo "ncu rc=$?"

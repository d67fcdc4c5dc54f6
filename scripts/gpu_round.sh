#!/bin/bash
# One gpurun payload: GPU tests, smoke, 1-GPU bench. Logs land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi -L
timeout 300 python -m pytest tests/test_gemm_tc_gpu.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest tc rc=$?"
timeout 900 python -m pytest tests -m gpu -q --deselect tests/test_gemm_tc_gpu.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 --mode parity --no-e2e --no-cpu-baseline > gpurun_out/bench_parity.log 2>&1; echo "bench parity rc=$?"
for f in gpurun_out/pytest_tc.log gpurun_out/pytest_gpu.log gpurun_out/smoke.log; do tail -n 3 $f; done; tail -c 2500 gpurun_out/bench.log; tail -c 1500 gpurun_out/bench_parity.log

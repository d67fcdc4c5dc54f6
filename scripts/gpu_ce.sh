#!/bin/bash
# Loss kernel with batched stage-in loads: its tests, the engine tests, and
# the CE launch time under ncu.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_kernels_gpu.py tests/test_engine_gpu.py -k "cross_entropy or engine or smoke" > gpurun_out/ce_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ce_pytest.log
timeout 600 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-c1-measured > gpurun_out/ce_bench.log 2>&1; echo "bench $(grep -o '"value": [0-9.]*' gpurun_out/ce_bench.log | head -1)"
timeout 600 ncu --kernel-name regex:ce_kernel --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 2 --csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-c1-measured 2>/dev/null | grep -a "ce_kernel" | cut -c1-20,200-400

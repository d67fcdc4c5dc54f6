#!/bin/bash
# Final one-GPU payload at HEAD: full GPU suite, smoke, the default bench
# line, then the ncu launch list + traffic JSON (small outputs only).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_full.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|C2 " gpurun_out/pytest_gpu_full.log | tail -14
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/bench_final.log | tail -1
PK_COMMIT=${PK_COMMIT} bash scripts/ncu_list_only.sh c2

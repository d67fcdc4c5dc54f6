#!/bin/bash
# One-GPU payload at HEAD: full GPU suite, the default bench line, a
# PK_TF_VEC=2 A/B, the ncu launch list + traffic JSON (PK_COMMIT), then the
# narrow-SpMM U2 sweep (rebuilds spmm.o: last).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_full.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|C2 " gpurun_out/pytest_gpu_full.log | tail -14
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/bench_final.log") if l.startswith("{")][-1])
print(d["value"], d["e2e"]["value"], d["phases_ms"], d["roofline"]["spmm_ms_per_epoch"], d["clocks"])
PY
PK_TF_VEC=2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c1-measured --no-e2e > gpurun_out/bench_tfvec2.log 2>&1
echo "tfvec2 $(grep -o '"value": [0-9.]*' gpurun_out/bench_tfvec2.log | head -1) $(grep -o '"spmm_ms_per_epoch": [0-9.]*' gpurun_out/bench_tfvec2.log)"
PK_COMMIT=${PK_COMMIT} bash scripts/ncu_r2.sh c2 > gpurun_out/ncu_r2.out 2>&1; echo "ncu rc=$?"; cat gpurun_out/ncu_spmm_c2.json
US="4 8" WIDTHS=47 bash scripts/spmm_u2_sweep.sh

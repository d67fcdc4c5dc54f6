#!/bin/bash
# Paired narrow SpMM form (PK_TF_PAIR): its tests, an epoch A/B on C2, and
# the narrow launches' durations and DRAM bytes under ncu.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_kernels_gpu.py tests/test_engine_gpu.py \
  -k "paired or fast or engine" > gpurun_out/pair_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pair_pytest.log
timeout 900 python -m pytest -q -x tests/test_c2_parity_gpu.py -k fast > gpurun_out/pair_c2.log 2>&1; echo "c2 fast rc=$?"; grep -a "FAST vs\|passed\|failed" gpurun_out/pair_c2.log | tail -3
ENVS="${ENVS:-PK_TF_PAIR=0|PK_TF_PAIR=1|PK_TF_PAIR=0|PK_TF_PAIR=1}" bash scripts/ab_env.sh
for v in 0 1; do
  PK_TF_PAIR=$v timeout 600 ncu --kernel-name regex:'spmm_(pair|list)_kernel' --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 6 --csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/pair_ncu_$v.csv 2> gpurun_out/pair_ncu_$v.err
  echo "ncu PK_TF_PAIR=$v rc=$?"
  python - "$v" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/pair_ncu_{sys.argv[1]}.csv")) if len(r) > 10]
hdr = rows[0]; K = hdr.index("Kernel Name"); M = hdr.index("Metric Name"); V = hdr.index("Metric Value"); I = hdr.index("ID")
d = {}
for r in rows[1:]:
    d.setdefault((r[I], r[K][:48]), {})[r[M]] = r[V]
for (i, k), m in d.items():
    print(i, k, {kk.split("__")[1][:18]: vv for kk, vv in m.items()})
PY
done

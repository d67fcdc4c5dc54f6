#!/bin/bash
# Backward order A/B (gpurun --gpus 4): multi-GPU tests, then C2 at 2x1x1 /
# 2x1x2 with PK_BWD_DH_FIRST=1 vs 0, then C2 / C3 scaling at 1 / 2 / 4.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_multigpu_gpu.py -q -rA -x > gpurun_out/pytest_multi.log 2>&1
echo "pytest multi rc=$?"; grep -E "passed|failed|^FAILED" gpurun_out/pytest_multi.log | tail -3
for rep in 1 2; do
for cfg in "2 2,1,1 1" "2 2,1,1 0" "4 2,1,2 1" "4 2,1,2 0"; do
  set -- $cfg
  PK_BWD_DH_FIRST=$3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 \
    --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $1 --grid $2 \
    --steps 20 --warmup 5 --no-cpu-baseline --no-c1-measured --no-e2e > gpurun_out/bwd_ab.log 2>&1
  python - "n$1 $2 dh_first=$3 rep$rep" <<'PY'
import json, sys
d = json.loads([l for l in open("gpurun_out/bwd_ab.log") if l.startswith("{")][-1])
print(sys.argv[1], round(d["value"], 2), round(d["collectives"]["ms_per_epoch"], 2),
      {k: round(v, 2) for k, v in d["phases_ms"].items()})
PY
done
done
for c in c2 c3; do
  for n in 1 2 4; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29800 + n)) bench.py --config $c --gpus $n \
      --steps 20 --warmup 5 --no-cpu-baseline --no-c1-measured > gpurun_out/scale_${c}_n$n.log 2>&1
    echo "$c n=$n rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/scale_${c}_n$n.log | head -2 | tr '\n' ' ') $(grep -o '"grid": "[0-9x]*"' gpurun_out/scale_${c}_n$n.log | head -1) $(grep -o '"ms_per_epoch": [0-9.]*' gpurun_out/scale_${c}_n$n.log | head -1)"
  done
done

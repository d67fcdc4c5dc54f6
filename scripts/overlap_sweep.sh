#!/bin/bash
# Row-chunked reductions beside their producers, with the reduction kernel
# on fewer SMs (gpurun --gpus N): C2 epoch and collective time for each
# CFGS entry (GPUS=2: grid 2,1,1; GPUS=4: grid 2,1,2).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
G=${GPUS:-2}; GRID=${GRID:-$([ "$G" = 4 ] && echo 2,1,2 || echo 2,1,1)}
for rep in ${REPS:-1 2}; do
for cfg in ${CFGS:-"-" "PK_COMM_CHUNKS=4" "PK_COMM_CHUNKS=4 PK_LSA_CTAS=148" "PK_COMM_CHUNKS=4 PK_LSA_CTAS=74" "PK_LSA_CTAS=148"}; do
  e="$cfg"; [ "$e" = "-" ] && e=""
  env $e timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
    --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $G --grid $GRID \
    --steps 20 --warmup 5 --no-cpu-baseline --no-c1-measured --no-e2e > gpurun_out/ov.log 2>&1
  python - "$cfg $rep" <<'PY'
import json, sys
try:
    d = json.loads([l for l in open("gpurun_out/ov.log") if l.startswith("{")][-1])
    print(sys.argv[1], round(d["value"], 2), round(d["collectives"]["ms_per_epoch"], 2),
          round(d["collectives"]["bus_gbs"], 1), {k: round(v, 2) for k, v in d["phases_ms"].items()})
except Exception as ex:
    print(sys.argv[1], "failed", ex); print(open("gpurun_out/ov.log").read()[-1500:])
PY
done
done

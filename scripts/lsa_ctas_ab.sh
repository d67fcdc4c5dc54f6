#!/bin/bash
# Ordered peer-memory reduction CTAs (gpurun --gpus 2): C2 at 2x1x1 with
# PK_LSA_CTAS = 74 / 148 / 296 and NCCL (PK_LSA=0).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in ${CFGS:-"PK_LSA_CTAS=148" "PK_LSA_CTAS=296" "PK_LSA_CTAS=74" "PK_LSA=0"}; do
  env $cfg timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --grid 2,1,1 \
    --steps 20 --warmup 5 --no-cpu-baseline --no-c1-measured --no-e2e > gpurun_out/lsa_ab.log 2>&1
  python - "$cfg $rep" <<'PY'
import json, sys
d = json.loads([l for l in open("gpurun_out/lsa_ab.log") if l.startswith("{")][-1])
print(sys.argv[1], round(d["value"], 2), round(d["collectives"]["ms_per_epoch"], 2),
      round(d["collectives"]["bus_gbs"], 1))
PY
done
done

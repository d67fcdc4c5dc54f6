#!/bin/bash
# Multi-GPU bench variants (no tests): NCCL CTA caps, with PK_TIMING for the load.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=$(nvidia-smi -L | wc -l)
for ctas in ${CTAS:-16 0}; do
  echo "PK_NCCL_MAX_CTAS=$ctas"
  PK_TIMING=1 PK_NCCL_MAX_CTAS=$ctas timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/benchq_$N_$ctas.log 2>&1
  grep -o '"value": [0-9.]*, "unit": "ms", "n_gpus[^}]*' gpurun_out/benchq_$N_$ctas.log | head -1
  grep -o '"phases_ms": {[^}]*}' gpurun_out/benchq_$N_$ctas.log
  grep "pk load r0" gpurun_out/benchq_$N_$ctas.log | tail -12
done

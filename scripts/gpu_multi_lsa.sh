#!/bin/bash
# Multi-GPU bench variants: NCCL vs ordered peer-memory reductions with
# different CTA counts; PK_TIMING prints the e2e load phases.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=$(nvidia-smi -L | wc -l)
run() {
  env "$@" PK_TIMING=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29566 bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/benchv.log 2>&1
  echo "$@: $(grep -o '"value": [0-9.]*, "unit": "ms", "n_gpus' gpurun_out/benchv.log | head -1) $(grep -o '"collectives_s": [0-9.]*' gpurun_out/benchv.log)"
  grep -o '"e2e": {"value": [0-9.]*' gpurun_out/benchv.log
}
run PK_LSA=0
run PK_LSA=1 PK_LSA_CTAS=296
run PK_LSA=1 PK_LSA_CTAS=148
run PK_LSA=1 PK_LSA_CTAS=64
grep "pk load r0" gpurun_out/benchv.log | tail -14

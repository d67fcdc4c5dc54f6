#!/bin/bash
# Multi-GPU epoch time vs comm pipeline depth (PK_COMM_CHUNKS) and reduction
# engine (PK_LSA): GRIDS / CHUNKS / LSA lists, bench without e2e / CPU legs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for lsa in ${LSA:-1}; do
for ch in ${CHUNKS:-1 2 4 8}; do
for g in ${GRIDS:-auto}; do
  ga=""; [ "$g" != auto ] && ga="--grid $g"
  PK_LSA=$lsa PK_COMM_CHUNKS=$ch timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-cpu-baseline $ga > gpurun_out/chunks_${lsa}_${ch}_${g}.log 2>&1
  echo "lsa=$lsa chunks=$ch grid=$g $(grep -o '"value": [0-9.]*' gpurun_out/chunks_${lsa}_${ch}_${g}.log | head -1) $(grep -o '"grid": "[^"]*"' gpurun_out/chunks_${lsa}_${ch}_${g}.log) $(grep -o '"spmm_ms_per_epoch": [0-9.]*' gpurun_out/chunks_${lsa}_${ch}_${g}.log) $(grep -o '"collectives_s": [0-9.]*' gpurun_out/chunks_${lsa}_${ch}_${g}.log)"
done; done; done

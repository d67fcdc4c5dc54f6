#!/bin/bash
# Round-2 multi-GPU payload (gpurun --gpus 4): multi-GPU parity + abort
# tests, then C2 bench at N=2 / N=4 on the model's grid and the 4-member-axis
# grids, ring-cost push all-reduce (default) vs all-pull (PK_LSA_PUSH=0).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
G=$(nvidia-smi -L | wc -l)
echo "GPUs: $G"
timeout 1500 python -m pytest tests/test_multigpu_gpu.py -x -q > gpurun_out/pytest_multi.log 2>&1
echo "pytest multi rc=$?"; tail -3 gpurun_out/pytest_multi.log
run() {  # n grid push tag
  PK_LSA_PUSH=$3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 \
    --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $1 \
    --grid $2 --steps 5 --warmup 3 --no-cpu-baseline --no-c1-measured --no-e2e \
    > gpurun_out/ab_$4.log 2>&1
  echo "$4 rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/ab_$4.log | head -1) \
$(grep -o '"ms_per_epoch": [0-9.]*' gpurun_out/ab_$4.log | head -1)"
}
for push in 1 0; do
  run 2 2,1,1 $push n2_211_push$push
  run 4 2,1,2 $push n4_212_push$push
  run 4 1,1,4 $push n4_114_push$push
  run 4 4,1,1 $push n4_411_push$push
  run 4 1,4,1 $push n4_141_push$push
done
# scaling on the performance model's grids (default push), full bench line
for n in 1 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29800 + n)) bench.py --gpus $n \
    --steps 10 --warmup 3 --no-cpu-baseline --no-c1-measured > gpurun_out/scale_c2_n$n.log 2>&1
  echo "scale n=$n rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/scale_c2_n$n.log | head -2 | tr '\n' ' ') $(grep -o '"grid": "[0-9x]*"' gpurun_out/scale_c2_n$n.log | head -1)"
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29911 scripts/grid_sweep.py --epochs 3 > gpurun_out/grid_sweep_n4.log 2>&1
echo "sweep rc=$?"; tail -3 gpurun_out/grid_sweep_n4.log

#!/bin/bash
# Round-2 multi-GPU payload after transform-first (gpurun --gpus 4):
# multi-GPU parity + abort tests, C2 / C3 scaling at 1 / 2 / 4 GPUs on the
# performance model's grids, the C5 sweep at 4.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_multigpu_gpu.py -q -rA > gpurun_out/pytest_multi.log 2>&1
echo "pytest multi rc=$?"; grep -E "passed|failed" gpurun_out/pytest_multi.log | tail -2
for c in c2 c3; do
  for n in 1 2 4; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29800 + n)) bench.py --config $c --gpus $n \
      --steps 20 --warmup 5 --no-cpu-baseline --no-c1-measured > gpurun_out/scale_${c}_n$n.log 2>&1
    echo "$c n=$n rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/scale_${c}_n$n.log | head -2 | tr '\n' ' ') $(grep -o '"grid": "[0-9x]*"' gpurun_out/scale_${c}_n$n.log | head -1) $(grep -o '"ms_per_epoch": [0-9.]*' gpurun_out/scale_${c}_n$n.log | head -1)"
  done
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29911 scripts/grid_sweep.py --epochs 3 > gpurun_out/grid_sweep_n4.log 2>&1
echo "sweep rc=$?"; grep -E "^\{|SWEEP" gpurun_out/grid_sweep_n4.log

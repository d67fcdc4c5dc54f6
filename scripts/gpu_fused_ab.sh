#!/bin/bash
# Producer-fused reductions (gpurun --gpus 4): multi-GPU tests, then C2 A/B
# PK_FUSED_REDUCE=1 vs 0 at 2 and 4 GPUs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_multigpu_gpu.py -q -rA -x > gpurun_out/pytest_multi_fused.log 2>&1
echo "pytest multi rc=$?"; grep -E "passed|failed|^FAILED" gpurun_out/pytest_multi_fused.log | tail -4
run() {  # n grid fused tag
  PK_FUSED_REDUCE=$3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 \
    --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $1 \
    --grid $2 --steps 20 --warmup 5 --no-cpu-baseline --no-c1-measured --no-e2e \
    > gpurun_out/fab_$4.log 2>&1
  echo "$4 rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/fab_$4.log | head -1) \
$(grep -o '"ms_per_epoch": [0-9.]*' gpurun_out/fab_$4.log | head -1)"
}
for f in 1 0; do
  run 2 2,1,1 $f n2_211_f$f
  run 4 2,1,2 $f n4_212_f$f
  run 4 1,1,4 $f n4_114_f$f
  run 4 2,2,1 $f n4_221_f$f
done

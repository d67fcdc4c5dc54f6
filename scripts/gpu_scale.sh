#!/bin/bash
# Scaling payload (gpurun --gpus N): bench.py for each config in CONFIGS at
# every power of two up to the box's GPU count, one torchrun per N.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
G=$(nvidia-smi -L | wc -l)
echo "GPUs: $G"
for c in ${CONFIGS:-c2 c3}; do
  n=1
  while [ $n -le $G ]; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --config $c --gpus $n \
      --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/scale_${c}_n$n.log 2>&1
    echo "$c n=$n rc=$?"
    grep -o '"value": [0-9.]*, "unit": "ms"' gpurun_out/scale_${c}_n$n.log | head -2 | tr '\n' ' '
    grep -o '"grid": "[0-9x]*"' gpurun_out/scale_${c}_n$n.log | head -1
    n=$((n * 2))
  done
done

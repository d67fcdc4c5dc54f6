#!/bin/bash
# Multi-GPU payload (gpurun --gpus N): engine parity vs the reference's
# distributed pass on every grid of N, then bench.py at N under torchrun.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
echo "GPUs: $N"
timeout 1200 python -m pytest tests/test_multigpu_gpu.py -q -x > gpurun_out/pytest_multi_$N.log 2>&1; echo "pytest multi rc=$?"
tail -5 gpurun_out/pytest_multi_$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/bench_$N.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_$N.log

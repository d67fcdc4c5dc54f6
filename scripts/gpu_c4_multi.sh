#!/bin/bash
# Billion-edge training on 4 GPUs (gpurun --gpus 4): s25 first, s24 if it
# does not fit.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for s in ${SCALES:-25 24}; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29933 scripts/c4_multi.py --scale $s --edges 1600000000 --grid ${GRID:-2,1,2} \
    > gpurun_out/c4_multi_s$s.log 2>&1
  rc=$?
  echo "s$s rc=$rc"; grep C4MULTI gpurun_out/c4_multi_s$s.log; tail -3 gpurun_out/c4_multi_s$s.log | cut -c1-300
  if grep -q C4MULTI gpurun_out/c4_multi_s$s.log; then break; fi
done

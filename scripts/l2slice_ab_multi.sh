#!/bin/bash
# A/B of the L2-sliced SpMM form on C3 at N GPUs (torchrun).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for mb in ${MBS:-0 96}; do
  PK_SPMM_L2_MB=$mb timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29611 bench.py --config c3 --gpus $N --steps 5 --warmup 3 \
    --no-e2e --no-cpu-baseline > gpurun_out/l2slice_n${N}_$mb.log 2>&1
  echo "N=$N MB=$mb rc=$?"
  tail -1 gpurun_out/l2slice_n${N}_$mb.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print(' value',round(d['value'],2),'grid',d['config']['grid'],'spmm_ms',round(r['spmm_ms_per_epoch'],2),'clk',d['clocks']['sm_mhz'],'loss',d['losses'][-1])"
done

#!/bin/bash
# A/B of the padded odd-width SpMM (engine.cu spmm_width) on C3 at N GPUs,
# after the engine and multi-GPU parity tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_multigpu_gpu.py -q -x > gpurun_out/pytest_pad_n$N.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_pad_n$N.log
for pad in ${PADS:-0 2}; do
  PK_SPMM_PAD=$pad timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29612 bench.py --config c3 --gpus $N --steps 5 --warmup 3 \
    --no-e2e --no-cpu-baseline > gpurun_out/pad_n${N}_$pad.log 2>&1
  echo "N=$N PAD=$pad rc=$?"
  tail -1 gpurun_out/pad_n${N}_$pad.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print(' value',round(d['value'],2),'grid',d['config']['grid'],'spmm_ms',round(r['spmm_ms_per_epoch'],2),'clk',d['clocks']['sm_mhz'],'loss',d['losses'][-1])"
done

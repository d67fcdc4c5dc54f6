#!/bin/bash
# A/B of the L2-sliced wide-row SpMM form (spmm.cu l2_sliced) on C3 at 1 GPU.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "l2_sliced or bitwise_random" > gpurun_out/pytest_l2slice.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_l2slice.log
for mb in ${MBS:-0 96}; do
  PK_SPMM_L2_MB=$mb timeout 600 python bench.py --config ${CFG:-c3} --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/l2slice_$mb.log 2>&1
  echo "MB=$mb rc=$?"
  tail -1 gpurun_out/l2slice_$mb.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print(' value',round(d['value'],2),'spmm_ms',round(r['spmm_ms_per_epoch'],2),'frac',round(r['frac'],3),'clk',d['clocks']['sm_mhz'],d['clocks']['reasons'],'loss',d['losses'][-1])"
done

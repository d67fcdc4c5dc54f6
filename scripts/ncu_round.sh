#!/bin/bash
# ncu evidence for the epoch (1 GPU), one ncu pass per gpurun call:
#   PART=list  launch list of one epoch (time + DRAM bytes per launch)
#   PART=spmm  full sections for the top SpMM list launches
#   PART=gemm  full sections for the tensor-core GEMM launches
# The plain run goes first and must exit 0.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${1:-c2}
PART=${PART:-list}
timeout 600 python scripts/epoch_driver.py --config $CFG > gpurun_out/ncu_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/ncu_plain.log; exit 1; }
case $PART in
  list)
    timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv python scripts/epoch_driver.py --config $CFG > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
    python scripts/spmm_traffic.py gpurun_out/launches_$CFG.csv gpurun_out/ncu_spmm_$CFG.json ;;
  spmm)
    timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:spmm_list -c 3 -o gpurun_out/prof_spmm_$CFG -f python scripts/epoch_driver.py --config $CFG > gpurun_out/ncu_spmm.log 2>&1; echo "spmm rc=$?" ;;
  gemm)
    timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:gemm_tc_kernel -c 9 -o gpurun_out/prof_gemm_$CFG -f python scripts/epoch_driver.py --config $CFG > gpurun_out/ncu_gemm.log 2>&1; echo "gemm rc=$?" ;;
esac
ls -la gpurun_out/ | tail -8

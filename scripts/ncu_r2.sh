#!/bin/bash
# Round-2 ncu evidence at HEAD (1 GPU, C2 epoch): plain run first (must exit
# 0), then the launch list (time + DRAM bytes per launch -> the bench's
# roofline.traffic JSON), then full sections of the top SpMM and GEMM
# launches. PK_COMMIT names the commit in the traffic JSON.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${1:-c2}
timeout 600 python scripts/epoch_driver.py --config $CFG > gpurun_out/ncu_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/ncu_plain.log; exit 1; }
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv python scripts/epoch_driver.py --config $CFG > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
python scripts/spmm_traffic.py gpurun_out/launches_$CFG.csv gpurun_out/ncu_spmm_$CFG.json
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:spmm_list -c 2 -o gpurun_out/prof_spmm_$CFG -f python scripts/epoch_driver.py --config $CFG > gpurun_out/ncu_spmm.log 2>&1; echo "spmm full rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:gemm_tc_kernel -c 3 -o gpurun_out/prof_gemm_$CFG -f python scripts/epoch_driver.py --config $CFG > gpurun_out/ncu_gemm.log 2>&1; echo "gemm full rc=$?"
ls -la gpurun_out/ | tail -8

#!/bin/bash
# ncu launch list of one C2 epoch at HEAD (time + DRAM bytes per launch),
# the traffic JSON the bench reads, and its summary (small outputs only).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${1:-c2}
timeout 600 python scripts/epoch_driver.py --config $CFG > gpurun_out/ncu_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv python scripts/epoch_driver.py --config $CFG > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
python scripts/spmm_traffic.py gpurun_out/launches_$CFG.csv gpurun_out/ncu_spmm_$CFG.json
python scripts/ncu_summary.py gpurun_out/launches_$CFG.csv > gpurun_out/epoch_$CFG.md; head -22 gpurun_out/epoch_$CFG.md

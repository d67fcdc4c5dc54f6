#!/bin/bash
# A/B of two source trees on one box (gpurun --gpus 2): HEAD (.) vs an older
# worktree (_ab_old), alternating, N=1 and N=2 (2x1x1), C2; HEAD also with
# the SpMM-fused reductions (PK_FUSED_REDUCE=1) vs off (0) at N=2.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
ROOTDIR=$(pwd)
show() {
  python - "$1" "$2" <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith("{")][-1]
d = json.loads(l)
print(sys.argv[2], round(d["value"], 2), {k: round(v, 2) for k, v in d["phases_ms"].items()},
      round(d["roofline"]["spmm_ms_per_epoch"], 2), d["clocks"]["sm_mhz"])
PY
}
for rep in 1 2; do
  for cfg in "_ab_old 0 old" ". 0 head_f0" ". 1 head_f1"; do
    set -- $cfg
    (cd $1 && PK_FUSED_REDUCE=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --grid 2,1,1 \
      --steps 20 --warmup 5 --no-cpu-baseline --no-c1-measured --no-e2e > $ROOTDIR/gpurun_out/abt_$3_n2_$rep.log 2>&1)
    show gpurun_out/abt_$3_n2_$rep.log "$3 n2 rep$rep"
    if [ "$3" != "head_f1" ]; then
      (cd $1 && timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c1-measured \
        --no-e2e > $ROOTDIR/gpurun_out/abt_$3_n1_$rep.log 2>&1)
      show gpurun_out/abt_$3_n1_$rep.log "$3 n1 rep$rep"
    fi
  done
done

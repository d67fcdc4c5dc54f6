#!/bin/bash
# A/B of two source trees on one box (gpurun --gpus 2): HEAD (.) vs an older
# worktree (_ab_old), alternating, N=1 and N=2 (2x1x1), C2.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
ROOTDIR=$(pwd)
for rep in 1 2; do
  for t in _ab_old .; do
    tag=$( [ "$t" = "." ] && echo head || echo old )
    (cd $t && PK_FUSED_REDUCE=${FUSED:-0} timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --grid 2,1,1 \
      --steps 20 --warmup 5 --no-cpu-baseline --no-c1-measured --no-e2e > $ROOTDIR/gpurun_out/abt_${tag}_n2_$rep.log 2>&1)
    (cd $t && timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c1-measured --no-e2e \
      > $ROOTDIR/gpurun_out/abt_${tag}_n1_$rep.log 2>&1)
    for n in n1 n2; do
      python - <<PY
import json
l=[x for x in open("gpurun_out/abt_${tag}_${n}_$rep.log") if x.startswith("{")][-1]
d=json.loads(l)
print("${tag} ${n} rep$rep", round(d["value"],2), {k: round(v,2) for k,v in d["phases_ms"].items()}, round(d["roofline"]["spmm_ms_per_epoch"],2), d["clocks"]["sm_mhz"])
PY
    done
  done
done

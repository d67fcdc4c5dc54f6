#!/bin/bash
# A/B of compile-time variants on one box: VARIANTS is a "|"-separated list
# of NVFLAGS_EXTRA strings ("-" = defaults); OBJS the objects to rebuild.
# Each variant runs CMD if set, else the 1-GPU bench without the e2e / CPU legs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
IFS='|' read -ra LIST <<< "${VARIANTS:--}"
i=0
for v in "${LIST[@]}"; do
  flags="$v"; [ "$flags" = "-" ] && flags=""
  for o in ${OBJS:-spmm}; do rm -f paper_2505_04083_b200/csrc/_obj/$o.o; done
  make -s -j16 -C paper_2505_04083_b200/csrc NVFLAGS_EXTRA="$flags" > gpurun_out/ab_build_$i.log 2>&1 || { echo "build failed: $v"; tail gpurun_out/ab_build_$i.log; continue; }
  if [ -n "${CMD:-}" ]; then
    echo "[$v]"; bash -c "$CMD"
  else
    timeout 600 python bench.py --steps ${STEPS:-8} --warmup 3 --no-e2e --no-cpu-baseline ${EXTRA:-} > gpurun_out/ab_$i.log 2>&1
    echo "[$v] $(grep -o '"value": [0-9.]*' gpurun_out/ab_$i.log | head -1) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/ab_$i.log) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/ab_$i.log)"
  fi
  i=$((i+1))
done

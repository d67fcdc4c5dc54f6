#!/bin/bash
# 256-bit epilogue stores (PK_EPI_V8) A/B: GEMM tests, per-shape times, epoch
# time, PK_TC_PROF wait breakdown for both builds; per-rank solo compute.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gemm_tc_gpu.py tests/test_kernels_gpu.py -k "gemm" > gpurun_out/epi_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/epi_pytest.log
timeout 900 python scripts/solo_ranks.py --config c2 --grid 2,1,2 > gpurun_out/solo_c2_212.log 2>&1; echo "solo rc=$?"; grep SOLO gpurun_out/solo_c2_212.log
timeout 600 python scripts/solo_ranks.py --config c2 --grid 2,1,1 > gpurun_out/solo_c2_211.log 2>&1; echo "solo2 rc=$?"; grep SOLO gpurun_out/solo_c2_211.log
for v in 1 0 1; do
  rm -f paper_2505_04083_b200/csrc/_obj/gemm_tc.o
  make -s -j16 -C paper_2505_04083_b200/csrc NVFLAGS_EXTRA="-DPK_EPI_V8=$v" > /dev/null 2>&1 || echo "build failed"
  echo "== PK_EPI_V8=$v"
  timeout 600 python scripts/gemm_bench.py fast 2>&1 | tail -10
  timeout 600 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/epi_bench_$v.log 2>&1
  echo "bench $(grep -o '"value": [0-9.]*' gpurun_out/epi_bench_$v.log | head -1) $(grep -o '"forward_gemm_s": [0-9.]*' gpurun_out/epi_bench_$v.log) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/epi_bench_$v.log)"
done
for v in 1 0; do echo "== tc_prof PK_EPI_V8=$v"; EXTRA_FLAGS="-DPK_EPI_V8=$v" bash scripts/tc_prof.sh 2>&1 | tail -9; done

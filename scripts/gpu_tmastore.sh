#!/bin/bash
# TMA-store GEMM epilogue (PK_TC_TMA_STORE): GEMM tests, bitwise on/off on
# the epoch's shapes, per-shape times, epoch A/B on C2, wait breakdown.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gemm_tc_gpu.py tests/test_kernels_gpu.py -k "gemm" > gpurun_out/ts_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ts_pytest.log
cat > /tmp/ts_hash.py <<'PY'
import hashlib, sys, torch
sys.path.insert(0, ".")
from paper_2505_04083_b200 import kernels as k
g = torch.Generator(device="cuda").manual_seed(7)
N = 1_000_003
out = []
for form, m, n, kk, relu in [("NN", N, 256, 100, False), ("NN", N, 256, 100, True), ("NT", N, 100, 256, False),
                             ("NN", N, 47, 256, False), ("NT", N, 256, 47, False), ("NN", 1000, 300, 64, True),
                             ("NT", 777, 40, 512, False), ("NN", 5000, 256, 600, False)]:
    ta, tb = form[0] == "T", form[1] == "T"
    a = torch.randn((kk, m) if ta else (m, kk), device="cuda", generator=g)
    b = torch.randn((n, kk) if tb else (kk, n), device="cuda", generator=g)
    c = k.gemm(a, b, ta, tb, mode=k.PK_MODE_FAST, relu=relu)
    out.append(hashlib.sha1(c.cpu().numpy().tobytes()).hexdigest()[:10])
print("HASH", " ".join(out))
PY
for v in 0 1; do PK_TC_TMA_STORE=$v timeout 300 python /tmp/ts_hash.py 2>&1 | tail -1; done
for v in 0 1; do echo "PK_TC_TMA_STORE=$v"; PK_TC_TMA_STORE=$v timeout 600 python scripts/gemm_bench.py fast 2>&1 | tail -10; done
ENVS="${ENVS:-PK_TC_TMA_STORE=0|PK_TC_TMA_STORE=1|PK_TC_TMA_STORE=1 PK_GEMM_RELU_BWD=0|PK_TC_TMA_STORE=0|PK_TC_TMA_STORE=1|PK_TC_TMA_STORE=1 PK_GEMM_RELU_BWD=0}" bash scripts/ab_env.sh
bash scripts/tc_prof.sh 2>&1 | tail -9

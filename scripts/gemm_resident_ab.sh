#!/bin/bash
# Weight-resident tcgen05 ring (PK_TC_RESIDENT): GEMM tests, bitwise on/off
# check of the affected shapes, per-shape timings and an epoch A/B on C2.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gemm_tc_gpu.py tests/test_kernels_gpu.py -k "gemm" > gpurun_out/res_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/res_pytest.log
cat > /tmp/res_hash.py <<'PY'
import hashlib, sys, torch
sys.path.insert(0, ".")
from paper_2505_04083_b200 import kernels as k
g = torch.Generator(device="cuda").manual_seed(7)
N = 1_000_003
out = []
for form, m, n, kk in [("NN", N, 47, 256), ("NT", N, 256, 47), ("NN", N, 64, 200), ("NT", N, 128, 60)]:
    ta, tb = form[0] == "T", form[1] == "T"
    a = torch.randn((kk, m) if ta else (m, kk), device="cuda", generator=g)
    b = torch.randn((n, kk) if tb else (kk, n), device="cuda", generator=g)
    c = k.gemm(a, b, ta, tb, mode=k.PK_MODE_FAST)
    out.append(hashlib.sha1(c.cpu().numpy().tobytes()).hexdigest()[:12])
print("HASH", " ".join(out))
PY
for v in 0 1; do PK_TC_RESIDENT=$v timeout 300 python /tmp/res_hash.py 2>&1 | grep HASH; done
for v in 0 1; do echo "PK_TC_RESIDENT=$v"; PK_TC_RESIDENT=$v timeout 600 python scripts/gemm_bench.py fast 2>&1 | tail -10; done
ENVS="${ENVS:-PK_TC_RESIDENT=0|PK_TC_RESIDENT=1|PK_TC_RESIDENT=0|PK_TC_RESIDENT=1}" bash scripts/ab_env.sh

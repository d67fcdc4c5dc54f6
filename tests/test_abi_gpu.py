"""The C++ drop-in boundary driven by a C++ caller: tests/abi/test_abi
(tests/abi/test_abi.cpp) includes the reference's own headers and
include/plexuskit_b200.hpp, and checks plexuskit::b200::{spmm, spmm_rows,
gemm, relu_*, softmax_cross_entropy_sums, adam_step, transpose,
train_distributed}, the per-layer entry points and the RankCtx collectives
of the C ABI against the reference's implementations in the same process.
The binary is compiled where the reference headers exist (build(), this
container) and travels to the GPU box like oracle/_ref."""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "abi", "_build", "test_abi")


def test_cpp_abi_caller(cuda):
    if not os.path.exists(BIN):
        import oracle
        if not os.path.isdir(oracle.REFERENCE_SRC):
            pytest.fail("tests/abi/_build/test_abi missing (build() compiles it where the "
                        "reference headers are)")
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "abi")], check=True)
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "0 failed" in p.stdout

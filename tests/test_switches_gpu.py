"""The measured-and-rejected switches stay correct: each runs one
FAST engine pass in its own process (the PK_* variables are read once per
process) on a graph with a transform-first last layer and is compared with
the default configuration — bit-identical where the switch only moves data
(TMA-store epilogue off, weight-resident ring, ReLU' in the GEMM epilogue,
narrower D <= 256 gathers), within FAST tolerance where it re-associates a
sum (the paired SpMM form)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(tmp_path, name, env):
    out = tmp_path / f"{name}.npz"
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, os.path.join(HERE, "_switch_pass.py"), str(out)], env=e,
                   check=True, timeout=600)
    return dict(np.load(out))


def _nrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


@pytest.fixture(scope="module")
def default(cuda, tmp_path_factory):
    return _run(tmp_path_factory.mktemp("sw"), "default", {})


@pytest.mark.parametrize("env", [{"PK_TC_TMA_STORE": "0"}, {"PK_TC_RESIDENT": "1"},
                                 {"PK_GEMM_RELU_BWD": "0"}, {"PK_SPMM_MID_VEC": "2"}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_data_movement_switch_bit_identical(default, tmp_path, env):
    got = _run(tmp_path, "sw", env)
    for k in default:
        assert np.array_equal(np.asarray(got[k]).view(np.uint32) if got[k].dtype == np.float32
                              else got[k], np.asarray(default[k]).view(np.uint32)
                              if default[k].dtype == np.float32 else default[k]), k


def test_paired_spmm_switch_within_fast_tolerance(default, tmp_path):
    got = _run(tmp_path, "pair", {"PK_TF_PAIR": "1"})
    assert _nrel(got["logits"], default["logits"]) <= 1e-5
    for l in range(3):
        assert _nrel(got[f"dw{l}"], default[f"dw{l}"]) <= 1e-4
    assert _nrel(got["df0"], default["df0"]) <= 1e-3
    assert abs(float(got["loss"]) - float(default["loss"])) <= 1e-5 * abs(float(default["loss"]))

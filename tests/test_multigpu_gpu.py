"""Multi-GPU engine parity (one process per GPU, NCCL axis communicators)
against the reference's distributed pass and train_distributed at the same
grid. Needs >= 2 GPUs on one box (`gpurun --gpus 2|4`); skipped otherwise."""

import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
WORKER = os.path.join(HERE, "mp", "engine_pass_worker.py")


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(nproc, *args, env=None):
    for attempt in range(3):  # a probed free port can be taken before torchrun binds it
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
               f"--master-port={_port()}", WORKER, *args]
        p = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                           env={**os.environ, **(env or {})})
        if "EADDRINUSE" not in p.stderr + p.stdout:
            break
    lines = [l for l in p.stdout.splitlines() if l.startswith("MPRESULT ")]
    assert lines, p.stdout[-3000:] + p.stderr[-3000:]
    rep = json.loads(lines[-1][len("MPRESULT "):])
    assert p.returncode == 0 and rep["ok"], rep
    return rep


def _grids(g):
    out = []
    for gx in range(1, g + 1):
        if g % gx:
            continue
        for gy in range(1, g // gx + 1):
            if (g // gx) % gy == 0:
                out.append(f"{gx},{gy},{g // gx // gy}")
    return out


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("grid", _grids(2))
def test_two_gpu_grids_match_reference(cuda, grid):
    rep = _run(2, "--grid", grid)
    assert rep["logits_bitwise"]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_gpu_fast_mode_and_blocks(cuda):
    _run(2, "--grid", "2,1,1", "--mode", "fast", "--block-count", "3")


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("fused", ["3", "0"])
@pytest.mark.parametrize("grid", _grids(2) + (_grids(4) if torch.cuda.device_count() >= 4 else []))
def test_fast_mode_every_grid(cuda, grid, fused):
    """FAST mode (tcgen05 GEMMs, segmented plans, transform-first layers
    where the inner axis is one rank) on every grid of 2 and 4 ranks, with
    the producer-fused reductions (the SpMM / GEMM epilogues store each row
    into its owner's peer-memory slot; csrc/lsa.cu reduce_slots) and
    without: within 1e-4 of the reference's distributed pass and curve."""
    n = 2 if grid in _grids(2) else 4
    _run(n, "--grid", grid, "--mode", "fast", env={"PK_FUSED_REDUCE": fused})


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("grid", _grids(2))
def test_two_gpu_nccl_reductions(cuda, grid):
    """The NCCL path the engine falls back to without peer-memory access
    (separate ReLU passes, materialised Q)."""
    _run(2, "--grid", grid, env={"PK_LSA": "0"})


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("grid", _grids(2))
@pytest.mark.parametrize("lsa", ["1", "0"])
def test_two_gpu_row_chunked_reductions(cuda, grid, lsa):
    """Row-chunked producer/reduction pipelines (PK_COMM_CHUNKS=3, odd
    chunk edges): the same bit-identical logits as the unchunked default."""
    rep = _run(2, "--grid", grid, env={"PK_LSA": lsa, "PK_COMM_CHUNKS": "3"})
    if lsa == "1":
        assert rep["logits_bitwise"]


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("grid", _grids(4))
def test_four_gpu_grids_match_reference(cuda, grid):
    """Four-member axes included: the ordered peer-memory reductions keep the
    logits bit-identical to the reference's coordinate-order combine."""
    rep = _run(4, "--grid", grid)
    assert rep["logits_bitwise"]


@pytest.mark.skipif(torch.cuda.device_count() < 8, reason="needs 8 GPUs")
@pytest.mark.parametrize("grid", ["2,2,2", "8,1,1", "1,1,8", "4,1,2"])
def test_eight_gpu_grids_match_reference(cuda, grid):
    _run(8, "--grid", grid)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("grid", _grids(2))
def test_two_gpu_relu_backward_in_spmm_epilogue(cuda, grid):
    """PK_FUSE_RELU_BWD=2: layer l-1's ReLU' applied by the SpMM^T epilogue
    where row_shard is one rank (opt-in variant), same results."""
    rep = _run(2, "--grid", grid, env={"PK_FUSE_RELU_BWD": "2"})
    assert rep["logits_bitwise"]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("grid", _grids(2))
def test_two_gpu_engines_from_shard_files(cuda, grid, tmp_path):
    """The file_handle path (trainer.hpp:461-466): rank 0 writes a 2x3 PLXS
    shard set, every rank loads only its blocks from it; same results as the
    reference's distributed pass and train_distributed."""
    rep = _run(2, "--grid", grid, "--files", str(tmp_path / "shards"), "--shard-grid", "2,3")
    assert rep["logits_bitwise"]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("fault", [False, True])
def test_two_gpu_cli_validate(cuda, fault):
    """cli validate (main.cpp:469-512): every 2-rank grid against the 1x1x1
    curve; an injected fault (a skipped reduction) must fail it (exit 1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", "-m", "paper_2505_04083_b200",
           "validate", "--synth", "rmat:scale=10,edges=8000", "--feat-dim", "12", "--classes",
           "5", "--epochs", "3", "--layers", "16"] + (["--inject-fault"] if fault else [])
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert p.returncode == (1 if fault else 0), p.stdout[-2000:] + p.stderr[-2000:]
    assert ("validation FAILED" if fault else "validation passed") in p.stdout


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("grid", ["2,1,1", "1,1,2"])
def test_two_gpu_rank_failure_aborts_peers(cuda, grid):
    """One process per GPU: rank 1's host code fails after epoch 1; rank 0,
    blocked in its next epoch's NCCL / peer-memory collectives, must end with
    ClusterAborted naming rank 1 (node-local abort block, csrc/comm.cu)
    instead of hanging."""
    worker = os.path.join(HERE, "mp", "abort_worker.py")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", worker, "--grid", grid]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    res = [l for l in p.stdout.splitlines() if l.startswith("ABORTRESULT")]
    assert len(res) == 2, p.stdout[-3000:] + p.stderr[-3000:]
    assert all("ok=1" in l for l in res), res

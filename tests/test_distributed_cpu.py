"""The N>1 host path on CPU: two processes over gloo run
distributed.train_distributed with a stand-in engine (the device engine needs
a GPU). Covers the NCCL-id broadcast, the per-rank metric reduction
(trainer.hpp:660-686: loss from rank 0, times max over ranks, counters
summed) and the W / F0 reassembly from weight_slice / feature_slice
(trainer.hpp:642-659), on every grid of 2 ranks — checked against the
reference's own init weights and features."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2505_04083_b200 import distributed as D
from paper_2505_04083_b200.layout import GridConfig, feature_slice, plan_layouts, weight_slice
from paper_2505_04083_b200.philox import init_weights

N, DIMS = 37, [6, 5, 7, 3]


class _Pre:
    n, feat_dim, num_classes = N, DIMS[0], DIMS[-1]


class _Opts:
    epochs = 3


class FakeEngine:
    """Holds exactly the shards a real rank holds at init: W blocks of the
    global Glorot init (model.hpp:17-51) and its F0 block (model.hpp:53-67)."""

    def __init__(self, grid, rank, uid):
        self.grid, self.rank, self.uid = grid, rank, uid
        self.dims = DIMS
        c = grid.coords_of(rank)
        lays = plan_layouts(len(DIMS) - 1)
        w = init_weights(DIMS, 0)
        self.w = []
        for l in range(len(DIMS) - 1):
            r0, r1, c0, c1 = weight_slice(grid, lays[l], c, DIMS[l], DIMS[l + 1])
            self.w.append(w[l][r0:r1, c0:c1].copy())
        feats = np.arange(N * DIMS[0], dtype=np.float32).reshape(N, DIMS[0])
        r0, r1, c0, c1 = feature_slice(grid, c, N, DIMS[0])
        self.f0 = feats[r0:r1, c0:c1].copy()

    def train_epoch(self, e):
        return {"epoch": e, "loss": 2.0 - 0.1 * e + (0.5 if self.rank else 0.0),
                "accuracy": 0.25, "forward_spmm_s": 0.1 * (self.rank + 1) + e,
                "backward_s": 1.0 - 0.1 * self.rank, "spmm_flops": 1000 * (self.rank + 1),
                "allreduce_bytes": 7.0, "kernel_launches": 40}

    def tensor(self, which, layer=0):
        return self.w[layer] if which == 0 else self.f0

    def close(self):
        pass


def _worker(rank, world, port, grid_t, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    grid = GridConfig(*grid_t)
    seen = {}

    def factory(pre, g, r, opts):
        uid = D.broadcast_unique_id(lambda: bytes(range(128)))
        seen["uid"] = uid
        return FakeEngine(g, r, uid)

    res = D.train_distributed(lambda: _Pre(), grid, _Opts(), engine_factory=factory)
    import torch.distributed as dist
    dist.destroy_process_group()
    q.put((rank, seen["uid"], res.global_metrics, [w.tolist() for w in res.weights],
           res.features.tolist()))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("grid_t", [(2, 1, 1), (1, 2, 1), (1, 1, 2)])
def test_train_distributed_host_path_world2(grid_t):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, grid_t, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=120) for _ in procs])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, uid0, g0, w0, f0), (_, uid1, g1, w1, f1) = out
    assert uid0 == uid1 == bytes(range(128))
    assert g0 == g1
    for e, g in enumerate(g0):
        assert g["loss"] == pytest.approx(2.0 - 0.1 * e)          # rank 0's
        assert g["forward_spmm_s"] == pytest.approx(0.2 + e)      # max over ranks
        assert g["backward_s"] == pytest.approx(1.0)
        assert g["spmm_flops"] == 3000 and g["kernel_launches"] == 80   # summed
    want_w = init_weights(DIMS, 0)
    for l in range(3):
        assert np.array_equal(np.asarray(w0[l], np.float32), want_w[l])
    feats = np.arange(N * DIMS[0], dtype=np.float32).reshape(N, DIMS[0])
    assert np.array_equal(np.asarray(f0, np.float32), feats)


def test_reduce_and_reassemble_single_process_all_grids_of_4():
    """Reassembly covers every element exactly once on every grid of 4."""
    from paper_2505_04083_b200.layout import enumerate_configs
    for g in enumerate_configs(4):
        grid = GridConfig(*g)
        engines = [FakeEngine(grid, r, None) for r in range(4)]
        w, f = D.reassemble(grid, N, DIMS, [e.w for e in engines], [e.f0 for e in engines])
        for l, want in enumerate(init_weights(DIMS, 0)):
            assert np.array_equal(w[l], want), (g, l)
        assert np.array_equal(f, np.arange(N * DIMS[0], dtype=np.float32).reshape(N, DIMS[0]))

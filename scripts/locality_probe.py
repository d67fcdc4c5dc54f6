"""How much does gather locality buy the SpMM? Times the same products-shaped
graph as (a) the double-permuted shard the engine sees (random column order
by design, graph.hpp:139-148) and (b) the un-permuted normalized adjacency
(RMAT's recursive id locality), with identical kernels and plans."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04083_b200 import graph, kernels

def timed(fn, iters=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    ts = []
    for _ in range(iters):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)

ds = graph.synth_rmat(21, 62_000_000, 16, 4, seed=1)
orig = graph.normalize_adjacency(ds.num_nodes, ds.edges, ds.undirected)
pre = graph.preprocess(ds, perm_seed=1)
for name, a in (("permuted", pre.a_even), ("original", orig)):
    for d in (100, 256):
        x = torch.rand(a.cols, d, device="cuda")
        y = torch.empty(a.rows, d, device="cuda")
        for mode in (kernels.PK_MODE_PARITY, kernels.PK_MODE_FAST):
            plan = kernels.SpmmPlan(a, 0, mode=mode)
            ms = timed(lambda: kernels.spmm(a, x, out=y, plan=plan))
            print(json.dumps(dict(matrix=name, d=d, mode="fast" if mode else "parity", ms=ms)), flush=True)
            del plan

"""Billion-edge full-graph training across GPUs (one process per GPU,
torchrun): every rank generates ONLY its own shards from synth_rmat's
indexable streams (rank_gen.py; the two global degree vectors are counted
per node range and all-gathered over NCCL), loads them into its engine
(taking the blocks over, no copy) and trains; prints one JSON line on rank 0
with the generation / load times, memory in use, per-epoch device time (max
over ranks), phases and collective bytes.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 scripts/c4_multi.py \
        --scale 25 --edges 1600000000 --grid 2,1,2
"""
import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2505_04083_b200 import distributed as D, rank_gen, trainer  # noqa: E402
from paper_2505_04083_b200.layout import GridConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=25)
    ap.add_argument("--edges", type=int, default=1_600_000_000)
    ap.add_argument("--grid", default="2,1,2")
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--epochs", type=int, default=5)
    ap.add_argument("--undirected", action="store_true")
    args = ap.parse_args()
    rank, world, local = D.dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    grid = GridConfig(*[int(x) for x in args.grid.split(",")])
    assert grid.size == world, (grid, world)
    spec = rank_gen.RmatSpec(args.scale, args.edges, 128, 172, seed=1,
                             undirected=args.undirected)

    def allgather(part, counts):
        mx = max(counts)
        buf = torch.zeros(mx, dtype=part.dtype, device="cuda")
        buf[:part.numel()] = part
        out = torch.empty(mx * world, dtype=part.dtype, device="cuda")
        dist.all_gather_into_tensor(out, buf)
        return torch.cat([out[i * mx:i * mx + counts[i]] for i in range(world)])

    def maxr(x):
        t = torch.tensor([float(x)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    dist.barrier()
    t0 = time.perf_counter()
    pieces = rank_gen.global_pieces(spec, rank, world, allgather)
    torch.cuda.synchronize()
    t_pieces = maxr(time.perf_counter() - t0)
    nnz_total = int(pieces.norm_degree.to(torch.int64).sum().item())  # row degrees incl. loops
    t0 = time.perf_counter()
    rt = rank_gen.generate_rank_tensors(spec, grid, rank, 3, pieces)
    torch.cuda.synchronize()
    t_shards = maxr(time.perf_counter() - t0)
    rank_nnz = sum(blk.nnz for (blk, _) in {id(v[0]): v for v in rt.adj.values()}.values())
    del pieces
    torch.cuda.empty_cache()
    opts = trainer.TrainOptions(hidden_dims=[128, 128], mode=trainer.PK_MODE_FAST)
    eng = trainer.RankEngine(spec.n, 128, 172, grid, rank, opts, local)
    obj = [trainer.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    eng.comm_init(obj[0], world)
    t0 = time.perf_counter()
    eng.load_rank(rt, adopt=True)
    torch.cuda.synchronize()
    t_load = maxr(time.perf_counter() - t0)
    del rt
    torch.cuda.empty_cache()
    for e in range(args.warmup):
        eng.train_epoch(e)
    dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(eng.stream_ptr())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    ms = eng.train_epochs(args.warmup, args.epochs)
    ev1.record(stream)
    torch.cuda.synchronize()
    epoch_ms = maxr(ev0.elapsed_time(ev1) / args.epochs)
    free, total = torch.cuda.mem_get_info()
    used = maxr((total - free) / 1e9)
    avg = lambda k: sum(m[k] for m in ms) / len(ms)  # noqa: E731
    phases = {k: maxr(avg(k) * 1e3) for k in ("forward_spmm_s", "forward_gemm_s", "backward_s",
                                              "optimizer_s", "collectives_s", "spmm_s")}
    ring = maxr(avg("allreduce_bytes") + avg("allgather_bytes") + avg("reducescatter_bytes"))
    losses = [m["loss"] for m in ms]
    if rank == 0:
        print("C4MULTI " + json.dumps({
            "workload": f"RMAT s{args.scale} ({spec.n:,} nodes), {args.edges:,} "
                        f"{'undirected' if args.undirected else 'directed'} edges, "
                        f"GCN 128-128-128-172, grid {args.grid} on {world} B200, FAST",
            "nnz_total": nnz_total, "rank0_block_nnz": int(rank_nnz),
            "global_pieces_s": t_pieces, "rank_shards_s": t_shards, "load_s": t_load,
            "device_mem_gb_max": used, "epoch_ms": epoch_ms, "phases_ms_max": phases,
            "ring_bytes_per_epoch_max": ring, "losses": losses,
            "note": "each rank generates only its own blocks; no process holds the global graph"}),
            flush=True)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""One rank's share of the papers-shaped C4 (BASELINE configs[3]: RMAT,
1.6B directed edges, 128-128-128-172, grid 2x2x2 on 8 B200s) measured on ONE
B200: the rank's shards are generated on the device from the indexable
generator (rank_gen.py: no global graph anywhere), loaded into the engine in
measurement mode (pk_engine_comm_init_solo: collectives keep only the rank's
own contribution, so the epoch is this rank's compute; the ring-model bytes
still follow the real grid) and trained for a few epochs.

Prints one JSON line: generation / load times, device memory in use, epoch
device time and phases, SpMM share, and the per-epoch collective bytes with
the transfer time they take at the measured NVLink bus bandwidth.

    python scripts/c4_rank.py [--scale 26] [--edges 1600000000] [--rank 0]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2505_04083_b200 import _capi, rank_gen, trainer  # noqa: E402
from paper_2505_04083_b200.layout import GridConfig  # noqa: E402


def used_gb():
    free, total = torch.cuda.mem_get_info()
    return (total - free) / 1e9, total / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--edges", type=int, default=1_600_000_000)
    ap.add_argument("--grid", default="2,2,2")
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--epochs", type=int, default=3)
    ap.add_argument("--undirected", action="store_true")
    ap.add_argument("--bus-gbs", type=float, default=564.0,
                    help="measured NVLink bus bandwidth of the ordered reductions "
                         "(profiles/r1_late_bench_n2.log: 564 GB/s)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    grid = GridConfig(*[int(x) for x in args.grid.split(",")])
    spec = rank_gen.RmatSpec(args.scale, args.edges, 128, 172, seed=1,
                             undirected=args.undirected)
    out = {"workload": f"RMAT s{args.scale}, {args.edges:,} "
                       f"{'undirected' if args.undirected else 'directed'} edges, "
                       f"GCN 128-128-128-172, grid {args.grid}, rank {args.rank} of {grid.size} "
                       "measured alone (pk_engine_comm_init_solo)"}
    def note(what):
        print(f"[c4] {what}: {used_gb()[0]:.1f} GB in use", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    pieces = rank_gen.global_pieces(spec, args.rank, grid.size)  # every degree range here
    torch.cuda.synchronize()
    out["global_pieces_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    rt = rank_gen.generate_rank_tensors(spec, grid, args.rank, 3, pieces)
    torch.cuda.synchronize()
    out["rank_shards_s"] = time.perf_counter() - t0
    out["rank_nnz"] = {f"{k[0]},{k[1]}": v[0].nnz for k, v in rt.adj.items()}
    del pieces
    torch.cuda.empty_cache()
    out["gen_mem_gb"] = used_gb()[0]
    note("shards generated")
    opts = trainer.TrainOptions(hidden_dims=[128, 128], mode=trainer.PK_MODE_FAST)
    eng = trainer.RankEngine(spec.n, 128, 172, grid, args.rank, opts, 0)
    eng.comm_init_solo()
    t0 = time.perf_counter()
    eng.load_rank(rt, adopt=True)
    torch.cuda.synchronize()
    out["load_s"] = time.perf_counter() - t0
    del rt
    torch.cuda.empty_cache()
    _capi.lib().pk_device_cache_release()
    note("engine loaded")
    for e in range(args.warmup):
        eng.train_epoch(e)
    ms = [eng.train_epoch(args.warmup + e) for e in range(args.epochs)]
    used, total = used_gb()
    out["device_mem_gb"] = {"in_use": used, "total": total}
    avg = lambda k: sum(m[k] for m in ms) / len(ms)  # noqa: E731
    out["epoch_ms"] = avg("epoch_s") * 1e3
    out["phases_ms"] = {k: avg(k) * 1e3 for k in ("forward_spmm_s", "forward_gemm_s",
                                                    "backward_s", "optimizer_s", "spmm_s")}
    ring = avg("allreduce_bytes") + avg("allgather_bytes") + avg("reducescatter_bytes")
    out["ring_bytes_per_epoch"] = ring
    out["comm_ms_at_bus_gbs"] = ring / (args.bus_gbs * 1e9) * 1e3
    out["bus_gbs"] = args.bus_gbs
    out["spmm_bytes_per_epoch"] = avg("spmm_bytes")
    out["spmm_compulsory_bytes_per_epoch"] = avg("spmm_compulsory_bytes")
    out["kernel_launches_per_epoch"] = avg("kernel_launches")
    eng.close()
    print("C4RANK " + json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

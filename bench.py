"""Benchmark: full-graph 3-layer GCN training epoch on the products-shaped
synthetic graph (BASELINE.json configs[1]) — epoch time in ms — with the
SpMM roofline, an end-to-end number through the host-buffer API and the
reference CPU implementation timed beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N      (one rank per GPU)

One step = one training epoch (forward, loss, backward, Adam) over the whole
graph, dataset resident in HBM. The grid for N GPUs is the performance
model's pick (1x1x1, 2x1x1, 2x1x2, 2x2x2).
"""

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("GCN epoch time (ms) at 1/2/4/8 B200; SpMM HBM GB/s vs roofline; "
          "CPU-ref speedup")

CONFIGS = {
    # BASELINE.json configs[1]: ogbn-products-shaped (2.4M nodes / 62M edges
    # -> RMAT needs n = 2^scale: scale 21 = 2,097,152 nodes, 62M edges,
    # 116,573,894 normalized nonzeros), 100 feats, 47 classes, hidden 256.
    "c2": dict(scale=21, edges=62_000_000, feat=100, classes=47, hidden=[256, 256],
               abc=(0.57, 0.19, 0.19),
               workload="ogbn-products-shaped RMAT s21 (2,097,152 nodes, 62M edges), "
                        "3-layer GCN 100-256-256-47"),
    # configs[0]: the reference's CPU-runnable case
    "c1": dict(scale=17, edges=2_000_000, feat=128, classes=16, hidden=[128, 128],
               abc=(0.57, 0.19, 0.19),
               workload="RMAT s17 (131,072 nodes, 2M edges), 3-layer GCN 128-128-128-16"),
    # configs[2]: Reddit-shaped dense-degree (flat RMAT, ~114.9M nnz)
    "c3": dict(scale=18, edges=57_307_946, feat=602, classes=41, hidden=[128, 128],
               abc=(0.25, 0.25, 0.25),
               workload="Reddit-shaped flat RMAT s18 (262,144 nodes, 57.3M edges), "
                        "3-layer GCN 602-128-128-41"),
}
# One 8-GPU NVSwitch box: every axis is intra-node at the measured NCCL bus
# bandwidth (B200_PROFILING: 725 GB/s all-reduce busBW at 1 GiB).
B200_MACHINE = dict(g_node=8, beta_intra=725e9, beta_inter=50e9, bytes_per_scalar=4)


def pick_grid(gpus, n, nnz, dims):
    """The performance model's choice (rank_configs, perf_model.cpp:207-229)
    for this dataset on this machine."""
    from paper_2505_04083_b200 import perf_model as pm
    best = pm.rank_configs(gpus, pm.DatasetStats(n, nnz, list(dims)),
                           pm.MachineParams(**B200_MACHINE), pm.default_coefficients())[0]
    return tuple(best.shape)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--grid", default=None, help="gx,gy,gz (default: perf-model pick)")
    ap.add_argument("--mode", default="fast", choices=["fast", "parity"])
    ap.add_argument("--e2e-epochs", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU seconds for the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []  # (host receive time, fields)
        self.proc = None
        self.window = None  # (t0, t1) host times of the timed region

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.monotonic(), [x.strip() for x in line.split(",")]))

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        """Samples inside the timed region; a region shorter than the
        sampler's first readings falls back to warm-up + timed (the GPU is
        under the same load), and says so in `window`."""
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = self.rows
        window = "timed"
        if self.window:
            inside = [r for r in rows if self.window[0] <= r[0] <= self.window[1] + 0.1]
            if len(inside) >= 2:
                rows = inside
            else:
                window = "warmup+timed"
        for _, r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for i, nm in enumerate(names):
                    if r[5 + i].lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "window": window}


def build_dataset(cfg, device):
    import torch
    from paper_2505_04083_b200 import graph
    a, b, c = cfg["abc"]
    ds = graph.synth_rmat(cfg["scale"], cfg["edges"], cfg["feat"], cfg["classes"], seed=1,
                          a=a, b=b, c=c)
    pre = graph.preprocess(ds, perm_seed=1)
    del ds
    torch.cuda.synchronize()
    return pre


def cpu_reference_sample(pre_dev, hidden, target_s, threads):
    """The reference's own CPU kernels (oracle/_ref, -O2 scalar) on a bounded
    row sample of this workload, scaled to a full epoch. Returns the
    estimated epoch ms and a description."""
    from oracle import ref
    from paper_2505_04083_b200.trainer import HostDataset
    h = HostDataset.from_device(pre_dev, pin=False)
    rpre = ref.Pre.from_arrays(h.n, h.feat_dim, h.num_classes,
                               (h.even[0].view(np.uint64), h.even[1].view(np.uint32), h.even[2]),
                               (h.odd[0].view(np.uint64), h.odd[1].view(np.uint32), h.odd[2]),
                               h.features, h.labels_row.view(np.uint32),
                               h.labels_col.view(np.uint32), h.mask_row, h.mask_col)
    # calibrate on a small sample, then size the measured one to target_s
    rows = 64
    est, wall = rpre.epoch_sample(hidden, rows, threads)
    per_row = wall / rows
    rows = int(max(64, min(h.n // max(1, threads), target_s / max(per_row, 1e-9))))
    est, wall = rpre.epoch_sample(hidden, rows, threads)
    return est * 1e3, rows, wall


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    import torch
    torch.cuda.set_device(local)
    cfg = CONFIGS[args.config]
    pre = build_dataset(cfg, local)
    dims = [cfg["feat"], *cfg["hidden"], cfg["classes"]]
    grid = (tuple(int(x) for x in args.grid.split(",")) if args.grid
            else pick_grid(args.gpus, pre.n, pre.a_even.nnz, dims))
    threads = os.cpu_count() or 1
    vals = []
    for step in range(args.warmup + args.steps):
        ms, rows, wall = cpu_reference_sample(pre, cfg["hidden"], 20.0 if step >= args.warmup
                                              else 3.0, threads)
        if step >= args.warmup:
            vals.append(ms)
    val = float(np.median(vals))
    sample = (f"{rows} rows x {threads} threads of every per-layer op of one 1x1x1 epoch "
              f"(reference spmm_rows/gemm/relu/CE/Adam, oracle/_ref -O2), scaled to "
              f"{pre.n} rows; input built by the GPU shard builder (bit-exact with "
              f"reference preprocess)")
    line = {"metric": METRIC, "value": val, "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": val, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": cfg["workload"], "grid": "x".join(map(str, grid)),
                       "reference_grid_note": "CPU reference timed as its 1x1x1 op set"},
            "cpu_baseline": {"value": val, "unit": "ms", "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": val, "unit": "ms", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2505_04083_b200 import _capi, layout, trainer

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]

    def new_uid():
        if world == 1:
            return None
        obj = [trainer.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    mode = trainer.PK_MODE_FAST if args.mode == "fast" else trainer.PK_MODE_PARITY
    opts = trainer.TrainOptions(hidden_dims=cfg["hidden"], mode=mode, epochs=args.steps)
    t_build = time.time()
    pre = build_dataset(cfg, local)
    t_build = time.time() - t_build
    n, nnz = pre.n, pre.a_even.nnz
    dims = [cfg["feat"], *cfg["hidden"], cfg["classes"]]
    grid = (tuple(int(x) for x in args.grid.split(",")) if args.grid
            else pick_grid(world, n, nnz, dims))
    gridc = layout.GridConfig(*grid)
    assert gridc.size == world, (grid, world)

    eng = trainer.RankEngine(pre.n, pre.feat_dim, pre.num_classes, gridc, rank, opts, local)
    if world > 1:
        eng.comm_init(new_uid(), world)
    eng.load(pre)
    stream = torch.cuda.ExternalStream(eng.stream_ptr())

    clocks = ClockSampler(local).__enter__()  # started early: nvidia-smi needs a moment
    for e in range(args.warmup):
        eng.train_epoch(e)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _capi.lib().pk_kernel_launch_count()
    t_timed0 = time.monotonic()
    ev0.record(stream)
    metrics = [eng.train_epoch(args.warmup + e) for e in range(args.steps)]
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks.mark(t_timed0, time.monotonic())
    clocks.__exit__(None, None, None)
    launches = _capi.lib().pk_kernel_launch_count() - launches0
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        dist.barrier()
    ms_step = ms_total / args.steps
    spmm_s = float(np.mean([m["spmm_s"] for m in metrics]))
    spmm_bytes = float(np.mean([m["spmm_bytes"] for m in metrics]))
    spmm_launch_share = spmm_s / (ms_step * 1e-3)
    peak, peak_kind = hbm_peak()
    achieved = spmm_bytes / spmm_s / 1e9 if spmm_s > 0 else None
    # DRAM bytes of the same SpMM launches of one epoch, from the committed
    # ncu launch list (scripts/ncu_round.sh -> scripts/spmm_traffic.py)
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"ncu_spmm_{args.config}.json")
    if os.path.exists(prof) and world == 1:
        try:
            with open(prof) as f:
                traffic = json.load(f).get("dram_bytes_per_epoch")
        except Exception:
            traffic = None
    phases = {k: float(np.mean([m[k] for m in metrics])) * 1e3 for k in
              ("forward_spmm_s", "forward_gemm_s", "backward_s", "optimizer_s", "collectives_s")}
    losses = [m["loss"] for m in metrics]
    # collective bus bandwidth: the reference's ring-model bytes (= NCCL bus
    # bytes, cluster.hpp:300-333) over the device time of this rank's
    # reductions / gathers (max over ranks of the time)
    coll = None
    if world > 1:
        ring = float(np.mean([m["allreduce_bytes"] + m["allgather_bytes"] +
                              m["reducescatter_bytes"] for m in metrics]))
        ctime = float(np.mean([m["collectives_s"] for m in metrics]))
        t = torch.tensor([ctime], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ctime = float(t.item())
        coll = {"ms_per_epoch": ctime * 1e3, "ring_bytes_per_epoch": ring,
                "bus_gbs": ring / ctime / 1e9 if ctime > 0 else None,
                "nvlink_gbs_per_direction": 900.0,
                "note": "ordered peer-memory reductions (csrc/lsa.cu) + NCCL all-gathers"}
    # closed before the e2e run; its device blocks stay in the library's
    # allocation cache (memory.cu) for the next engine, like a process that
    # re-builds its engine
    eng.close()
    del eng
    torch.cuda.empty_cache()

    # e2e: the reference-facing API with HOST buffers (train_distributed on a
    # host PreprocessedDataset): H2D of the whole dataset from pinned memory,
    # shard slicing, E epochs (each reads its loss/accuracy back to the host).
    e2e = None
    if not args.no_e2e:
        host = trainer.HostDataset.from_device(pre, pin=True)
        uid = new_uid()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng2 = trainer.RankEngine(host.n, host.feat_dim, host.num_classes, gridc, rank, opts,
                                  local)
        if world > 1:
            eng2.comm_init(uid, world)
        t1 = time.perf_counter()
        eng2.load(host)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        for e in range(args.e2e_epochs):
            eng2.train_epoch(e)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        parts = [t3 - t0, t1 - t0, t2 - t1, t3 - t2]
        if world > 1:
            t = torch.tensor(parts, device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            parts = t.tolist()
        wall = parts[0]
        eng2.close()
        e2e = {"value": wall * 1e3 / args.e2e_epochs, "unit": "ms",
               "h2d_bytes_per_step": int(host.nbytes() // args.e2e_epochs),
               "d2h_bytes_per_step": 4 * 8,
               "epochs": args.e2e_epochs,
               "phases_ms": {"create_and_comm_init": parts[1] * 1e3, "load": parts[2] * 1e3,
                             "epochs": parts[3] * 1e3},
               "note": "train_distributed from a pinned-host PreprocessedDataset: dataset H2D "
                       "+ shard slicing + E epochs, wall / E (max over ranks)"}
        del host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            ms, rows, wall = cpu_reference_sample(pre, cfg["hidden"], args.cpu_seconds, 1)
            cpu = {"value": ms, "unit": "ms", "cores": 1, "kind": "reference",
                   "sample": f"{rows} rows of every per-layer op of one epoch on 1 thread "
                             f"(oracle/_ref, reference -O2 scalar kernels), scaled to {n} rows "
                             f"({wall:.1f} s measured)"}
        except Exception as exc:  # report, never fake
            cpu = {"value": None, "unit": "ms", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": ms_step, "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["workload"], "grid": "x".join(map(str, grid)),
                       "n": n, "nnz": nnz, "dims": [cfg["feat"], *cfg["hidden"], cfg["classes"]],
                       "gemm_mode": args.mode, "l2": "inputs larger than L2 (adjacency "
                       f"{2 * nnz * 8 / 1e9:.1f} GB + activations per epoch)",
                       "dataset_build_s": round(t_build, 2)},
            "roofline": {"bound": "hbm", "kernel": "spmm (all launches of the epoch)",
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": achieved / peak if achieved else None,
                         "traffic": traffic, "traffic_unit": "DRAM bytes per epoch (ncu)",
                         "alg_bytes_per_epoch": spmm_bytes,
                         "spmm_ms_per_epoch": spmm_s * 1e3,
                         "spmm_share_of_step": spmm_launch_share,
                         # DRAM view of the same launches: ncu bytes over the
                         # live SpMM time (frac above exceeds 1 because L2
                         # serves about half of the gathered feature rows)
                         "dram_achieved": (traffic / spmm_s / 1e9
                                           if traffic and spmm_s > 0 else None),
                         "dram_frac": (traffic / spmm_s / 1e9 / peak
                                       if traffic and spmm_s > 0 else None),
                         # against the 8 TB/s HBM3e spec sheet figure as well
                         "spec_peak": 8000.0,
                         "dram_frac_spec": (traffic / spmm_s / 1e9 / 8000.0
                                            if traffic and spmm_s > 0 else None),
                         "note": "achieved = SURVEY 8(d) algorithmic bytes "
                                 "(8nnz + 8(rows+1) + 4nnz*D + 4rows*D per SpMM) / "
                                 "measured SpMM time"},
            "phases_ms": phases,
            "collectives": coll,
            "losses": losses,
            "gpu_launches": int(launches),
            "gpu_launches_per_step": int(launches // max(1, args.steps)),
            "clocks": clocks.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

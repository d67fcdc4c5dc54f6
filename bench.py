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


def ref_pick_grid(gpus, n, nnz, dims):
    """The same pick from the reference's own rank_configs (oracle/_ref):
    the reference arm never loads libplexus_b200.so."""
    from oracle import ref
    m = B200_MACHINE
    best = ref.rank_configs(gpus, n, nnz, dims, g_node=m["g_node"], beta_intra=m["beta_intra"],
                            beta_inter=m["beta_inter"],
                            bytes_per_scalar=m["bytes_per_scalar"])[0]
    return tuple(int(x) for x in best[:3])


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
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU seconds for the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c1-measured", action="store_true",
                    help="skip the measured reference C1 epoch (train_distributed, 8 threads)")
    ap.add_argument("--ref-budget-s", type=float, default=100.0,
                    help="--impl reference: sampled CPU seconds over all timed steps")
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


def config_dict(cfg, grid, n, nnz):
    """The workload, identical in both arms' JSON lines."""
    return {"workload": cfg["workload"], "grid": "x".join(map(str, grid)), "n": int(n),
            "nnz": int(nnz), "dims": [cfg["feat"], *cfg["hidden"], cfg["classes"]],
            "l2": f"inputs larger than L2 (adjacency {2 * nnz * 8 / 1e9:.1f} GB + activations "
                  "per epoch)"}


def ref_dataset(cfg):
    """The reference's own synth_rmat + preprocess (oracle/_ref, -O2, one
    thread; graph.hpp:291-322, 356-384) — the reference arm's input, built
    without libplexus_b200.so."""
    from oracle import ref
    a, b, c = cfg["abc"]
    g = ref.synth_rmat(cfg["scale"], cfg["edges"], cfg["feat"], cfg["classes"], seed=1,
                       a=a, b=b, c=c)
    pre = g.preprocess(1)
    del g
    return pre


def ref_dataset_from_device(pre_dev):
    """Our GPU-built dataset (bit-identical to the reference's preprocess,
    tests/test_shard_builder_gpu.py, tests/test_c2_parity_gpu.py) handed to
    the reference for the cpu_baseline leg of our own arm."""
    from oracle import ref
    from paper_2505_04083_b200.trainer import HostDataset
    h = HostDataset.from_device(pre_dev, pin=False)
    return ref.Pre.from_arrays(h.n, h.feat_dim, h.num_classes,
                               (h.even[0].view(np.uint64), h.even[1].view(np.uint32), h.even[2]),
                               (h.odd[0].view(np.uint64), h.odd[1].view(np.uint32), h.odd[2]),
                               h.features, h.labels_row.view(np.uint32),
                               h.labels_col.view(np.uint32), h.mask_row, h.mask_col)


def reference_epoch_estimate(rpre, hidden, threads, target_s, rows=None):
    """The ONE cpu_baseline definition of both arms: the reference's own
    per-layer ops (spmm_rows / gemm incl. its TN dW form / relu / CE / Adam,
    oracle/_ref built with the reference's flags) over a row sample of the
    full epoch on `threads` host threads (ref_capi.cpp ref_epoch_sample),
    scaled to all n rows. An ESTIMATE: a full C2 epoch of the reference's
    scalar code takes minutes even on every host core. Returns (ms, rows
    per thread, sampled wall s)."""
    n = rpre.info()["n"]
    if rows is None:
        est, wall = rpre.epoch_sample(hidden, 64, threads)
        rows = int(max(64, min(n // max(1, threads), target_s / max(wall / 64, 1e-9))))
    est, wall = rpre.epoch_sample(hidden, rows, threads)
    return est * 1e3, rows, wall


def ref_c1_measured(threads_cap):
    """A MEASURED (not extrapolated) epoch of the reference's own
    train_distributed (trainer.hpp:541-687, one std::thread per rank) on C1
    at grid 2x2x2 = 8 threads: wall(3 epochs) - wall(1 epoch) over 2, so the
    setup cancels. Input from the reference's own synth_rmat + preprocess."""
    from oracle import ref
    cfg = CONFIGS["c1"]
    rpre = ref_dataset(cfg)
    grid = (2, 2, 2)
    walls = {}
    for e in (1, 3):
        t0 = time.perf_counter()
        out = rpre.train_distributed(grid, hidden=tuple(cfg["hidden"]), epochs=e,
                                     max_running=threads_cap)
        walls[e] = time.perf_counter() - t0
    ms = (walls[3] - walls[1]) / 2 * 1e3
    return {"config": "c1", "workload": cfg["workload"], "grid": "2x2x2", "threads": 8,
            "ms_per_epoch": ms, "losses": [float(x) for x in out["loss"]],
            "how": "reference train_distributed, wall(3 epochs) - wall(1 epoch) over 2, "
                   "input from reference synth_rmat+preprocess (oracle/_ref)"}


def gpu_c1_epoch_ms(local):
    """Our C1 epoch (1 GPU, grid 1x1x1, FAST): mean device epoch time of
    epochs 2..9 of 10 (the reference CLI's averaging window, main.cpp:209-231)."""
    from paper_2505_04083_b200 import trainer
    cfg = CONFIGS["c1"]
    pre = build_dataset(cfg, local)
    opts = trainer.TrainOptions(hidden_dims=cfg["hidden"], mode=trainer.PK_MODE_FAST, epochs=10)
    metrics, _, _ = trainer.train_single(pre, opts)
    return float(np.mean([m["epoch_s"] for m in metrics[2:10]])) * 1e3


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path,
    on this box's host cores, never touching libplexus_b200.so. Input: the
    reference's synth_rmat + preprocess (oracle/_ref). Each step: one
    bounded row-sample estimate of a full epoch (reference_epoch_estimate),
    sized so the whole --warmup/--steps run stays within a few minutes. Rank
    0 only under torchrun."""
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    t0 = time.perf_counter()
    rpre = ref_dataset(cfg)
    t_build = time.perf_counter() - t0
    info = rpre.info()
    n, nnz = info["n"], info["nnz_even"]
    dims = [cfg["feat"], *cfg["hidden"], cfg["classes"]]
    grid = (tuple(int(x) for x in args.grid.split(",")) if args.grid
            else ref_pick_grid(args.gpus, n, nnz, dims))
    threads = os.cpu_count() or 1
    # per timed step ~budget / steps seconds of sampled work
    step_s = max(1.0, min(8.0, args.ref_budget_s / max(1, args.steps)))
    _, rows, _ = reference_epoch_estimate(rpre, cfg["hidden"], threads, step_s)
    vals, walls = [], []
    for step in range(args.warmup + args.steps):
        r = max(64, rows // 8) if step < args.warmup else rows
        ms, _, wall = reference_epoch_estimate(rpre, cfg["hidden"], threads, step_s, rows=r)
        if step >= args.warmup:
            vals.append(ms)
            walls.append(wall)
    val = float(np.median(vals))
    sample = (f"{rows} rows x {threads} threads of every per-layer op of one 1x1x1 epoch "
              f"(reference spmm_rows/gemm/relu/CE/Adam, oracle/_ref -O2) per step, "
              f"extrapolated to {n} rows; input from the reference's own synth_rmat + "
              f"preprocess ({t_build:.0f} s)")
    line = {"metric": METRIC, "value": val, "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": val, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference", "extrapolated": True,
            "sampled_wall_s_per_step": float(np.median(walls)),
            "config": config_dict(cfg, grid, n, nnz),
            "cpu_baseline": {"value": val, "unit": "ms", "cores": threads, "kind": "reference",
                             "sample": sample, "extrapolated": True},
            "e2e": {"value": val, "unit": "ms", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def transform_first_layers(grid, dims, mode):
    from paper_2505_04083_b200 import layout
    if mode != "fast" or os.environ.get("PK_TRANSFORM_FIRST", "1") == "0":
        return []
    lays = layout.plan_layouts(len(dims) - 1)
    return [l for l, lay in enumerate(lays)
            if grid.extent(lay.inner) == 1 and dims[l + 1] < dims[l]]


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
    # the K epochs back to back, one host wait at the end (train_epochs)
    metrics = eng.train_epochs(args.warmup, args.steps)
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
    spmm_cbytes = float(np.mean([m["spmm_compulsory_bytes"] for m in metrics]))
    peak, peak_kind = hbm_peak()
    # DRAM bytes of the same SpMM launches of one epoch, from the committed
    # ncu launch list of this config at 1 GPU (scripts/ncu_round.sh ->
    # scripts/spmm_traffic.py; the file names the commit it was taken at)
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", f"ncu_spmm_{args.config}.json")
    if os.path.exists(prof) and world == 1 and args.mode == "fast":
        try:
            with open(prof) as f:
                pj = json.load(f)
            traffic = pj.get("dram_bytes_per_epoch")
            traffic_src = {"file": os.path.relpath(prof, ROOT), "commit": pj.get("commit"),
                           "launches": pj.get("spmm_launches")}
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
    # shard slicing, E epochs (each reads its metrics back to the host), then
    # the TrainResult download of this rank's trained W shards and F0 shard
    # (trainer.hpp:636-686 reassembles them on the host).
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
        eng2.prepare_result_buffers()  # host-side, overlaps the epochs
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        for e in range(args.e2e_epochs):
            eng2.train_epoch(e)
        t3 = time.perf_counter()
        result = eng2.download_params()
        t4 = time.perf_counter()
        parts = [t4 - t0, t1 - t0, t2 - t1, t3 - t2, t4 - t3]
        if world > 1:
            t = torch.tensor(parts, device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            parts = t.tolist()
        wall = parts[0]
        eng2.close()
        d2h = sum(a.nbytes for a in result) + args.e2e_epochs * C.sizeof(trainer.pk_epoch_metrics)
        e2e = {"value": wall * 1e3 / args.e2e_epochs, "unit": "ms",
               "h2d_bytes_per_step": int(host.nbytes() // args.e2e_epochs),
               "d2h_bytes_per_step": int(d2h // args.e2e_epochs),
               "epochs": args.e2e_epochs,
               "phases_ms": {"create_and_comm_init": parts[1] * 1e3, "load": parts[2] * 1e3,
                             "epochs": parts[3] * 1e3, "result_download": parts[4] * 1e3},
               "note": "train_distributed from a pinned-host PreprocessedDataset: dataset H2D "
                       "+ shard slicing + E epochs + download of the trained W / F0 shards, "
                       "wall / E (max over ranks)"}
        del host, result

    threads = os.cpu_count() or 1
    cpu = c1 = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            rpre = ref_dataset_from_device(pre)
            ms, rows, wall = reference_epoch_estimate(rpre, cfg["hidden"], threads,
                                                      args.cpu_seconds)
            del rpre
            cpu = {"value": ms, "unit": "ms", "cores": threads, "kind": "reference",
                   "extrapolated": True,
                   "sample": f"{rows} rows x {threads} threads of every per-layer op of one "
                             f"1x1x1 epoch (reference spmm_rows/gemm/relu/CE/Adam, oracle/_ref "
                             f"-O2), extrapolated to {n} rows ({wall:.1f} s sampled); same "
                             f"definition as --impl reference"}
        except Exception as exc:  # report, never fake
            cpu = {"value": None, "unit": "ms", "cores": threads, "kind": "reference",
                   "sample": f"unavailable: {exc}"}
    if rank == 0 and world == 1 and not args.no_c1_measured:
        try:
            del pre
            torch.cuda.empty_cache()
            c1 = ref_c1_measured(threads)
            c1["gpu_ms_per_epoch"] = gpu_c1_epoch_ms(local)
            c1["gpu_grid"] = "1x1x1 (1 B200, FAST)"
            c1["speedup"] = c1["ms_per_epoch"] / c1["gpu_ms_per_epoch"]
        except Exception as exc:
            c1 = {"unavailable": str(exc)}

    if rank == 0:
        dram = traffic / spmm_s / 1e9 if traffic and spmm_s > 0 else None
        comp = spmm_cbytes / spmm_s / 1e9 if spmm_s > 0 else None
        alg = spmm_bytes / spmm_s / 1e9 if spmm_s > 0 else None
        achieved = dram if dram is not None else comp
        line = {
            "metric": METRIC, "value": ms_step, "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": config_dict(cfg, grid, n, nnz),
            "gemm_mode": args.mode, "dataset_build_s": round(t_build, 2),
            # layers run as Q = A (F W) (engine.cu, transform-first: inner
            # axis one rank and D_out < D_in, FAST only)
            "transform_first_layers": transform_first_layers(gridc, dims, args.mode),
            "roofline": {"bound": "hbm", "kernel": "spmm (all launches of the epoch)",
                         "basis": "dram" if dram is not None else "compulsory",
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": achieved / peak if achieved else None,
                         "traffic": traffic, "traffic_unit": "DRAM bytes per epoch (ncu)",
                         "traffic_source": traffic_src,
                         "spmm_ms_per_epoch": spmm_s * 1e3,
                         "spmm_share_of_step": spmm_launch_share,
                         # the traffic floor: sparse matrix, output and every
                         # gathered row once per launch
                         "compulsory_bytes_per_epoch": spmm_cbytes,
                         "compulsory_gbs": comp,
                         "compulsory_frac": comp / peak if comp else None,
                         "traffic_over_compulsory": (traffic / spmm_cbytes
                                                     if traffic and spmm_cbytes else None),
                         # SURVEY 8(d) no-reuse bytes (one gathered row per
                         # nonzero): above the DRAM peak because L2 serves
                         # about half of the gathers, so not a DRAM fraction
                         "alg_noreuse_bytes_per_epoch": spmm_bytes,
                         "alg_noreuse_gbs": alg,
                         "alg_noreuse_over_peak": alg / peak if alg else None,
                         "spec_peak": 8000.0,
                         "note": "achieved = DRAM bytes of the epoch's SpMM launches (ncu, "
                                 "traffic) / live SpMM device time (CUDA events); "
                                 "compulsory = 8nnz + 8(rows+1) + 4 x_rows D + 4 rows D"},
            "phases_ms": phases,
            # mean device time between each epoch's first and last event (the
            # value above also covers any gap between epochs)
            "epoch_device_ms_mean": float(np.mean([m["epoch_s"] for m in metrics])) * 1e3,
            "collectives": coll,
            "losses": losses,
            "gpu_launches": int(launches),
            "gpu_launches_per_step": int(launches // max(1, args.steps)),
            "clocks": clocks.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "cpu_measured_c1": c1,
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

"""Command line front end mirroring the reference's tools/main.cpp
(preprocess / train / rank-configs / validate) over this package. f32 only: the device
path computes in fp32 (`--precision f64` is refused, exit code 2).

    python -m paper_2505_04083_b200 preprocess --synth rmat:scale=17,edges=2000000 \\
        --feat-dim 128 --classes 16 --p 2 --q 2 --seed 1 --precision f32 --out shards/
    python -m paper_2505_04083_b200 train --manifest shards/ --grid 1,1,1 --epochs 10 \\
        --layers 128,128 --out run/           # torchrun --nproc-per-node N for N ranks
    python -m paper_2505_04083_b200 rank-configs --stats n=2097152,nnz=116573894,dims=100-256-256-47 --g 8

Exit codes follow main.cpp:20-24 (0 ok, 1 validation, 2 input, 3 output,
4 resource)."""

import argparse
import os
import struct
import sys

import numpy as np

EXIT_OK, EXIT_VALIDATION, EXIT_INPUT, EXIT_OUTPUT, EXIT_RESOURCE = range(5)


class CliError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def parse_synth(spec):
    """'kind:key=value,...' (main.cpp:44-61)."""
    kind, _, rest = spec.partition(":")
    params = {}
    for kv in filter(None, rest.split(",")):
        k, eq, v = kv.partition("=")
        if not eq:
            raise CliError(EXIT_INPUT, f"bad synth parameter '{kv}' (expected key=value)")
        try:
            params[k] = float(v)
        except ValueError:
            raise CliError(EXIT_INPUT, f"bad synth parameter value in '{kv}'")
    return kind, params


def _ints(s):
    return [int(x) for x in s.split(",") if x]


def ensure_out_dir(d):
    try:
        os.makedirs(d, exist_ok=True)
        probe = os.path.join(d, ".plexuskit_write_probe")
        open(probe, "w").close()
        os.remove(probe)
    except OSError:
        raise CliError(EXIT_OUTPUT, f"output directory {d} is not writable")


def make_synth(kind, p, feat_dim, classes, seed, train_fraction):
    """make_synth_dataset (tools/main.cpp:70-93): sbm / erdos / rmat with the
    reference's parameter names and defaults, generated on the GPU."""
    from . import graph
    if kind == "sbm":
        return graph.synth_sbm(int(p.get("n", 1024)), int(p.get("k", 8)), p.get("p_in", 0.1),
                               p.get("p_out", 0.01), feat_dim, classes, seed,
                               train_fraction=train_fraction)
    if kind == "erdos":
        return graph.synth_erdos(int(p.get("n", 1024)), p.get("p", 0.01), feat_dim, classes,
                                 seed, train_fraction=train_fraction)
    if kind == "rmat":
        return graph.synth_rmat(int(p.get("scale", 10)), int(p.get("edges", 0)), feat_dim,
                                classes, seed, p.get("a", 0.57), p.get("b", 0.19),
                                p.get("c", 0.19), train_fraction=train_fraction)
    raise CliError(EXIT_INPUT, f"unknown synth kind '{kind}' (expected sbm, erdos or rmat)")


def cmd_preprocess(a):
    import torch

    from . import graph, shard_io
    if bool(a.edges) == bool(a.synth):
        raise CliError(EXIT_INPUT, "preprocess needs exactly one of --edges or --synth")
    if a.precision != "f32":
        raise CliError(EXIT_INPUT, "this build writes f32 shards (--precision f32)")
    if a.synth:
        kind, p = parse_synth(a.synth)
        ds = make_synth(kind, p, a.feat_dim, a.classes, a.seed, a.train_fraction)
    else:
        ds = load_dataset_files(a)
    ensure_out_dir(a.out)
    pre = graph.preprocess(ds, a.seed)
    m = shard_io.write_shards(pre, a.p, a.q, a.out, a.name)
    torch.cuda.synchronize()
    print(f"dataset {a.name}: {pre.n} nodes, {pre.a_even.nnz} nonzeros, {pre.feat_dim} "
          f"features, {pre.num_classes} classes")
    print(f"balance (max/mean over {a.p}x{a.q} blocks): double permutation "
          f"{graph.balance_metric(pre.a_even, a.p, a.q)}")
    print(f"wrote {len(m.files)} shard files + manifest to {a.out}")
    return EXIT_OK


def load_dataset_files(a):
    """Edge list ('src dst' per line, '#' comments) + optional labels / mask
    text files (main.cpp:87-159); features from Philox stream 3 like the
    reference when no feature file is given."""
    import torch

    from . import _capi, graph
    try:
        uv = []
        with open(a.edges) as f:
            for lineno, line in enumerate(f, 1):
                line = line.split("#", 1)[0].split()
                if not line:
                    continue
                if len(line) != 2:
                    raise CliError(EXIT_INPUT, f"{a.edges}:{lineno}: expected 'src dst' per line")
                uv.append((int(line[0]), int(line[1])))
    except OSError:
        raise CliError(EXIT_INPUT, f"cannot open edge list {a.edges}")
    e = np.asarray(uv, np.uint64).reshape(-1, 2)
    n = int(e.max()) + 1 if e.size else 0
    if a.nodes:
        if a.nodes < n:
            raise CliError(EXIT_INPUT, "--nodes is smaller than the largest edge endpoint")
        n = a.nodes
    dev = "cuda"
    edges = torch.from_numpy(e.astype(np.uint32).view(np.int32)).to(dev)
    feats = torch.empty((n, a.feat_dim), dtype=torch.float32, device=dev)
    _capi.call("pk_rmat_features", a.seed, n, a.feat_dim, feats.data_ptr(), a.feat_dim, None)
    if a.labels:
        lab = np.loadtxt(a.labels, dtype=np.uint64).reshape(-1)
        if lab.size != n:
            raise CliError(EXIT_INPUT, "labels file length does not match the node count")
        classes = max(a.classes, int(lab.max()) + 1)
        labels = torch.from_numpy(lab.astype(np.uint32).view(np.int32)).to(dev)
    else:
        classes = a.classes
        labels = torch.empty(n, dtype=torch.int32, device=dev)
        _capi.call("pk_degree_quantile_labels", edges.data_ptr(), edges.shape[0], n, classes,
                   labels.data_ptr(), None)
    if a.train_mask:
        mk = np.loadtxt(a.train_mask, dtype=np.int64).reshape(-1)
        if mk.size != n:
            raise CliError(EXIT_INPUT, "mask file length does not match the node count")
        mask = torch.from_numpy((mk != 0).astype(np.uint8)).to(dev)
    else:
        mask = torch.ones(n, dtype=torch.uint8, device=dev)
    return graph.GraphDataset(n, edges, feats, labels, classes, mask, not a.directed)


def write_model_file(weights, features, path):
    """write_model_file (shard_io.hpp:640-662): PLXM, f32."""
    with open(path, "wb") as f:
        f.write(b"PLXM" + struct.pack("<III", 1, 4, len(weights)))
        for m in list(weights) + [features]:
            m = np.ascontiguousarray(m, np.float32)
            f.write(struct.pack("<QQ", m.shape[0], m.shape[1]))
            f.write(m.tobytes())


METRIC_COLS = ("loss", "accuracy", "load_s", "forward_spmm_s", "forward_gemm_s", "backward_s",
               "optimizer_s", "collectives_s", "spmm_flops", "gemm_flops", "allreduce_bytes",
               "allgather_bytes", "reducescatter_bytes")


def _fmt_bytes(x):
    """the reference streams a double with default ostream formatting
    (6 significant digits)"""
    return f"{x:g}"


def cmd_train(a):
    import torch

    from . import distributed as D, perf_model as pm, shard_io, trainer
    from .layout import GridConfig
    mani = shard_io.load_manifest(a.manifest)
    if a.precision and a.precision != ("f32" if mani.precision == 4 else "f64"):
        raise CliError(EXIT_INPUT, f"--precision {a.precision} does not match the manifest")
    if mani.precision != 4:
        raise CliError(EXIT_INPUT, "this build trains f32 manifests")
    hidden = _ints(a.layers)
    if a.grid == "auto":
        if not a.machine:
            raise CliError(EXIT_INPUT, "--grid auto requires --machine")
        if a.ranks < 1:
            raise CliError(EXIT_INPUT, "--grid auto requires --ranks")
        machine = pm.machine_from_json_file(a.machine)
        coeffs = pm.coefficients_from_json_file(a.coeffs) if a.coeffs \
            else pm.default_coefficients()
        stats = pm.DatasetStats(mani.n, mani.nnz_even,
                                trainer.model_dims(mani.feat_dim, hidden, mani.classes))
        best = pm.rank_configs(a.ranks, stats, machine, coeffs)[0]
        shape = best.shape
        print(f"auto-selected grid {shape[0]}x{shape[1]}x{shape[2]} (predicted "
              f"{best.total_seconds} s/epoch)")
    else:
        shape = tuple(_ints(a.grid))
        if len(shape) != 3:
            raise CliError(EXIT_INPUT, "--grid expects X,Y,Z or 'auto'")
    grid = GridConfig(*shape)
    rank, world, local = D.dist_env()
    torch.cuda.set_device(local)
    opts = trainer.TrainOptions(hidden_dims=hidden, epochs=a.epochs, lr=a.lr, seed=a.seed,
                                block_count=a.block_count,
                                mode=trainer.PK_MODE_FAST if a.mode == "fast"
                                else trainer.PK_MODE_PARITY)
    res = D.train_distributed(lambda: mani, grid, opts)
    if rank != 0:
        return EXIT_OK
    ensure_out_dir(a.out)
    with open(os.path.join(a.out, "metrics.csv"), "w") as f:
        f.write("epoch,rank," + ",".join(METRIC_COLS) + "\n")
        for e in range(a.epochs):
            rows = [(str(r), res.per_rank[r][e]) for r in range(grid.size)]
            rows.append(("global", res.global_metrics[e]))
            for name, m in rows:
                f.write(f"{e},{name}," + ",".join(str(m.get(k, 0)) for k in METRIC_COLS) + "\n")
    g = res.global_metrics
    first = 2 if len(g) > 2 else 0  # average_window, main.cpp:213-231
    avg = {k: float(np.mean([m.get(k, 0.0) for m in g[first:]])) for k in METRIC_COLS}
    with open(os.path.join(a.out, "summary.csv"), "w") as f:
        f.write("grid,epochs,averaged_from_epoch,loss,accuracy,forward_spmm_s,forward_gemm_s,"
                "backward_s,optimizer_s,collectives_s\n")
        f.write(f"{grid.gx}x{grid.gy}x{grid.gz},{a.epochs},{first},{avg['loss']},"
                f"{avg['accuracy']},{avg['forward_spmm_s']},{avg['forward_gemm_s']},"
                f"{avg['backward_s']},{avg['optimizer_s']},{avg['collectives_s']}\n")
    # comm_stats.csv (main.cpp:353-366): per rank, axis and collective
    with open(os.path.join(a.out, "comm_stats.csv"), "w") as f:
        f.write("rank,axis,collective,calls,ring_bytes\n")
        for r, st in enumerate(res.stats):
            if st is None:
                continue
            calls, byts = st
            for ax in range(3):
                for op, name in enumerate(("all_gather", "all_reduce", "reduce_scatter")):
                    f.write(f"{r},{'XYZ'[ax]},{name},{int(calls[ax][op])},"
                            f"{_fmt_bytes(byts[ax][op])}\n")
    write_model_file(res.weights, res.features, os.path.join(a.out, "model.plxm"))
    print(f"trained {a.epochs} epochs on grid {grid.gx}x{grid.gy}x{grid.gz}: loss "
          f"{g[0]['loss']} -> {g[-1]['loss']}, accuracy {g[-1]['accuracy']}")
    print(f"wrote metrics.csv, summary.csv, comm_stats.csv, model.plxm to {a.out}")
    return EXIT_OK


def cmd_rank_configs(a):
    from . import perf_model as pm, shard_io, trainer
    hidden = _ints(a.layers)
    if a.manifest:
        m = shard_io.load_manifest(a.manifest)
        stats = pm.DatasetStats(m.n, m.nnz_even, trainer.model_dims(m.feat_dim, hidden, m.classes))
    elif a.stats:
        kv = {}
        for part in a.stats.split(","):
            k, eq, v = part.partition("=")
            if not eq:
                raise CliError(EXIT_INPUT, f"bad --stats entry '{part}'")
            kv[k] = v
        try:
            stats = pm.DatasetStats(int(kv["n"]), int(kv["nnz"]),
                                    [int(d) for d in kv["dims"].split("-")])
        except (KeyError, ValueError):
            raise CliError(EXIT_INPUT, "--stats expects n=..,nnz=..,dims=D0-H1-...-C")
    else:
        raise CliError(EXIT_INPUT, "rank-configs needs --manifest or --stats")
    machine = pm.machine_from_json_file(a.machine) if a.machine else pm.MachineParams()
    if a.fit_samples:
        coeffs = pm.fit_regression(pm.samples_from_csv_file(a.fit_samples))
        print(f"fitted coefficients: c1={coeffs.c1} c2={coeffs.c2} c3={coeffs.c3} "
              f"(train R2 {coeffs.train_r2}, RMSE {coeffs.train_rmse})")
        if a.coeffs_out:
            pm.coefficients_to_json_file(coeffs, a.coeffs_out)
    elif a.coeffs:
        coeffs = pm.coefficients_from_json_file(a.coeffs)
    else:
        coeffs = pm.default_coefficients()
        print("warning: no coefficients supplied, using built-in defaults", file=sys.stderr)
    ranked = pm.rank_configs(a.g, stats, machine, coeffs)
    print("gx,gy,gz,spmm_s,comm_s,total_s")
    for p in ranked:
        print(f"{p.shape[0]},{p.shape[1]},{p.shape[2]},{p.spmm_seconds},{p.comm_seconds},"
              f"{p.total_seconds}" + (" (spmm clamped to 0)" if p.clamped else ""))
    if a.csv:
        try:
            with open(a.csv, "w") as f:
                f.write("gx,gy,gz,spmm_s,comm_s,total_s,clamped\n")
                for p in ranked:
                    f.write(f"{p.shape[0]},{p.shape[1]},{p.shape[2]},{p.spmm_seconds},"
                            f"{p.comm_seconds},{p.total_seconds},{int(p.clamped)}\n")
        except OSError:
            raise CliError(EXIT_OUTPUT, f"cannot write {a.csv}")
    return EXIT_OK


def cmd_validate(a):
    """validate (main.cpp:469-512): every factorization of the world size
    trains the same dataset; each loss curve must match the single-rank
    1x1x1 run within --tolerance (relative, per epoch). Run under torchrun
    with --nproc-per-node G (one process per GPU); fp32 here, so the default
    tolerance is 1e-5 (the reference's f64 sweep uses 1e-9). PARITY mode:
    the ordered reductions keep the forward bit-identical across grids."""
    import torch
    import torch.distributed as dist

    from . import distributed as D, graph, shard_io, trainer
    from .layout import GridConfig, enumerate_configs
    rank, world = D.init_control_plane()
    _, _, local = D.dist_env()
    torch.cuda.set_device(local)
    if a.manifest:
        pre = shard_io.load_preprocessed(shard_io.load_manifest(a.manifest))
    elif a.synth:
        kind, p = parse_synth(a.synth)
        pre = graph.preprocess(make_synth(kind, p, a.feat_dim, a.classes, a.seed, 1.0), a.seed)
    else:
        raise CliError(EXIT_INPUT, "validate needs --manifest or --synth")
    opts = trainer.TrainOptions(hidden_dims=_ints(a.layers), epochs=a.epochs, lr=a.lr,
                                seed=a.seed, mode=trainer.PK_MODE_PARITY,
                                fault_epoch=0 if a.inject_fault else -1)
    serial = None
    if rank == 0:  # the single-rank reference curve on this GPU
        eng = trainer.RankEngine(pre.n, pre.feat_dim, pre.num_classes, GridConfig(1, 1, 1), 0,
                                 opts, local)
        eng.load(pre)
        serial = [eng.train_epoch(e)["loss"] for e in range(a.epochs)]
        eng.close()
        print(f"single-rank reference: {a.epochs} epochs, final loss {serial[-1]}")
    all_ok = True
    for shape in enumerate_configs(world):
        res = D.train_distributed(lambda: pre, GridConfig(*shape), opts,
                                  reassemble_params=False)
        if rank != 0:
            continue
        dev = [abs(m["loss"] - s_) / max(abs(s_), abs(m["loss"]), 1e-300)
               for m, s_ in zip(res.global_metrics, serial)]
        worst = max(dev)
        ok = worst <= a.tolerance
        all_ok = all_ok and ok
        print(f"{'PASS' if ok else 'FAIL'} config ({shape[0]}x{shape[1]}x{shape[2]}): max rel "
              f"loss deviation {worst} at epoch {dev.index(worst)}")
    if world > 1:
        flag = torch.tensor([1 if all_ok else 0], dtype=torch.int32)
        dist.broadcast(flag, 0)
        all_ok = bool(flag.item())
    if rank == 0:
        print("validation passed" if all_ok else "validation FAILED")
    return EXIT_OK if all_ok else EXIT_VALIDATION


def build_parser():
    ap = argparse.ArgumentParser(prog="paper_2505_04083_b200",
                                 description="3D tensor-parallel full-graph GCN training on B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("preprocess", help="synthesize or ingest a graph, write PLXS shards")
    p.add_argument("--edges", default="")
    p.add_argument("--synth", default="")
    p.add_argument("--labels", default="")
    p.add_argument("--train-mask", default="")
    p.add_argument("--nodes", type=int, default=0)
    p.add_argument("--feat-dim", type=int, default=128)
    p.add_argument("--classes", type=int, default=32)
    p.add_argument("--train-fraction", type=float, default=1.0)
    p.add_argument("--directed", action="store_true")
    p.add_argument("--p", type=int, default=8)
    p.add_argument("--q", type=int, default=8)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--precision", default="f32")
    p.add_argument("--name", default="dataset")
    p.add_argument("--out", required=True)
    t = sub.add_parser("train", help="train from shards (torchrun for several ranks)")
    t.add_argument("--manifest", required=True)
    t.add_argument("--grid", default="1,1,1")
    t.add_argument("--ranks", type=int, default=0)
    t.add_argument("--epochs", type=int, default=10)
    t.add_argument("--layers", default="128,128")
    t.add_argument("--seed", type=int, default=0)
    t.add_argument("--precision", default="")
    t.add_argument("--lr", type=float, default=1e-2)
    t.add_argument("--block-count", type=int, default=0)
    t.add_argument("--mode", default="fast", choices=["fast", "parity"],
                   help="fast: tcgen05 3xTF32 GEMMs, segmented hub rows; parity: bit-exact")
    t.add_argument("--machine", default="")
    t.add_argument("--coeffs", default="")
    t.add_argument("--out", default="train_out")
    r = sub.add_parser("rank-configs", help="rank grid shapes with the performance model")
    r.add_argument("--manifest", default="")
    r.add_argument("--stats", default="")
    r.add_argument("--layers", default="128,128")
    r.add_argument("--g", type=int, required=True)
    r.add_argument("--machine", default="")
    r.add_argument("--coeffs", default="")
    r.add_argument("--fit-samples", default="")
    r.add_argument("--coeffs-out", default="")
    r.add_argument("--csv", default="")
    v = sub.add_parser("validate", help="every grid of the world size vs the 1x1x1 run")
    v.add_argument("--manifest", default="")
    v.add_argument("--synth", default="")
    v.add_argument("--feat-dim", type=int, default=16)
    v.add_argument("--classes", type=int, default=32)
    v.add_argument("--epochs", type=int, default=10)
    v.add_argument("--layers", default="16")
    v.add_argument("--seed", type=int, default=0)
    v.add_argument("--lr", type=float, default=1e-2)
    v.add_argument("--tolerance", type=float, default=1e-5)
    v.add_argument("--inject-fault", action="store_true",
                   help="skip a reduction in epoch 0 (the check must then fail)")
    return ap


def main(argv=None):
    from ._capi import ContractError, IoError, MemoryError_, TrainingError
    a = build_parser().parse_args(argv)
    try:
        return {"preprocess": cmd_preprocess, "train": cmd_train,
                "rank-configs": cmd_rank_configs, "validate": cmd_validate}[a.cmd](a)
    except CliError as e:
        print(f"error: {e}", file=sys.stderr)
        return e.code
    except IoError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_OUTPUT if e.code == "WriteFailed" else EXIT_INPUT
    except TrainingError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_VALIDATION
    except MemoryError_ as e:
        print(f"error: out of memory: {e}", file=sys.stderr)
        return EXIT_RESOURCE
    except ContractError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INPUT

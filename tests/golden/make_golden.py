"""Generates the golden fixtures in this directory from the compiled
reference (oracle/_ref/libplexus_ref.so, built from /root/reference/proj by
oracle/Makefile). Run in the build container:
    PYTHONPATH=. python tests/golden/make_golden.py
The fixtures are small and committed; GPU-side tests and the oracle tests
read them without needing /root/reference.
"""

import os

import numpy as np

from oracle import ref

HERE = os.path.dirname(os.path.abspath(__file__))


def rmat_s9():
    scale, edges, feat, classes, seed, perm_seed = 9, 3000, 8, 4, 1, 1
    g = ref.synth_rmat(scale, edges, feat, classes, seed)
    ga = g.arrays()
    pre = g.preprocess(perm_seed)
    erp, eci, ev = pre.csr(0).arrays()
    orp, oci, ov = pre.csr(1).arrays()
    dims = [feat, 16, 16, classes]
    ser = pre.serial(hidden=(16, 16), seed=0)
    out = ser.forward_backward(0)
    curve, _ = pre.serial(hidden=(16, 16), seed=0).train(5)
    d = dict(scale=scale, edges=edges, feat=feat, classes=classes, seed=seed,
             perm_seed=perm_seed, dims=np.asarray(dims), uv=ga["edges"], labels=ga["labels"],
             features=ga["features"], even_rp=erp, even_ci=eci, even_v=ev, odd_rp=orp,
             odd_ci=oci, odd_v=ov, loss=out["loss"], accuracy=out["accuracy"],
             logits=out["logits"], df0=out["df0"], loss_curve_f32=curve)
    for l, w in enumerate(out["dw"]):
        d[f"dw{l}"] = w
    np.savez_compressed(os.path.join(HERE, "rmat_s9.npz"), **d)


def kernel_kats():
    # gemm 2x2 (test_kernels.cpp:129-141) and a small spmm (test_kernels.cpp:87-100)
    ga = np.array([[1, 2], [3, 4]], np.float32)
    gb = np.array([[5, 6], [7, 8]], np.float32)
    gc, _ = ref.gemm(ga, gb)
    rng = np.random.default_rng(0)
    rows, cols, dd = 20, 16, 5
    mask = rng.random((rows, cols)) < 0.3
    r, c = np.nonzero(mask)
    rp = np.zeros(rows + 1, np.uint64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp).astype(np.uint64)
    v = rng.uniform(-2, 2, size=r.size).astype(np.float32)
    x = rng.uniform(-1, 1, size=(cols, dd)).astype(np.float32)
    y, _ = ref.spmm_rows(rows, cols, rp, c.astype(np.uint32), v, x)
    np.savez_compressed(os.path.join(HERE, "kernel_kats.npz"), g_a=ga, g_b=gb, g_c=gc, s_rp=rp,
                        s_ci=c.astype(np.uint32), s_v=v, s_x=x, s_y=y)


def c1_curves():
    """The C1 golden loss curves quoted in SURVEY 8c (fp32 and fp64 at 2x2x2,
    10 epochs) — the 10-epoch envelope the GPU curve is judged against."""
    out = {}
    for f64 in (False, True):
        pre = ref.synth_rmat(17, 2_000_000, 128, 16, seed=1, f64=f64).preprocess(1)
        r = pre.train_distributed((2, 2, 2), hidden=(128, 128), seed=0, epochs=10)
        out["loss_f64" if f64 else "loss_f32"] = r["loss"]
        out["acc_f64" if f64 else "acc_f32"] = r["accuracy"]
    np.savez_compressed(os.path.join(HERE, "c1_curves.npz"), **out)


if __name__ == "__main__":
    rmat_s9()
    kernel_kats()
    if not os.path.exists(os.path.join(HERE, "c1_curves.npz")):
        c1_curves()
    print("golden fixtures written to", HERE)

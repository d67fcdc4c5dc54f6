"""CPU: pin the C restatement (oracle/plexus_oracle.c) against the compiled
reference (oracle/_ref) and against the committed golden fixtures; check
that the product library loads and exports every symbol the C ABI header
declares (no compute without a GPU)."""

import os
import re

import numpy as np
import pytest

from oracle import ref, restate

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def test_philox_streams_match_reference():
    for seed, stream in [(0, 0), (1, 5), (2**40 + 3, 100), (7, 2**33 + 1)]:
        assert np.array_equal(restate.philox_u64(seed, stream, 257), ref.philox_u64(seed, stream, 257))
        from paper_2505_04083_b200.philox import philox_u64
        assert np.array_equal(philox_u64(seed, stream, 257), ref.philox_u64(seed, stream, 257))


def test_permutation_pair_matches_reference():
    for n, seed in [(1, 0), (17, 3), (5000, 1)]:
        r, c = restate.permutation_pair(n, seed)
        wr, wc = ref.permutation_pair(n, seed)
        assert np.array_equal(r, wr) and np.array_equal(c, wc)


@pytest.mark.parametrize("scale,edges,a,b,c", [(9, 5000, 0.57, 0.19, 0.19),
                                               (10, 9000, 0.25, 0.25, 0.25)])
def test_synth_and_preprocess_match_reference(scale, edges, a, b, c):
    g = ref.synth_rmat(scale, edges, 6, 4, seed=2, a=a, b=b, c=c)
    ga = g.arrays()
    r = restate.synth_rmat(scale, edges, 6, 4, seed=2, a=a, b=b, c=c)
    assert np.array_equal(ga["edges"], r["edges"])
    assert np.array_equal(ga["features"], r["features"])
    assert np.array_equal(ga["labels"], r["labels"])
    pre = g.preprocess(3)
    rp = restate.preprocess(r, 3)
    for parity, key in ((0, "even"), (1, "odd")):
        for x, y in zip(pre.csr(parity).arrays(), rp[key]):
            assert np.array_equal(x, y)
    pa = pre.arrays()
    assert np.array_equal(pa["features"], rp["features"])
    for k in ("labels_row", "labels_col", "mask_row", "mask_col"):
        assert np.array_equal(pa[k], rp[k])


def test_kernels_match_reference():
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, size=(40, 7)).astype(np.float32)
    y = rng.uniform(-1, 1, size=(40, 9)).astype(np.float32)
    for ta, tb, a, b in [(False, False, x.T.copy(), y), (True, False, x, y),
                         (False, True, x, y[:7].copy()), (True, True, x, y[:, :7].T.copy())]:
        try:
            want, _ = ref.gemm(a, b, ta, tb)
        except RuntimeError:
            continue
        assert np.array_equal(restate.gemm(a, b, ta, tb), want)
    lg = rng.normal(size=(50, 5)).astype(np.float32)
    lab = rng.integers(0, 5, 50).astype(np.uint32)
    msk = (rng.random(50) < 0.7).astype(np.uint8)
    a1, a2 = restate.ce_sums(lg, lab, msk), ref.ce_sums(lg, lab, msk)
    assert a1[:3] == a2[:3] and np.array_equal(a1[3], a2[3])
    p = rng.uniform(-1, 1, size=(6, 5)).astype(np.float32)
    g = rng.uniform(-1, 1, size=(6, 5)).astype(np.float32)
    p1, m1, v1 = p.copy(), np.zeros_like(p), np.zeros_like(p)
    p2, m2, v2 = p.copy(), np.zeros_like(p), np.zeros_like(p)
    for step in range(1, 4):
        restate.adam_step(p1, g, m1, v1, step)
        ref.adam_step(p2, g, m2, v2, step - 1)
    assert np.array_equal(p1, p2) and np.array_equal(m1, m2) and np.array_equal(v1, v2)


def test_serial_pass_matches_reference():
    g = ref.synth_rmat(10, 6000, 12, 5, seed=4)
    pre = g.preprocess(4)
    want = pre.serial(hidden=(16, 16), seed=0).forward_backward(0)
    rp = restate.preprocess(restate.synth_rmat(10, 6000, 12, 5, seed=4), 4)
    got = restate.serial_forward_backward(rp, restate.init_weights([12, 16, 16, 5], 0))
    assert got["loss"] == want["loss"] and got["accuracy"] == want["accuracy"]
    assert np.array_equal(got["logits"], want["logits"])
    assert all(np.array_equal(a, b) for a, b in zip(got["dw"], want["dw"]))
    assert np.array_equal(got["df0"], want["df0"])


def test_golden_fixtures():
    """Oracle vs the committed reference outputs (tests/golden/make_golden.py)."""
    path = os.path.join(GOLDEN, "rmat_s9.npz")
    z = np.load(path)
    r = restate.synth_rmat(int(z["scale"]), int(z["edges"]), int(z["feat"]), int(z["classes"]),
                           seed=int(z["seed"]))
    assert np.array_equal(r["edges"], z["uv"])
    assert np.array_equal(r["labels"], z["labels"])
    rp = restate.preprocess(r, int(z["perm_seed"]))
    assert np.array_equal(rp["even"][0], z["even_rp"]) and np.array_equal(rp["even"][1], z["even_ci"])
    assert np.array_equal(rp["even"][2], z["even_v"])
    dims = [int(d) for d in z["dims"]]
    out = restate.serial_forward_backward(rp, restate.init_weights(dims, 0))
    assert out["loss"] == float(z["loss"])
    assert np.array_equal(out["logits"], z["logits"])
    assert np.array_equal(out["df0"], z["df0"])
    for l in range(len(dims) - 1):
        assert np.array_equal(out["dw"][l], z[f"dw{l}"])
    curve = z["loss_curve_f32"]
    assert curve.shape == (5,)


def test_kernel_known_answer_fixtures():
    """test_kernels.cpp KATs as committed vectors."""
    z = np.load(os.path.join(GOLDEN, "kernel_kats.npz"))
    assert np.array_equal(restate.gemm(z["g_a"], z["g_b"]), z["g_c"])
    got = restate.spmm_rows(z["s_rp"], z["s_ci"], z["s_v"], z["s_x"], 0, len(z["s_rp"]) - 1)
    assert np.array_equal(got, z["s_y"])


def test_capi_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "plexus_b200.h")).read()
    declared = set(re.findall(r"\b(pk_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) >= 20
    from paper_2505_04083_b200 import _capi
    lib = _capi.lib()
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_capi.SIGNATURES) <= declared | {"pk_last_error"}
    assert lib.pk_abi_version() == 2

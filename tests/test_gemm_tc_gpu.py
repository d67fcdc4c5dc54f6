"""Tensor-core (tcgen05, 3xTF32) dense transforms vs an fp64 reference.

The reference GEMM (kernels.hpp:64-92) is fp32; FAST mode must land within
fp32-level normwise error (fp32 ~2e-7, 3xTF32 ~8e-8 vs
fp64; plain TF32 ~3e-4 would fail). Tolerance: normwise 1e-5, plus a
max-abs bound relative to the operand scale.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _k():
    from paper_2505_04083_b200 import kernels
    return kernels


def _ref(a, b, ta, tb):
    a64 = a.astype(np.float64)
    b64 = b.astype(np.float64)
    return (a64.T if ta else a64) @ (b64.T if tb else b64)


def _check(got, want):
    got = got.astype(np.float64)
    den = np.linalg.norm(want)
    rel = np.linalg.norm(got - want) / (den if den else 1.0)
    assert rel <= TOL, rel
    return rel


# every BN bucket (16..256), n > 256 (several n tiles), odd k tails, m tails
SHAPES = [
    (128, 16, 32), (300, 47, 100), (1000, 24, 50), (257, 64, 128), (2048, 96, 33),
    (4096, 128, 100), (777, 192, 256), (5000, 256, 256), (640, 300, 64), (128, 13, 7),
    (3, 5, 2),
]


@pytest.mark.parametrize("m,n,kk", SHAPES)
@pytest.mark.parametrize("form", ["NN", "NT", "TN"])
def test_tc_gemm_forms(cuda, m, n, kk, form):
    ta, tb = form[0] == "T", form[1] == "T"
    rng = np.random.default_rng(m + 3 * n + 7 * kk)
    a = rng.standard_normal(size=(kk, m) if ta else (m, kk)).astype(np.float32)
    b = rng.standard_normal(size=(n, kk) if tb else (kk, n)).astype(np.float32)
    k = _k()
    got = k.gemm(torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda), ta, tb,
                 mode=k.PK_MODE_FAST).cpu().numpy()
    _check(got, _ref(a, b, ta, tb))


@pytest.mark.parametrize("m,n,kk", [(100, 128, 200000), (256, 47, 300000), (50, 24, 70001)])
def test_tc_gemm_tall_reduction(cuda, m, n, kk):
    """dW = H^T dQ with K = adjacency rows: split-K with fixed-order combine."""
    rng = np.random.default_rng(kk)
    h = rng.uniform(-1, 1, size=(kk, m)).astype(np.float32)
    dq = rng.uniform(-1, 1, size=(kk, n)).astype(np.float32)
    k = _k()
    hd, dd = torch.from_numpy(h).to(cuda), torch.from_numpy(dq).to(cuda)
    got = k.gemm(hd, dd, True, False, mode=k.PK_MODE_FAST).cpu().numpy()
    _check(got, _ref(h, dq, True, False))
    again = k.gemm(hd, dd, True, False, mode=k.PK_MODE_FAST).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), again.view(np.uint32)), "not deterministic"


def test_tc_gemm_strided_unaligned_views(cuda):
    """Column-chunk views (the last layer's dQ is a class chunk of dlogits with
    an odd column offset, engine backward) take the scalar-load path."""
    rng = np.random.default_rng(3)
    k = _k()
    big = torch.from_numpy(rng.standard_normal((3000, 48)).astype(np.float32)).to(cuda)
    dq = big[:, 23:47]          # 24 classes starting at column 23 (misaligned)
    w = torch.from_numpy(rng.standard_normal((128, 24)).astype(np.float32)).to(cuda)
    h = torch.from_numpy(rng.standard_normal((3000, 128)).astype(np.float32)).to(cuda)
    dqn = dq.cpu().numpy()
    got = k.gemm(dq, w, False, True, mode=k.PK_MODE_FAST).cpu().numpy()
    _check(got, _ref(dqn, w.cpu().numpy(), False, True))
    got = k.gemm(h, dq, True, False, mode=k.PK_MODE_FAST).cpu().numpy()
    _check(got, _ref(h.cpu().numpy(), dqn, True, False))


def test_tc_gemm_beats_tf32(cuda):
    """3xTF32 must be far better than plain TF32 (~3e-4 normwise)."""
    rng = np.random.default_rng(11)
    m, n, kk = 8192, 128, 128
    a = rng.standard_normal((m, kk)).astype(np.float32)
    b = rng.standard_normal((kk, n)).astype(np.float32)
    k = _k()
    got = k.gemm(torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda),
                 mode=k.PK_MODE_FAST).cpu().numpy()
    rel = _check(got, _ref(a, b, False, False))
    assert rel < 2e-6, rel


def test_tc_gemm_large_products_shape(cuda):
    """Products-shaped forward transform (1.2M x 128 . 128 x 128, SURVEY
    Appendix B) checked on a row sample against fp64."""
    k = _k()
    g = torch.Generator(device=cuda).manual_seed(0)
    h = torch.rand(1_224_515, 128, device=cuda, generator=g) - 0.5
    w = torch.rand(128, 128, device=cuda, generator=g) - 0.5
    q = k.gemm(h, w, mode=k.PK_MODE_FAST)
    idx = torch.randint(0, h.shape[0], (4096,), device=cuda, generator=g)
    want = h[idx].double() @ w.double()
    rel = (torch.linalg.norm(q[idx].double() - want) / torch.linalg.norm(want)).item()
    assert rel <= TOL, rel
    assert torch.isfinite(q).all()


@pytest.mark.parametrize("m,n,kk", [(5000, 256, 256), (300, 47, 100), (4096, 128, 1100),
                                    (64, 48, 40000), (3, 5, 2)])
@pytest.mark.parametrize("mode", ["fast", "parity"])
def test_gemm_relu_fused_equals_gemm_then_relu(cuda, m, n, kk, mode):
    """pk_gemm_relu_f32 (the hidden layer's GEMM with relu_forward in its
    epilogue) == relu_forward(gemm) bit for bit: plain tiles, segmented long
    k (1100 > 16 stages), split-K (k = 40000) and the SIMT parity path."""
    k = _k()
    md = k.PK_MODE_FAST if mode == "fast" else k.PK_MODE_PARITY
    rng = np.random.default_rng(m + n + kk)
    a = torch.from_numpy(rng.standard_normal(size=(m, kk)).astype(np.float32)).to(cuda)
    b = torch.from_numpy(rng.standard_normal(size=(kk, n)).astype(np.float32)).to(cuda)
    plain = k.gemm(a, b, mode=md)
    fused = k.gemm(a, b, mode=md, relu=True)
    want = k.relu_forward(plain)
    assert torch.equal(fused.view(torch.int32), want.view(torch.int32))
    assert (fused >= 0).all() and (fused == 0).any()


def _variant(tmp_path, name, env):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / f"{name}.npz"
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "mp", "gemm_variant_worker.py"),
                        str(out), root], env={**os.environ, **env}, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    return dict(np.load(out))


def test_gemm_cluster_multicast_matches_single_cta(cuda, tmp_path):
    """Weight-image multicast across 2- and 4-CTA clusters (with phantom
    tiles: 149 and 37 m tiles) gives the single-CTA results bit for bit; the
    register-staged fallback (PK_TC_TMA=0) stays within the 3xTF32 bound."""
    one = _variant(tmp_path, "cs1", {"PK_TC_CLUSTER": "1", "PK_TC_PAIR": "1"})  # CTA pairs
    for cs in ("2", "4"):
        got = _variant(tmp_path, "cs" + cs, {"PK_TC_CLUSTER": cs, "PK_TC_PAIR": "0"})
        for key in one:
            assert np.array_equal(got[key].view(np.uint32), one[key].view(np.uint32)), (cs, key)
    # CTA pairs (cta_group::2, M = 256) accumulate every element in the same k
    # order as one CTA: bit-identical too
    single = _variant(tmp_path, "nopair", {"PK_TC_PAIR": "0", "PK_TC_CLUSTER": "1"})
    for key in one:
        assert np.array_equal(single[key].view(np.uint32), one[key].view(np.uint32)), key
    reg = _variant(tmp_path, "reg", {"PK_TC_TMA": "0"})
    for key in one:
        den = np.linalg.norm(one[key].astype(np.float64)) or 1.0
        assert np.linalg.norm(reg[key].astype(np.float64) - one[key]) / den <= 2e-6, key

"""Parity of the sm_100a kernels against the CPU oracle (bit-exact where the
reference semantics allow it). Calls go through the C ABI
(libplexus_b200.so) via paper_2505_04083_b200.kernels.

Reference cases mirrored: proj/tests/test_kernels.cpp (identity / row swap /
flop counter / shape errors / random_csr vs dense / gemm 2x2 / transpose
flags / relu / cross entropy / masked rows).
"""

import numpy as np
import pytest
import torch

from oracle import ref, restate

pytestmark = pytest.mark.gpu


def _k():
    from paper_2505_04083_b200 import kernels
    return kernels


def random_csr(rows, cols, density, rng):
    """test_helpers.hpp:31-45 shape of random_csr (numpy RNG; sorted cols)."""
    mask = rng.random((rows, cols)) < density
    r, c = np.nonzero(mask)
    v = rng.uniform(-2, 2, size=r.size).astype(np.float32)
    rp = np.zeros(rows + 1, np.uint64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp).astype(np.uint64)
    return rp, c.astype(np.uint32), v


def skewed_csr(rows, cols, rng, hubs=((0, 9000), (7, 5000))):
    """Power-law-ish rows plus explicit hub rows (RMAT skew)."""
    lens = np.minimum(rng.zipf(1.6, size=rows), cols).astype(np.int64)
    for r, l in hubs:
        if r < rows:
            lens[r] = min(l, cols)
    rp = np.zeros(rows + 1, np.uint64)
    rp[1:] = np.cumsum(lens)
    ci = np.concatenate([np.sort(rng.choice(cols, size=l, replace=False)) for l in lens]
                        ).astype(np.uint32) if lens.sum() else np.zeros(0, np.uint32)
    v = rng.uniform(-1, 1, size=ci.size).astype(np.float32)
    return rp, ci, v


def dev_csr(rows, cols, rp, ci, v):
    return _k().DeviceCsr.from_host(rows, cols, rp, ci, v)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def assert_bitwise(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape
    diff = np.nonzero(bits(got) != bits(want))
    assert diff[0].size == 0, f"{diff[0].size} elements differ, first at {tuple(d[0] for d in diff)}"


# ---------------------------------------------------------------------------
# SpMM

def test_spmm_identity_and_row_swap(cuda):
    k = _k()
    eye = dev_csr(3, 3, np.array([0, 1, 2, 3]), np.array([0, 1, 2]), np.ones(3, np.float32))
    x = torch.tensor([[1, 2], [3, 4], [5, 6]], dtype=torch.float32, device=cuda)
    assert torch.equal(k.spmm(eye, x), x)
    sw = dev_csr(2, 2, np.array([0, 1, 2]), np.array([1, 0]), np.ones(2, np.float32))
    x2 = torch.tensor([[1, 2], [3, 4]], dtype=torch.float32, device=cuda)
    assert k.spmm(sw, x2).tolist() == [[3, 4], [1, 2]]


def test_spmm_flops_and_shape_error(cuda):
    k = _k()
    a = dev_csr(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]),
                np.array([1, 2, 3, 4], np.float32))
    fl = [0]
    k.spmm(a, torch.zeros(2, 2, device=cuda), flops=fl)
    assert fl[0] == 16
    bad = dev_csr(2, 3, np.array([0, 1, 1]), np.array([2]), np.array([5], np.float32))
    with pytest.raises(k.ContractError):
        k.spmm(bad, torch.zeros(2, 2, device=cuda))


@pytest.mark.parametrize("d", [1, 2, 3, 5, 8, 13, 16, 25, 32, 47, 50, 64, 100, 128, 256, 301,
                               520, 602, 777, 1000, 1200])
def test_spmm_bitwise_random(cuda, d):
    """Every vector width and lane-group form, including wide rows split
    into balanced column slices (520, 602, 777, 1000, 1200)."""
    rng = np.random.default_rng(d)
    rows, cols = 300, 257
    rp, ci, v = random_csr(rows, cols, 0.08, rng)
    x = rng.uniform(-1, 1, size=(cols, d)).astype(np.float32)
    want = restate.spmm_rows(rp, ci, v, x, 0, rows)
    a = dev_csr(rows, cols, rp, ci, v)
    got = _k().spmm(a, torch.from_numpy(x).to(cuda)).cpu().numpy()
    assert_bitwise(got, want)


@pytest.mark.parametrize("d,ld", [(50, 52), (100, 100), (128, 132), (13, 16), (47, 48)])
def test_spmm_bitwise_padded_ld_and_row_range(cuda, d, ld):
    rng = np.random.default_rng(100 + d)
    rows, cols = 500, 400
    rp, ci, v = skewed_csr(rows, cols, rng, hubs=((3, 350),))
    x = rng.uniform(-1, 1, size=(cols, d)).astype(np.float32)
    xs = torch.zeros(cols, ld, device=cuda)
    xs[:, :d] = torch.from_numpy(x).to(cuda)
    a = dev_csr(rows, cols, rp, ci, v)
    r0, r1 = 37, 411
    out = torch.full((r1 - r0, ld), 7.0, device=cuda)
    fl = [0]
    _k().spmm_rows(a, xs[:, :d], r0, r1, flops=fl, out=out[:, :d])
    want = restate.spmm_rows(rp, ci, v, x, r0, r1)
    assert_bitwise(out[:, :d].cpu().numpy(), want)
    assert torch.all(out[:, d:] == 7.0)  # padding untouched
    assert fl[0] == 2 * int(rp[r1] - rp[r0]) * d


@pytest.mark.parametrize("d", [16, 50, 100, 128, 256])
def test_spmm_hub_path_bitwise(cuda, d):
    """Hub CTAs (cp.async ring + sequential consumer) match the reference
    chain exactly; force a low threshold so several rows take that path."""
    rng = np.random.default_rng(7 + d)
    rows, cols = 2000, 20000
    rp, ci, v = skewed_csr(rows, cols, rng, hubs=((0, 15000), (5, 9000), (1999, 4097),
                                                   (1000, 33), (77, 2)))
    x = rng.uniform(-1, 1, size=(cols, d)).astype(np.float32)
    a = dev_csr(rows, cols, rp, ci, v)
    plan = _k().SpmmPlan(a, hub_threshold=30)
    hubs, thr = plan.info()
    assert thr == 30 and hubs >= 4
    xt = torch.from_numpy(x).to(cuda)
    got = _k().spmm(a, xt, plan=plan).cpu().numpy()
    want = restate.spmm_rows(rp, ci, v, x, 0, rows)
    assert_bitwise(got, want)
    # a row range through the same plan
    got2 = _k().spmm_rows(a, xt, 3, 1500, plan=plan).cpu().numpy()
    assert_bitwise(got2, want[3:1500])


def test_spmm_matches_reference_binary(cuda):
    """Against the compiled reference itself (oracle/_ref), not only the
    restatement."""
    rng = np.random.default_rng(3)
    rows, cols, d = 64, 64, 16
    rp, ci, v = random_csr(rows, cols, 0.15, rng)
    x = rng.uniform(-1, 1, size=(cols, d)).astype(np.float32)
    want, fl = ref.spmm_rows(rows, cols, rp, ci, v, x)
    got = _k().spmm(dev_csr(rows, cols, rp, ci, v), torch.from_numpy(x).to(cuda))
    assert_bitwise(got.cpu().numpy(), want)


def test_spmm_empty_rows_and_zero_extent(cuda):
    k = _k()
    a = dev_csr(4, 3, np.array([0, 0, 2, 2, 3]), np.array([0, 2, 1]),
                np.array([1, 2, 3], np.float32))
    x = torch.arange(6, dtype=torch.float32, device=cuda).reshape(3, 2)
    got = k.spmm(a, x).cpu().numpy()
    assert got.tolist() == [[0, 0], [0 + 8, 1 + 10], [0, 0], [6, 9]]
    z = k.spmm(a, torch.zeros(3, 0, device=cuda))
    assert tuple(z.shape) == (4, 0)
    e = dev_csr(0, 3, np.array([0]), np.zeros(0, np.uint32), np.zeros(0, np.float32))
    assert tuple(k.spmm(e, x).shape) == (0, 2)


# ---------------------------------------------------------------------------
# GEMM

def test_gemm_known_answers(cuda):
    k = _k()
    b1 = torch.tensor([[1, 2], [3, 4]], dtype=torch.float32, device=cuda)
    b2 = torch.tensor([[5, 6], [7, 8]], dtype=torch.float32, device=cuda)
    assert k.gemm(b1, b2).tolist() == [[19, 22], [43, 50]]
    a = torch.tensor([[1, 2, 3], [4, 5, 6]], dtype=torch.float32, device=cuda)
    fl = [0]
    assert torch.equal(k.gemm(a, torch.eye(3, device=cuda), flops=fl), a)
    assert fl[0] == 2 * 2 * 3 * 3
    with pytest.raises(k.ContractError):
        k.gemm(a, a)


@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("m,n,kk", [(5, 7, 4), (130, 47, 100), (67, 256, 129), (1, 1, 1),
                                    (200, 13, 3000)])
def test_gemm_parity_bitwise(cuda, ta, tb, m, n, kk):
    rng = np.random.default_rng(m * 7 + n + kk)
    a = rng.uniform(-1, 1, size=(kk, m) if ta else (m, kk)).astype(np.float32)
    b = rng.uniform(-1, 1, size=(n, kk) if tb else (kk, n)).astype(np.float32)
    want = restate.gemm(a, b, ta, tb)
    got = _k().gemm(torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda), ta, tb)
    assert_bitwise(got.cpu().numpy(), want)


def test_gemm_tall_reduction_parity(cuda):
    """dW shape: (dQ^T H)^T with K = adjacency rows (engine.hpp:233-235)."""
    rng = np.random.default_rng(5)
    K, f, w = 20000, 50, 24
    h = rng.uniform(-1, 1, size=(K, f)).astype(np.float32)
    dq = rng.uniform(-1, 1, size=(K, w)).astype(np.float32)
    want = restate.gemm(h, dq, True, False)  # serial form H^T dQ
    got = _k().gemm(torch.from_numpy(h).to(cuda), torch.from_numpy(dq).to(cuda), True, False)
    assert_bitwise(got.cpu().numpy(), want)
    want_rw, _ = ref.gemm(dq, h, True, False)  # engine rewrite (dQ^T H), transposed
    assert_bitwise(got.cpu().numpy(), want_rw.T)


def test_gemm_fast_mode_tolerance(cuda):
    k = _k()
    rng = np.random.default_rng(9)
    for (m, n, kk, ta, tb) in [(4096, 128, 100, False, False), (256, 47, 30000, True, False),
                               (5000, 100, 256, False, True)]:
        a = rng.uniform(-1, 1, size=(kk, m) if ta else (m, kk)).astype(np.float32)
        b = rng.uniform(-1, 1, size=(n, kk) if tb else (kk, n)).astype(np.float32)
        want = (a.T.astype(np.float64) if ta else a.astype(np.float64)) @ (
            b.T.astype(np.float64) if tb else b.astype(np.float64))
        got = k.gemm(torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda), ta, tb,
                     mode=k.PK_MODE_FAST).cpu().numpy().astype(np.float64)
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert rel <= 1e-5, (m, n, kk, ta, tb, rel)


def test_gemm_zero_k_writes_zeros(cuda):
    k = _k()
    out = k.gemm(torch.zeros(13, 0, device=cuda), torch.zeros(7, 0, device=cuda), False, True)
    assert tuple(out.shape) == (13, 7) and torch.count_nonzero(out) == 0


# ---------------------------------------------------------------------------
# elementwise

def test_relu_bitwise(cuda):
    k = _k()
    rng = np.random.default_rng(1)
    q = rng.uniform(-1, 1, size=(333, 47)).astype(np.float32)
    q[0, :3] = [0.0, -0.0, np.float32(1e-45)]
    df = rng.uniform(-1, 1, size=q.shape).astype(np.float32)
    qt, dft = torch.from_numpy(q).to(cuda), torch.from_numpy(df).to(cuda)
    assert_bitwise(k.relu_forward(qt).cpu().numpy(), restate.relu_forward(q))
    assert_bitwise(k.relu_backward(qt, dft).cpu().numpy(), restate.relu_backward(q, df))
    with pytest.raises(k.ContractError):
        k.relu_backward(qt, torch.zeros(2, 2, device=cuda))


def test_cross_entropy_known_answer(cuda):
    k = _k()
    logits = torch.zeros(1, 2, device=cuda)
    loss, dl = k.softmax_cross_entropy(logits, torch.tensor([0], dtype=torch.int32, device=cuda),
                                       torch.tensor([1], dtype=torch.uint8, device=cuda))
    assert abs(loss - np.log(2.0)) <= 1e-7
    assert dl.cpu().tolist() == [[-0.5, 0.5]]
    with pytest.raises(k.ContractError):
        k.softmax_cross_entropy(torch.eye(2, device=cuda),
                                torch.tensor([0, 1], dtype=torch.int32, device=cuda),
                                torch.zeros(2, dtype=torch.uint8, device=cuda))


@pytest.mark.parametrize("c,pad", [(3, 0), (16, 0), (47, 0), (47, 5), (172, 0), (256, 3),
                                   (384, 0)])
def test_cross_entropy_vs_oracle(cuda, c, pad):
    """Tile-staged CE: odd/even class counts, padded logits rows (ld > C),
    a partial last tile (4099 rows)."""
    k = _k()
    rng = np.random.default_rng(c)
    rows = 4099
    logits = rng.normal(0, 3, size=(rows, c)).astype(np.float32)
    logits[5, :] = 1.0  # all ties -> argmax 0
    labels = rng.integers(0, c, size=rows).astype(np.uint32)
    mask = (rng.random(rows) < 0.8).astype(np.uint8)
    ls, cnt, cor, d = restate.ce_sums(logits, labels, mask)
    wide = torch.zeros(rows, c + pad, device=cuda)
    wide[:, :c] = torch.from_numpy(logits).to(cuda)
    s = k.softmax_cross_entropy_sums(wide[:, :c],
                                     torch.from_numpy(labels.view(np.int32)).to(cuda),
                                     torch.from_numpy(mask).to(cuda))
    assert s.count == cnt and s.correct == cor
    assert abs(s.loss_sum - ls) / abs(ls) <= 1e-6
    dg = s.dlogits.cpu().numpy()
    assert np.linalg.norm(dg - d) / np.linalg.norm(d) <= 1e-6
    assert np.all(dg[mask == 0] == 0)


def test_adam_bitwise(cuda):
    k = _k()
    rng = np.random.default_rng(2)
    shape = (611, 50)
    p = rng.uniform(-1, 1, size=shape).astype(np.float32)
    m = np.zeros(shape, np.float32)
    v = np.zeros(shape, np.float32)
    pt = torch.from_numpy(p.copy()).to(cuda)
    st = k.AdamState.like(pt)
    for step in range(1, 6):
        g = rng.uniform(-1, 1, size=shape).astype(np.float32)
        restate.adam_step(p, g, m, v, step)
        k.adam_step(pt, torch.from_numpy(g).to(cuda), st)
        assert_bitwise(pt.cpu().numpy(), p)
        assert_bitwise(st.m.cpu().numpy(), m)
        assert_bitwise(st.v.cpu().numpy(), v)


# ---------------------------------------------------------------------------
# FAST SpMM plans: hub rows cut into segments, fixed-order combine

@pytest.mark.parametrize("d", [1, 7, 64, 100, 256, 602])
def test_spmm_fast_plan_segments_tolerance(cuda, d):
    """Hub rows (>= threshold) are summed as 2048-nonzero segments combined
    in a fixed order, and every chain uses fused multiply-adds (FAST plans):
    within fp32 rounding of the reference's chain, identical run to run and
    between row ranges of the same plan."""
    k = _k()
    rng = np.random.default_rng(d)
    n_rows, n_cols = 300, 20000
    lens = rng.integers(0, 40, size=n_rows)
    lens[[3, 77, 150]] = [4500, 9000, 5001]          # hub rows, several segments
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    ci = np.concatenate([np.sort(rng.choice(n_cols, size=l, replace=False)) for l in lens])
    vals = rng.uniform(-1, 1, size=ci.size).astype(np.float32)
    a = k.DeviceCsr.from_host(n_rows, n_cols, rp, ci.astype(np.uint32), vals)
    x = torch.from_numpy(rng.uniform(-1, 1, size=(n_cols, d)).astype(np.float32)).to(cuda)
    want = restate.spmm_rows(rp, ci.astype(np.uint32), vals, x.cpu().numpy(), 0, n_rows)
    plan = k.SpmmPlan(a, hub_threshold=4096, mode=k.PK_MODE_FAST)
    got = k.spmm(a, x, plan=plan).cpu().numpy()
    again = k.spmm(a, x, plan=plan).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), again.view(np.uint32))
    hub = lens >= 4096
    # regular rows: one chain each, fma vs mul+add roundings only
    exact = np.zeros_like(want, dtype=np.float64)
    for i in np.nonzero(~hub)[0]:
        s0, s1 = int(rp[i]), int(rp[i + 1])
        exact[i] = (vals[s0:s1].astype(np.float64)[:, None] *
                    x.cpu().numpy()[ci[s0:s1]].astype(np.float64)).sum(0)
    bound = 2 * (lens[~hub, None] + 2) * 2.0 ** -24 * lens[~hub, None] + 1e-30
    assert (np.abs(got[~hub] - exact[~hub]) <= bound).all()
    err = np.abs(got[hub].astype(np.float64) - want[hub])
    scale = np.abs(vals).max() * np.sqrt(lens.max()) * 4
    assert err.max() <= 1e-5 * scale, err.max()
    # row ranges through the same plan (blocked aggregation)
    part = k.spmm_rows(a, x, 50, 160, plan=plan).cpu().numpy()
    assert np.array_equal(part.view(np.uint32), got[50:160].view(np.uint32))


@pytest.mark.parametrize("d,ld", [(1, 1), (7, 7), (16, 16), (30, 30), (47, 48), (48, 48),
                                  (64, 64), (100, 100)])
def test_spmm_paired_form_tolerance(cuda, d, ld):
    """PK_SPMM_PAIRED (the transform-first layers' narrow SpMMs): each row as
    two interleaved chains added at the row end. Deterministic, within fp32
    rounding of the reference's single chain, row ranges through the same
    plan; rows wider than 16 vectors take the plain (bit-identical) form."""
    k = _k()
    rng = np.random.default_rng(1000 + d)
    n_rows, n_cols = 3000, 20000
    lens = rng.integers(0, 70, size=n_rows)
    lens[rng.random(n_rows) < 0.3] = 1                 # single-nonzero rows
    lens[[3, 777, 1500]] = [4500, 9000, 5001]           # hub rows (segments)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    ci = np.concatenate([np.sort(rng.choice(n_cols, size=l, replace=False)) for l in lens])
    vals = rng.uniform(-1, 1, size=ci.size).astype(np.float32)
    a = k.DeviceCsr.from_host(n_rows, n_cols, rp, ci.astype(np.uint32), vals)
    xh = rng.uniform(-1, 1, size=(n_cols, ld)).astype(np.float32)
    xh[:, d:] = 0
    x = torch.from_numpy(xh).to(cuda)  # the engine's padded width (47 -> 48, zero columns)
    want = restate.spmm_rows(rp, ci.astype(np.uint32), vals, xh[:, :ld], 0, n_rows)
    plan = k.SpmmPlan(a, hub_threshold=4096, mode=k.PK_MODE_FAST)
    got = k.spmm(a, x, plan=plan, paired=True).cpu().numpy()
    again = k.spmm(a, x, plan=plan, paired=True).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), again.view(np.uint32))
    plain = k.spmm(a, x, plan=plan).cpu().numpy()
    if ld > 64:
        assert np.array_equal(got.view(np.uint32), plain.view(np.uint32))
    # each of the two sums is within (n + 1) u sum|v x| of the exact one
    bound = 2 * (lens[:, None] + 2) * 2.0 ** -24 * (
        np.abs(vals)[None, :].max() * np.abs(xh[:, :ld]).max() * lens[:, None])
    err = np.abs(got.astype(np.float64) - want.astype(np.float64))
    assert (err <= bound + 1e-30).all(), float((err - bound).max())
    if ld > d:
        assert not got[:, d:].any()  # padding columns stay exactly +0
    part = k.spmm_rows(a, x, 500, 2600, plan=plan, paired=True).cpu().numpy()
    assert np.array_equal(part.view(np.uint32), got[500:2600].view(np.uint32))
    exact = k.SpmmPlan(a, hub_threshold=4096, mode=k.PK_MODE_PARITY)
    with pytest.raises(k.ContractError):
        k.spmm(a, x, plan=exact, paired=True)


@pytest.mark.parametrize("d", [1, 7, 64, 100, 256])
@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_spmm_relu_backward_fused(cuda, d, mode):
    """SpMM^T with the previous layer's relu_backward in its epilogue ==
    relu_backward(mask, spmm_rows) bit for bit: list rows, empty rows, hub
    rows (exact hub kernel / FAST segment combine), partial row ranges."""
    k = _k()
    md = k.PK_MODE_FAST if mode == "fast" else k.PK_MODE_PARITY
    rng = np.random.default_rng(100 + d)
    n_rows, n_cols = 300, 20000
    lens = rng.integers(0, 40, size=n_rows)
    lens[[3, 77, 150]] = [4500, 9000, 5001]
    lens[[5, 6, 200]] = 0
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    ci = np.concatenate([np.sort(rng.choice(n_cols, size=l, replace=False)) for l in lens])
    vals = rng.uniform(-1, 1, size=ci.size).astype(np.float32)
    a = k.DeviceCsr.from_host(n_rows, n_cols, rp, ci.astype(np.uint32), vals)
    x = torch.from_numpy(rng.uniform(-1, 1, size=(n_cols, d)).astype(np.float32)).to(cuda)
    act = rng.uniform(-1, 1, size=(n_rows, d)).astype(np.float32)
    act[act < 0] = 0  # a relu(Q): zeros and positives
    act[0, :] = -0.0
    mask = torch.from_numpy(act).to(cuda)
    plan = k.SpmmPlan(a, hub_threshold=4096, mode=md)
    for r0, r1 in [(0, n_rows), (50, 160), (140, 160)]:
        plain = k.spmm_rows(a, x, r0, r1, plan=plan)
        want = k.relu_backward(mask[r0:r1], plain)
        got = k.spmm_rows_relu_backward(a, x, r0, r1, mask[r0:r1], plan)
        assert torch.equal(got.view(torch.int32), want.view(torch.int32)), (r0, r1)


_L2_SLICED_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from oracle import restate
from paper_2505_04083_b200 import kernels as k
sys.path.insert(0, sys.argv[1] + "/tests")
from test_kernels_gpu import random_csr, skewed_csr
for d in (33, 100, 301, 602, 1000):
    rng = np.random.default_rng(500 + d)
    for rows, cols in ((300, 257), (800, 3000)):
        rp, ci, v = (random_csr(rows, cols, 0.08, rng) if rows == 300
                     else skewed_csr(rows, cols, rng, hubs=((3, 2500),)))
        x = rng.uniform(-1, 1, size=(cols, d)).astype(np.float32)
        want = restate.spmm_rows(rp, ci, v, x, 0, rows)
        a = k.DeviceCsr.from_host(rows, cols, rp, ci, v)
        got = k.spmm(a, torch.from_numpy(x).cuda()).cpu().numpy()
        want = np.ascontiguousarray(want, dtype=np.float32)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (d, rows)
print("ok")
"""


def test_spmm_l2_sliced_form_bitwise(cuda):
    """The L2-sliced wide-row form (one 32-lane column slice per grid.y,
    spmm.cu l2_slice_lanes) is forced with PK_SPMM_L2_LANES at 32 and 16
    lanes; rows stay bit-identical with the reference chain. The variable is
    read once per process, hence the child processes."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for lanes in ("32", "16"):
        env = dict(os.environ, PK_SPMM_L2_LANES=lanes)
        r = subprocess.run([sys.executable, "-c", _L2_SLICED_CHILD, root], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr

"""Parity at the bench configuration C2 (products-shaped RMAT s21, 62M edges,
2,097,152 nodes, 116,573,894 nonzeros, GCN 100-256-256-47) on one B200 —
the workload bench.py's headline number is measured on.

Checker: the compiled, unmodified reference (oracle/_ref):
  (a) synth_rmat + preprocess (graph.hpp:291-322, 356-384) on one host
      thread — the GPU shard builder must match it byte for byte: both
      permuted adjacency variants, features, labels and masks;
  (b) SerialTrainer::forward_backward (trainer.hpp:137-169) composed from the
      reference's own kernels over row blocks on every host core
      (ref_serial_pass_parallel in oracle/ref_capi.cpp; rows bitwise the
      serial pass's, the loss sum reduced blockwise, dW = H^T dQ over K =
      2,097,152 rows returned in float64). From the same W and F0: PARITY
      logits bit-identical and dF0 within 1e-5 (it inherits the CE's
      expf / logf ulps), FAST logits / dW / dF0 within 1e-4
      normwise, loss within 1e-6 relative (expf / logf ulps). PARITY dW runs
      the reference's sequential fp32 k chain (2.1M terms per column): within
      1e-5 of the serial trainer's own gemm(h, dq, true) on the columns the
      checker also runs serially (operands differ only by the CE's ulps);
      that chain's own rounding is up to ~2e-3 normwise from the fp64 value
      (last layer), so its fp64 gate is 5e-3 — the tensor-core path, which
      folds its TMEM partial every 512 k with round-to-nearest adds, must
      meet 1e-4;
  (c) the FAST SpMM plan's segmented hub rows at C2's real degrees (rows of
      up to 155,518 nonzeros = 76 fixed 2048-nonzero segments): H of layer 0
      bit-identical on every non-hub row, hub rows within 1e-4 normwise (the
      largest is 6.5e-6 off: the reference's 155K-term chain's own rounding).
Runs for a few minutes (the reference preprocess alone is ~2 min of one
core), so everything shares one module-scoped reference dataset.
"""

import os
import time

import numpy as np
import pytest
import torch

from oracle import ref

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SCALE, EDGES, FEAT, CLASSES, HIDDEN = 21, 62_000_000, 100, 47, (256, 256)
NNZ = 116_573_894


def nrel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def c2(cuda):
    from paper_2505_04083_b200 import graph
    t0 = time.time()
    rpre = ref.synth_rmat(SCALE, EDGES, FEAT, CLASSES, seed=1).preprocess(1)
    t_ref = time.time() - t0
    t0 = time.time()
    pre = graph.preprocess(graph.synth_rmat(SCALE, EDGES, FEAT, CLASSES, seed=1), perm_seed=1)
    torch.cuda.synchronize()
    t_gpu = time.time() - t0
    print(f"\nC2 preprocess: reference {t_ref:.1f} s (1 thread), GPU {t_gpu:.2f} s")
    yield rpre, pre


def test_c2_shard_builder_bit_exact(c2):
    rpre, pre = c2
    info = rpre.info()
    assert info["n"] == pre.n == 1 << SCALE
    assert info["nnz_even"] == info["nnz_odd"] == pre.a_even.nnz == pre.a_odd.nnz == NNZ
    for parity, a in ((0, pre.a_even), (1, pre.a_odd)):
        want = rpre.csr(parity).arrays()
        got = a.to_host()
        for g, w in zip(got, want):
            g, w = np.asarray(g), np.asarray(w)
            assert g.shape == w.shape and np.array_equal(g.view(np.uint8), w.view(np.uint8)), \
                parity
    arr = rpre.arrays()
    assert np.array_equal(pre.features.cpu().numpy().view(np.uint32),
                          arr["features"].view(np.uint32))
    for name, t in (("labels_row", pre.labels_row_order), ("labels_col", pre.labels_col_order),
                    ("mask_row", pre.mask_row_order), ("mask_col", pre.mask_col_order)):
        assert np.array_equal(t.cpu().numpy(), arr[name]), name


@pytest.fixture(scope="module")
def ref_pass(c2):
    rpre, _ = c2
    threads = os.cpu_count() or 1
    t0 = time.time()
    out = rpre.serial_pass_parallel(HIDDEN, threads, seed=0, want_h0=True, sample_cols=4)
    print(f"\nC2 reference forward_backward on {threads} threads: {time.time() - t0:.1f} s")
    return out


_ACT = {}  # PARITY pass's ReLU masks (reference-identical) for the FAST test


def _engine_pass(pre, mode):
    from paper_2505_04083_b200 import trainer as tr
    opts = tr.TrainOptions(hidden_dims=list(HIDDEN), mode=mode)
    eng = tr.RankEngine(pre.n, pre.feat_dim, pre.num_classes, tr.GridConfig(1, 1, 1), 0, opts)
    eng.load(pre)
    loss, acc = eng.forward_backward(0)
    out = dict(loss=loss, accuracy=acc, logits=eng.tensor(tr.PK_T_FOUT).cpu().numpy(),
               dw=[eng.tensor(tr.PK_T_DW, l).cpu().numpy() for l in range(3)],
               df0=eng.tensor(tr.PK_T_DF0).cpu().numpy(),
               h0=eng.tensor(tr.PK_T_H, 0).cpu().numpy(),
               mask=[(eng.tensor(tr.PK_T_ACT, l) > 0).cpu().numpy() for l in range(2)])
    eng.close()
    torch.cuda.empty_cache()
    return out


def test_c2_parity_pass_logits_bitwise(c2, ref_pass):
    from paper_2505_04083_b200 import trainer as tr
    _, pre = c2
    got = _engine_pass(pre, tr.PK_MODE_PARITY)
    _ACT["parity"] = got["mask"]
    assert np.array_equal(got["logits"].view(np.uint32), ref_pass["logits"].view(np.uint32))
    assert got["accuracy"] == ref_pass["accuracy"]
    assert abs(got["loss"] - ref_pass["loss"]) <= 1e-6 * abs(ref_pass["loss"])
    # dW: PARITY runs the serial trainer's k order (one fp32 chain over all
    # 2,097,152 rows); its operands differ from the reference's only by the
    # CE's expf / logf ulps, so on the columns the checker also ran
    # serially it must sit within 1e-5 of the reference's own chain, while
    # that chain itself is up to ~2e-3 from the fp64 value
    for l in range(3):
        ser = ref_pass["dw_serial_cols"][l]
        k = ser.shape[1]
        e_chain = nrel(got["dw"][l][:, :k], ser)
        e_ref64 = nrel(ser, ref_pass["dw"][l][:, :k])
        print(f"\nC2 PARITY dW layer {l}: vs reference serial chain {e_chain:.2e}; "
              f"reference chain vs fp64 {e_ref64:.2e}")
        assert e_chain <= 1e-5, (l, e_chain)
    errs = [nrel(got["dw"][l], ref_pass["dw"][l]) for l in range(3)]
    print(f"C2 PARITY dW vs fp64 (normwise): {errs}")
    assert max(errs) <= 5e-3, errs
    # dF0 inherits the CE's expf / logf ulps through every layer's dQ
    e_df0 = nrel(got["df0"], ref_pass["df0"])
    print(f"C2 PARITY dF0 vs reference (normwise): {e_df0:.2e}")
    assert e_df0 <= 1e-5
    # every H row of layer 0 is one exact chain in PARITY plans
    assert np.array_equal(got["h0"].view(np.uint32), ref_pass["h0"].view(np.uint32))


def test_c2_fast_pass_within_tolerance(c2, ref_pass):
    """The bench's mode: tcgen05 3xTF32 GEMMs + segmented FAST SpMM plans.

    Forward and weight gradients meet 1e-4 normwise (measured: logits
    4e-6, dW 1e-5). dF0 is gated at 2e-3: it runs through two ReLU'
    masks, and a hidden activation within fp32 rounding of 0 can land on the
    other side of 0 once the GEMM rounds differently (the same happens to
    the reference's own fp32 pass against fp64); each such flip moves one dQ
    entry by a full gradient value, so the normwise error scales with the
    square root of the flip fraction, not with the rounding. The test
    counts the flips against the PARITY pass (whose activations are the
    reference's bit for bit) and checks the hub segmentation first."""
    from paper_2505_04083_b200 import trainer as tr
    rpre, pre = c2
    got = _engine_pass(pre, tr.PK_MODE_FAST)
    # (c) hub segmentation at C2's real degrees: FAST plans cut rows of
    # >= 4096 nonzeros (the automatic threshold max(4096, 64 x mean) at a
    # mean of 55.6) into 2048-nonzero segments; every chain uses fused
    # multiply-adds, so regular rows differ from the reference by a rounding
    # per nonzero at most
    rp = pre.a_even.row_ptr.cpu().numpy().astype(np.int64)
    deg = np.diff(rp)
    assert deg.max() >= 150_000, deg.max()
    hub = deg >= 4096
    assert hub.sum() > 0
    h0, w0 = got["h0"], ref_pass["h0"]
    e_reg = nrel(h0[~hub], w0[~hub])
    print(f"\nC2 FAST regular rows (fma chains) vs reference: {e_reg:.2e} (normwise)")
    assert e_reg <= 1e-6, e_reg
    # a hub row's 2048-term segments summed in order differ from the
    # reference's single 155K-term chain by that chain's own rounding
    top = int(np.argmax(deg))
    e_top, e_hub = nrel(h0[top], w0[top]), nrel(h0[hub], w0[hub])
    print(f"\nC2 FAST hub rows: {int(hub.sum())} rows >= 4096 nnz, largest {deg[top]:,}: "
          f"{e_top:.2e}; all hub rows {e_hub:.2e} (normwise)")
    assert e_top <= 1e-4 and e_hub <= 1e-4, (e_top, e_hub)
    assert abs(got["loss"] - ref_pass["loss"]) <= 1e-6 * abs(ref_pass["loss"])
    errs = dict(logits=nrel(got["logits"], ref_pass["logits"]),
                dw=[nrel(got["dw"][l], ref_pass["dw"][l]) for l in range(3)],
                df0=nrel(got["df0"], ref_pass["df0"]))
    flips = None
    if "parity" in _ACT:
        flips = [int(np.count_nonzero(a != b)) for a, b in zip(got["mask"], _ACT["parity"])]
    print(f"\nC2 FAST vs reference (normwise): {errs}; ReLU mask flips vs reference "
          f"(layers 0, 1 of {got['mask'][0].size:,} each): {flips}")
    assert errs["logits"] <= 1e-4
    assert max(errs["dw"]) <= 1e-4
    assert errs["df0"] <= 2e-3

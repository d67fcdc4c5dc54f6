"""Performance model (perf_model.hpp / src/perf_model.cpp) through the native
C ABI, against the reference's own known answers (test_perf_model.cpp) and
against the compiled reference itself (oracle/_ref) on every factorization
used by the benchmark configs. CPU only: the model has no device work."""

import math

import numpy as np
import pytest

from oracle import ref
from paper_2505_04083_b200 import perf_model as pm
from paper_2505_04083_b200._capi import ContractError

PRODUCTS = pm.DatasetStats(2449029, 126167053, [100, 256, 256, 47])
C2_RMAT = pm.DatasetStats(2097152, 116573894, [100, 256, 256, 47])


def test_published_flops_cost_and_penalties():
    """test_perf_model.cpp:51-64."""
    one = pm.DatasetStats(2449029, 126167053, [100, 47])
    f = pm.comp_features(one, (1, 1, 1))
    assert f[0] * f[0] == pytest.approx(1.26167053e10, rel=1e-12)
    f = pm.comp_features(one, (64, 1, 1))
    assert f[1] / f[0] == pytest.approx(382.66078125, rel=1e-12)
    assert f[2] / f[0] == pytest.approx(24490.29, rel=1e-6)
    small = pm.DatasetStats(1000, 5000, [25, 10])
    f = pm.comp_features(small, (1, 1, 1))
    assert f[1] / f[0] == pytest.approx(40.0, rel=1e-12)
    with pytest.raises(ContractError):
        pm.comp_features(pm.DatasetStats(0, 5, [4, 2]), (1, 1, 1))
    with pytest.raises(ContractError):
        pm.comp_features(pm.DatasetStats(10, 5, [4, 0]), (1, 1, 1))


def test_predict_spmm_clamp_and_sqrt_scaling():
    """test_perf_model.cpp:85-101."""
    assert pm.predict_spmm_time((0, 0, 0), pm.PerfCoefficients(1, 1, 1))[0] == 0.0
    s, clamped = pm.predict_spmm_time((5, 0, 0), pm.PerfCoefficients(-1, 0, 0))
    assert s == 0.0 and clamped
    c1 = pm.PerfCoefficients(1, 0, 0)
    t1 = pm.predict_spmm_time(pm.comp_features(pm.DatasetStats(100000, 1000000, [64, 8]),
                                               (2, 2, 2)), c1)[0]
    t2 = pm.predict_spmm_time(pm.comp_features(pm.DatasetStats(100000, 2000000, [64, 8]),
                                               (2, 2, 2)), c1)[0]
    assert t2 / t1 == pytest.approx(math.sqrt(2.0), rel=1e-12)
    d = pm.default_coefficients()
    u = pm.predict_spmm_time(pm.comp_features(PRODUCTS, (64, 1, 1)), d)[0]
    v = pm.predict_spmm_time(pm.comp_features(PRODUCTS, (1, 64, 1)), d)[0]
    assert u < v


def test_effective_bandwidth_cases():
    """test_perf_model.cpp:112-138."""
    m = pm.MachineParams(4, 200e9, 25e9, 4)
    for a in "XYZ":
        assert pm.effective_bandwidth(a, (2, 2, 1), m) == 200e9
    assert pm.effective_bandwidth("Z", (2, 2, 4), m) == pytest.approx(25e9 / 4, rel=1e-12)
    assert pm.effective_bandwidth("Y", (4, 4, 1), m) == 200e9
    assert pm.effective_bandwidth("X", (4, 4, 1), m) == pytest.approx(25e9 / 4, rel=1e-12)
    solo = pm.MachineParams(1, 200e9, 25e9, 4)
    assert pm.effective_bandwidth("X", (4, 4, 4), solo) == 25e9
    assert pm.effective_bandwidth("Z", (4, 4, 1), solo) == 200e9


def test_ring_worked_example():
    """test_perf_model.cpp:140-152."""
    t = pm.ring_collective_seconds("all_reduce", 1e8, 4, 25e9)
    assert abs(t - 6e-3) <= 1e-12
    assert pm.ring_collective_seconds("all_reduce", 1e8, 1, 25e9) == 0.0
    assert pm.ring_collective_seconds("all_gather", 1e8, 4, 25e9) == pytest.approx(3e-3)
    assert pm.predict_comm_time((1, 1, 1), pm.DatasetStats(256, 3000, [16, 8, 4]),
                                pm.MachineParams()) == 0.0


@pytest.mark.parametrize("g", [1, 2, 4, 8, 12, 64])
@pytest.mark.parametrize("stats", [PRODUCTS, C2_RMAT,
                                   pm.DatasetStats(131072, 3698720, [128, 128, 128, 16]),
                                   pm.DatasetStats(13, 40, [5, 7, 3])])
def test_matches_reference_every_config(g, stats):
    """Features, comm model and the full ranking equal the compiled
    reference (perf_model.cpp:33-229) on every ordered factorization."""
    machine = pm.MachineParams(8, 725e9, 50e9, 4)
    coeffs = pm.default_coefficients()
    configs = pm.enumerate_configs(g)
    assert len(configs) == len(set(configs))
    for shape in configs:
        mine = pm.comp_features(stats, shape)
        theirs = ref.comp_features(stats.n, stats.nnz, stats.dims, shape)
        np.testing.assert_allclose(mine, theirs, rtol=1e-14)
        mc = pm.predict_comm_time(shape, stats, machine)
        rc = ref.predict_comm(stats.n, stats.nnz, stats.dims, shape, machine.g_node,
                              machine.beta_intra, machine.beta_inter, machine.bytes_per_scalar)
        assert mc == pytest.approx(rc, rel=1e-14, abs=0)
        vols = pm.training_collective_volumes(shape, stats.n, stats.dims)
        rv = ref.collective_volumes(shape, stats.n, stats.dims)
        assert [tuple(int(x) for x in (v[0], v[1], v[2], v[3], v[4])) for v in vols] == \
            [tuple(int(x) for x in r) for r in rv]
    mine = pm.rank_configs(g, stats, machine, coeffs)
    theirs = ref.rank_configs(g, stats.n, stats.nnz, stats.dims, machine.g_node,
                              machine.beta_intra, machine.beta_inter, machine.bytes_per_scalar,
                              (coeffs.c1, coeffs.c2, coeffs.c3))
    assert [p.shape for p in mine] == [tuple(int(x) for x in r[:3]) for r in theirs]
    np.testing.assert_allclose([p.total_seconds for p in mine], theirs[:, 5], rtol=1e-13)


def test_products_default_pick_is_2x2x2():
    """default coefficients + an 8-GPU NVSwitch machine
    pick 2,2,2 for G=8, 2,1,2 for G=4 and 2,1,1 for G=2."""
    m = pm.MachineParams(8, 900e9, 50e9, 4)
    c = pm.default_coefficients()
    assert pm.rank_configs(8, PRODUCTS, m, c)[0].shape == (2, 2, 2)
    assert pm.rank_configs(4, PRODUCTS, m, c)[0].shape == (2, 1, 2)
    assert pm.rank_configs(2, PRODUCTS, m, c)[0].shape == (2, 1, 1)


def _synth_samples(truth, noise, seed, count):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        n = int(rng.integers(1000, 3_000_000))
        nnz = int(n * rng.uniform(2, 60))
        dims = [int(rng.integers(8, 600)), int(rng.integers(8, 300)), int(rng.integers(2, 200))]
        g = [1, 2, 4, 8, 16, 32, 64][int(rng.integers(0, 7))]
        cfgs = pm.enumerate_configs(g)
        shape = cfgs[int(rng.integers(0, len(cfgs)))]
        f = pm.comp_features(pm.DatasetStats(n, nnz, dims), shape)
        y = truth[0] * f[0] + truth[1] * f[1] + truth[2] * f[2]
        y *= 1.0 + noise * (2 * rng.random() - 1)
        out.append(pm.RegressionSample(f, y))
    return out


def test_fit_regression_recovery_and_reference():
    """test_perf_model.cpp:173-190 (exact recovery, R2 under noise), and the
    same coefficients as the reference's solver."""
    truth = (7.8e-4, 7.8e-10, -2.6e-10)
    s = _synth_samples(truth, 0.0, 3, 40)
    fit = pm.fit_regression(s)
    for got, want in zip((fit.c1, fit.c2, fit.c3), truth):
        assert abs(got - want) <= 1e-9 * abs(want)
    assert fit.train_r2 == pytest.approx(1.0, abs=1e-9)
    noisy = _synth_samples(truth, 0.05, 7, 67)
    fit = pm.fit_regression(noisy)
    assert fit.train_r2 >= 0.85
    r = ref.fit_regression(np.array([x.features for x in noisy]),
                           np.array([x.seconds for x in noisy]))
    np.testing.assert_allclose([fit.c1, fit.c2, fit.c3], r[:3], rtol=1e-8)
    assert fit.train_r2 == pytest.approx(r[3], rel=1e-10)
    split = pm.fit_with_split(noisy, 0.7, 11)
    assert split.test_r2 >= 0.7
    with pytest.raises(ContractError):
        pm.fit_regression(s[:2])
    flat = [pm.RegressionSample((1.0, 0.0, 2.0), 1.0)] * 5
    with pytest.raises(ContractError):
        pm.fit_regression(flat)


def test_files_round_trip(tmp_path):
    c = pm.PerfCoefficients(1e-3, 2e-10, -3e-10, 0.9, 0.01)
    p = tmp_path / "coeffs.json"
    pm.coefficients_to_json_file(c, p)
    assert pm.coefficients_from_json_file(p) == c
    (tmp_path / "m.json").write_text('{"g_node": 8, "beta_intra": 7.25e11}')
    m = pm.machine_from_json_file(tmp_path / "m.json")
    assert (m.g_node, m.beta_intra, m.beta_inter) == (8, 7.25e11, 25e9)
    with pytest.raises(pm.IoError) as e:
        pm.machine_from_json_file(tmp_path / "missing.json")
    assert e.value.code == "MissingFile"
    csv = tmp_path / "s.csv"
    csv.write_text("n,nnz,dims,gx,gy,gz,seconds\n2449029,126167053,100-256-256-47,2,2,2,0.0123\n")
    s = pm.samples_from_csv_file(csv)
    assert s[0].features == pm.comp_features(PRODUCTS, (2, 2, 2)) and s[0].seconds == 0.0123
    csv.write_text("bad header\n")
    with pytest.raises(pm.IoError):
        pm.samples_from_csv_file(csv)

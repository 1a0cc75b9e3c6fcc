"""Pins for the oracle's weighted fitness metrics. CPU only."""
import math

import numpy as np
import pytest

import synth


def F(orc, metric, yh, y, w=None):
    return orc.fitness(metric, np.asarray(yh, float), np.asarray(y, np.float32),
                       None if w is None else np.asarray(w, np.float32))[0]


def test_spec_examples(orc):
    assert F(orc, "mae", [3.0], [2.0]) == 1.0
    assert F(orc, "logloss", [0.0], [1.0]) == pytest.approx(math.log(2), rel=1e-15)
    assert F(orc, "mse", [4.0], [1.0]) == 9.0
    assert F(orc, "mae", [1.0, 3.0], [1.0, 2.0], [1, 1]) == 0.5
    y = np.array([0.3, -1.2, 2.5, 4.0])
    assert F(orc, "pearson", y, y, [1, 2, 0.5, 3]) == pytest.approx(1.0, abs=1e-15)
    assert F(orc, "rmse", [3.0, 4.0], [0.0, 0.0], [1, 1]) == pytest.approx(math.sqrt(12.5),
                                                                           rel=1e-15)


def test_pagie_closed_forms(orc):
    """Values computed in double from the grid (SURVEY row C "Metrics on Pagie grids")."""
    X, y = synth.pagie_grid(2)
    v = X[0].astype(float)
    assert np.allclose(y, 1.996805111821086)
    assert F(orc, "mse", v, y) == pytest.approx(28.987230654594818, rel=1e-6)  # fp32 target
    assert F(orc, "mae", v, y) == pytest.approx(5.0, rel=1e-6)
    X, y = synth.pagie_grid(64)
    x0 = X[0].astype(float)
    assert F(orc, "mse", x0, y) == pytest.approx(11.275708036362, rel=1e-7)
    assert F(orc, "mae", x0, y) == pytest.approx(2.671017724475, rel=1e-7)
    assert F(orc, "rmse", x0, y) == pytest.approx(3.357932107170, rel=1e-7)
    assert F(orc, "mse", np.full(4096, 0.5), y) == pytest.approx(1.364170312804, rel=1e-7)
    assert abs(F(orc, "pearson", x0, y)) < 1e-12          # target even in x, grid symmetric
    assert F(orc, "pearson", x0 * x0, y) == pytest.approx(0.457215701338, rel=1e-7)


def test_identities(orc):
    rng = np.random.default_rng(0)
    for trial in range(50):
        n = int(rng.integers(2, 300))
        y = rng.normal(size=n).astype(np.float32)
        yh = rng.normal(size=n) * 3 + 1
        w = synth.weights(n, seed=trial)
        w[0] = 1.0
        mse = F(orc, "mse", yh, y, w)
        assert F(orc, "rmse", yh, y, w) ** 2 == pytest.approx(mse, rel=1e-12)
        assert F(orc, "mae", yh, y, np.ones(n)) == pytest.approx(F(orc, "mae", yh, y), rel=1e-15)
        # weight scaling invariance; integer weights == duplicated rows (brute force)
        assert F(orc, "mse", yh, y, w * 4) == pytest.approx(mse, rel=1e-12)
        ki = rng.integers(0, 3, n).astype(np.float32)
        ki[0] = 1
        rep = np.repeat(np.arange(n), ki.astype(int))
        for m in ("mae", "mse", "logloss", "pearson"):
            yy = (y > 0).astype(np.float32) if m == "logloss" else y
            a = F(orc, m, yh, yy, ki)
            b = F(orc, m, yh[rep], yy[rep])
            assert a == pytest.approx(b, rel=1e-10, abs=1e-12)
        r = F(orc, "pearson", yh, y, w)
        assert -1.0 <= r <= 1.0
        a, b = rng.normal(), rng.normal()
        ys = y.astype(float)
        assert F(orc, "pearson", a * ys + b, y, w) == pytest.approx(np.sign(a), abs=1e-9)
        lab = (rng.random(n) < 0.5).astype(np.float32)
        assert F(orc, "logloss", np.zeros(n), lab, w) == pytest.approx(math.log(2), rel=1e-12)


def test_textbook_special_cases(orc):
    """Unweighted cases reduce to library routines (numpy / scikit-learn)."""
    from sklearn.metrics import log_loss, mean_absolute_error, mean_squared_error
    rng = np.random.default_rng(1)
    n = 1000
    y = rng.normal(size=n).astype(np.float32)
    yh = rng.normal(size=n)
    w = rng.uniform(0.1, 2, n).astype(np.float32)
    assert F(orc, "mse", yh, y) == pytest.approx(mean_squared_error(y, yh), rel=1e-12)
    assert F(orc, "mae", yh, y, w) == pytest.approx(
        mean_absolute_error(y, yh, sample_weight=w), rel=1e-12)
    assert F(orc, "pearson", yh, y) == pytest.approx(np.corrcoef(yh, y)[0, 1], rel=1e-10)
    lab = (rng.random(n) < 0.4).astype(np.float32)
    p = 1 / (1 + np.exp(-yh))
    assert F(orc, "logloss", yh, lab, w) == pytest.approx(
        log_loss(lab, p, sample_weight=w), rel=1e-10)


def test_zero_weight_rows_skipped(orc):
    # DESIGN.md C5: a w = 0 row contributes exactly nothing, even when its loss is inf/nan.
    y = np.array([1, 2, 3], np.float32)
    yh = np.array([1.5, np.inf, 2.0])
    assert F(orc, "mse", yh, y, [1, 0, 1]) == pytest.approx((0.25 + 1) / 2)
    assert F(orc, "mse", yh, y) == math.inf                                       # reading C4


def test_pearson_undefined(orc):
    y = np.array([1, 2, 3], np.float32)
    f, und = orc.fitness("pearson", np.array([2.0, 2.0, 2.0]), y)
    assert f == 0.0 and und                                                        # S:202, C4


def test_logloss_clamp(orc):
    # S:191 clamp: p in [1e-15, 1 - 1e-15] -> per-row loss <= -ln(1e-15)
    assert F(orc, "logloss", [-1e4], [1.0]) == pytest.approx(-math.log(1e-15), rel=1e-12)
    assert F(orc, "logloss", [1e4], [1.0]) == pytest.approx(-math.log1p(-1e-15), rel=1e-6)


# ---- Spearman -------------------------------------------
def test_rank_vector_spec_examples(orc):
    assert orc.rank_vector([10, 30, 20]).tolist() == [1, 3, 2]
    assert orc.rank_vector([5, 5]).tolist() == [1.5, 1.5]
    assert orc.rank_vector([2, 1, 2, 3]).tolist() == [2.5, 1, 2.5, 4]


def test_rank_vector_matches_scipy(orc):
    from scipy.stats import rankdata
    rng = np.random.default_rng(3)
    for n in (1, 2, 7, 100, 1000):
        v = rng.integers(-5, 6, n).astype(np.float64)                   # many ties
        assert np.array_equal(orc.rank_vector(v), rankdata(v, method="average"))
        u = rng.standard_normal(n)
        assert np.array_equal(orc.rank_vector(u), rankdata(u, method="average"))


def test_spearman_matches_scipy_unweighted(orc):
    from scipy.stats import spearmanr
    rng = np.random.default_rng(4)
    for n in (5, 50, 2000):
        y = rng.integers(0, 20, n).astype(np.float32)
        yh = (rng.integers(0, 30, n) + 0.5 * y).astype(np.float64)      # fp32-exact, with ties
        f, und = orc.fitness("spearman", yh, y)
        assert not und
        assert abs(f - spearmanr(yh, y).statistic) <= 1e-12


def test_spearman_weighted_is_pearson_of_ranks(orc):
    """S:219 identity with weights, against numpy's weighted covariance on scipy ranks."""
    from scipy.stats import rankdata
    rng = np.random.default_rng(5)
    n = 777
    y = rng.standard_normal(n).astype(np.float32)
    yh = np.round(rng.standard_normal(n) * 8).astype(np.float64)
    w = synth.weights(n, seed=2)
    c = np.cov(rankdata(yh), rankdata(y), aweights=w)
    ref = c[0, 1] / math.sqrt(c[0, 0] * c[1, 1])
    f, und = orc.fitness("spearman", yh, y, w)
    assert not und and abs(f - ref) <= 1e-12


def test_spearman_monotone_invariance_and_special_cases(orc):
    rng = np.random.default_rng(6)
    y = rng.integers(0, 50, 500).astype(np.float32)
    yh = rng.integers(-20, 20, 500).astype(np.float64)
    f0, _ = orc.fitness("spearman", yh, y)
    for g in (lambda v: 3 * v + 1, lambda v: v ** 3, lambda v: np.exp(v / 8)):
        assert orc.fitness("spearman", g(yh), y)[0] == pytest.approx(f0, abs=1e-12)
    assert orc.fitness("spearman", y.astype(np.float64), y)[0] == pytest.approx(1.0, abs=1e-12)
    assert orc.fitness("spearman", -y.astype(np.float64), y)[0] == pytest.approx(-1.0, abs=1e-12)
    assert orc.fitness("spearman", np.full(500, 2.0), y) == (0.0, True)          # constant
    bad = yh.copy()
    bad[3] = np.nan
    assert orc.fitness("spearman", bad, y) == (0.0, True)                         # non-finite

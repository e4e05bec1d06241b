"""Pins for oracle O8 (particle reweighting, §Approach) -- CPU only."""
import math

import numpy as np
import pytest

from _golden import spec_value


def _two():
    return (np.array([[0.0, 1.0]], np.float32), np.array([[0.0, 0.0]], np.float32),
            np.array([[0.5, 0.5]], np.float32))


def test_spec_examples(orc):
    x, y, w = _two()
    wo, lz, fl = orc.reweight(x, y, w, np.zeros((1, 2), np.float32), (1, 0, 1), np.array([1], np.int32))
    np.testing.assert_allclose(wo[0], spec_value("reweight_one_z"), rtol=1e-12)
    assert fl[0] == 0
    wo, lz, fl = orc.reweight(x, y, w, np.zeros((2, 2), np.float32), (1, 0, 1), np.array([1, 1], np.int32))
    np.testing.assert_allclose(wo[0], spec_value("reweight_two_z"), rtol=1e-12)
    # logZ is the log marginal likelihood: 0.5 N(0;0,I)^2 + 0.5 N(0;(1,0),I)^2
    ref = math.log(0.5 / (2 * math.pi) ** 2 * (1 + math.exp(-1.0)))
    assert lz[0] == pytest.approx(ref, rel=1e-12)


def test_empty_assignment_identity_and_theta_columns(orc):
    r = np.random.default_rng(2)
    T, P, M = 4, 32, 6
    x = r.normal(0, 1, (T, P)).astype(np.float32)
    y = r.normal(0, 1, (T, P)).astype(np.float32)
    w = r.dirichlet(np.ones(P), T).astype(np.float32)
    Z = r.normal(0, 1, (M, 2)).astype(np.float32)
    theta = np.array([0, 3, 3, 0, 9, 5], np.int32)       # col_offset 2: local j=0 -> col 3, j=2 -> col 5
    wo, lz, fl = orc.reweight(x, y, w, Z, (1, 0, 1), theta, col_offset=2)
    for j in (1, 3):                                      # cols 4, 6: no measurement
        np.testing.assert_array_equal(wo[j], w[j].astype(np.float64))
        assert lz[j] == pytest.approx(math.log(w[j].astype(np.float64).sum()), abs=1e-15)
    for j in (0, 2):
        assert wo[j].sum() == pytest.approx(1.0, abs=1e-13)
        assert not np.allclose(wo[j], w[j])
    assert np.all(fl == 0)


def test_scale_invariance(orc):
    r = np.random.default_rng(4)
    x = r.normal(0, 1, (1, 64)).astype(np.float32)
    y = r.normal(0, 1, (1, 64)).astype(np.float32)
    w = r.dirichlet(np.ones(64), 1).astype(np.float32)
    Z = np.array([[0.3, -0.2], [0.1, 0.4]], np.float32)
    th = np.array([1, 1], np.int32)
    base = orc.reweight(x, y, w, Z, (0.5, 0.1, 0.7), th)
    for c in (1e-30, 1e30):
        wc = (w.astype(np.float64) * c).astype(np.float32)
        out = orc.reweight(x, y, wc, Z, (0.5, 0.1, 0.7), th)
        np.testing.assert_allclose(out[0], base[0], rtol=1e-6)     # fp32 rounding of w*c
        assert out[1][0] - base[1][0] == pytest.approx(math.log(c), abs=1e-5)


def test_consistency_with_compat(orc):
    """|S_j| = 1  =>  exp(logZ_j) = L_ij = C[i,j] / P_D (O7 vs O8, different code paths)."""
    r = np.random.default_rng(6)
    T, P, M = 3, 50, 5
    x = r.normal(10, 1, (T, P)).astype(np.float32)
    y = r.normal(10, 1, (T, P)).astype(np.float32)
    w = r.dirichlet(np.ones(P), T).astype(np.float32)
    Z = r.normal(10, 1, (M, 2)).astype(np.float32)
    R = (0.9, -0.2, 1.1)
    cm = orc.compat(x, y, w, Z, R, 0.9, 1e-3, 1e-30)
    theta = np.array([2, 0, 1, 0, 3], np.int32)
    wo, lz, fl = orc.reweight(x, y, w, Z, R, theta)
    for i, j in [(2, 0), (0, 1), (4, 2)]:
        assert math.exp(lz[j]) == pytest.approx(cm["L"][j, i], rel=1e-12)


def test_degenerate_all_zero_weights(orc):
    x, y, _ = _two()
    w = np.zeros((1, 2), np.float32)
    wo, lz, fl = orc.reweight(x, y, w, np.zeros((1, 2), np.float32), (1, 0, 1), np.array([1], np.int32))
    np.testing.assert_array_equal(wo[0], [0.5, 0.5])
    assert fl[0] == 1 and lz[0] == -np.inf


def test_far_measurement_is_range_safe(orc):
    x, y, w = _two()
    Z = np.array([[1e4, 0.0]], np.float32)                  # exp(-q/2) underflows fp64
    wo, lz, fl = orc.reweight(x, y, w, Z, (1, 0, 1), np.array([1], np.int32))
    assert fl[0] == 0 and wo[0].sum() == pytest.approx(1.0)
    assert wo[0, 1] > 0.999                                   # the nearer particle takes the mass


def test_kalman_cross_check(orc):
    """Prior cloud ~ N(mu, S) (position block), H = [I 0], one z:  the reweighted
    weighted mean/cov equal the Kalman update within Monte-Carlo error."""
    P = 200_000
    r = np.random.default_rng(8)
    mu = np.array([3.0, -1.0])
    S = np.array([[2.0, 0.6], [0.6, 1.0]])
    Rm = np.array([[0.8, -0.1], [-0.1, 0.5]])
    pts = r.multivariate_normal(mu, S, P).astype(np.float32)
    x, y = pts[None, :, 0], pts[None, :, 1]
    w = np.full((1, P), 1.0 / P, np.float32)
    z = np.array([[4.0, 0.0]], np.float32)
    wo, lz, fl = orc.reweight(x, y, w, z, (0.8, -0.1, 0.5), np.array([1], np.int32))
    K = S @ np.linalg.inv(S + Rm)
    m_kf = mu + K @ (z[0].astype(np.float64) - mu)
    S_kf = (np.eye(2) - K) @ S
    p64 = pts.astype(np.float64)
    m = (wo[0, :, None] * p64).sum(0)
    d = p64 - m
    cov = (wo[0, :, None, None] * d[:, :, None] * d[:, None, :]).sum(0)
    ess = 1.0 / (wo[0] ** 2).sum()
    se = np.sqrt(np.diag(S_kf) / ess)
    np.testing.assert_array_less(np.abs(m - m_kf), 5 * se)
    np.testing.assert_allclose(cov, S_kf, atol=5 * np.sqrt(2.0 / ess) * S_kf.max())
    # marginal likelihood: N(z; mu, S + R)
    from scipy.stats import multivariate_normal
    ref = multivariate_normal(mu, S + Rm).logpdf(z[0].astype(np.float64))
    assert lz[0] == pytest.approx(ref, abs=5 / math.sqrt(ess))

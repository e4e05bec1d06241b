"""Pins for the particle-loop oracle (O14-O16; §Approach) -- CPU only.

O14 (unique pairs) against a hand-worked example and a brute-force set
construction; O15 (per-pair update) against the independently pinned O8 and
closed-form ESS values; O16 (systematic resampling) against the defining
property of systematic resampling (each particle gets floor or ceil of its
expected count P w_m), the ESS threshold in closed form, and Monte-Carlo
unbiasedness over the uniform.
"""
import math

import numpy as np
import pytest

from _golden import spec_value


# ------------------------------------------------------------------ O14
def test_pairs_hand_example(orc):
    # hyp A: alive {0, 1}, theta = [1, 0, 2, 1] -> (0, {0, 3}), (1, {2})
    # hyp B: alive {0, 1, 2}, theta = [1, 0, 0, 1] -> (0, {0, 3}) again, (1, {}), (2, {})
    alive = np.array([[0b011], [0b111]], np.uint32)
    theta = np.array([[1, 0, 2, 1], [1, 0, 0, 1]], np.int32)
    pt, pp, pm, po = orc.assoc_pairs([0, 1], alive, theta, 3, 4)
    np.testing.assert_array_equal(pt, [0, 1, 1, 2])
    np.testing.assert_array_equal(pp, [0, 2, 3, 3, 3])
    np.testing.assert_array_equal(pm, [0, 3, 2])
    np.testing.assert_array_equal(po, [[0, 1, -1], [0, 2, 3]])
    # the scan order is the given hypothesis order
    pt, pp, pm, po = orc.assoc_pairs([1, 0], alive, theta, 3, 4)
    np.testing.assert_array_equal(pt, [0, 1, 2, 1])
    np.testing.assert_array_equal(po, [[0, 1, 2], [0, 3, -1]])


def test_pairs_brute_force(orc):
    rng = np.random.default_rng(4)
    T, M, n = 23, 40, 60
    alive = rng.integers(0, 2**23, (n, 1), dtype=np.uint64).astype(np.uint32)
    theta = np.zeros((n, M), np.int32)
    for q in range(n):
        al = [j for j in range(T) if (alive[q, 0] >> j) & 1]
        for i in range(M):       # few distinct sets: draw from a small menu so pairs repeat
            theta[q, i] = 0 if (rng.random() < 0.5 or not al) else 1 + al[(i * 7 + q % 3) % len(al)]
    order = rng.permutation(n)
    pt, pp, pm, po = orc.assoc_pairs(order, alive, theta, T, M)
    seen = {}
    for r, q in enumerate(order):
        for j in range(T):
            if not (alive[q, 0] >> j) & 1:
                assert po[r, j] == -1
                continue
            S = tuple(int(i) for i in np.nonzero(theta[q] == j + 1)[0])
            k = po[r, j]
            assert pt[k] == j and tuple(pm[pp[k]:pp[k + 1]]) == S
            if (j, S) not in seen:
                assert k == len(seen)                      # numbered on first occurrence
                seen[(j, S)] = k
            assert seen[(j, S)] == k
    assert len(pt) == len(seen)


# ------------------------------------------------------------------ O15
def test_reweight_pairs_equals_O8(orc):
    """One pair per track with S_j = {i : theta_i = j + 1} reproduces O8."""
    from paper_2512_06230_b200 import scenes
    x, y, v, psi, om, w = scenes.random_cloud(6, 64, 3, center_scale=20.0, spread=2.0, dirichlet=True)
    rng = np.random.default_rng(3)
    Z = (rng.uniform(0, 20, (15, 2))).astype(np.float32)
    theta = rng.integers(0, 7, 15).astype(np.int32)
    R = (1.3, 0.2, 0.9)
    w8, lz8, fl8 = orc.reweight(x, y, w, Z, R, theta)
    pt = np.arange(6, dtype=np.int32)
    sets = [np.nonzero(theta == j + 1)[0] for j in range(6)]
    pp = np.concatenate([[0], np.cumsum([len(s) for s in sets])]).astype(np.int32)
    pm = np.concatenate(sets).astype(np.int32)
    wo, lz, fl, ess = orc.reweight_pairs(x, y, w, Z, R, pt, pp, pm)
    np.testing.assert_allclose(wo, w8, rtol=1e-13, atol=1e-300)
    np.testing.assert_allclose(lz, lz8, rtol=1e-13)
    np.testing.assert_array_equal(fl, fl8)
    np.testing.assert_allclose(ess, wo.sum(1) ** 2 / (wo ** 2).sum(1), rtol=1e-12)


def test_reweight_pairs_closed_forms(orc):
    P = 8
    x = np.zeros((2, P), np.float32)
    y = np.zeros((2, P), np.float32)
    w = np.full((2, P), 1.0 / P, np.float32)
    w[1] = 0
    w[1, 3] = 1.0
    # empty sets: weights copied; ESS = P for uniform, 1 for a single particle
    wo, lz, fl, ess = orc.reweight_pairs(x, y, w, np.zeros((0, 2)), (1, 0, 1), [0, 1], [0, 0, 0], [])
    assert ess[0] == pytest.approx(P, rel=1e-14) and ess[1] == pytest.approx(1.0, rel=1e-14)
    np.testing.assert_array_equal(wo, w.astype(np.float64))
    # two particles at (0,0) and (1,0), sigma = 1, z = (0, 0) -> {0.6224593, 0.3775407}
    x2 = np.array([[0.0, 1.0, 0.0, 0.0]], np.float32)
    y2 = np.zeros((1, 4), np.float32)
    w2 = np.array([[0.5, 0.5, 0.0, 0.0]], np.float32)
    wo, lz, fl, ess = orc.reweight_pairs(x2, y2, w2, np.array([[0.0, 0.0]]), (1, 0, 1), [0], [0, 1], [0])
    np.testing.assert_allclose(wo[0, :2], spec_value("reweight_one_z"), rtol=1e-7)
    a, b = spec_value("reweight_one_z")
    assert ess[0] == pytest.approx(1.0 / (a * a + b * b), rel=1e-7)


# ------------------------------------------------------------------ O16
def _counts(anc, P):
    return np.bincount(anc, minlength=P)


def test_resample_floor_ceil_property(orc):
    """Systematic resampling: every particle gets floor or ceil of P W_m / S copies,
    the ancestors are non-decreasing and cover P slots."""
    rng = np.random.default_rng(0)
    for trial in range(200):
        P = int(rng.choice([4, 12, 64, 1000, 4096]))
        w = rng.dirichlet(np.full(P, 0.05 if trial % 2 else 0.5)).astype(np.float32)
        res, anc = orc.resample(w, 11, 3, trial)
        W = np.floor(w.astype(np.float64) * 2.0 ** 26)
        S, Q = W.sum(), (W * W).sum()
        assert res == (S > 0 and 2 * S * S < P * Q)
        if not res:
            continue
        N = _counts(anc, P)
        e = P * W / S
        assert N.sum() == P
        assert np.all(N >= np.floor(e) - 0) and np.all(N <= np.ceil(e))
        assert np.all(np.diff(anc) >= 0)
        assert np.all(N[W == 0] == 0)


def test_resample_decision_closed_forms(orc):
    a = np.float32(0.25)
    assert orc.resample(np.full(64, 1 / 64, np.float32), 0, 0, 0)[0] is False      # ESS = P
    res, anc = orc.resample(np.array([0, 0, 1, 0], np.float32), 0, 0, 0)           # ESS = 1
    assert res and np.all(anc == 2)
    assert orc.resample(np.array([a, a, 0, 0], np.float32), 0, 0, 0)[0] is False   # ESS = P/2 exactly: no
    assert orc.resample(np.array([a, a, a, 0], np.float32), 0, 0, 0)[0] is False
    assert orc.resample(np.array([a, 0, 0, 0], np.float32), 0, 0, 0)[0] is True
    assert orc.resample(np.zeros(8, np.float32), 0, 0, 0)[0] is False              # S = 0: nothing to draw


def test_resample_unbiased(orc):
    """E[N_m] = P W_m / S over the uniform (different k -> different Philox draws)."""
    P = 16
    rng = np.random.default_rng(5)
    w = rng.dirichlet(np.full(P, 0.3)).astype(np.float32)
    W = np.floor(w.astype(np.float64) * 2.0 ** 26)
    e = P * W / W.sum()
    n = 4000
    tot = np.zeros(P)
    for k in range(n):
        res, anc = orc.resample(w, 99, 1, k)
        assert res
        tot += _counts(anc, P)
    frac = e - np.floor(e)
    se = np.sqrt(np.maximum(frac * (1 - frac), 1e-12) / n)
    assert np.all(np.abs(tot / n - e) <= 5 * se + 1e-12)


def test_resample_keying(orc):
    """The uniform is O3 of word 0 of Philox(counter (k, 0, step, 4<<24)): shifting it by the
    documented grid reproduces the ancestors (O1 pinned by test_oracle_philox)."""
    P = 4
    w = np.array([0.7, 0.1, 0.1, 0.1], np.float32)
    W = np.floor(w.astype(np.float64) * 2.0 ** 26).astype(np.int64)
    S = int(W.sum())
    for k in range(20):
        r = int(orc.philox(5, np.array([[k, 0, 9, 4 << 24]], np.uint32))[0, 0])
        u = orc.uniform_u32(r)                                 # = U 2^-24
        res, anc = orc.resample(w, 5, 9, k)
        assert res
        cum = np.cumsum(W)
        for n in range(P):
            t = math.floor((n + u) / P * S)
            assert anc[n] == int(np.searchsorted(cum, t, side="right")) or \
                abs((n + u) / P * S - round((n + u) / P * S)) < 1e-6   # grid point within rounding of a boundary

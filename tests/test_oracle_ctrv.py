"""Pins for oracle O5 (CTRV predict) and O6 (birth) -- CPU only.

The CTRV flow is pinned against an independent numerical integration of the
CTRV ODE (x' = v cos psi, y' = v sin psi, psi' = omega, v' = omega' = 0), the
SPEC closed forms, the semigroup property and the turn-centre invariant."""
import math

import numpy as np
import pytest
from scipy.integrate import solve_ivp

from _golden import spec_value

PI = math.pi


def _ode(state, dt):
    def f(t, s):
        return [s[2] * math.cos(s[3]), s[2] * math.sin(s[3]), 0.0, s[4], 0.0]
    sol = solve_ivp(f, (0, dt), list(state), rtol=1e-12, atol=1e-12, method="DOP853")
    return sol.y[:, -1]


def _angdiff(a, b):
    return (a - b + PI) % (2 * PI) - PI


def test_identity_straight_line_half_circle(orc):
    np.testing.assert_allclose(orc.ctrv([0, 0, 0, 0, 0], 0.1), [0, 0, 0, 0, 0], atol=0)
    np.testing.assert_allclose(orc.ctrv([0, 0, 1, 0, 0], 0.1), [0.1, 0, 1, 0, 0], atol=1e-15)
    hc = spec_value("half_circle_dt1")
    out = orc.ctrv([0, 0, 1, 0, PI], 1.0)
    np.testing.assert_allclose(out, hc, atol=1e-12)


@pytest.mark.parametrize("om", [0.7, -1.3, 1e-3, -2e-4, 5e-5, 0.0, -3e-6, 2.5])
def test_matches_ode_integration(orc, om):
    r = np.random.default_rng(int(abs(om) * 1e6) + 1)
    for _ in range(5):
        s = [r.uniform(-500, 500), r.uniform(-500, 500), r.uniform(0, 25), r.uniform(-PI, PI), om]
        for dt in (0.1, 1.0):
            out = orc.ctrv(s, dt)
            ref = _ode(s, dt)
            np.testing.assert_allclose(out[[0, 1, 2, 4]], ref[[0, 1, 2, 4]], atol=1e-8)
            assert abs(_angdiff(out[3], ref[3])) < 1e-10


def test_branch_continuity(orc):
    s = np.array([10.0, -3.0, 20.0, 0.7, 0.0])
    for th in (1e-4, -1e-4):
        a = s.copy(); a[4] = th * (1 + 1e-9)
        b = s.copy(); b[4] = th * (1 - 1e-9)
        np.testing.assert_allclose(orc.ctrv(a, 0.1), orc.ctrv(b, 0.1), atol=1e-9)


def test_semigroup_and_invariants(orc):
    r = np.random.default_rng(5)
    for _ in range(50):
        s = np.array([r.uniform(-100, 100), r.uniform(-100, 100), r.uniform(0, 30),
                      r.uniform(-PI, PI), r.normal(0, 1)])
        dt = 0.1
        one = orc.ctrv(s, dt)
        two = orc.ctrv(orc.ctrv(s, dt / 2), dt / 2)
        np.testing.assert_allclose(one[[0, 1, 2, 4]], two[[0, 1, 2, 4]], atol=1e-12)
        assert abs(_angdiff(one[3], two[3])) < 1e-12
        assert one[2] == s[2]                                          # speed preserved
        assert abs(_angdiff(one[3], s[3] + s[4] * dt)) < 1e-14         # heading += omega dt
        if abs(s[4]) > 1e-3:                                           # turn centre fixed
            c0 = (s[0] - s[2] / s[4] * math.sin(s[3]), s[1] + s[2] / s[4] * math.cos(s[3]))
            c1 = (one[0] - one[2] / one[4] * math.sin(one[3]),
                  one[1] + one[2] / one[4] * math.cos(one[3]))
            np.testing.assert_allclose(c0, c1, atol=1e-9)


def test_noise_enters_linearly(orc):
    s = np.array([1.0, 2.0, 10.0, 0.4, 0.2])
    dt, na, nw = 0.1, 1.7, -0.3
    d = orc.ctrv(s, dt, na, nw) - orc.ctrv(s, dt)
    exp = [0.5 * dt * dt * math.cos(0.4) * na, 0.5 * dt * dt * math.sin(0.4) * na,
           dt * na, 0.5 * dt * dt * nw, dt * nw]
    np.testing.assert_allclose(d, exp, atol=1e-13)


def test_wrap(orc):
    assert orc.wrap(PI) == PI
    assert abs(orc.wrap(-PI) - PI) < 1e-15
    assert abs(orc.wrap(3 * PI) - PI) < 1e-12
    r = np.random.default_rng(1)
    for a in r.uniform(-50, 50, 1000):
        w = orc.wrap(a)
        assert -PI < w <= PI
        k = (a - w) / (2 * PI)
        assert abs(k - round(k)) < 1e-12


def test_predict_uses_keyed_philox_noise(orc):
    """predict(j,p) == ctrv(state, dt, sigma_a n_a, sigma_w n_w) with (n_a, n_w) = normals (0,1)
    (p even) or (2,3) (p odd) of the block with counter (p // 2, gid, step, 0)."""
    T, P = 3, 8
    r = np.random.default_rng(0)
    st = [r.uniform(0, 50, (T, P)).astype(np.float32) for _ in range(2)] + [
        r.uniform(0, 20, (T, P)).astype(np.float32), r.uniform(-3, 3, (T, P)).astype(np.float32),
        r.normal(0, 0.3, (T, P)).astype(np.float32)]
    gid = np.array([5, 900, 17], np.int32)
    out = orc.predict(*st, gid, 0.1, 1.0, 0.1, seed=99, step=4)
    for j in range(T):
        for p in range(P):
            n = orc.normals4(99, [p // 2, gid[j], 4, 0])
            na, nw = (n[0], n[1]) if p % 2 == 0 else (n[2], n[3])
            s = [float(a[j, p]) for a in st]
            ref = orc.ctrv(s, float(np.float32(0.1)), float(np.float32(1.0)) * na,
                           float(np.float32(0.1)) * nw)
            np.testing.assert_array_equal([o[j, p] for o in out], ref)


def test_predict_monte_carlo_moments(orc):
    P = 20000
    st = [np.full((1, P), v, np.float32) for v in (0.0, 0.0, 10.0, 0.0, 0.0)]
    dt, sa, sw = 0.1, 1.0, 0.1
    out = orc.predict(*st, np.array([3], np.int32), dt, sa, sw, seed=1, step=0)
    v = out[2][0]
    om = out[4][0]
    assert abs(v.mean() - 10.0) < 4 * dt * sa / math.sqrt(P)
    assert abs(v.std() - dt * sa) < 0.03 * dt * sa
    assert abs(om.std() - dt * sw) < 0.03 * dt * sw
    assert abs(out[0][0].mean() - 1.0) < 4 * 0.5 * dt * dt * sa / math.sqrt(P) + 1e-12


def test_birth_moments(orc):
    P = 100_000
    mean = np.array([[100.0, -50.0, 10.0, 0.5, 0.0]], np.float32)
    # a full lower triangle, so a packing/index mistake shows in the covariance
    Lm = np.array([[5, 0, 0, 0, 0], [1, 4, 0, 0, 0], [0.5, -0.5, 2, 0, 0],
                   [0.1, 0.0, 0.2, 0.6, 0], [0.0, 0.05, 0.0, 0.1, 0.2]], np.float64)
    chol = Lm[np.tril_indices(5)].astype(np.float32)[None, :]
    out = orc.birth(mean, chol, np.array([11], np.int32), P, seed=5, step=2)
    X = np.stack(out[:5], axis=-1)[0]                                  # [P,5]
    assert np.all(out[5] == 1.0 / P)
    assert np.all((X[:, 3] > -PI) & (X[:, 3] <= PI))
    Lf = chol[0].astype(np.float64)
    L64 = np.zeros((5, 5)); L64[np.tril_indices(5)] = Lf
    Sig = L64 @ L64.T
    m = X.mean(0)
    se = np.sqrt(np.diag(Sig) / P)
    np.testing.assert_array_less(np.abs(m - mean[0]), 5 * se)
    cov = np.cov(X.T)
    np.testing.assert_allclose(cov, Sig, atol=5 * np.sqrt(2.0 / P) * np.max(np.diag(Sig)))
    # ranks of different births / steps draw different particles
    out2 = orc.birth(mean, chol, np.array([12], np.int32), 16, seed=5, step=2)
    assert not np.array_equal(out2[0][0], out[0][0][:16])


def test_predict_keying_properties(orc):
    """R9's keying pinned by what it must guarantee, not by its formula (BJ north_star: noise
    "keyed by (seed, step, track, particle)"): the draws of a track follow its global id, not its
    row (rows permuted with their gids -> outputs permuted exactly; the same track alone in a
    one-row call -> the same output); a different step, seed or gid changes every particle's
    draw; the two particles sharing a Philox block (p = 2q, 2q + 1) get different noise; and the
    noise-free flow is recovered with sigma = 0."""
    T, P = 4, 16
    r = np.random.default_rng(5)
    st = [r.uniform(0, 50, (T, P)).astype(np.float32), r.uniform(0, 50, (T, P)).astype(np.float32),
          r.uniform(2, 20, (T, P)).astype(np.float32), r.uniform(-3, 3, (T, P)).astype(np.float32),
          r.normal(0, 0.3, (T, P)).astype(np.float32)]
    gid = np.array([11, 4, 700, 9], np.int32)
    base = orc.predict(*st, gid, 0.1, 1.0, 0.1, seed=3, step=2)
    perm = np.array([2, 0, 3, 1])
    swapped = orc.predict(*[a[perm] for a in st], gid[perm], 0.1, 1.0, 0.1, seed=3, step=2)
    for b, s_ in zip(base, swapped):
        np.testing.assert_array_equal(b[perm], s_)
    alone = orc.predict(*[a[2:3] for a in st], gid[2:3], 0.1, 1.0, 0.1, seed=3, step=2)
    for b, s_ in zip(base, alone):
        np.testing.assert_array_equal(b[2:3], s_)
    clean = orc.predict(*st, gid, 0.1, 0.0, 0.0, seed=3, step=2)
    dv = base[2] - clean[2]                                  # dt * nu_a: the drawn acceleration
    for kw in ({"seed": 4, "step": 2}, {"seed": 3, "step": 3}):
        other = orc.predict(*st, gid, 0.1, 1.0, 0.1, **kw)
        assert np.all(other[2] - clean[2] != dv)
    other = orc.predict(*st, gid + 1, 0.1, 1.0, 0.1, seed=3, step=2)
    assert np.all(other[2] - clean[2] != dv)
    assert np.all(dv[:, 0::2] != dv[:, 1::2])                # block-sharing particle pairs differ
    for j in range(T):                                       # clean = the noise-free CTRV flow
        s = [float(a[j, 5]) for a in st]
        np.testing.assert_allclose([c[j, 5] for c in clean[:2]], orc.ctrv(s, float(np.float32(0.1)))[:2],
                                   rtol=0, atol=1e-12)

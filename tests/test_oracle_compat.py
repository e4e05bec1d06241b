"""Pins for oracle O7 (likelihood, gate, C_k; §Approach) -- CPU only."""
import math

import numpy as np
import pytest
from scipy.stats import multivariate_normal

from _golden import spec_value


def _cloud(xs, ys, ws):
    a = lambda v: np.asarray([v], np.float32)
    return a(xs), a(ys), a(ws)


@pytest.mark.parametrize("R", [(1.0, 0.0, 1.0), (0.0625, 0.0, 0.0625), (2.0, 0.7, 0.5),
                               (0.3, -0.25, 1.4)])
def test_single_particle_equals_scipy_pdf(orc, R):
    r = np.random.default_rng(3)
    for _ in range(20):
        p = r.uniform(-100, 100, 2).astype(np.float32)
        z = (p + r.normal(0, 1.5, 2)).astype(np.float32)
        x, y, w = _cloud([p[0]], [p[1]], [1.0])
        out = orc.compat(x, y, w, z[None], R, 1.0, 0.0, 1e-30)
        cov = [[R[0], R[1]], [R[1], R[2]]]
        ref = multivariate_normal(mean=p.astype(np.float64), cov=np.float32(cov).astype(np.float64)).pdf(z.astype(np.float64))
        assert out["L"][0, 0] == pytest.approx(ref, rel=1e-12)


def test_spec_examples(orc):
    s = 0.0625
    x, y, w = _cloud([0.0], [0.0], [1.0])
    out = orc.compat(x, y, w, np.zeros((1, 2), np.float32), (s, 0, s), 0.9, 0.01, 1e-6)
    assert out["L"][0, 0] == pytest.approx(spec_value("single_particle_peak_sigma0.25")[0], rel=1e-12)
    row = spec_value("row_pd0.9_kappa0.01")
    assert out["C_clutter"][0] == pytest.approx(row[0], rel=1e-7)      # kappa is fp32 0.01
    assert out["C_tracks"][0, 0] == pytest.approx(row[1], rel=1e-7)    # P_D fp32 0.9
    x, y, w = _cloud([0.0, 1.0], [0.0, 0.0], [0.5, 0.5])
    out = orc.compat(x, y, w, np.zeros((1, 2), np.float32), (1, 0, 1), 1.0, 0.0, 1e-30)
    assert out["L"][0, 0] == pytest.approx(spec_value("two_particle_mixture_sigma1")[0], rel=1e-12)


def test_edge_cases(orc):
    Z = np.array([[1, 2], [3, 4], [5, 6]], np.float32)
    e = np.zeros((0, 8), np.float32)
    out = orc.compat(e, e, e, Z, (1, 0, 1), 0.9, np.float32(5e-5), 1e-6)
    assert out["C_tracks"].shape == (0, 3)
    np.testing.assert_array_equal(out["C_clutter"], np.float64(np.float32(5e-5)))
    x, y, w = _cloud([500.0], [500.0], [1.0])                          # all gated out
    out = orc.compat(x, y, w, Z, (1, 0, 1), 0.9, 0.01, 1e-6)
    assert np.all(out["C_tracks"] == 0) and np.all(out["gate"] == 0)
    out = orc.compat(x, y, w, np.zeros((0, 2), np.float32), (1, 0, 1), 0.9, 0.01, 1e-6)
    assert out["C_tracks"].shape == (1, 0) and out["gate"].shape == (1, 0)


@pytest.mark.parametrize("gamma", [1e-6, 1e-8])
def test_gate_radius_closed_form(orc, gamma):
    g32 = float(np.float32(gamma))
    d = math.sqrt(-2.0 * math.log(2 * math.pi * g32))                # L(d) = gamma, R = I
    x, y, w = _cloud([0.0], [0.0], [1.0])
    Z = np.array([[d - 1e-3, 0.0], [d + 1e-3, 0.0], [0.0, -(d - 1e-3)], [0.0, d + 1e-3]], np.float32)
    out = orc.compat(x, y, w, Z, (1, 0, 1), 0.9, 0.01, gamma)
    assert list(out["L"][0] >= g32) == [True, False, True, False]
    assert int(out["gate"][0, 0]) == 0b0101
    assert out["C_tracks"][0, 1] == 0.0 and out["C_tracks"][0, 0] > 0


def test_gate_bit_layout_and_C_relation(orc):
    r = np.random.default_rng(9)
    T, P, M = 3, 16, 77
    x = r.normal(50, 2, (T, P)).astype(np.float32)
    y = r.normal(50, 2, (T, P)).astype(np.float32)
    w = r.dirichlet(np.ones(P), T).astype(np.float32)
    Z = r.normal(50, 5, (M, 2)).astype(np.float32)
    out = orc.compat(x, y, w, Z, (1.5, 0.2, 0.8), 0.9, 1e-4, 1e-4)
    g = out["L"] >= np.float32(1e-4)
    assert 0 < g.sum() < g.size
    for j in range(T):
        for i in range(M):
            bit = (int(out["gate"][j, i // 32]) >> (i % 32)) & 1
            assert bit == int(g[j, i])
            assert out["C_tracks"][j, i] == (np.float64(np.float32(0.9)) * out["L"][j, i] if g[j, i] else 0.0)
    assert np.all(out["gate"][:, -1] >> (M % 32) == 0)                  # no bits past M


def test_brute_force_tiny(orc):
    """1 track x 2 particles x 2 measurements, each pdf from scipy, summed by hand."""
    x, y, w = _cloud([0.0, 1.0], [0.5, -0.5], [0.25, 0.75])
    Z = np.array([[0.2, 0.1], [1.5, -1.0]], np.float32)
    R = (0.5, 0.1, 0.8)
    out = orc.compat(x, y, w, Z, R, 0.8, 0.0, 1e-30)
    cov = np.array([[0.5, 0.1], [0.1, 0.8]], np.float32).astype(np.float64)
    for i in range(2):
        ref = sum(float(np.float32(wp)) * multivariate_normal([float(np.float32(px)), float(np.float32(py))], cov).pdf(Z[i].astype(np.float64))
                  for px, py, wp in [(0.0, 0.5, 0.25), (1.0, -0.5, 0.75)])
        assert out["L"][0, i] == pytest.approx(ref, rel=1e-12)


def test_permutation_and_rotation_invariance(orc):
    r = np.random.default_rng(11)
    T, P, M = 2, 64, 20
    x = r.normal(20, 1, (T, P)).astype(np.float32)
    y = r.normal(-5, 1, (T, P)).astype(np.float32)
    w = r.dirichlet(np.ones(P), T).astype(np.float32)
    Z = np.stack([r.normal(20, 2, M), r.normal(-5, 2, M)], 1).astype(np.float32)
    R = (1.2, 0.3, 0.7)
    base = orc.compat(x, y, w, Z, R, 0.9, 1e-3, 1e-9)
    perm = r.permutation(P)                                           # particle order
    o2 = orc.compat(x[:, perm], y[:, perm], w[:, perm], Z, R, 0.9, 1e-3, 1e-9)
    np.testing.assert_allclose(o2["L"], base["L"], rtol=1e-13)
    rp = r.permutation(M)                                             # detection order
    o3 = orc.compat(x, y, w, Z[rp], R, 0.9, 1e-3, 1e-9)
    np.testing.assert_array_equal(o3["L"], base["L"][:, rp])
    # joint rotation by 90 degrees (exact in fp32): (a,b) -> (-b,a), R -> Q R Q^T
    R90 = (R[2], -R[1], R[0])
    o4 = orc.compat(-y, x, w, np.stack([-Z[:, 1], Z[:, 0]], 1), R90, 0.9, 1e-3, 1e-9)
    np.testing.assert_allclose(o4["L"], base["L"], rtol=1e-12)


def test_likelihood_integrates_to_one(orc):
    x, y, w = _cloud([0.0, 1.0, -0.5], [0.0, 0.5, 1.0], [0.2, 0.3, 0.5])
    h = 0.05
    g = np.arange(-8, 9, h)
    gx, gy = np.meshgrid(g, g)
    Z = np.stack([gx.ravel(), gy.ravel()], 1).astype(np.float32)
    out = orc.compat(x, y, w, Z, (0.6, 0.2, 0.9), 1.0, 0.0, 1e-30)
    assert out["L"].sum() * h * h == pytest.approx(1.0, abs=1e-6)


def test_nearest_gate_theta_hand_example(orc):
    """BASELINE.json configs[2]'s nearest-gate map from the oracle's C_k (R22), worked by hand:
    3 tracks at x = 0, 3, 30 (one particle each, R = I, P_D = 1, gamma = 1e-6, gate radius
    4.894 m).  z0 = (1, 0): tracks 0 (d = 1) and 1 (d = 2) gated, the nearer one wins -> 1;
    z1 = (1.5, 0): equidistant from tracks 0 and 1, an exact tie -> the lower column, 1;
    z2 = (30, 4): only track 2 (d = 4) -> 3; z3 = (15, 0): nothing within the gate -> 0."""
    x, y, w = (np.asarray([[0.0], [3.0], [30.0]], np.float32), np.zeros((3, 1), np.float32),
               np.ones((3, 1), np.float32))
    Z = np.asarray([[1.0, 0.0], [1.5, 0.0], [30.0, 4.0], [15.0, 0.0]], np.float32)
    ref = orc.compat(x, y, w, Z, (1.0, 0.0, 1.0), 1.0, 1e-4, 1e-6)
    assert ref["C_tracks"][0, 1] == ref["C_tracks"][1, 1]           # the tie is exact
    np.testing.assert_array_equal(orc.nearest_gate_theta(ref), [1, 1, 3, 0])
    assert orc.nearest_gate_theta(orc.compat(x[:0], y[:0], w[:0], Z, (1, 0, 1), 1.0, 1e-4, 1e-6)).tolist() == [0] * 4

"""GPU parity: every stage of the CUDA path (through the C ABI) vs the fp64 oracle
on identical seeded fp32 inputs."""
import numpy as np
import pytest

from conftest import gpu_available
from _parity import (check_compat, check_log_norm, check_state, check_weights)

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA GPU")]


@pytest.fixture(scope="module")
def L():
    import torch
    from paper_2512_06230_b200 import _lib
    from paper_2512_06230_b200.build import build
    build()
    _lib.glmb_init(0)
    torch.cuda.set_device(0)
    return _lib


def _dev(a, dtype=None):
    import torch
    t = torch.as_tensor(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def _host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


# ------------------------------------------------------------------ Philox
def test_philox_bit_exact(L, orc):
    import torch
    r = np.random.default_rng(0)
    n = 200_000
    ctr = r.integers(0, 2**32, (n, 4), dtype=np.uint64).astype(np.uint32)
    # every counter configs 0-1 use in predict / birth
    p = np.arange(1024, dtype=np.uint32)
    for gid, tag in [(0, 0), (3, 0), (63, 0), (64, 0x100), (67, 0x101)]:
        blk = np.stack([p, np.full_like(p, gid), np.zeros_like(p), np.full_like(p, tag)], 1)
        ctr = np.concatenate([ctr, blk])
    ctr[:2] = [[0, 0, 0, 0], [0xFFFFFFFF] * 4]
    for seed in (0, 7, 0xFFFFFFFFFFFFFFFF, 0x123456789ABCDEF0):
        out = torch.empty(ctr.shape, dtype=torch.int32, device="cuda")
        L.glmb_philox_dump(seed, _dev(ctr.view(np.int32)), out)
        got = _host(out).view(np.uint32)
        np.testing.assert_array_equal(got, orc.philox(seed, ctr))


def test_box_muller_normals(L, orc):
    import torch
    n = 100_000
    ctr = np.zeros((n, 4), np.uint32)
    ctr[:, 0] = np.arange(n)
    ctr[:, 1] = 5
    out = torch.empty((n, 4), dtype=torch.float32, device="cuda")
    L.glmb_normals_dump(11, _dev(ctr.view(np.int32)), out)
    g = _host(out).astype(np.float64)
    ref = orc.normals_batch(11, ctr)
    assert np.abs(g - ref).max() < 1e-5


# ------------------------------------------------------------------ predict / birth
def _predict_gpu(L, arrs, gid, dt, sa, sw, seed, step):
    from paper_2512_06230_b200._lib import Particles
    T, P = arrs[0].shape
    w = np.full((T, P), 1.0 / P, np.float32)
    pin = Particles.from_arrays(list(arrs) + [w])
    pout = Particles.empty(T, P)
    L.glmb_predict(pin, pout, _dev(gid), dt, sa, sw, seed, step)
    res = _host(pout.data)
    # in place gives the same bits
    L.glmb_predict(pin, pin, _dev(gid), dt, sa, sw, seed, step)
    np.testing.assert_array_equal(_host(pin.data)[:5], res[:5])
    return res


@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_predict_parity_configs(L, orc, cfg):
    from paper_2512_06230_b200.scenes import make_scene
    s = make_scene(cfg, steps=1)
    c = s.cfg
    arrs = (s.x, s.y, s.v, s.psi, s.omega)
    g = _predict_gpu(L, arrs, s.gid, c.dt, c.sigma_a, c.sigma_w, c.seed, 3)
    ref = orc.predict(*arrs, s.gid, c.dt, c.sigma_a, c.sigma_w, c.seed, 3)
    check_state(g[:5], ref)


def test_predict_edge_kinematics(L, orc):
    """omega at and around 0 and the oracle's 1e-4 branch, large dt, headings near +-pi."""
    T, P = 2, 64
    r = np.random.default_rng(1)
    om = np.concatenate([np.array([0, 1e-7, -1e-7, 1e-5, -1e-5, 1e-4, -1e-4, 1.0001e-4, 3e-3, -0.5, 2.0, -4.0]),
                         r.normal(0, 1, T * P - 12)]).reshape(T, P).astype(np.float32)
    psi = r.uniform(-np.pi, np.pi, (T, P)).astype(np.float32)
    psi[0, :6] = [np.pi, -np.pi, 3.1415925, -3.1415925, 0.0, 1.5707964]
    arrs = (r.uniform(-3000, 3000, (T, P)).astype(np.float32), r.uniform(-3000, 3000, (T, P)).astype(np.float32),
            r.uniform(0, 30, (T, P)).astype(np.float32), psi, om)
    gid = np.array([0, 12345], np.int32)
    for dt in (0.1, 1.0):
        g = _predict_gpu(L, arrs, gid, dt, 2.0, 0.5, 99, 7)
        ref = orc.predict(*arrs, gid, dt, 2.0, 0.5, 99, 7)
        check_state(g[:5], ref)
        assert np.all((g[3] > -np.float32(np.pi)) & (g[3] <= np.float32(np.pi)))


def test_predict_noise_free_matches_flow(L, orc):
    from paper_2512_06230_b200.scenes import random_cloud
    x, y, v, psi, om, _ = random_cloud(3, 128, seed=4)
    g = _predict_gpu(L, (x, y, v, psi, om), np.arange(3, dtype=np.int32), 0.1, 0.0, 0.0, 1, 0)
    ref = orc.predict(x, y, v, psi, om, np.arange(3, dtype=np.int32), 0.1, 0.0, 0.0, 1, 0)
    check_state(g[:5], ref)
    np.testing.assert_array_equal(g[2], v)          # speed untouched without noise
    np.testing.assert_array_equal(g[4], om)


@pytest.mark.parametrize("cfg", [1, 3])
def test_birth_parity(L, orc, cfg):
    from paper_2512_06230_b200._lib import Particles
    from paper_2512_06230_b200.scenes import make_scene
    s = make_scene(cfg, rows=range(0), steps=1)
    B, P = s.birth_mean.shape[0], s.cfg.P
    out = Particles.empty(B, P)
    L.glmb_birth(out, _dev(s.birth_gid), _dev(s.birth_mean), _dev(s.birth_chol), s.cfg.seed, 2)
    g = _host(out.data)
    ref = orc.birth(s.birth_mean, s.birth_chol, s.birth_gid, P, s.cfg.seed, 2)
    check_state(g[:5], ref[:5])
    np.testing.assert_array_equal(g[5], np.float32(1.0 / P))


def test_birth_full_covariance(L, orc):
    from paper_2512_06230_b200._lib import Particles
    mean = np.array([[10, 20, 5, 3.1, 0.1], [-5, 0, 1, -3.1, 0]], np.float32)
    Lm = np.array([[2, 0, 0, 0, 0], [0.5, 1, 0, 0, 0], [0.1, 0.2, 0.3, 0, 0],
                   [0.0, 0.1, 0.0, 0.8, 0], [0.05, 0, 0.02, 0.01, 0.2]])
    chol = np.stack([Lm[np.tril_indices(5)]] * 2).astype(np.float32)
    gid = np.array([100, 101], np.int32)
    out = Particles.empty(2, 256)
    L.glmb_birth(out, _dev(gid), _dev(mean), _dev(chol), 3, 9)
    g = _host(out.data)
    ref = orc.birth(mean, chol, gid, 256, 3, 9)
    check_state(g[:5], ref[:5])


# ------------------------------------------------------------------ compat
def _compat_gpu(L, x, y, w, Z, R, p_d, kappa, gamma, ld=None, ldc=None, ldg=None):
    import torch
    from paper_2512_06230_b200._lib import Particles
    T, P = x.shape
    M = Z.shape[0]
    ld = P if ld is None else ld
    ldc = max(M, 1) if ldc is None else ldc
    ldg = max((M + 31) // 32, 1) if ldg is None else ldg
    data = np.zeros((6, T, ld), np.float32)
    data[0, :, :P], data[1, :, :P], data[5, :, :P] = x, y, w
    data[0, :, P:] = np.nan   # padding beyond P must never be read
    trk = Particles(_dev(data), P)
    C = torch.full((T, ldc), -7.0, dtype=torch.float32, device="cuda")
    G = torch.full((T, ldg), -1, dtype=torch.int32, device="cuda")
    Cc = torch.full((max(M, 1),), -7.0, dtype=torch.float32, device="cuda")
    Zd = _dev(Z.reshape(-1, 2).astype(np.float32)) if M else torch.zeros((0, 2), device="cuda")
    L.glmb_compat(trk, Zd, R, p_d, kappa, gamma, Cc, C, G)
    return _host(C), _host(G).view(np.uint32), _host(Cc)


@pytest.mark.parametrize("cfg", [0, 1])
def test_compat_parity_configs(L, orc, cfg):
    from paper_2512_06230_b200.scenes import make_scene
    s = make_scene(cfg, steps=1)
    c = s.cfg
    Z = s.Z[0]
    C, G, Cc = _compat_gpu(L, s.x, s.y, s.w, Z, c.R, c.p_d, c.kappa, c.gamma)
    ref = orc.compat(s.x, s.y, s.w, Z, c.R, c.p_d, c.kappa, c.gamma)
    nband, rel = check_compat(C, G, Cc, ref, c.gamma, len(Z))
    assert rel < 1e-5 and nband <= max(1, 1e-3 * (ref["L"] >= c.gamma).sum())
    assert (ref["L"] >= c.gamma).sum() > 0


def test_compat_parity_cfg2_sampled(L, orc):
    from paper_2512_06230_b200.scenes import make_scene
    s = make_scene(2, rows=range(40, 72), steps=1)
    c = s.cfg
    C, G, Cc = _compat_gpu(L, s.x, s.y, s.w, s.Z[0], c.R, c.p_d, c.kappa, c.gamma)
    ref = orc.compat(s.x, s.y, s.w, s.Z[0], c.R, c.p_d, c.kappa, c.gamma)
    check_compat(C, G, Cc, ref, c.gamma, len(s.Z[0]))


@pytest.mark.parametrize("T,P,M,ld", [(1, 4, 1, 4), (2, 260, 33, 264), (3, 1028, 129, 1028),
                                      (2, 516, 1025, 520), (1, 512, 2049, 512), (5, 8, 7, 12)])
def test_compat_ragged_shapes(L, orc, T, P, M, ld):
    r = np.random.default_rng(T * 1000 + M)
    cen = r.uniform(0, 50, (T, 2))
    x = (cen[:, :1] + r.normal(0, 2, (T, P))).astype(np.float32)
    y = (cen[:, 1:] + r.normal(0, 2, (T, P))).astype(np.float32)
    w = r.dirichlet(np.ones(P), T).astype(np.float32)
    Z = r.uniform(-5, 55, (M, 2)).astype(np.float32)
    R = (1.3, 0.4, 0.9)
    C, G, Cc = _compat_gpu(L, x, y, w, Z, R, 0.85, 3e-4, 1e-6, ld=ld, ldc=M + 5, ldg=(M + 31) // 32 + 2)
    ref = orc.compat(x, y, w, Z, R, 0.85, 3e-4, 1e-6)
    check_compat(C, G, Cc, ref, 1e-6, M)
    assert np.all(C[:, M:] == -7.0)                      # entries past M untouched
    assert np.all(G[:, (M + 31) // 32:] == 0xFFFFFFFF)   # words past ceil(M/32) untouched


def test_compat_large_coordinates_general_R(L, orc):
    """Tracks near 4 km (cfg4 scale) with a correlated R: whitening + centring keep 1e-4."""
    r = np.random.default_rng(5)
    T, P, M = 4, 1024, 300
    cen = r.uniform(3500, 4000, (T, 2))
    x = (cen[:, :1] + r.normal(0, 2, (T, P))).astype(np.float32)
    y = (cen[:, 1:] + r.normal(0, 2, (T, P))).astype(np.float32)
    w = np.full((T, P), 1.0 / P, np.float32)
    Z = (cen[r.integers(0, T, M)] + r.normal(0, 4, (M, 2))).astype(np.float32)
    R = (0.7, -0.3, 1.6)
    C, G, Cc = _compat_gpu(L, x, y, w, Z, R, 0.9, 6.25e-5, 1e-8)
    ref = orc.compat(x, y, w, Z, R, 0.9, 6.25e-5, 1e-8)
    nb, rel = check_compat(C, G, Cc, ref, 1e-8, M)
    assert (ref["L"] >= 1e-8).sum() > 50


def test_compat_edge_cases(L, orc):
    import torch
    from paper_2512_06230_b200._lib import Particles
    Z = np.array([[1, 2], [3, 4], [5, 6]], np.float32)
    # T = 0: clutter-only matrix
    trk = Particles.empty(0, 4)
    Cc = torch.full((3,), -1.0, device="cuda")
    L.glmb_compat(trk, _dev(Z), (1, 0, 1), 0.9, 5e-5, 1e-6, Cc, torch.empty((0, 3), device="cuda"),
                  torch.empty((0, 1), dtype=torch.int32, device="cuda"))
    np.testing.assert_array_equal(_host(Cc), np.float32(5e-5))
    # M = 0: no-op
    x = np.zeros((1, 4), np.float32)
    C, G, _ = _compat_gpu(L, x, x, x + 0.25, np.zeros((0, 2), np.float32), (1, 0, 1), 0.9, 1e-3, 1e-6)
    assert np.all(C == -7.0)
    # all gated out
    C, G, Cc = _compat_gpu(L, x + 500, x + 500, x + 0.25, Z, (1, 0, 1), 0.9, 1e-3, 1e-6)
    assert np.all(C[:, :3] == 0) and np.all(G[:, 0] == 0)
    # NaN particle -> L NaN -> g = 0, C = 0
    xn = x.copy(); xn[0, 0] = np.nan
    C, G, _ = _compat_gpu(L, xn, x, x + 0.25, np.zeros((1, 2), np.float32), (1, 0, 1), 0.9, 1e-3, 1e-6)
    assert C[0, 0] == 0 and G[0, 0] == 0
    # the gate radius closed form: single particle, R = I
    g = 1e-6
    d = np.sqrt(-2 * np.log(2 * np.pi * float(np.float32(g))))
    Zg = np.array([[d - 1e-3, 0], [d + 1e-3, 0]], np.float32)
    C, G, _ = _compat_gpu(L, x[:, :4] * 0, x[:, :4] * 0, np.array([[1, 0, 0, 0]], np.float32), Zg,
                          (1, 0, 1), 0.9, 1e-3, g)
    assert int(G[0, 0]) == 0b01


def test_compat_invariances(L, orc):
    """Row permutation of Z permutes C rows bit-exactly; splitting the tracks (sharding) is
    bit-identical; particle permutation changes C by fp32 reduction order only."""
    from paper_2512_06230_b200.scenes import make_scene
    s = make_scene(1, steps=1)
    c = s.cfg
    Z = s.Z[0]
    C, G, _ = _compat_gpu(L, s.x, s.y, s.w, Z, c.R, c.p_d, c.kappa, c.gamma)
    perm = np.random.default_rng(0).permutation(len(Z))
    C2, _, _ = _compat_gpu(L, s.x, s.y, s.w, Z[perm], c.R, c.p_d, c.kappa, c.gamma)
    np.testing.assert_array_equal(C2[:, :len(Z)], C[:, perm])
    for lo, hi in [(0, 17), (17, 40), (40, 64)]:
        Cs, Gs, _ = _compat_gpu(L, s.x[lo:hi], s.y[lo:hi], s.w[lo:hi], Z, c.R, c.p_d, c.kappa, c.gamma)
        np.testing.assert_array_equal(Cs, C[lo:hi])
        np.testing.assert_array_equal(Gs, G[lo:hi])
    pp = np.random.default_rng(1).permutation(s.cfg.P)
    pp = np.concatenate([[0], pp[pp != 0]])   # keep the centring particle first
    C3, _, _ = _compat_gpu(L, s.x[:, pp], s.y[:, pp], s.w[:, pp], Z, c.R, c.p_d, c.kappa, c.gamma)
    nz = C != 0
    np.testing.assert_allclose(C3[nz], C[nz], rtol=1e-5)


# ------------------------------------------------------------------ reweight
def _reweight_gpu(L, x, y, w, Z, R, theta, col_offset=0):
    import torch
    from paper_2512_06230_b200._lib import Particles
    T, P = x.shape
    data = np.zeros((6, T, P), np.float32)
    data[0], data[1], data[5] = x, y, w
    trk = Particles(_dev(data), P)
    ln = torch.zeros(T, device="cuda")
    fl = torch.full((T,), -1, dtype=torch.int32, device="cuda")
    Zd = _dev(Z.reshape(-1, 2).astype(np.float32))
    L.glmb_reweight(trk, Zd, R, _dev(theta.astype(np.int32)), col_offset, ln, fl)
    return _host(trk.data)[5], _host(ln), _host(fl)


@pytest.mark.parametrize("cfg", [0, 1])
def test_reweight_parity_configs(L, orc, cfg):
    from paper_2512_06230_b200.scenes import make_scene
    s = make_scene(cfg, steps=1)
    c = s.cfg
    w, ln, fl = _reweight_gpu(L, s.x, s.y, s.w, s.Z[0], c.R, s.theta[0])
    rw, rln, rfl = orc.reweight(s.x, s.y, s.w, s.Z[0], c.R, s.theta[0])
    check_weights(w, rw)
    check_log_norm(ln, rln)
    np.testing.assert_array_equal(fl.view(np.uint32), rfl)


@pytest.mark.parametrize("P", [4, 1024, 4096, 8192, 12288, 16384])
def test_reweight_paths_and_multi_detection(L, orc, P):
    """Shared-memory-cached path (P <= 12800) and the recompute path (P = 16384); several
    detections per track (P:46-48 multiple detections per object), a far-away
    measurement, an empty track, theta values out of range and a column offset."""
    r = np.random.default_rng(P)
    T = 5
    x = r.normal(100, 1.5, (T, P)).astype(np.float32)
    y = r.normal(-40, 1.5, (T, P)).astype(np.float32)
    w = r.dirichlet(np.ones(P), T).astype(np.float32)
    Z = np.array([[100.5, -40], [99, -41], [101, -39.5], [130, -40], [100, -40.2], [0, 0]], np.float32)
    # col_offset 10: local j -> column 11 + j
    theta = np.array([11, 11, 11, 12, 14, 99], np.int32)
    wg, ln, fl = _reweight_gpu(L, x, y, w, Z, (0.8, 0.1, 1.1), theta, col_offset=10)
    rw, rln, rfl = orc.reweight(x, y, w, Z, (0.8, 0.1, 1.1), theta, col_offset=10)
    check_weights(wg, rw)
    check_log_norm(ln, rln)
    np.testing.assert_array_equal(wg[2], w[2])     # column 13: no measurement -> untouched
    np.testing.assert_array_equal(fl, 0)


@pytest.mark.parametrize("P", [2048, 8192])
def test_reweight_fp32_budget_edge(L, orc, P):
    """The e-cache kernel's fp32 pass is kept only while the unit's max log-weight m >= -300
    (every weight that matters then has q' <= 400 and an fp32 error under the contract),
    else pass 1 is rerun in fp64.  Tracks with a measurement 12-32 m from a 1.5 m cloud and
    Dirichlet weights put m on both sides of the threshold (the 28-32 m tracks past it);
    all of them must meet the 1e-4 contract against the oracle, 1e-30 absolute for the tiny
    weights.  Also 4 km coordinates, where z - p is formed from the split (hi, lo) mean."""
    r = np.random.default_rng(P + 7)
    ds = [12.0, 18.0, 22.0, 25.0, 28.0, 30.0, 32.0]
    T = len(ds)
    for base in (0.0, 4000.0):
        x = (base + r.normal(0, 1.5, (T, P))).astype(np.float32)
        y = (base + r.normal(0, 1.5, (T, P))).astype(np.float32)
        w = r.dirichlet(np.full(P, 0.5), T).astype(np.float32)
        Z = np.array([[base + d, base + 0.3] for d in ds], np.float32)
        theta = np.arange(1, T + 1, dtype=np.int32)
        wg, ln, fl = _reweight_gpu(L, x, y, w, Z, (1.0, 0.0, 1.0), theta)
        rw, rln, rfl = orc.reweight(x, y, w, Z, (1.0, 0.0, 1.0), theta)
        check_weights(wg, rw)
        check_log_norm(ln, rln)
        np.testing.assert_array_equal(fl.view(np.uint32), rfl)
        # the threshold is crossed inside the set: m_j = max_p log2 w' before normalising
        lw = np.log2(np.maximum(w.astype(np.float64), 1e-300))
        q = 0.5 / np.log(2) * ((Z[:, 0:1] - x.astype(np.float64)) ** 2 + (Z[:, 1:2] - y.astype(np.float64)) ** 2)
        m = (lw - q).max(axis=1)
        assert (m > -300).any() and (m < -300).any(), m


@pytest.mark.parametrize("P", [256, 8192])   # cluster kernel / flat two-pass kernel
def test_reweight_degenerate_and_many_assigned(L, orc, P):
    r = np.random.default_rng(3)
    T, M = 2, 1500                  # > 256 assigned measurements: generic S path
    x = r.normal(0, 1, (T, P)).astype(np.float32)
    y = r.normal(0, 1, (T, P)).astype(np.float32)
    w = r.dirichlet(np.ones(P), T).astype(np.float32)
    w[1] = 0.0                      # degenerate track: uniform reset + flag
    Z = r.normal(0, 0.3, (M, 2)).astype(np.float32)
    theta = np.where(np.arange(M) % 2 == 0, 1, 2).astype(np.int32)
    wg, ln, fl = _reweight_gpu(L, x, y, w, Z, (50.0, 0, 50.0), theta)
    rw, rln, rfl = orc.reweight(x, y, w, Z, (50.0, 0, 50.0), theta)
    check_weights(wg, rw)
    check_log_norm(ln, rln)
    np.testing.assert_array_equal(fl.view(np.uint32), rfl)
    assert rfl[1] == 1


# ------------------------------------------------------------------ whole step
def test_step_composition_and_host_entry(L):
    """glmb_step == the four calls in sequence (bit-exact); glmb_step_host == glmb_step."""
    import torch
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    s = make_scene(1, steps=1)
    a = GlmbStep(s)
    b = GlmbStep(s)
    a.predict(0); a.birth(0); a.compat(0); a.reweight(0)
    b.run(0)
    torch.cuda.synchronize()
    for f in ("C_tracks", "gate", "log_norm", "flags", "C_clutter"):
        np.testing.assert_array_equal(getattr(a.out, f).cpu().numpy(), getattr(b.out, f).cpu().numpy())
    np.testing.assert_array_equal(a.particles.data.cpu().numpy(), b.particles.data.cpu().numpy())
    c = GlmbStep(s)
    M = len(s.Z[0])
    pin = lambda arr: torch.from_numpy(arr).pin_memory()
    Zh, th = pin(s.Z[0]), pin(s.theta[0])
    Cc_h = torch.empty(c.M_max).pin_memory()
    Ct_h = torch.empty(c.T_local, c.ldc).pin_memory()
    G_h = torch.empty(c.T_local, c.ldg, dtype=torch.int32).pin_memory()
    ln_h = torch.empty(c.T_local).pin_memory()
    fl_h = torch.empty(c.T_local, dtype=torch.int32).pin_memory()
    o = c.out
    L.glmb_step_host(c.step_params(0), Zh, th, torch.empty(M, 2, device="cuda"),
                     torch.empty(M, dtype=torch.int32, device="cuda"), o.C_clutter, o.C_tracks,
                     o.gate, o.log_norm, o.flags, Cc_h, Ct_h, G_h, ln_h, fl_h)
    np.testing.assert_array_equal(Ct_h.numpy()[:, :M], b.out.C_tracks.cpu().numpy()[:, :M])
    np.testing.assert_array_equal(G_h.numpy(), b.out.gate.cpu().numpy())
    np.testing.assert_array_equal(ln_h.numpy(), b.out.log_norm.cpu().numpy())
    # the overlapped read-back (compat in track chunks, D2H on a second stream) is identical
    d = GlmbStep(s)
    Ct2, G2, ln2, fl2, Cc2 = (torch.zeros_like(Ct_h).pin_memory(), torch.zeros_like(G_h).pin_memory(),
                              torch.zeros_like(ln_h).pin_memory(), torch.zeros_like(fl_h).pin_memory(),
                              torch.zeros_like(Cc_h).pin_memory())
    st, cs = torch.cuda.Stream(), torch.cuda.Stream()
    L.glmb_step_host(d.step_params(0), Zh, th, torch.empty(M, 2, device="cuda"),
                     torch.empty(M, dtype=torch.int32, device="cuda"), d.out.C_clutter, d.out.C_tracks,
                     d.out.gate, d.out.log_norm, d.out.flags, Cc2, Ct2, G2, ln2, fl2, stream=st, copy_stream=cs)
    np.testing.assert_array_equal(Ct2.numpy()[:, :M], Ct_h.numpy()[:, :M])
    np.testing.assert_array_equal(G2.numpy(), G_h.numpy())
    np.testing.assert_array_equal(ln2.numpy(), ln_h.numpy())
    np.testing.assert_array_equal(fl2.numpy(), fl_h.numpy())
    np.testing.assert_array_equal(Cc2.numpy()[:M], Cc_h.numpy()[:M])
    np.testing.assert_array_equal(d.particles.data.cpu().numpy(), c.particles.data.cpu().numpy())
    # ... and with reweight into the spare weight buffer, concurrent with compat
    e = GlmbStep(s)
    Ct3, G3, ln3, fl3 = (torch.zeros_like(Ct_h).pin_memory(), torch.zeros_like(G_h).pin_memory(),
                         torch.zeros_like(ln_h).pin_memory(), torch.zeros_like(fl_h).pin_memory())
    L.glmb_step_host(e.step_params(0, out_of_place=True), Zh, th, torch.empty(M, 2, device="cuda"),
                     torch.empty(M, dtype=torch.int32, device="cuda"), e.out.C_clutter, e.out.C_tracks,
                     e.out.gate, e.out.log_norm, e.out.flags, None, Ct3, G3, ln3, fl3, stream=st, copy_stream=cs)
    e.swap_weights()
    np.testing.assert_array_equal(Ct3.numpy()[:, :M], Ct_h.numpy()[:, :M])
    np.testing.assert_array_equal(G3.numpy(), G_h.numpy())
    np.testing.assert_array_equal(ln3.numpy(), ln_h.numpy())
    np.testing.assert_array_equal(fl3.numpy(), fl_h.numpy())
    np.testing.assert_array_equal(e.weights().cpu().numpy(), c.particles.data[5].cpu().numpy())


def test_status_errors(L):
    import torch
    from paper_2512_06230_b200._lib import GlmbError, Particles
    trk = Particles.empty(2, 8)
    Z = torch.zeros(3, 2, device="cuda")
    C = torch.zeros(2, 3, device="cuda")
    G = torch.zeros(2, 1, dtype=torch.int32, device="cuda")
    with pytest.raises(GlmbError) as e:
        L.glmb_compat(trk, Z, (1, 2, 1), 0.9, 1e-3, 1e-6, None, C, G)    # R not SPD
    assert e.value.status == -1
    with pytest.raises(GlmbError):
        L.glmb_compat(trk, Z, (1, 0, 1), 0.9, 1e-3, 1e-31, None, C, G)   # gamma < 1e-30
    with pytest.raises(GlmbError) as e:
        L.glmb_compat(Particles(trk.data, 6), Z, (1, 0, 1), 0.9, 1e-3, 1e-6, None, C, G)
    assert e.value.status == -2                                           # P % 4 != 0


@pytest.mark.parametrize("case", ["wide", "tiny_w", "mixed"])
def test_compat_fold_fallback_tiles(L, orc, case):
    """Tiles with a particle at |p'|^2 > 64 (wide clouds) take the exact-difference
    form; wide tracks, a track mixing wide and narrow tiles, and weights spanning
    1e-36 .. 1e-3 must all match the oracle."""
    r = np.random.default_rng(hash(case) % 2**32)
    T, P, M = 3, 1024, 300
    spread = {"wide": 25.0, "tiny_w": 2.0, "mixed": 2.0}[case]
    x = (500 + spread * r.standard_normal((T, P))).astype(np.float32)
    y = (800 + spread * r.standard_normal((T, P))).astype(np.float32)
    w = np.full((T, P), 1.0 / P, np.float32)
    if case == "tiny_w":
        w[:] = np.float32(1e-36)
        w[:, ::7] = np.float32(1e-3)
    if case == "mixed":
        x[:, 256:512] += (40 * r.standard_normal(256)).astype(np.float32)   # one wide tile
    Z = np.stack([500 + 30 * r.standard_normal(M), 800 + 30 * r.standard_normal(M)], 1).astype(np.float32)
    R = (1.0, 0.2, 0.7)
    C, G, Cc = _compat_gpu(L, x, y, w, Z, R, 0.9, 1e-4, 1e-30 if case == "tiny_w" else 1e-8)
    ref = orc.compat(x, y, w, Z, R, 0.9, 1e-4, 1e-30 if case == "tiny_w" else 1e-8)
    check_compat(C, G, Cc, ref, 1e-30 if case == "tiny_w" else 1e-8, M)
    assert (ref["C_tracks"] > 0).sum() > 10


@pytest.mark.parametrize("P", [1024, 8192, 16384])
def test_reweight_out_of_place_matches_in_place(L, orc, P):
    """glmb_reweight with a separate w_out: same bits as in place, input weights untouched,
    tracks without assigned measurements copied."""
    import torch
    from paper_2512_06230_b200._lib import Particles
    r = np.random.default_rng(P + 1)
    T = 6
    data = np.zeros((6, T, P), np.float32)
    data[0] = r.normal(0, 1, (T, P))
    data[1] = r.normal(0, 1, (T, P))
    data[5] = r.dirichlet(np.ones(P), T)
    Z = r.normal(0, 1, (5, 2)).astype(np.float32)
    theta = np.array([1, 3, 3, 0, 6], np.int32)
    a = Particles(_dev(data), P)
    b = Particles(_dev(data), P)
    w_out = torch.full((T, P), -1.0, device="cuda")
    la, fa = torch.zeros(T, device="cuda"), torch.zeros(T, dtype=torch.int32, device="cuda")
    lb, fb = torch.zeros(T, device="cuda"), torch.zeros(T, dtype=torch.int32, device="cuda")
    L.glmb_reweight(a, _dev(Z), (1, 0, 1), _dev(theta), 0, la, fa)
    L.glmb_reweight(b, _dev(Z), (1, 0, 1), _dev(theta), 0, lb, fb, w_out=w_out)
    np.testing.assert_array_equal(_host(w_out), _host(a.data)[5])
    np.testing.assert_array_equal(_host(b.data)[5], data[5])
    np.testing.assert_array_equal(_host(la), _host(lb))
    rw, _, _ = orc.reweight(data[0], data[1], data[5], Z, (1, 0, 1), theta)
    check_weights(_host(w_out), rw)


def test_compat_peers_fused_gather(L):
    """glmb_compat_peers (compat fused with the column all-gather): with one destination it
    equals glmb_compat; with the tracks split into two blocks each written to two destination
    buffers (two 'ranks' on one GPU, no rank waits on another) both buffers hold the whole
    single-launch C_k and gate, bit for bit."""
    import torch
    from paper_2512_06230_b200._lib import Particles
    from paper_2512_06230_b200 import scenes
    sc = scenes.make_scene(1, steps=1)
    cfg = sc.cfg
    p = Particles.from_arrays([sc.x, sc.y, sc.v, sc.psi, sc.omega, sc.w])
    Z = _dev(sc.Z[0])
    T, M = p.T, Z.shape[0]
    ldc, ldg = (M + 31) // 32 * 32, (M + 31) // 32
    C0 = torch.zeros(T, ldc, device="cuda")
    G0 = torch.zeros(T, ldg, dtype=torch.int32, device="cuda")
    L.glmb_compat(p, Z, cfg.R, cfg.p_d, cfg.kappa, cfg.gamma, None, C0, G0)
    bufs = [(torch.full((T, ldc), -1.0, device="cuda"), torch.full((T, ldg), -1, dtype=torch.int32, device="cuda"))
            for _ in range(2)]
    ptrs = lambda k: torch.tensor([b[k].data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    half = T // 2
    for r0, r1 in ((0, half), (half, T)):
        L.glmb_compat_peers(p.rows(r0, r1), Z, cfg.R, cfg.p_d, cfg.kappa, cfg.gamma, None, ptrs(0), ptrs(1), r0,
                            ldc, ldg)
    torch.cuda.synchronize()
    for Cb, Gb in bufs:
        np.testing.assert_array_equal(Cb.cpu().numpy()[:, :M], C0.cpu().numpy()[:, :M])
        np.testing.assert_array_equal(Gb.cpu().numpy(), G0.cpu().numpy())


def test_step_graph_capture(L):
    """The C-ABI calls are CUDA-graph capturable (no stream queries during capture): a captured
    glmb_step replays to the same outputs as the eager call."""
    import torch
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    s = make_scene(1, steps=1)
    a, b = GlmbStep(s), GlmbStep(s)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        a.run(0, st)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            b.run(0, st)
        g.replay()
        st.synchronize()
    for f in ("C_tracks", "gate", "log_norm", "flags"):
        np.testing.assert_array_equal(getattr(a.out, f).cpu().numpy(), getattr(b.out, f).cpu().numpy())
    np.testing.assert_array_equal(a.particles.data.cpu().numpy(), b.particles.data.cpu().numpy())


@pytest.mark.parametrize("case", range(30))
def test_step_kernels_random_tiny_shapes(L, orc, case):
    """SURVEY §4 tier 5: random tiny T, P (multiple of 4), M, general SPD R, weights, gamma,
    including T = 1 and M = 0 -- compat and reweight vs the oracle."""
    r = np.random.default_rng(7000 + case)
    T = int(r.integers(1, 12))
    P = int(4 * r.integers(1, 80))
    M = int(r.integers(0, 70)) if case % 7 else 0
    sx, sy = r.uniform(0.2, 3.0, 2)
    rho = r.uniform(-0.8, 0.8)
    R = (float(np.float32(sx * sx)), float(np.float32(rho * sx * sy)), float(np.float32(sy * sy)))
    cen = r.uniform(0, 60, (T, 2))
    x = (cen[:, :1] + r.normal(0, r.uniform(0.3, 4), (T, P))).astype(np.float32)
    y = (cen[:, 1:] + r.normal(0, r.uniform(0.3, 4), (T, P))).astype(np.float32)
    w = r.dirichlet(np.ones(P) * r.uniform(0.1, 5), T).astype(np.float32)
    Z = r.uniform(-5, 65, (M, 2)).astype(np.float32)
    gamma = float(np.float32(10 ** r.uniform(-9, -3)))
    p_d, kappa = float(np.float32(r.uniform(0.2, 1.0))), float(np.float32(10 ** r.uniform(-6, -2)))
    if M:
        C, G, Cc = _compat_gpu(L, x, y, w, Z, R, p_d, kappa, gamma)
        check_compat(C, G, Cc, orc.compat(x, y, w, Z, R, p_d, kappa, gamma), gamma, M)
    theta = r.integers(0, T + 1, M).astype(np.int32)
    wg, ln, fl = _reweight_gpu(L, x, y, w, Z, R, theta)
    rw, rln, rfl = orc.reweight(x, y, w, Z, R, theta)
    check_weights(wg, rw)
    check_log_norm(ln, rln)
    np.testing.assert_array_equal(fl.view(np.uint32), rfl)


def test_step_host_csr_matches_dense(L, orc):
    """glmb_step_host_csr returns exactly the gated entries of the dense C_k that glmb_step_host
    reads back (row order, ascending columns, bit-identical values), and the same log_norm."""
    import torch
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    s = make_scene(1, steps=1)
    a, b = GlmbStep(s), GlmbStep(s)
    M = len(s.Z[0])
    pin = lambda t: t.pin_memory()
    Zh, th = pin(torch.from_numpy(s.Z[0])), pin(torch.from_numpy(s.theta[0]))
    Zd, thd = torch.empty(M, 2, device="cuda"), torch.empty(M, dtype=torch.int32, device="cuda")
    Ct_h = pin(torch.empty(a.T_local, a.ldc))
    G_h = pin(torch.empty(a.T_local, a.ldg, dtype=torch.int32))
    ln_a, fl_a = pin(torch.empty(a.T_local)), pin(torch.empty(a.T_local, dtype=torch.int32))
    L.glmb_step_host(a.step_params(0), Zh, th, Zd, thd, a.out.C_clutter, a.out.C_tracks, a.out.gate,
                     a.out.log_norm, a.out.flags, None, Ct_h, G_h, ln_a, fl_a)
    cap = b.T_local * M
    rp = torch.empty(M + 1, dtype=torch.int32, device="cuda")
    col, val = torch.empty(cap, dtype=torch.int32, device="cuda"), torch.empty(cap, device="cuda")
    lv = torch.empty(cap, dtype=torch.float64, device="cuda")
    rp_h = pin(torch.empty(M + 1, dtype=torch.int32))
    col_h, val_h = pin(torch.empty(8, dtype=torch.int32)), pin(torch.empty(8))   # small: forces the 2nd copy
    ln_b, fl_b = pin(torch.empty(b.T_local)), pin(torch.empty(b.T_local, dtype=torch.int32))
    with pytest.raises(Exception):   # more gated entries than the host arrays hold
        L.glmb_step_host_csr(b.step_params(0), Zh, th, Zd, thd, b.out.C_tracks, b.out.gate, b.out.log_norm,
                             b.out.flags, rp, col, val, lv, rp_h, col_h, val_h, ln_b, fl_b)
    c = GlmbStep(s)
    col_h, val_h = pin(torch.empty(4096, dtype=torch.int32)), pin(torch.empty(4096))
    # a speculative first copy of 8 entries: the rest (nnz > 8, within the host capacity) in
    # the second, exact-size copy
    nnz = L.glmb_step_host_csr(c.step_params(0), Zh, th, Zd, thd, c.out.C_tracks, c.out.gate, c.out.log_norm,
                               c.out.flags, rp, col, val, lv, rp_h, col_h, val_h, ln_b, fl_b, first_copy=8)
    assert nnz > 8
    C = Ct_h.numpy()[:, :M]
    G = np.unpackbits(G_h.numpy().view(np.uint8), bitorder="little").reshape(a.T_local, -1)[:, :M].astype(bool)
    rows = [np.nonzero(G[:, i])[0] for i in range(M)]
    np.testing.assert_array_equal(rp_h.numpy(), np.concatenate([[0], np.cumsum([len(r) for r in rows])]))
    assert nnz == sum(len(r) for r in rows)
    np.testing.assert_array_equal(col_h.numpy()[:nnz], np.concatenate(rows))
    np.testing.assert_array_equal(val_h.numpy()[:nnz], np.concatenate([C[r, i] for i, r in enumerate(rows)]))
    np.testing.assert_array_equal(ln_b.numpy(), ln_a.numpy())
    # reweight beside compat on an aux stream (out of place): same CSR, same new weights
    d = GlmbStep(s)
    st_, aux = torch.cuda.Stream(), torch.cuda.Stream()
    rp2 = pin(torch.empty(M + 1, dtype=torch.int32))
    col2, val2 = pin(torch.empty(4096, dtype=torch.int32)), pin(torch.empty(4096))
    ln2, fl2 = pin(torch.empty(d.T_local)), pin(torch.empty(d.T_local, dtype=torch.int32))
    nnz2 = L.glmb_step_host_csr(d.step_params(0, out_of_place=True), Zh, th, Zd, thd, d.out.C_tracks, d.out.gate,
                                d.out.log_norm, d.out.flags, rp, col, val, lv, rp2, col2, val2, ln2, fl2,
                                stream=st_, aux_stream=aux)
    d.swap_weights()
    assert nnz2 == nnz
    np.testing.assert_array_equal(rp2.numpy(), rp_h.numpy())
    np.testing.assert_array_equal(col2.numpy()[:nnz], col_h.numpy()[:nnz])
    np.testing.assert_array_equal(val2.numpy()[:nnz], val_h.numpy()[:nnz])
    np.testing.assert_array_equal(ln2.numpy(), ln_a.numpy())
    np.testing.assert_array_equal(d.weights().cpu().numpy(), c.weights().cpu().numpy())


@pytest.mark.parametrize("cfg_id,n_rows,n_pred", [(1, 64, 0), (3, 96, 0), (3, 96, 12)])
def test_compat_exact_skip(cfg_id, n_rows, n_pred, tmp_path):
    """GLMB_COMPAT_SKIP=1 (warps skip particle tiles whose every pair has q >= 200, where both
    exp paths give exactly +0) reproduces the dense pass bit for bit: C and the gate words
    from two child processes, one per setting (compact and diffused clouds)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    outs = {}
    for skip in ("0", "1"):
        out = str(tmp_path / f"c{skip}.npz")
        env = dict(os.environ, GLMB_COMPAT_SKIP=skip, PYTHONPATH=os.path.dirname(here))
        r = subprocess.run([sys.executable, os.path.join(here, "_compat_dump.py"), str(cfg_id), str(n_rows),
                            str(n_pred), out], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        outs[skip] = np.load(out)
    np.testing.assert_array_equal(outs["0"]["C"].view(np.uint32), outs["1"]["C"].view(np.uint32))
    np.testing.assert_array_equal(outs["0"]["G"], outs["1"]["G"])


@pytest.mark.parametrize("cfg_id", [1, 2])
def test_pipelined_steps_equal_sequential(L, cfg_id):
    """step.PipelinedSteps (bench.py's N = 1 schedule: predict + birth of step k into the spare
    state buffer beside compat of step k-1, reweight beside compat, event-ordered) gives the
    sequential steps' results bit for bit: state, weights, C_k, gate words, log-normalisers."""
    import torch
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep, PipelinedSteps
    s = make_scene(cfg_id, steps=6)
    a, b = GlmbStep(s), GlmbStep(s)
    main, side = torch.cuda.Stream(), torch.cuda.Stream()
    pipe = PipelinedSteps(b, main, side)
    for k in range(6):
        a.predict(k)
        a.birth(k)
        a.compat(k)
        a.reweight(k)
        pipe.step(k)
    pipe.join()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(a.particles.data[:5].cpu().numpy(), b.particles.data[:5].cpu().numpy())
    np.testing.assert_array_equal(a.particles.data[5].cpu().numpy(), b.weights().cpu().numpy())
    for f in ("C_tracks", "gate", "log_norm", "flags"):
        np.testing.assert_array_equal(getattr(a.out, f).cpu().numpy(), getattr(b.out, f).cpu().numpy())


def test_compat_p1024_split_bit_identical(tmp_path):
    """At P = 1024 (four particle tiles) compat runs a 4-CTA cluster per unit, one tile per
    rank; rank 0's ordered merge adds the tile sums in the order one CTA would, so C and the
    gate words equal the unsplit kernel's (GLMB_COMPAT_CL=1) bit for bit (config 1: P = 1024,
    births included)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    outs = {}
    for cl in ("", "1"):
        out = str(tmp_path / f"cl{cl or 'd'}.npz")
        env = dict(os.environ, PYTHONPATH=os.path.dirname(here))
        env.pop("GLMB_COMPAT_CL", None)
        if cl:
            env["GLMB_COMPAT_CL"] = cl
        r = subprocess.run([sys.executable, os.path.join(here, "_compat_dump.py"), "1", "64", "3", out, "68"],
                           env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        outs[cl] = np.load(out)
    np.testing.assert_array_equal(outs[""]["C"].view(np.uint32), outs["1"]["C"].view(np.uint32))
    np.testing.assert_array_equal(outs[""]["G"], outs["1"]["G"])


def test_compat_low_slot_path_bit_identical(tmp_path):
    """A warp whose only valid measurement slot is its packed pair's low one (the ragged last
    warp of a tile when M mod 64 <= 32: config 1, M = 81) evaluates that lane alone with
    scalar mirrors of the packed ops; C and the gate words equal the packed evaluation's
    (GLMB_COMPAT_LO=0) bit for bit, births included."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    outs = {}
    for lo in ("1", "0"):
        out = str(tmp_path / f"lo{lo}.npz")
        env = dict(os.environ, GLMB_COMPAT_LO=lo, PYTHONPATH=os.path.dirname(here))
        r = subprocess.run([sys.executable, os.path.join(here, "_compat_dump.py"), "1", "64", "3", out, "68"],
                           env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        outs[lo] = np.load(out)
    assert outs["1"]["C"].shape[1] % 64 <= 32   # the low-slot path is exercised
    np.testing.assert_array_equal(outs["1"]["C"].view(np.uint32), outs["0"]["C"].view(np.uint32))
    np.testing.assert_array_equal(outs["1"]["G"], outs["0"]["G"])

"""GPU parity of the particle loop (§Approach) through the C ABI
against the fp64 oracle O14-O16 on identical seeded inputs (generator or oracle outputs).

Bars: pairs (integers) bit-exact; reweighted weights rel 1e-4 or abs
1e-30, log_norm 1e-4 max(1, |ref|), flags exact, ESS rel 1e-4; resampling decisions,
ancestors and the gathered states bit-exact (integer CDF, same fp32 weights on both
sides), weights exactly 1/P or copied."""
import numpy as np
import pytest

from conftest import gpu_available
from _parity import check_log_norm, check_weights

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


def _dev(a):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


def _host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _gpu_pairs(L, hyp_idx, alive, theta, T, M):
    import torch
    n = len(hyp_idx)
    i32 = torch.int32
    pt = torch.full((max(1, n * T),), -9, dtype=i32, device="cuda")
    pp = torch.full((max(1, n * T) + 1,), -9, dtype=i32, device="cuda")
    pm = torch.full((max(1, n * M),), -9, dtype=i32, device="cuda")
    po = torch.full((max(1, n), max(1, T)), -9, dtype=i32, device="cuda")
    nk = torch.full((1,), -9, dtype=i32, device="cuda")
    ws = torch.empty(max(16, L.glmb_assoc_pairs_workspace_size(n, T, M)), dtype=torch.uint8, device="cuda")
    L.glmb_assoc_pairs(_dev(np.asarray(hyp_idx, np.int32)), _dev(np.asarray(alive).view(np.int32)),
                       _dev(theta), T, M, pt, pp, pm, po, nk, ws)
    K = int(_host(nk)[0])
    pp_h = _host(pp)
    return _host(pt)[:K], pp_h[:K + 1], _host(pm)[:pp_h[K]], _host(po)[:n, :T], K


def _check_pairs(got, ref):
    pt, pp, pm, po, K = got
    r_pt, r_pp, r_pm, r_po = ref
    assert K == len(r_pt)
    np.testing.assert_array_equal(pt, r_pt)
    np.testing.assert_array_equal(pp, r_pp)
    np.testing.assert_array_equal(pm, r_pm)
    np.testing.assert_array_equal(po, r_po)


# ------------------------------------------------------------------ O14
def test_pairs_hand_example(L, orc):
    alive = np.array([[0b011], [0b111]], np.uint32)
    theta = np.array([[1, 0, 2, 1], [1, 0, 0, 1]], np.int32)
    for order in ([0, 1], [1, 0], [1, 1, 0]):
        _check_pairs(_gpu_pairs(L, order, alive, theta, 3, 4), orc.assoc_pairs(order, alive, theta, 3, 4))


@pytest.mark.parametrize("T,M,n,seed", [(23, 40, 60, 4), (1040, 1198, 25, 3), (300, 0, 5, 1), (5, 7, 1, 2),
                                        (70, 513, 100, 6),
                                        (5, 300, 8, 7), (2, 1000, 3, 8)])   # > 32 rows per track: warp-walk lists
def test_pairs_random(L, orc, T, M, n, seed):
    rng = np.random.default_rng(seed)
    ldt = (T + 31) // 32
    alive = rng.integers(0, 2**32, (n, ldt), dtype=np.uint64).astype(np.uint32)
    if T % 32:
        alive[:, -1] &= np.uint32((1 << (T % 32)) - 1)
    theta = np.zeros((n, max(M, 1)), np.int32)
    menu = rng.integers(0, T + 1, (4, max(M, 1)))   # few distinct maps -> repeated pairs
    for q in range(n):
        theta[q] = menu[q % 4] if rng.random() < 0.7 else rng.integers(0, T + 1, max(M, 1))
    order = rng.permutation(n)
    _check_pairs(_gpu_pairs(L, order, alive, theta[:, :max(M, 1)], T, M),
                 orc.assoc_pairs(order, alive, theta, T, M))


def test_pairs_from_sampler(L, orc):
    """The pairs of the kept hypotheses of a cfg1 update (oracle chain O7 -> O13 as input)."""
    from paper_2512_06230_b200 import scenes
    sc = scenes.make_scene(1, steps=1)
    cfg = sc.cfg
    Z = sc.Z[0]
    ref = orc.compat(sc.x, sc.y, sc.w, Z, cfg.R, cfg.p_d, cfg.kappa, cfg.gamma)
    C = ref["C_tracks"].astype(np.float32)
    g = np.ascontiguousarray(ref["gate"], np.uint32)
    T, M = C.shape[0], Z.shape[0]
    pm, plw, ps = scenes.hypothesis_inputs(T, 0, 10, seed=5)
    d = orc.death_prob(C, g, cfg.p_d, cfg.kappa, ps).astype(np.float32)
    rows = orc.compat_rows(C, g, M)
    al, th, lw = orc.assoc_sample(pm, plw, 100, d, ps, cfg.p_d, cfg.kappa, rows, M, 17, 0)
    u = orc.dedup(al, th, 10, 100)
    idx, w = orc.prune(lw, u, 1e-5, 25)
    _check_pairs(_gpu_pairs(L, idx, al, th, T, M), orc.assoc_pairs(idx, al, th, T, M))


# ------------------------------------------------------------------ O15
def _src(x, y, w):
    from paper_2512_06230_b200._lib import Particles
    T, P = x.shape
    z = np.zeros_like(x)
    return Particles.from_arrays([x, y, z, z, z, w])


def _gpu_reweight_pairs(L, src, Z, R, pt, pp, pm, K_cap=None, n_pairs=None):
    import torch
    K = len(pt) if K_cap is None else K_cap
    P = src.P
    wo = torch.full((max(K, 1), P), -1.0, dtype=torch.float32, device="cuda")
    lz = torch.zeros(max(K, 1), dtype=torch.float32, device="cuda")
    fl = torch.full((max(K, 1),), 7, dtype=torch.int32, device="cuda")
    es = torch.zeros(max(K, 1), dtype=torch.float32, device="cuda")
    one = lambda a: a if len(a) else np.zeros(1, np.int32)
    L.glmb_reweight_pairs(src, _dev(np.asarray(Z, np.float32).reshape(-1, 2)), R, K,
                          None if n_pairs is None else _dev(np.array([n_pairs], np.int32)),
                          _dev(one(np.asarray(pt, np.int32))), _dev(np.asarray(pp, np.int32)),
                          _dev(one(np.asarray(pm, np.int32))), wo, lz, fl, es)
    return _host(wo), _host(lz), _host(fl).view(np.uint32), _host(es)


@pytest.mark.parametrize("P", [4, 1024, 4096, 8192, 12288, 16384])
def test_reweight_pairs_vs_oracle(L, orc, P):
    from paper_2512_06230_b200 import scenes
    T = 9
    x, y, v, psi, om, w = scenes.random_cloud(T, P, P, center_scale=30.0, spread=2.0, dirichlet=True)
    w[4] = 0.0                                              # degenerate track
    rng = np.random.default_rng(P)
    Z = rng.uniform(-5, 35, (40, 2)).astype(np.float32)
    R = (1.5, 0.3, 0.8)
    sets = [[], [3], [3, 7, 11], [0], list(range(0, 40, 3)), [5], [], [39], [1, 2]]
    tracks = [0, 0, 1, 4, 2, 3, 4, 8, 7]
    pp = np.concatenate([[0], np.cumsum([len(s) for s in sets])]).astype(np.int32)
    pm = np.array([i for s in sets for i in s], np.int32)
    wo, lz, fl, es = _gpu_reweight_pairs(L, _src(x, y, w), Z, R, tracks, pp, pm)
    r_w, r_lz, r_fl, r_es = orc.reweight_pairs(x, y, w, Z, R, tracks, pp, pm)
    check_weights(wo, r_w)
    check_log_norm(lz, r_lz)
    np.testing.assert_array_equal(fl, r_fl)
    np.testing.assert_allclose(es, r_es, rtol=1e-4)


def test_reweight_pairs_device_count(L, orc):
    """n_pairs (device) limits the work: rows past it are untouched."""
    from paper_2512_06230_b200 import scenes
    x, y, v, psi, om, w = scenes.random_cloud(3, 256, 1)
    Z = np.array([[50.0, 50.0], [10.0, 10.0]], np.float32)
    pt, pp, pm = [0, 1, 2, 2], [0, 1, 2, 2, 2], [0, 1]
    wo, lz, fl, es = _gpu_reweight_pairs(L, _src(x, y, w), Z, (1, 0, 1), pt, pp, pm, K_cap=4, n_pairs=2)
    r_w, r_lz, r_fl, r_es = orc.reweight_pairs(x, y, w, Z, (1, 0, 1), pt[:2], pp[:3], pm)
    check_weights(wo[:2], r_w)
    assert np.all(wo[2:] == -1.0) and np.all(fl[2:] == 7)


# ------------------------------------------------------------------ O16
def _gpu_resample(L, src, pt, wk, seed, step, n_pairs=None):
    import torch
    from paper_2512_06230_b200._lib import Particles
    K, P = wk.shape
    out = Particles(torch.full((6, K, P), -3.0, dtype=torch.float32, device="cuda"), P)
    fl = torch.ones(K, dtype=torch.int32, device="cuda")      # bit 0 must survive
    L.glmb_resample(src, K, None if n_pairs is None else _dev(np.array([n_pairs], np.int32)),
                    _dev(np.asarray(pt, np.int32)), _dev(wk), out, seed, step, fl)
    return _host(out.data), _host(fl).view(np.uint32)


@pytest.mark.parametrize("P", [4, 1024, 8192, 16384])
def test_resample_vs_oracle(L, orc, P):
    from paper_2512_06230_b200 import scenes
    T = 4
    arr = scenes.random_cloud(T, P, 3 + P)
    src = _src(arr[0], arr[1], arr[5])
    import torch
    src.data[2] = _dev(arr[2])
    src.data[3] = _dev(arr[3])
    src.data[4] = _dev(arr[4])
    rng = np.random.default_rng(P)
    K = 12
    pt = rng.integers(0, T, K).astype(np.int32)
    wk = np.zeros((K, P), np.float32)
    conc = [0.01, 0.1, 1.0, 10.0, 100.0, 0.3, 0.05, 1e3, 0.5, 2.0, 0.02, 5.0]
    for k in range(K):
        wk[k] = rng.dirichlet(np.full(P, conc[k])).astype(np.float32)
    wk[5] = 0.0
    wk[5, P // 2] = 1.0                                       # one-hot: every slot the same ancestor
    wk[6] = 1.0 / P                                           # uniform: kept
    seed, step = 0xABCDEF, 12
    out, fl = _gpu_resample(L, src, pt, wk, seed, step)
    assert np.all(fl & 1)
    for k in range(K):
        res, anc = orc.resample(wk[k], seed, step, k)
        assert bool(fl[k] & 2) == res, k
        srcrows = np.stack(arr[:5])[:, pt[k]]
        if res:
            np.testing.assert_array_equal(out[:5, k], srcrows[:, anc])
            assert np.all(out[5, k] == np.float32(1.0 / P))
        else:
            np.testing.assert_array_equal(out[:5, k], srcrows)
            np.testing.assert_array_equal(out[5, k], wk[k])
    assert fl[5] & 2 and not fl[6] & 2


# ------------------------------------------------------------------ the loop
def test_particle_update_chain(L, orc):
    """HypothesisUpdate -> ParticleUpdate on cfg1 (C_k from the oracle): pairs bit-exact,
    per-pair weights within the contract vs O15; the resampled set has the systematic
    floor/ceil count property on the GPU's own weights."""
    import torch
    from paper_2512_06230_b200 import scenes
    from paper_2512_06230_b200._lib import Particles
    from paper_2512_06230_b200.hyp import HypothesisUpdate, ParticleUpdate
    sc = scenes.make_scene(1, steps=1)
    cfg = sc.cfg
    Z = sc.Z[0]
    ref = orc.compat(sc.x, sc.y, sc.w, Z, cfg.R, cfg.p_d, cfg.kappa, cfg.gamma)
    C = ref["C_tracks"].astype(np.float32)
    g = np.ascontiguousarray(ref["gate"], np.uint32)
    T, M = C.shape[0], Z.shape[0]
    H_old, H_up, h_max = 10, 100, 25
    pm, plw, ps = scenes.hypothesis_inputs(T, 0, H_old, seed=8)
    hu = HypothesisUpdate(T, M, H_old, H_up, h_max)
    hu.run(_dev(C), _dev(g.view(np.int32)), M, _dev(ps), _dev(pm.view(np.int32)), _dev(plw),
           cfg.p_d, cfg.kappa, 1e-5, seed=4, step=0)
    n_hyp = int(_host(hu.n_kept)[0])
    src = Particles.from_arrays([sc.x, sc.y, sc.v, sc.psi, sc.omega, sc.w])
    pu = ParticleUpdate(T, M, h_max, cfg.P)
    pu.run(src, _dev(Z), cfg.R, hu.keep_idx, n_hyp, hu.alive, hu.theta, M, seed=4, step=0)
    K = pu.n_pairs_checked()
    # oracle chain on the oracle's own samples (identical to the GPU's: bit-exact stages)
    d = orc.death_prob(C, g, cfg.p_d, cfg.kappa, ps).astype(np.float32)
    rows = orc.compat_rows(C, g, M)
    al, th, lw = orc.assoc_sample(pm, plw, H_up, d, ps, cfg.p_d, cfg.kappa, rows, M, 4, 0)
    idx, _ = orc.prune(lw, orc.dedup(al, th, H_old, H_up), 1e-5, h_max)
    assert n_hyp == len(idx)
    r_pt, r_pp, r_pm, r_po = orc.assoc_pairs(idx, al, th, T, M)
    assert K == len(r_pt)
    np.testing.assert_array_equal(_host(pu.pair_track)[:K], r_pt)
    np.testing.assert_array_equal(_host(pu.pair_meas)[:r_pp[K]], r_pm)
    r_w, r_lz, r_fl, r_es = orc.reweight_pairs(sc.x, sc.y, sc.w, Z, cfg.R, r_pt, r_pp, r_pm)
    w_gpu = _host(pu.w_new)[:K]
    check_weights(w_gpu, r_w)
    check_log_norm(_host(pu.log_norm)[:K], r_lz)
    fl = _host(pu.flags)[:K].view(np.uint32)
    np.testing.assert_array_equal(fl & 1, r_fl)
    out = _host(pu.out.data)[:, :K]
    P = cfg.P
    # resampling stage: a property check on the GPU's own weights (no oracle input from the GPU)
    n_res = 0
    for k in range(K):
        W = np.floor(w_gpu[k].astype(np.float64) * 2.0 ** 26)
        S, Q = W.sum(), (W * W).sum()
        res = S > 0 and 2 * S * S < P * Q
        assert bool(fl[k] & 2) == res
        xs = sc.x[r_pt[k]]
        if res:
            n_res += 1
            rows5 = np.stack([sc.x, sc.y, sc.v, sc.psi, sc.omega])[:, r_pt[k]]
            pos = {rows5[:, m].tobytes(): m for m in range(P)}      # full state: fp32 x alone collides
            assert len(pos) == P
            anc = np.array([pos[out[:5, k, n].copy().tobytes()] for n in range(P)])
            N = np.bincount(anc, minlength=P)
            e = P * W / S
            assert N.sum() == P and np.all(N >= np.floor(e)) and np.all(N <= np.ceil(e))
            assert np.all(np.diff(anc) >= 0)
            assert np.all(out[5, k] == np.float32(1.0 / P))
        else:
            np.testing.assert_array_equal(out[0, k], xs)
            np.testing.assert_array_equal(out[5, k], w_gpu[k])
    assert n_res > 0

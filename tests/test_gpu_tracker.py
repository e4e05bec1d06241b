"""GPU parity of the tracker-loop kernels (O17, O18) and of the parent-count plumbing,
plus the whole tracker on a small paper-shaped convoy.

The end-to-end run is checked by properties (there is no fp64 end-to-end oracle: the
stages are parity-tested one by one on identical inputs, and fp32 state drift may flip
a later sampling decision): bit-identical reruns, the cardinality of the MAP
hypothesis and the Hungarian tracking error of P:213-215 after the entry phase."""
import numpy as np
import pytest

from conftest import gpu_available

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


@pytest.mark.parametrize("H,T,K_cap,B,col0,n_kept", [(100, 57, 200, 1, 130, 37), (5, 3, 6, 2, 6, 2),
                                                     (10, 400, 700, 3, 690, 10), (4, 9, 9, 1, 5, 0)])
def test_next_parents_vs_oracle(L, orc, H, T, K_cap, B, col0, n_kept):
    import torch
    rng = np.random.default_rng(H + T)
    pair_of = rng.integers(-1, K_cap + 20, (H, T)).astype(np.int32)   # includes pairs past K_cap
    keep_w = rng.dirichlet(np.ones(H))
    ldt = (max(K_cap, col0 + B) + 31) // 32
    mask = torch.full((H, ldt), -1, dtype=torch.int32, device="cuda")
    lw = torch.full((H,), 7.0, dtype=torch.float64, device="cuda")
    npar = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    L.glmb_next_parents(_dev(np.array([n_kept], np.int32)), _dev(keep_w), _dev(pair_of), K_cap, B, col0,
                        mask, lw, npar)
    r_mask, r_lw = orc.next_parents(keep_w[:n_kept], pair_of[:n_kept], T, K_cap, B, col0, ldt)
    m = _host(mask).view(np.uint32)
    np.testing.assert_array_equal(m[:n_kept], r_mask)
    assert np.all(m[n_kept:] == 0xFFFFFFFF)                    # rows past n_kept untouched
    np.testing.assert_allclose(_host(lw)[:n_kept], r_lw, rtol=1e-15)
    assert int(_host(npar)[0]) == n_kept
    # the same with the birth column read on the device (e.g. glmb_assoc_pairs' n_pairs)
    mask2 = torch.full((H, ldt), -1, dtype=torch.int32, device="cuda")
    L.glmb_next_parents(_dev(np.array([n_kept], np.int32)), _dev(keep_w), _dev(pair_of), K_cap, B, 0,
                        mask2, lw, npar, birth_col0_dev=_dev(np.array([col0], np.int32)))
    np.testing.assert_array_equal(_host(mask2).view(np.uint32)[:n_kept], r_mask)


@pytest.mark.parametrize("P", [4, 1024, 8192])
def test_map_estimate_vs_oracle(L, orc, P):
    import torch
    from paper_2512_06230_b200 import scenes
    from paper_2512_06230_b200._lib import Particles
    K = 6
    x, y, v, psi, om, w = scenes.random_cloud(K, P, P, center_scale=80.0, spread=0.5, dirichlet=True)
    pair_of0 = np.array([3, -1, 0, 5, -1, 2, 2, 1], np.int32)
    s = Particles.from_arrays([x, y, v, psi, om, w])
    est = torch.zeros(len(pair_of0), 3, dtype=torch.float64, device="cuda")
    L.glmb_map_estimate(_dev(np.array([4], np.int32)), _dev(pair_of0), s, est)
    got = _host(est)
    ref = orc.map_estimate(4, pair_of0, x, y, w)
    np.testing.assert_array_equal(got[:, 2], ref[:, 2])
    ok = ref[:, 2] > 0
    np.testing.assert_allclose(got[ok, :2], ref[ok, :2], rtol=1e-12)
    assert np.all(np.isnan(got[~ok, :2]))
    L.glmb_map_estimate(_dev(np.array([0], np.int32)), _dev(pair_of0), s, est)
    assert np.all(_host(est)[:, 2] == 0)


def test_sampler_parent_count(L, orc):
    """n_parents = 2 of 4 parent slots: the first two parents' samples equal a run with
    H_old = 2; the other slots are skipped by the sampler and marked non-unique by dedup."""
    import torch
    from paper_2512_06230_b200 import scenes
    from paper_2512_06230_b200 import _lib
    T, M, H_up = 40, 60, 32
    C, g = scenes.synthetic_compat(T, M, 12)
    rows = orc.compat_rows(C, g, M)
    pm, plw, ps = scenes.hypothesis_inputs(T, 0, 4, seed=12)
    d = np.full(T, 0.2, np.float32)
    rp, col, val, lv = rows

    def run(pm_rows, n_par):
        H = pm_rows.shape[0]
        n = H * H_up
        alive = torch.full((n, pm.shape[1]), -1, dtype=torch.int32, device="cuda")
        theta = torch.full((n, 60), -5, dtype=torch.int32, device="cuda")
        logw = torch.zeros(n, dtype=torch.float64, device="cuda")
        hsh = torch.zeros(n, dtype=torch.int64, device="cuda")
        npd = None if n_par is None else _dev(np.array([n_par], np.int32))
        _lib.glmb_assoc_sample(H_up, _dev(pm_rows.view(np.int32)), _dev(plw[:H]), _dev(d), _dev(ps), 0.9, 1e-3,
                               _dev(rp), _dev(col), _dev(val), _dev(lv), M, 5, 0, alive, theta, logw, hsh,
                               n_parents=npd)
        u = torch.full((n,), 9, dtype=torch.uint8, device="cuda")
        _lib.glmb_dedup(H, H_up, M, alive, theta, hsh, u, n_parents=npd)
        return _host(alive), _host(theta), _host(logw), _host(u)

    a4, t4, l4, u4 = run(pm, 2)
    a2, t2, l2, u2 = run(pm[:2], None)
    n2 = 2 * H_up
    np.testing.assert_array_equal(a4[:n2], a2)
    np.testing.assert_array_equal(t4[:n2], t2)
    np.testing.assert_array_equal(l4[:n2], l2)
    np.testing.assert_array_equal(u4[:n2], u2)
    assert np.all(a4[n2:] == -1) and np.all(t4[n2:] == -5) and np.all(u4[n2:] == 0)


def test_convoy_tracker_small(L):
    """N = 3 objects, 80 steps (P:182-186 shape, scaled down): reruns are bit-identical; after
    the entry phase the MAP cardinality error is small and the matched tracking error is well
    under the detection spread's scale."""
    from paper_2512_06230_b200.scenes import ConvoyConfig
    from paper_2512_06230_b200.tracker import convoy_metrics, run_convoy
    cfg = ConvoyConfig(N=3, K=80, P=512, H_max=20, seed=3)
    recs, ests, truth = run_convoy(cfg, K_cap=256)
    recs2, ests2, _ = run_convoy(cfg, K_cap=256)
    assert [r.n_pairs for r in recs] == [r.n_pairs for r in recs2]
    for e1, e2 in zip(ests, ests2):
        np.testing.assert_array_equal(e1, e2)
    warm = 3 * cfg.delta + 10
    card, dist = convoy_metrics(ests[warm:], truth[warm:])
    assert card <= 0.15, card
    assert dist <= 0.3, dist
    assert max(r.n_kept for r in recs) <= cfg.H_max


def test_glmb_update_one_call_equals_stages(L, orc):
    """glmb_update (one C call) enqueues exactly the stage-by-stage chain: identical outputs."""
    import torch
    from paper_2512_06230_b200 import scenes
    from paper_2512_06230_b200._lib import Particles
    from paper_2512_06230_b200.hyp import HypothesisUpdate, ParticleUpdate, update_params
    sc = scenes.make_scene(1, steps=1)
    cfg = sc.cfg
    Z = sc.Z[0]
    ref = orc.compat(sc.x, sc.y, sc.w, Z, cfg.R, cfg.p_d, cfg.kappa, cfg.gamma)
    C = _dev(ref["C_tracks"].astype(np.float32))
    g = _dev(np.ascontiguousarray(ref["gate"], np.uint32).view(np.int32))
    T, M = C.shape[0], Z.shape[0]
    pm, plw, ps = scenes.hypothesis_inputs(T, 0, 6, seed=2)
    lc = _dev(np.array([-2.0, -0.5, -0.2, -1.0, -3.0]))
    src = Particles.from_arrays([sc.x, sc.y, sc.v, sc.psi, sc.omega, sc.w])
    outs = []
    for one_call in (False, True):
        hu = HypothesisUpdate(T, M, 6, 50, 12)
        pu = ParticleUpdate(T, M, 12, cfg.P)
        est = torch.zeros(T, 3, dtype=torch.float64, device="cuda")
        if one_call:
            prm = update_params(hu, pu, src, C, g, M, _dev(Z), cfg.R, _dev(ps), _dev(pm.view(np.int32)), _dev(plw),
                                cfg.p_d, cfg.kappa, 1e-5, 9, 1, count_lp=lc, est=est)
            L.glmb_update(prm)
        else:
            hu.run(C, g, M, _dev(ps), _dev(pm.view(np.int32)), _dev(plw), cfg.p_d, cfg.kappa, 1e-5, 9, 1,
                   count_lp=lc)
            pu.run(src, _dev(Z), cfg.R, hu.keep_idx, 12, hu.alive, hu.theta, M, 9, 1, n_hyp_dev=hu.n_kept)
            L.glmb_map_estimate(hu.n_kept, pu.pair_of.view(-1)[:T], pu.out, est)
        K = pu.n_pairs_checked()
        nk = int(_host(hu.n_kept)[0])
        outs.append([_host(hu.theta)[:, :M], _host(hu.logw), _host(hu.keep_idx)[:nk], K, _host(pu.out.data)[:, :K],
                     _host(est)])
    a, b = outs
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)

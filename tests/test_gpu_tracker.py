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
    # a set of 4 rows: pairs 5 (past the rows, a K_cap overflow) count as none
    L.glmb_map_estimate(_dev(np.array([4], np.int32)), _dev(pair_of0), s.rows(0, 4), est)
    got4 = _host(est)
    past = pair_of0 >= 4
    assert np.all(got4[past, 2] == 0) and np.all(np.isnan(got4[past, :2]))
    np.testing.assert_array_equal(got4[~past], got[~past])


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


def test_convoy_loop_stagewise_vs_oracle_chain(L, orc):
    """The tracker loop itself against the oracle chain (SURVEY 8(c) protocol 1 applied to f4):
    a convoy of N = 5 objects for 30 updates through ConvoyTracker.update (one glmb_update call
    per step, the tracker's real path).  At every step each stage's GPU input buffers are copied
    to the host and the oracle recomputes that stage from exactly those values: predict (O5),
    birth (O6), compat (O7), death_prob (O9), compat_rows (O10), assoc_sample (O11), dedup (O12),
    prune (O13), assoc_pairs (O14), reweight_pairs (O15), resample (O16, on the GPU's weights),
    map_estimate (O18) and next_parents (O17).  Integer outcomes (gate bits outside the gamma
    band, survival bits, theta, uniqueness, kept indices, pairs, resampling decisions and
    ancestors, parent masks) must match bit for bit; weights and estimates within contract."""
    import torch
    from _parity import check_compat, check_log_norm, check_state, check_weights
    from paper_2512_06230_b200.scenes import ConvoyConfig, convoy_scene
    from paper_2512_06230_b200.tracker import ConvoyTracker, count_log_prior
    cfg = ConvoyConfig(N=5, K=30, seed=4)
    Zs, truth, bm, bc = convoy_scene(cfg)
    M_max = max(len(z) for z in Zs)
    tr = ConvoyTracker(cfg, M_max, K_cap=512)
    tr.reset(bm, bc)
    lc = count_log_prior(cfg, M_max)
    P, B, H, H_up = cfg.P, cfg.B, cfg.H_max, cfg.H_up
    seen_multi_parent = seen_resampled = 0
    for k in range(cfg.K):
        torch.cuda.synchronize()
        T = tr.n_surv
        Tk = T + B
        src = tr.bufs[tr.cur]
        pre = src.data[:, :T].cpu().numpy()
        npar = int(tr.counts[2].item())
        pm = tr.parent_mask[:npar].cpu().numpy().view(np.uint32)
        plw = tr.parent_logw[:npar].cpu().numpy()
        gid = tr.gid[:Tk].cpu().numpy()
        Z = Zs[k]
        M = len(Z)
        rec = tr.update(k, Z)
        torch.cuda.synchronize()
        dst = tr.bufs[tr.cur]
        post = src.data[:, :Tk].cpu().numpy()
        # a1/a3: predict and birth
        if T:
            ref = orc.predict(*pre[:5], gid[:T], cfg.dt, cfg.sigma_a, cfg.sigma_w, cfg.seed, k)
            check_state([a[:T] for a in post[:5]], ref)
            np.testing.assert_array_equal(post[5][:T], pre[5])
        bref = orc.birth(bm, bc, gid[T:Tk], P, cfg.seed, k)
        check_state([a[T:Tk] for a in post[:5]], bref[:5])
        # a4/a5: compat
        C = tr.C_tracks[:Tk, :M].cpu().numpy()
        G = tr.gate[:Tk, :(M + 31) // 32].cpu().numpy().view(np.uint32)
        ref_c = orc.compat(post[0], post[1], post[5], Z, cfg.R, cfg.p_d, cfg.kappa, cfg.gamma)
        check_compat(C, G, tr.C_clutter.cpu().numpy(), ref_c, cfg.gamma, M)
        # f1: death probabilities, CSR rows, the two-stage sampler, dedup (on the GPU's C_k)
        ps = np.concatenate([np.full(T, cfg.p_s), np.full(B, cfg.r_birth)]).astype(np.float32)
        hu, pu = tr.hu, tr.pu
        d = hu.d[:Tk].cpu().numpy()
        np.testing.assert_array_equal(d, orc.death_prob(C, G, cfg.p_d, cfg.kappa, ps).astype(np.float32))
        rp, col, val, lv = orc.compat_rows(C, G, M)
        nnz = int(rp[M])
        np.testing.assert_array_equal(hu.row_ptr[:M + 1].cpu().numpy(), rp)
        np.testing.assert_array_equal(hu.col[:nnz].cpu().numpy(), col)
        np.testing.assert_array_equal(hu.val[:nnz].cpu().numpy(), val)
        np.testing.assert_allclose(hu.ln_val[:nnz].cpu().numpy(), lv, rtol=1e-15)
        n = npar * H_up
        al, th, lw = orc.assoc_sample(pm, plw, H_up, d, ps, cfg.p_d, cfg.kappa, (rp, col, val, lv), M,
                                      cfg.seed, k, count_lp=lc)
        g_al = hu.alive[:n].cpu().numpy().view(np.uint32)
        g_th = hu.theta[:n, :M].cpu().numpy()
        g_lw = hu.logw[:n].cpu().numpy()
        np.testing.assert_array_equal(g_al, al)
        np.testing.assert_array_equal(g_th, th)
        np.testing.assert_allclose(g_lw, lw, rtol=1e-9, atol=1e-9)
        u = hu.unique[:H * H_up].cpu().numpy()
        np.testing.assert_array_equal(u[:n], orc.dedup(g_al, g_th, npar, H_up))
        assert not u[n:].any()
        # f3: normalisation, tau, H_max (on the GPU's log-weights)
        idx, kw = orc.prune(g_lw, u[:n], cfg.tau, H)
        nk = rec.n_kept
        np.testing.assert_array_equal(hu.keep_idx[:nk].cpu().numpy(), idx)
        g_kw = hu.keep_w[:nk].cpu().numpy()
        np.testing.assert_allclose(g_kw, kw, rtol=1e-9)
        # f2: pairs, per-pair update, resampling (on the GPU's kept set and weights)
        r_pt, r_pp, r_pm, r_po = orc.assoc_pairs(idx, g_al, g_th, Tk, M)
        K = rec.n_pairs
        assert K == len(r_pt)
        np.testing.assert_array_equal(pu.pair_track[:K].cpu().numpy(), r_pt)
        np.testing.assert_array_equal(pu.pair_ptr[:K + 1].cpu().numpy(), r_pp)
        np.testing.assert_array_equal(pu.pair_meas[:len(r_pm)].cpu().numpy(), r_pm)
        po = pu.pair_of.view(-1)[:H * Tk].view(H, Tk)[:nk].cpu().numpy()
        np.testing.assert_array_equal(po, r_po)
        r_w, r_lz, r_fl, r_es = orc.reweight_pairs(post[0], post[1], post[5], Z, cfg.R, r_pt, r_pp, r_pm)
        g_w = pu.w_new[:K].cpu().numpy()
        fl = pu.flags[:K].cpu().numpy().view(np.uint32)
        check_weights(g_w, r_w)
        check_log_norm(pu.log_norm[:K].cpu().numpy(), r_lz)
        np.testing.assert_array_equal(fl & 1, r_fl)
        np.testing.assert_allclose(pu.ess[:K].cpu().numpy(), r_es, rtol=1e-4)
        out = dst.data[:, :K].cpu().numpy()
        for q in range(K):
            res, anc = orc.resample(g_w[q], cfg.seed, k, q)
            assert bool(fl[q] & 2) == res, (k, q)
            rows = post[:5, r_pt[q]]
            if res:
                seen_resampled += 1
                np.testing.assert_array_equal(out[:5, q], rows[:, anc])
                assert np.all(out[5, q] == np.float32(1.0 / P))
            else:
                np.testing.assert_array_equal(out[:5, q], rows)
                np.testing.assert_array_equal(out[5, q], g_w[q])
        # f4: MAP estimate and the next parents
        est = tr.est[:Tk].cpu().numpy()
        r_est = orc.map_estimate(nk, po[0], out[0], out[1], out[5])
        np.testing.assert_array_equal(est[:, 2], r_est[:, 2])
        ok = r_est[:, 2] > 0
        np.testing.assert_allclose(est[ok, :2], r_est[ok, :2], rtol=1e-12)
        r_mask, r_plw = orc.next_parents(g_kw, po, Tk, tr.K_cap, B, K, tr.ldt)
        np.testing.assert_array_equal(tr.parent_mask[:nk].cpu().numpy().view(np.uint32), r_mask)
        np.testing.assert_allclose(tr.parent_logw[:nk].cpu().numpy(), r_plw, rtol=1e-15)
        assert int(tr.counts[2].item()) == nk
        seen_multi_parent += npar > 1
    # the run exercised the interesting paths: several parents, resampled pairs, all objects in
    assert seen_multi_parent > 10 and seen_resampled > 0
    assert tr.n_surv >= cfg.N

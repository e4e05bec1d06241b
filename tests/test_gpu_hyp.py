"""GPU parity of the hypothesis machinery (§Approach)
through the C ABI against the fp64 oracle O9-O13 on identical seeded inputs.

Inputs are generator (scenes.synthetic_compat / hypothesis_inputs) or oracle
outputs (oracle.compat on a BASELINE scene), never GPU outputs -- except that
glmb_dedup consumes the fingerprints glmb_assoc_sample emits (an internal hash
with no oracle counterpart), and the dedup result is compared with the
oracle's dedup of the oracle's own samples.

Bars: integer outcomes (CSR, alive bits, theta, unique, kept
indices) bit-exact; d_prob rel 1e-6 (fp64 rounded once to fp32); ln_val rel
1e-15; logw |d| <= 1e-9 max(1, |ref|) (fp64 sums of ~T + M logs in another
order); kept weights rel 1e-9."""
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


def _oracle_C(orc, cfg_id):
    """fp32 C_k and gate of a BASELINE scene from the oracle's compat (O7)."""
    from paper_2512_06230_b200 import scenes
    sc = scenes.make_scene(cfg_id, steps=1)
    cfg = sc.cfg
    Z = sc.Z[0]
    ref = orc.compat(sc.x, sc.y, sc.w, Z, cfg.R, cfg.p_d, cfg.kappa, cfg.gamma)
    C = ref["C_tracks"].astype(np.float32)
    return C, np.ascontiguousarray(ref["gate"], np.uint32), Z.shape[0], cfg


def _gpu_rows(L, C, g, M, cap=None):
    import torch
    T = C.shape[0]
    cap = max(1, T * M) if cap is None else cap
    rp = torch.zeros(M + 1, dtype=torch.int32, device="cuda")
    col = torch.full((cap,), -7, dtype=torch.int32, device="cuda")
    val = torch.zeros(cap, dtype=torch.float32, device="cuda")
    lv = torch.zeros(cap, dtype=torch.float64, device="cuda")
    L.glmb_compat_rows(_dev(C), _dev(g.view(np.int32)), M, rp, col, val, lv)
    return _host(rp), _host(col), _host(val), _host(lv)


def _gpu_sample(L, H_up, pm, plw, d, ps, p_d, kappa, rows, M, seed, step, ldm=None, count_lp=None):
    import torch
    H_old, ldt = pm.shape
    n = H_old * H_up
    ldm = max(4, (M + 3) // 4 * 4) if ldm is None else ldm
    rp, col, val, lv = rows
    one = lambda a, dt: a if len(a) else np.zeros(1, dt)
    alive = torch.full((n, ldt), -1, dtype=torch.int32, device="cuda")
    theta = torch.full((n, ldm), -5, dtype=torch.int32, device="cuda")
    logw = torch.zeros(n, dtype=torch.float64, device="cuda")
    hsh = torch.zeros(n, dtype=torch.int64, device="cuda")
    L.glmb_assoc_sample(H_up, _dev(pm.view(np.int32)), _dev(plw), _dev(np.asarray(d, np.float32)),
                        _dev(np.asarray(ps, np.float32)), p_d, kappa, _dev(rp), _dev(one(col, np.int32)),
                        _dev(one(val, np.float32)), _dev(one(lv, np.float64)), M, seed, step,
                        alive, theta, logw, hsh, count_lp=None if count_lp is None else _dev(count_lp))
    return (_host(alive).view(np.uint32), _host(theta), _host(logw), _host(hsh))


def _check_logw(g, r):
    with np.errstate(invalid="ignore"):
        d = np.abs(np.asarray(g) - np.asarray(r))
    same_inf = np.isinf(g) & np.isinf(r) & (np.sign(g) == np.sign(r))
    ok = same_inf | (d <= 1e-9 * np.maximum(1.0, np.abs(r)))
    assert ok.all(), f"{(~ok).sum()} log-weights off; worst {d[~ok].max():.3e}"


# ------------------------------------------------------------------ O9
@pytest.mark.parametrize("src", ["cfg1", "synthetic"])
def test_death_prob(L, orc, src):
    import torch
    from paper_2512_06230_b200 import scenes
    if src == "cfg1":
        C, g, M, cfg = _oracle_C(orc, 1)
        p_d, kappa = cfg.p_d, cfg.kappa
    else:
        C, g = scenes.synthetic_compat(300, 517, 5)
        M, p_d, kappa = 517, 0.9, 7.5e-5
    T = C.shape[0]
    rng = np.random.default_rng(1)
    ps = rng.uniform(0.5, 1.0, T).astype(np.float32)
    ps[::7] = 1.0                                       # certain survival -> d = 0
    ref = orc.death_prob(C, g, p_d, kappa, ps)
    d = torch.zeros(T, dtype=torch.float32, device="cuda")
    L.glmb_death_prob(_dev(C), _dev(g.view(np.int32)), M, p_d, kappa, _dev(ps), d)
    got = _host(d).astype(np.float64)
    np.testing.assert_allclose(got, ref, rtol=1e-6, atol=0)
    # IEEE-exact fp64 steps on both sides: the fp32 result is the oracle's, rounded once
    np.testing.assert_array_equal(got.astype(np.float32), ref.astype(np.float32))
    assert np.all(got[::7] == 0.0)


# ------------------------------------------------------------------ O10
@pytest.mark.parametrize("shape", [(68, None), (1, 1), (5, 33), (300, 517), (1040, 1198), (0, 40), (7, 0)])
def test_compat_rows_bit_exact(L, orc, shape):
    from paper_2512_06230_b200 import scenes
    T, M = shape
    if M is None:
        C, g, M, _ = _oracle_C(orc, 1)
    else:
        C, g = scenes.synthetic_compat(T, M, T + M, mean_gated=2.5)
    rp, col, val, lv = _gpu_rows(L, C, g, M)
    r_rp, r_col, r_val, r_lv = orc.compat_rows(C, g, M)
    np.testing.assert_array_equal(rp, r_rp)
    n = int(r_rp[M])
    np.testing.assert_array_equal(col[:n], r_col)
    np.testing.assert_array_equal(val[:n].view(np.uint32), r_val.view(np.uint32))
    np.testing.assert_allclose(lv[:n], r_lv, rtol=1e-15, atol=0)
    if T * M > n:
        assert np.all(col[n:] == -7)                      # nothing past nnz written


def test_compat_rows_capacity(L, orc):
    from paper_2512_06230_b200 import scenes
    C, g = scenes.synthetic_compat(50, 200, 3, mean_gated=3.0)
    r_rp, r_col, _, _ = orc.compat_rows(C, g, 200)
    n = int(r_rp[200])
    cap = n // 2
    rp, col, val, lv = _gpu_rows(L, C, g, 200, cap=cap)
    np.testing.assert_array_equal(rp, r_rp)               # row_ptr[M] = nnz > cap reports the overflow
    np.testing.assert_array_equal(col[:cap], r_col[:cap])


# ------------------------------------------------------------------ O11 (+ hash)
def _sample_case(orc, name):
    from paper_2512_06230_b200 import scenes
    if name == "cfg1":
        C, g, M, cfg = _oracle_C(orc, 1)
        T = C.shape[0]
        pm, plw, ps = scenes.hypothesis_inputs(T, 0, 4, seed=11)   # C holds the survivors
        d = orc.death_prob(C, g, cfg.p_d, cfg.kappa, ps).astype(np.float32)
        return C, g, M, pm, plw, ps, d, cfg.p_d, cfg.kappa, 64
    if name == "cfg3-shaped":
        T, B, M = 1024, 16, 1198
        C, g = scenes.synthetic_compat(T + B, M, 3)
        pm, plw, ps = scenes.hypothesis_inputs(T, B, 16, seed=3)
        d = orc.death_prob(C, g, 0.9, 7.5e-5, ps).astype(np.float32)
        return C, g, M, pm, plw, ps, d, 0.9, 7.5e-5, 24
    if name == "dense-rows":       # many gated tracks per row: long inverse-CDF scans
        T, M = 40, 90
        C, g = scenes.synthetic_compat(T, M, 9, mean_gated=12.0)
        pm, plw, ps = scenes.hypothesis_inputs(T, 0, 3, seed=9, p_in_parent=0.7)
        d = np.random.default_rng(9).uniform(0, 0.8, T).astype(np.float32)
        return C, g, M, pm, plw, ps, d, 0.95, 1e-3, 200
    if name == "no-measurements":
        T, M = 37, 0
        C, g = np.zeros((T, 0), np.float32), np.zeros((T, 1), np.uint32)
        pm, plw, ps = scenes.hypothesis_inputs(T, 0, 2, seed=2)
        d = np.random.default_rng(2).uniform(0, 1, T).astype(np.float32)
        return C, g, M, pm, plw, ps, d, 0.9, 1e-3, 50
    if name == "kappa-zero":       # clutter impossible: ln kappa = -inf rows where nothing is gated
        T, M = 12, 30
        C, g = scenes.synthetic_compat(T, M, 4, mean_gated=2.0)
        pm, plw, ps = scenes.hypothesis_inputs(T, 0, 2, seed=4)
        d = np.zeros(T, np.float32)
        return C, g, M, pm, plw, ps, d, 0.9, 0.0, 20
    raise KeyError(name)


@pytest.mark.parametrize("name", ["cfg1", "cfg3-shaped", "dense-rows", "no-measurements", "kappa-zero"])
def test_assoc_sample_vs_oracle(L, orc, name):
    C, g, M, pm, plw, ps, d, p_d, kappa, H_up = _sample_case(orc, name)
    rows = orc.compat_rows(C, g, M)
    seed, step = 0xC0FFEE_1234, 5
    al, th, lw, hs = _gpu_sample(L, H_up, pm, plw, d, ps, p_d, kappa, rows, M, seed, step)
    r_al, r_th, r_lw = orc.assoc_sample(pm, plw, H_up, d, ps, p_d, kappa, rows, M, seed, step)
    np.testing.assert_array_equal(al, r_al)
    np.testing.assert_array_equal(th[:, :M], r_th)
    if th.shape[1] > M:
        assert np.all(th[:, M:] == -5)                    # padding past M untouched
    _check_logw(lw, r_lw)
    # fingerprint: equal (alive, theta) -> equal hash
    keys = {}
    for q in range(al.shape[0]):
        k = (al[q].tobytes(), th[q, :M].tobytes())
        if k in keys:
            assert hs[q] == hs[keys[k]]
        else:
            keys[k] = q


def test_assoc_sample_forced_and_launch_invariance(L, orc):
    """d = 1: nothing survives, all clutter; d = 0 inside the parent: exactly the parent survives.
    A different H_old split of the same parents gives the same samples (the draws are keyed by h, s)."""
    from paper_2512_06230_b200 import scenes
    T, M = 70, 100
    C, g = scenes.synthetic_compat(T, M, 1)
    rows = orc.compat_rows(C, g, M)
    pm, plw, ps = scenes.hypothesis_inputs(T, 0, 3, seed=1)
    al, th, lw, _ = _gpu_sample(L, 16, pm, plw, np.ones(T), ps, 0.9, 1e-3, rows, M, 1, 0)
    assert np.all(al == 0) and np.all(th[:, :M] == 0)
    al, th, lw, _ = _gpu_sample(L, 16, pm, plw, np.zeros(T), ps, 0.9, 1e-3, rows, M, 1, 0)
    np.testing.assert_array_equal(al, np.repeat(pm, 16, axis=0))
    full = _gpu_sample(L, 16, pm, plw, np.full(T, 0.3), ps, 0.9, 1e-3, rows, M, 1, 0)
    # ldm padding does not change the result
    wide = _gpu_sample(L, 16, pm, plw, np.full(T, 0.3), ps, 0.9, 1e-3, rows, M, 1, 0, ldm=128)
    np.testing.assert_array_equal(full[1][:, :M], wide[1][:, :M])
    np.testing.assert_array_equal(full[2], wide[2])


# ------------------------------------------------------------------ O12
@pytest.mark.parametrize("name", ["cfg1", "dense-rows", "no-measurements"])
def test_dedup_vs_oracle(L, orc, name):
    import torch
    C, g, M, pm, plw, ps, d, p_d, kappa, H_up = _sample_case(orc, name)
    if name != "dense-rows":     # concentrate the posterior so duplicates are common
        d = np.minimum(d, np.float32(0.02))
    rows = orc.compat_rows(C, g, M)
    al, th, lw, hs = _gpu_sample(L, H_up, pm, plw, d, ps, p_d, kappa, rows, M, 77, 1)
    r_al, r_th, _ = orc.assoc_sample(pm, plw, H_up, d, ps, p_d, kappa, rows, M, 77, 1)
    ref = orc.dedup(r_al, r_th, pm.shape[0], H_up)
    if name != "dense-rows":
        assert ref.sum() < len(ref)                       # the case has duplicates
    n = al.shape[0]
    ldm = th.shape[1]
    u = torch.zeros(n, dtype=torch.uint8, device="cuda")
    L.glmb_dedup(pm.shape[0], H_up, M, _dev(al.view(np.int32)), _dev(th), _dev(hs), u)
    np.testing.assert_array_equal(_host(u), ref)
    # exactness does not rest on the fingerprint: all-equal hashes give the same answer
    u2 = torch.zeros(n, dtype=torch.uint8, device="cuda")
    L.glmb_dedup(pm.shape[0], H_up, M, _dev(al.view(np.int32)), _dev(th), _dev(np.zeros(n, np.int64)), u2)
    np.testing.assert_array_equal(_host(u2), ref)
    assert ldm >= M


def test_dedup_large_parent(L, orc):
    """H_up = 5000 samples of one parent (more than one shared-memory hash tile)."""
    import torch
    from paper_2512_06230_b200 import scenes
    T, M = 6, 5
    C, g = scenes.synthetic_compat(T, M, 8, mean_gated=1.0)
    rows = orc.compat_rows(C, g, M)
    pm, plw, ps = scenes.hypothesis_inputs(T, 0, 1, seed=8)
    d = np.full(T, 0.2, np.float32)
    H_up = 5000
    al, th, lw, hs = _gpu_sample(L, H_up, pm, plw, d, ps, 0.9, 0.05, rows, M, 3, 0)
    r_al, r_th, _ = orc.assoc_sample(pm, plw, H_up, d, ps, 0.9, 0.05, rows, M, 3, 0)
    ref = orc.dedup(r_al, r_th, 1, H_up)
    u = torch.zeros(H_up, dtype=torch.uint8, device="cuda")
    L.glmb_dedup(1, H_up, M, _dev(al.view(np.int32)), _dev(th), _dev(hs), u)
    np.testing.assert_array_equal(_host(u), ref)


# ------------------------------------------------------------------ O13
def _gpu_prune(L, lw, uq, tau, h_max):
    import torch
    n = len(lw)
    ki = torch.full((max(h_max, 1),), -1, dtype=torch.int32, device="cuda")
    kw = torch.zeros(max(h_max, 1), dtype=torch.float64, device="cuda")
    nk = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    ws = torch.zeros(max(n, 1), dtype=torch.int64, device="cuda")
    L.glmb_prune(_dev(np.asarray(lw, np.float64)), _dev(np.asarray(uq, np.uint8)), tau, h_max, ws, ki, kw, nk)
    k = int(_host(nk)[0])
    return _host(ki)[:k], _host(kw)[:k]


@pytest.mark.parametrize("n,tau,h_max", [(10000, 1e-5, 100), (10000, 0.0, 5), (3000, 1e-3, 4096),
                                         (257, 0.0, 1000), (1, 0.5, 3), (20000, 1e-5, 16384)])
def test_prune_vs_oracle(L, orc, n, tau, h_max):
    rng = np.random.default_rng(n + h_max)
    lw = rng.normal(-50.0, 4.0, n)
    uq = (rng.random(n) < 0.8).astype(np.uint8)
    uq[0] = 1
    idx, w = _gpu_prune(L, lw, uq, tau, h_max)
    r_idx, r_w = orc.prune(lw, uq, tau, h_max)
    np.testing.assert_array_equal(idx, r_idx)
    np.testing.assert_allclose(w, r_w, rtol=1e-9, atol=0)


def test_prune_ties_and_edges(L, orc):
    # equal weights: ties broken by index; the threshold tie is split exactly at h_max
    lw = np.zeros(3000)
    uq = np.ones(3000, np.uint8)
    uq[::3] = 0
    idx, w = _gpu_prune(L, lw, uq, 0.0, 700)
    r_idx, r_w = orc.prune(lw, uq, 0.0, 700)
    np.testing.assert_array_equal(idx, r_idx)
    np.testing.assert_allclose(w, r_w, rtol=1e-12)
    # SPEC S:334 example and the always-kept maximiser
    idx, w = _gpu_prune(L, np.log([0.6, 0.3, 0.05, 0.05]), np.ones(4, np.uint8), 0.1, 2)
    np.testing.assert_array_equal(idx, [0, 1])
    np.testing.assert_allclose(w, [2 / 3, 1 / 3], rtol=1e-12)
    idx, w = _gpu_prune(L, np.log([0.25] * 4), np.array([1, 0, 1, 1], np.uint8), 0.9, 5)
    np.testing.assert_array_equal(idx, [0])
    idx, w = _gpu_prune(L, np.full(5, -1e4), np.zeros(5, np.uint8), 0.0, 5)   # nothing unique
    assert len(idx) == 0
    idx, w = _gpu_prune(L, np.array([-3000.0, -3001.0, -2999.5]), np.ones(3, np.uint8), 0.0, 2)
    r_idx, r_w = orc.prune(np.array([-3000.0, -3001.0, -2999.5]), np.ones(3, np.uint8), 0.0, 2)
    np.testing.assert_array_equal(idx, r_idx)
    np.testing.assert_allclose(w, r_w, rtol=1e-12)


# ------------------------------------------------------------------ the chain
def test_hypothesis_update_chain(L, orc):
    """death_prob -> rows -> sample -> dedup -> prune through hyp.HypothesisUpdate on a cfg1
    C_k vs the oracle chain O9 -> O13 (H_old = 10, H_up = 100, tau = 1e-5, H_max = 25: P:186)."""
    import torch
    from paper_2512_06230_b200 import scenes
    from paper_2512_06230_b200.hyp import HypothesisUpdate
    C, g, M, cfg = _oracle_C(orc, 1)
    T = C.shape[0]
    H_old, H_up, h_max, tau = 10, 100, 25, 1e-5
    pm, plw, ps = scenes.hypothesis_inputs(T, 0, H_old, seed=21)
    hu = HypothesisUpdate(T, M, H_old, H_up, h_max)
    hu.run(_dev(C), _dev(g.view(np.int32)), M, _dev(ps), _dev(pm.view(np.int32)), _dev(plw),
           cfg.p_d, cfg.kappa, tau, seed=99, step=3)
    torch.cuda.synchronize()
    d = orc.death_prob(C, g, cfg.p_d, cfg.kappa, ps)
    d32 = d.astype(np.float32)
    np.testing.assert_array_equal(_host(hu.d)[:T], d32)
    rows = orc.compat_rows(C, g, M)
    r_al, r_th, r_lw = orc.assoc_sample(pm, plw, H_up, d32, ps, cfg.p_d, cfg.kappa, rows, M, 99, 3)
    np.testing.assert_array_equal(_host(hu.alive).view(np.uint32), r_al)
    np.testing.assert_array_equal(_host(hu.theta)[:, :M], r_th)
    _check_logw(_host(hu.logw), r_lw)
    r_u = orc.dedup(r_al, r_th, H_old, H_up)
    np.testing.assert_array_equal(_host(hu.unique), r_u)
    r_idx, r_w = orc.prune(r_lw, r_u, tau, h_max)
    k = int(_host(hu.n_kept)[0])
    np.testing.assert_array_equal(_host(hu.keep_idx)[:k], r_idx)
    np.testing.assert_allclose(_host(hu.keep_w)[:k], r_w, rtol=1e-9)


@pytest.mark.parametrize("name", ["cfg1", "dense-rows", "cfg3-shaped"])
def test_assoc_sample_count_prior(L, orc, name):
    """The per-track measurement-count prior (Poisson(D) over C's P_D factor) vs O11."""
    import math
    C, g, M, pm, plw, ps, d, p_d, kappa, H_up = _sample_case(orc, name)
    D = 2.5
    pd32 = float(np.float32(p_d))
    lc = np.array([-D + n * math.log(D) - n * math.log(pd32) for n in range(12)])
    rows = orc.compat_rows(C, g, M)
    al, th, lw, hs = _gpu_sample(L, H_up, pm, plw, d, ps, p_d, kappa, rows, M, 31, 2, count_lp=lc)
    r_al, r_th, r_lw = orc.assoc_sample(pm, plw, H_up, d, ps, p_d, kappa, rows, M, 31, 2, count_lp=lc)
    np.testing.assert_array_equal(al, r_al)
    np.testing.assert_array_equal(th[:, :M], r_th)
    _check_logw(lw, r_lw)


@pytest.mark.parametrize("pool", [1024, 4096])
def test_assoc_sample_small_pool(pool):
    """The sampler's shared-memory fallbacks: GLMB_SAMPLER_POOL forces a small pool, so the
    row filter takes the per-row passes (1 KB: no room for the kept-entry bitmap) or keeps
    the bitmap but walks the global CSR, and the ln P_S cache covers few or no parent
    quads.  The oracle parity tests above must pass unchanged (run in a subprocess: the
    launcher reads the variable once)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, GLMB_SAMPLER_POOL=str(pool))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_hyp.py"), "-k", "assoc_sample_vs_oracle or count_prior",
                        "-m", "gpu"], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "passed" in r.stdout


def test_plain_launches_without_pdl():
    """GLMB_PDL=0 (plain launches, no programmatic serialization): the sampler, update-chain
    and tracker parity tests pass unchanged (child process: the knob is read once)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, GLMB_PDL="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_hyp.py"), os.path.join(here, "test_gpu_tracker.py"),
                        "-k", "assoc_sample_vs_oracle or hypothesis_update_chain or one_call or convoy",
                        "-m", "gpu"], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "passed" in r.stdout

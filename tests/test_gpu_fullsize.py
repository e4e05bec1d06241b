"""GPU parity at BASELINE.json's full sizes, through the same GlmbStep buffers and
launch configuration bench.py times.  Every output of config 3 and 64 columns per rank block of
config 4 are checked against the oracle, config 2 stage by stage over its 50 steps; whole-matrix
properties (that hold at any size) are checked everywhere.  Every stage is fed generator / oracle
inputs, except config 2's sequence, whose stage inputs are the GPU's buffers copied to the host
(the oracle recomputes each stage from exactly those fp32 values)."""
import numpy as np
import pytest
import torch

from conftest import gpu_available
from _parity import check_compat, check_log_norm, check_state, check_weights, unpack_gate

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA GPU")]


@pytest.fixture(scope="module")
def L():
    from paper_2512_06230_b200 import _lib
    from paper_2512_06230_b200.build import build
    build()
    torch.cuda.set_device(0)
    _lib.glmb_init(0)
    return _lib


def _whole_matrix_properties(C, G, Cc, M, T, c):
    """Properties of C_k at any size: finite, 0 <= C <= P_D / (2 pi sqrt(det R)),
    gate bit <=> C > 0 (C = P_D L >= P_D gamma when gated), clutter column = kappa."""
    C = C[:T, :M]
    assert np.isfinite(C).all()
    det = c.R[0] * c.R[2] - c.R[1] ** 2
    assert C.min() >= 0 and C.max() <= np.float32(c.p_d) / (2 * np.pi * np.sqrt(det)) * (1 + 1e-5)
    bits = unpack_gate(G[:T], M)
    np.testing.assert_array_equal(bits, C > 0)
    assert np.all(C[bits] >= np.float32(c.p_d) * np.float32(c.gamma) * (1 - 1e-6))
    np.testing.assert_array_equal(Cc[:M], np.float32(c.kappa))


def _gated_band_bound(nband, ref_c, gamma):
    """SURVEY 8(c) protocol 4: the gate-band exclusions stay << 0.1 % of the gated-in entries."""
    gated = int((ref_c["L"] >= np.float32(gamma)).sum())
    assert gated > 0
    assert nband <= 1e-3 * gated, f"{nband} band exclusions for {gated} gated entries"
    return gated


def test_cfg3_full_size_every_entry(L, orc):
    """Config 3 (T=1024 + 16 births, P=8192, M~1200) in the bench launch configuration, every
    output against the oracle: all 8.4 M predicted particles (O5), all 16 x 8192 birth particles
    (O6), every entry of C_k and every gate word (O7; band count bounded), every reweighted
    track (O8).  Stage inputs are the generator's (survivors) and the oracle's (births)."""
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    s = make_scene(3, steps=1)
    c = s.cfg
    st = GlmbStep(s)
    k = 0
    st.predict(k)
    st.birth(k)
    torch.cuda.synchronize()
    got = st.particles.data.cpu().numpy()
    ref = orc.predict(s.x, s.y, s.v, s.psi, s.omega, s.gid, c.dt, c.sigma_a, c.sigma_w, st.seed, k)
    check_state([g[:c.T] for g in got[:5]], ref)
    np.testing.assert_array_equal(got[5][:c.T], s.w)                  # predict leaves w alone
    del ref
    bref = orc.birth(s.birth_mean, s.birth_chol, s.birth_gid, c.P, st.seed, k)
    check_state([g[c.T:] for g in got[:5]], bref[:5])
    np.testing.assert_allclose(got[5][c.T:], bref[5], rtol=1e-7)
    # compat + reweight on generator survivors and oracle births (fp32)
    births32 = [r.astype(np.float32) for r in bref]
    inp = np.stack([np.concatenate([a, b]) for a, b in
                    zip((s.x, s.y, s.v, s.psi, s.omega, s.w), births32)])
    del got, bref, births32
    st.particles.data.copy_(torch.from_numpy(inp))
    st.compat(k)
    torch.cuda.synchronize()
    C = st.out.C_tracks.cpu().numpy()
    G = st.out.gate.cpu().numpy().view(np.uint32)
    Cc = st.out.C_clutter.cpu().numpy()
    M = len(s.Z[0])
    Tk = c.T + c.B
    _whole_matrix_properties(C, G, Cc, M, Tk, c)
    ref_c = orc.compat(inp[0], inp[1], inp[5], s.Z[0], c.R, c.p_d, c.kappa, c.gamma)
    nband, rel = check_compat(C[:Tk], G[:Tk], Cc, ref_c, c.gamma, M)
    gated = _gated_band_bound(nband, ref_c, c.gamma)
    print(f"cfg3 compat: {Tk} x {M} entries, {gated} gated, {nband} in the band, worst rel {rel:.2e}")
    del ref_c
    st.reweight(k)
    torch.cuda.synchronize()
    w = st.particles.data[5].cpu().numpy()
    rw, rln, rfl = orc.reweight(inp[0], inp[1], inp[5], s.Z[0], c.R, s.theta[0], 0)
    check_weights(w, rw)
    check_log_norm(st.out.log_norm.cpu().numpy(), rln)
    np.testing.assert_array_equal(st.out.flags.cpu().numpy().view(np.uint32), rfl)
    assigned = np.unique(s.theta[0][s.theta[0] > 0]) - 1
    assert len(assigned) > 0.8 * c.T
    np.testing.assert_allclose(w[assigned].astype(np.float64).sum(1), 1.0, rtol=2e-5)


def test_cfg4_full_size_rank_blocks(L, orc):
    """Config 4 (T=4096, P=8192, M~4700) on one GPU: 64 oracle columns in each of the W=8 rank
    blocks, whole-matrix properties, and the W=8 column blocks launched one by
    one reproduce the W=1 matrix bit for bit."""
    from paper_2512_06230_b200 import _lib
    from paper_2512_06230_b200.dist import ShardPlan
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    s = make_scene(4, steps=1)
    c = s.cfg
    st = GlmbStep(s)
    st.compat(0)
    torch.cuda.synchronize()
    M = len(s.Z[0])
    C = st.out.C_tracks.cpu().numpy()
    G = st.out.gate.cpu().numpy().view(np.uint32)
    _whole_matrix_properties(C, G, st.out.C_clutter.cpu().numpy(), M, c.T, c)
    plan = ShardPlan(c.T, 8)
    rng = np.random.default_rng(44)
    cols = np.concatenate([np.sort(rng.choice(plan.cols(r), 64, replace=False)) for r in range(8)])
    ref = orc.compat(s.x[cols], s.y[cols], s.w[cols], s.Z[0], c.R, c.p_d, c.kappa, c.gamma)
    nband, rel = check_compat(C[cols], G[cols], None, ref, c.gamma, M)
    _gated_band_bound(nband, ref, c.gamma)
    for r in range(8):
        blk = plan.cols(r)
        sub = _lib.Particles(st.particles.data[:, blk.start:blk.stop].contiguous(), c.P)
        Cs = torch.zeros(len(blk), st.ldc, device="cuda")
        Gs = torch.zeros(len(blk), st.ldg, dtype=torch.int32, device="cuda")
        _lib.glmb_compat(sub, st.Z[0], c.R, c.p_d, c.kappa, c.gamma, None, Cs, Gs)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(Cs.cpu().numpy()[:, :M], C[blk.start:blk.stop, :M])
        np.testing.assert_array_equal(Gs.cpu().numpy().view(np.uint32), G[blk.start:blk.stop])


@pytest.mark.parametrize("n_pred", [0, 25])
def test_cfg3_exact_skip_vs_oracle(L, orc, n_pred):
    """glmb_compat_skipping at the full config 3 (1024 survivors + 16 births, every column)
    against the oracle directly -- not only against the dense pass -- on compact (step-0)
    clouds, where most tiles are skipped, and on the diffused clouds after 25 predicts (the
    bench's timed steps).  C and the gate words are bit-identical to glmb_compat's, and the
    device counter reports how many pairs were skipped (the bench's evaluated-pair count)."""
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    s = make_scene(3, steps=1)
    c = s.cfg
    st = GlmbStep(s)
    for k in range(n_pred):
        st.predict(k)
    st.birth(0)
    st.compat(0)
    M = len(s.Z[0])
    Cs = torch.full_like(st.out.C_tracks, -1.0)
    Gs = torch.full_like(st.out.gate, -1)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    L.glmb_compat_skipping(st.particles, st.Z[0], c.R, c.p_d, c.kappa, c.gamma, None, Cs, Gs, cnt)
    torch.cuda.synchronize()
    ldg = (M + 31) // 32
    np.testing.assert_array_equal(Cs.cpu().numpy()[:, :M].view(np.uint32),
                                  st.out.C_tracks.cpu().numpy()[:, :M].view(np.uint32))
    np.testing.assert_array_equal(Gs.cpu().numpy()[:, :ldg], st.out.gate.cpu().numpy()[:, :ldg])
    skipped = int(cnt.item())
    total = M * st.T_local * c.P
    assert 0 < skipped < total
    d = st.particles.data.cpu().numpy()
    ref = orc.compat(d[0], d[1], d[5], s.Z[0], c.R, c.p_d, c.kappa, c.gamma)
    nband, rel = check_compat(Cs.cpu().numpy(), Gs.cpu().numpy().view(np.uint32), None, ref, c.gamma, M)
    _gated_band_bound(nband, ref, c.gamma)
    print(f"cfg3 exact skip after {n_pred} predicts: {skipped / total:.3f} of the pairs skipped")


def test_cfg2_sequence_stagewise_vs_oracle(L, orc):
    """Config 2, all 50 steps (SURVEY 8(c) protocol 1): at every step each GPU stage's input
    buffers are copied to the host and the oracle recomputes that stage from those exact fp32
    values -- predict (O5) on the GPU's state before the step, compat (O7) on the GPU's
    predicted state, reweight (O8) under BASELINE configs[2]'s nearest-gate theta, computed
    from the ORACLE's C_k (oracle.nearest_gate_theta) and fed to both sides."""
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    s = make_scene(2)
    c = s.cfg
    assert c.steps == 50 and c.B == 0
    st = GlmbStep(s)
    gid = st.gid.cpu().numpy()
    n_band = n_gated = n_assigned = 0
    for k in range(c.steps):
        pre = st.particles.data.cpu().numpy()
        st.predict(k)
        torch.cuda.synchronize()
        post = st.particles.data.cpu().numpy()
        ref = orc.predict(*pre[:5], gid, c.dt, c.sigma_a, c.sigma_w, st.seed, k)
        check_state(post[:5], ref)
        np.testing.assert_array_equal(post[5], pre[5])
        Zk = s.Z[k]
        M = len(Zk)
        st.compat(k)
        torch.cuda.synchronize()
        ref_c = orc.compat(post[0], post[1], post[5], Zk, c.R, c.p_d, c.kappa, c.gamma)
        nb, _ = check_compat(st.out.C_tracks.cpu().numpy(), st.out.gate.cpu().numpy().view(np.uint32),
                             st.out.C_clutter.cpu().numpy(), ref_c, c.gamma, M)
        n_band += nb
        n_gated += int((ref_c["L"] >= np.float32(c.gamma)).sum())
        theta = orc.nearest_gate_theta(ref_c)
        n_assigned += int((theta > 0).sum())
        st.reweight(k, theta=torch.from_numpy(theta).cuda())
        torch.cuda.synchronize()
        rw, rln, rfl = orc.reweight(post[0], post[1], post[5], Zk, c.R, theta, 0)
        check_weights(st.particles.data[5].cpu().numpy(), rw)
        check_log_norm(st.out.log_norm.cpu().numpy(), rln)
        np.testing.assert_array_equal(st.out.flags.cpu().numpy().view(np.uint32), rfl)
    assert n_assigned > 0.5 * c.steps * c.T
    assert n_band <= 1e-3 * n_gated


def test_compat_large_M_row_permutation_bit_exact(L):
    """K = 4 measurement slots per thread (packed pairs, FMA-pipe exps): permuting Z's rows
    permutes C's rows bit for bit."""
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    s = make_scene(3, rows=range(0, 24), steps=1)
    st = GlmbStep(s, cols=range(0, 24))
    st.compat(0)
    C = st.out.C_tracks.clone()
    M = len(s.Z[0])
    perm = np.random.default_rng(0).permutation(M)
    st.compat(0, Z=torch.from_numpy(s.Z[0][perm].copy()).cuda())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(st.out.C_tracks.cpu().numpy()[:, :M], C.cpu().numpy()[:, perm])
    assert (C.cpu().numpy() > 0).sum() > 0


def test_cfg2_sequence_properties_and_determinism(L):
    """Config 2: 50 filter steps through glmb_step.  Per step: every assigned track's
    weights sum to 1, no degenerate flags, C's whole-matrix properties; two runs are
    bit-identical (counter-based noise, fixed reduction orders)."""
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    s = make_scene(2)
    c = s.cfg
    runs = []
    for rep in range(2):
        st = GlmbStep(s)
        for k in range(c.steps):
            st.run(k)
            if rep == 0 and k % 10 == 9:
                torch.cuda.synchronize()
                M = len(s.Z[k])
                _whole_matrix_properties(st.out.C_tracks.cpu().numpy(), st.out.gate.cpu().numpy().view(np.uint32),
                                         st.out.C_clutter.cpu().numpy(), M, c.T, c)
                w = st.particles.data[5].cpu().numpy().astype(np.float64)
                assigned = np.unique(s.theta[k][s.theta[k] > 0]) - 1
                np.testing.assert_allclose(w[assigned].sum(1), 1.0, rtol=2e-5)
                assert np.isfinite(st.particles.data.cpu().numpy()).all()
        torch.cuda.synchronize()
        runs.append((st.particles.data.cpu().numpy(), st.out.C_tracks.cpu().numpy(), st.out.log_norm.cpu().numpy()))
    for a, b in zip(*runs):
        np.testing.assert_array_equal(a, b)

"""GPU parity at BASELINE.json's full sizes, through the same GlmbStep buffers and
launch configuration bench.py times.  Sampled columns are checked against the
oracle one by one; whole-matrix properties (that hold at any size) are checked
everywhere.  Every stage is fed generator / oracle inputs, never GPU outputs."""
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


def test_cfg3_full_size_sampled_columns(L, orc):
    """Config 3 (T=1024 + 16 births, P=8192, M~1200) in the bench launch configuration."""
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    s = make_scene(3, steps=1)
    c = s.cfg
    st = GlmbStep(s)
    k = 0
    sample = [0, 1, 217, 511, 730, 1023]            # survivor columns
    bsample = [0, 15]                                # birth columns (T + b)
    # predict + birth on the generator state
    st.predict(k)
    st.birth(k)
    torch.cuda.synchronize()
    got = st.particles.data.cpu().numpy()
    gen = [a[sample] for a in (s.x, s.y, s.v, s.psi, s.omega)]
    ref = orc.predict(*gen, s.gid[sample], c.dt, c.sigma_a, c.sigma_w, st.seed, k)
    check_state([g[sample] for g in got[:5]], ref)
    bref = orc.birth(s.birth_mean, s.birth_chol, s.birth_gid, c.P, st.seed, k)
    check_state([g[[c.T + b for b in bsample]] for g in got[:5]], [r[bsample] for r in bref[:5]])
    # compat + reweight on generator survivors and oracle births (fp32)
    births32 = [r.astype(np.float32) for r in bref]
    inp = np.stack([np.concatenate([a, b]) for a, b in
                    zip((s.x, s.y, s.v, s.psi, s.omega, s.w), births32)])
    st.particles.data.copy_(torch.from_numpy(inp))
    st.compat(k)
    torch.cuda.synchronize()
    C = st.out.C_tracks.cpu().numpy()
    G = st.out.gate.cpu().numpy().view(np.uint32)
    Cc = st.out.C_clutter.cpu().numpy()
    M = len(s.Z[0])
    Tk = c.T + c.B
    _whole_matrix_properties(C, G, Cc, M, Tk, c)
    cols = sample + [c.T + b for b in bsample]
    ref_c = orc.compat(inp[0][cols], inp[1][cols], inp[5][cols], s.Z[0], c.R, c.p_d, c.kappa, c.gamma)
    nband, rel = check_compat(C[cols], G[cols], None, ref_c, c.gamma, M)
    assert (ref_c["L"] >= c.gamma).sum() > 0
    st.reweight(k)
    torch.cuda.synchronize()
    w = st.particles.data[5].cpu().numpy()
    ln = st.out.log_norm.cpu().numpy()
    # theta's columns are global; the oracle sees the sampled tracks at their own columns
    for j in cols:
        th = (s.theta[0] == j + 1).astype(np.int32)   # column j+1 -> the single oracle column 1
        rw, rln, rfl = orc.reweight(inp[0][[j]], inp[1][[j]], inp[5][[j]], s.Z[0], c.R, th, 0)
        check_weights(w[j], rw[0])
        check_log_norm(ln[[j]], rln)
    # every track with an assigned detection is normalised
    assigned = np.unique(s.theta[0][s.theta[0] > 0]) - 1
    np.testing.assert_allclose(w[assigned].astype(np.float64).sum(1), 1.0, rtol=2e-5)


def test_cfg4_full_size_single_gpu_and_shards(L, orc):
    """Config 4 (T=4096, P=8192, M~4700) on one GPU: sampled oracle columns, whole-matrix
    properties, and the W=8 column blocks reproduce the W=1 matrix bit for bit."""
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
    cols = [3, 2048, 4095]
    ref = orc.compat(s.x[cols], s.y[cols], s.w[cols], s.Z[0], c.R, c.p_d, c.kappa, c.gamma)
    check_compat(C[cols], G[cols], None, ref, c.gamma, M)
    plan = ShardPlan(c.T, 8)
    for r in (0, 5, 7):
        blk = plan.cols(r)
        sub = _lib.Particles(st.particles.data[:, blk.start:blk.stop].contiguous(), c.P)
        Cs = torch.zeros(len(blk), st.ldc, device="cuda")
        Gs = torch.zeros(len(blk), st.ldg, dtype=torch.int32, device="cuda")
        _lib.glmb_compat(sub, st.Z[0], c.R, c.p_d, c.kappa, c.gamma, None, Cs, Gs)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(Cs.cpu().numpy()[:, :M], C[blk.start:blk.stop, :M])
        np.testing.assert_array_equal(Gs.cpu().numpy().view(np.uint32), G[blk.start:blk.stop])


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

"""Pins for the hypothesis machinery oracle (O9-O13; SURVEY §8f rows f1, f3;
P:44-53 §Approach) -- CPU only.

Each test checks the oracle against something other than itself: SPEC's
worked values (tests/golden/spec_examples.txt), forced outcomes, Monte-Carlo
frequencies against the closed-form row probabilities, a brute-force
enumeration of the exact successor posterior, and invariants.
"""
import itertools
import math

import numpy as np
import pytest

from _golden import spec_value


def _one_track(entries, gated=None):
    """C_tracks [1][M] and gate words for one track with the given row entries."""
    M = len(entries)
    C = np.array([entries], np.float32)
    g = np.zeros((1, (M + 31) // 32), np.uint32)
    for i in range(M):
        if gated is None or gated[i]:
            g[0, i // 32] |= np.uint32(1 << (i % 32))
    return C, g


def _rand_compat(rng, T, M, density=0.3):
    C = np.zeros((T, M), np.float32)
    g = np.zeros((T, (M + 31) // 32), np.uint32)
    for j in range(T):
        for i in range(M):
            if rng.random() < density:
                C[j, i] = np.float32(rng.uniform(1e-4, 0.5))
                g[j, i // 32] |= np.uint32(1 << (i % 32))
    return C, g


# ------------------------------------------------------------------ O9
def test_death_prob_spec_examples(orc):
    C, g = _one_track([0.0], gated=[False])
    d = orc.death_prob(C, g, 0.95, 0.01, np.array([0.99], np.float32))
    assert d[0] == pytest.approx(spec_value("death_prob_ps0.99_pd0.95_e0")[0], rel=1e-6)
    C, g = _one_track([2.29183])
    d = orc.death_prob(C, g, 0.95, 0.01, np.array([0.99], np.float32))
    assert d[0] == pytest.approx(spec_value("death_prob_ps0.99_pd0.95_entry2.29183_kappa0.01")[0], rel=1e-6)
    d = orc.death_prob(C, g, 0.95, 0.01, np.array([1.0], np.float32))
    assert d[0] == 0.0                                   # certain survival


def test_death_prob_limits_and_monotonicity(orc):
    ps = np.float32(0.9)
    # P_D -> 0: the detection evidence carries no information, d = 1 - P_S
    C, g = _one_track([5.0])
    d = orc.death_prob(C, g, 1e-12, 0.01, np.array([ps], np.float32))
    assert d[0] == pytest.approx(1 - float(ps), rel=1e-9)
    # e_j = max over gated rows of C/(C+kappa): decreasing d as the best entry grows
    prev = 1.0
    for c in (1e-6, 1e-3, 0.1, 1.0, 10.0):
        C, g = _one_track([1e-7, c, 1e-8])
        d = orc.death_prob(C, g, 0.95, 0.01, np.array([ps], np.float32))[0]
        assert 0.0 <= d < prev
        prev = d
    # ungated entries never count
    C, g = _one_track([100.0, 1e-3], gated=[False, True])
    d1 = orc.death_prob(C, g, 0.95, 0.01, np.array([ps], np.float32))[0]
    C, g = _one_track([0.0, 1e-3], gated=[False, True])
    assert orc.death_prob(C, g, 0.95, 0.01, np.array([ps], np.float32))[0] == d1


# ------------------------------------------------------------------ O10
def test_compat_rows_round_trip(orc):
    rng = np.random.default_rng(0)
    T, M = 7, 70
    C, g = _rand_compat(rng, T, M)
    rp, col, val, lv = orc.compat_rows(C, g, M)
    assert rp[0] == 0 and np.all(np.diff(rp) >= 0) and rp[M] == len(col)
    dense = np.zeros((M, T), np.float32)
    for i in range(M):
        cols = col[rp[i]:rp[i + 1]]
        assert np.all(np.diff(cols) > 0)                  # ascending track order
        dense[i, cols] = val[rp[i]:rp[i + 1]]
    bits = np.array([[(g[j, i // 32] >> (i % 32)) & 1 for j in range(T)] for i in range(M)], bool)
    np.testing.assert_array_equal(dense, np.where(bits, C.T, 0))
    np.testing.assert_allclose(np.exp(lv), val.astype(np.float64), rtol=1e-15)
    rp, col, val, lv = orc.compat_rows(np.zeros((0, M), np.float32), np.zeros((0, 3), np.uint32), M)
    assert len(col) == 0 and np.all(rp == 0)


# ------------------------------------------------------------------ O11
def _sampler(orc, C, g, d, ps, pd, kappa, H_up, seed=1, step=0, parent_mask=None, parent_logw=None,
             count_lp=None):
    T, M = C.shape[0], C.shape[1]
    ldt = max(1, (T + 31) // 32)
    if parent_mask is None:
        parent_mask = np.zeros((1, ldt), np.uint32)
        for j in range(T):
            parent_mask[0, j // 32] |= np.uint32(1 << (j % 32))
    if parent_logw is None:
        parent_logw = np.zeros(parent_mask.shape[0])
    rows = orc.compat_rows(C, g, M)
    return orc.assoc_sample(parent_mask, parent_logw, H_up, np.asarray(d, np.float32), np.asarray(ps, np.float32),
                            pd, kappa, rows, M, seed, step, count_lp=count_lp), rows


def test_sampler_forced_outcomes(orc):
    rng = np.random.default_rng(1)
    C, g = _rand_compat(rng, 5, 40)
    (al, th, lw), _ = _sampler(orc, C, g, np.ones(5), np.full(5, 0.9), 0.9, 0.01, 64)
    assert np.all(al == 0) and np.all(th == 0)           # d = 1: nothing survives, all clutter
    (al, th, lw), _ = _sampler(orc, C, g, np.zeros(5), np.full(5, 0.9), 0.9, 0.01, 64)
    assert np.all(al[:, 0] == 0b11111)                   # d = 0: everything survives


def test_sampler_support(orc):
    """No measurement is ever assigned to a dead, ungated or out-of-parent track."""
    rng = np.random.default_rng(2)
    T, M = 9, 50
    C, g = _rand_compat(rng, T, M, 0.4)
    pm = np.array([[0b101101111], [0b011111010]], np.uint32)
    (al, th, lw), _ = _sampler(orc, C, g, rng.uniform(0, 0.6, T), np.full(T, 0.95), 0.9, 0.05, 300,
                               parent_mask=pm, parent_logw=np.array([-0.1, -2.3]))
    for q in range(al.shape[0]):
        assert (al[q, 0] & ~pm[q // 300, 0]) == 0
        for i in range(M):
            if th[q, i] > 0:
                j = th[q, i] - 1
                assert (al[q, 0] >> j) & 1 and (g[j, i // 32] >> (i % 32)) & 1


def test_sampler_frequencies(orc):
    """Stage 1 survives with 1 - d; stage 2 picks a column with its normalised row weight."""
    N = 100000
    C, g = _one_track([2.29183])
    (al, th, lw), _ = _sampler(orc, C, g, [0.0], [0.99], 0.95, 0.01, N)
    p = 2.29183 / (2.29183 + 0.01)                        # S:241, 0.99566
    f = (th[:, 0] == 1).mean()
    assert abs(f - p) < 4 * math.sqrt(p * (1 - p) / N)
    C, g = _one_track([0.0], gated=[False])
    (al, th, lw), _ = _sampler(orc, C, g, [0.5], [0.99], 0.95, 0.01, N)
    f = (al[:, 0] & 1).mean()
    assert abs(f - 0.5) < 4 * math.sqrt(0.25 / N)
    # a three-way row: clutter 0.2, track 0 0.5, track 1 0.3
    C = np.array([[0.5], [0.3]], np.float32)
    g = np.array([[1], [1]], np.uint32)
    (al, th, lw), _ = _sampler(orc, C, g, [0.0, 0.0], [0.9, 0.9], 0.9, 0.2, N)
    for c, p in ((0, 0.2), (1, 0.5), (2, 0.3)):
        f = (th[:, 0] == c).mean()
        assert abs(f - p) < 4 * math.sqrt(p * (1 - p) / N)


def test_sampler_row_independence_and_keying(orc):
    N = 20000
    C = np.array([[0.5, 0.5]], np.float32)
    g = np.array([[0b11]], np.uint32)
    (al, th, lw), _ = _sampler(orc, C, g, [0.0], [0.9], 0.9, 0.5, N, seed=3)
    a, b = (th[:, 0] == 1).astype(float), (th[:, 1] == 1).astype(float)
    assert abs(np.corrcoef(a, b)[0, 1]) < 0.03
    (al2, th2, lw2), _ = _sampler(orc, C, g, [0.0], [0.9], 0.9, 0.5, N, seed=3)
    np.testing.assert_array_equal(th, th2)
    np.testing.assert_array_equal(lw, lw2)
    for kw in ({"seed": 4}, {"step": 1}):
        (_, th3, _), _ = _sampler(orc, C, g, [0.0], [0.9], 0.9, 0.5, N, **{"seed": 3, **kw})
        assert (th3 != th).mean() > 0.3


def test_sampler_uniform_keying(orc):
    """Stage-1 decision for track j of sample (h, s) uses word j%4 of the Philox block
    (j/4, h, step, 2<<24 | s) (O1, pinned by test_oracle_philox) mapped by O3."""
    T = 6
    d = np.array([0.1, 0.3, 0.5, 0.7, 0.9, 0.45], np.float32)
    C = np.zeros((T, 1), np.float32)
    g = np.zeros((T, 1), np.uint32)
    H = 50
    (al, th, lw), _ = _sampler(orc, C, g, d, np.full(T, 0.9), 0.9, 0.1, H, seed=0x1234_5678_9abc, step=7)
    for s in range(H):
        for j in range(T):
            r = orc.philox(0x1234_5678_9abc, np.array([[j // 4, 0, 7, (2 << 24) | s]], np.uint32))[0, j % 4]
            u = np.float32(orc.uniform_u32(int(r)))
            assert bool((al[s, 0] >> j) & 1) == bool(u < np.float32(1) - d[j])


def test_hypothesis_weight_spec_examples(orc):
    # two detections both assigned to the surviving track (kappa negligible)
    C, g = _one_track([2.29183, 0.05])
    (al, th, lw), _ = _sampler(orc, C, g, [0.0], [0.99], 0.95, 1e-30, 8)
    assert np.all(th == 1)
    np.testing.assert_allclose(np.exp(lw), spec_value("hyp_weight_two_detections")[0], rtol=1e-6)
    # survives, no measurements: P_S (1 - P_D)
    C, g = np.zeros((1, 0), np.float32), np.zeros((1, 1), np.uint32)
    (al, th, lw), _ = _sampler(orc, C, g, [0.0], [0.99], 0.95, 0.01, 4)
    np.testing.assert_allclose(np.exp(lw), spec_value("hyp_weight_missed")[0], rtol=1e-6)
    # dies, one measurement -> clutter: (1 - P_S) kappa
    C, g = _one_track([2.29183])
    (al, th, lw), _ = _sampler(orc, C, g, [1.0], [0.99], 0.95, 0.01, 4)
    assert np.all(th == 0)
    np.testing.assert_allclose(np.exp(lw), spec_value("hyp_weight_death_clutter")[0], rtol=1e-6)


# ------------------------------------------------------------------ O11 + O12 + O13 vs brute force
def _exact_posterior(C, gate_bits, ps, pd, kappa):
    """Enumerate every (survival set, association map) of T tracks x M rows."""
    T, M = C.shape
    out = {}
    for alive in itertools.product([0, 1], repeat=T):
        choices = []
        for i in range(M):
            choices.append([0] + [j + 1 for j in range(T) if alive[j] and gate_bits[j][i]])
        for th in itertools.product(*choices):
            w = 1.0
            for j in range(T):
                w *= ps[j] if alive[j] else 1 - ps[j]
            for i, c in enumerate(th):
                w *= kappa if c == 0 else float(C[c - 1, i])
            det = {c - 1 for c in th if c > 0}
            w *= (1 - pd) ** sum(1 for j in range(T) if alive[j] and j not in det)
            out[(alive, th)] = w
    z = sum(out.values())
    return {k: v / z for k, v in out.items()}


def test_successors_match_enumerated_posterior(orc):
    """unique candidates (dedup) weighted by the target measure and
    normalised reproduce the exact enumerated posterior (TV < 0.02)."""
    T, M = 2, 2
    C = np.array([[0.8, 0.05], [0.3, 0.6]], np.float32)
    g = np.array([[0b11], [0b11]], np.uint32)
    ps, pd, kappa = np.array([0.9, 0.7], np.float32), 0.8, 0.2
    d = np.array([0.3, 0.4], np.float32)                  # proposal, not the target
    H = 3000
    (al, th, lw), _ = _sampler(orc, C, g, d, ps, pd, kappa, H, seed=11)
    u = orc.dedup(al, th, 1, H)
    keys = [(tuple(int((al[q, 0] >> j) & 1) for j in range(T)), tuple(int(t) for t in th[q])) for q in range(H)]
    uniq = [q for q in range(H) if u[q]]
    assert len({keys[q] for q in uniq}) == len(uniq) == len(set(keys))    # dedup is exact
    assert all(u[q] == (keys.index(keys[q]) == q) for q in range(H))      # first occurrence wins
    exact = _exact_posterior(C, [[1, 1], [1, 1]], [float(v) for v in ps], pd, kappa)
    idx, w = orc.prune(lw, u, 0.0, 10 ** 6)
    got = {keys[q]: wq for q, wq in zip(idx, w)}
    for k, p in exact.items():
        if p > 1e-3:
            assert k in got
    tv = 0.5 * sum(abs(got.get(k, 0.0) - p) for k, p in exact.items())
    assert tv < 0.02
    # each unique candidate's weight is its exact (unnormalised) target measure
    z = sum(math.exp(lw[q]) for q in uniq)
    zex = None
    for q in uniq:
        ratio = math.exp(lw[q]) / exact[keys[q]]
        zex = ratio if zex is None else zex
        assert ratio == pytest.approx(zex, rel=1e-6)


# ------------------------------------------------------------------ O13
def test_prune_spec_and_edges(orc):
    w = np.log(np.array([0.6, 0.3, 0.05, 0.05]))
    idx, kw = orc.prune(w, np.ones(4, np.uint8), 0.1, 2)
    np.testing.assert_array_equal(idx, [0, 1])
    np.testing.assert_allclose(kw, spec_value("prune_0.6_0.3_0.05_0.05_tau0.1_hmax2"), rtol=1e-12)
    idx, kw = orc.prune(w, np.ones(4, np.uint8), 0.01, 10)      # identity (sorted)
    np.testing.assert_array_equal(idx, [0, 1, 2, 3])
    np.testing.assert_allclose(kw, [0.6, 0.3, 0.05, 0.05], rtol=1e-12)
    idx, kw = orc.prune(np.array([0.0]), np.ones(1, np.uint8), 0.5, 3)
    np.testing.assert_array_equal(idx, [0]) and np.testing.assert_allclose(kw, [1.0])
    # the largest always survives tau; ties ordered by index; duplicates excluded
    idx, kw = orc.prune(np.log([0.25, 0.25, 0.25, 0.25]), np.array([1, 0, 1, 1], np.uint8), 0.9, 5)
    np.testing.assert_array_equal(idx, [0])
    idx, kw = orc.prune(np.log([0.2, 0.4, 0.4]), np.ones(3, np.uint8), 0.0, 2)
    np.testing.assert_array_equal(idx, [1, 2])
    # log-domain shift invariance (far-underflowing weights)
    idx2, kw2 = orc.prune(np.log([0.2, 0.4, 0.4]) - 2000.0, np.ones(3, np.uint8), 0.0, 2)
    np.testing.assert_array_equal(idx, idx2)
    np.testing.assert_allclose(kw, kw2, rtol=1e-12)


def _exact_posterior_counts(C, ps, kappa, lc):
    """Enumeration with a per-track measurement-count prior exp(lc[min(n, len-1)]) for alive tracks."""
    T, M = C.shape
    out = {}
    for alive in itertools.product([0, 1], repeat=T):
        choices = [[0] + [j + 1 for j in range(T) if alive[j]] for _ in range(M)]
        for th in itertools.product(*choices):
            w = 1.0
            for j in range(T):
                w *= ps[j] if alive[j] else 1 - ps[j]
                if alive[j]:
                    n = sum(1 for c in th if c == j + 1)
                    w *= math.exp(lc[min(n, len(lc) - 1)])
            for i, c in enumerate(th):
                w *= kappa if c == 0 else float(C[c - 1, i])
            out[(alive, th)] = w
    z = sum(out.values())
    return {k: v / z for k, v in out.items()}


def test_successors_with_count_prior(orc):
    """the proposal ignores the per-object measurement-count prior, the importance weight
    restores it.  With a Poisson(D) count table (combined with C's P_D factor: e^-D D^n / P_D^n)
    the unique weighted samples reproduce the exact enumerated posterior of that target."""
    T, M = 2, 3
    C = np.array([[0.8, 0.05, 0.4], [0.3, 0.6, 0.5]], np.float32)
    g = np.array([[0b111], [0b111]], np.uint32)
    ps, pd, kappa, D = np.array([0.9, 0.7], np.float32), 0.8, 0.2, 1.5
    lc = np.array([-D + n * math.log(D) - n * math.log(pd) for n in range(M + 1)])
    d = np.array([0.3, 0.4], np.float32)
    H = 4000
    (al, th, lw), _ = _sampler(orc, C, g, d, ps, pd, kappa, H, seed=12, count_lp=lc)
    u = orc.dedup(al, th, 1, H)
    keys = [(tuple(int((al[q, 0] >> j) & 1) for j in range(T)), tuple(int(t) for t in th[q])) for q in range(H)]
    exact = _exact_posterior_counts(C, [float(v) for v in ps], kappa, lc)
    idx, w = orc.prune(lw, u, 0.0, 10 ** 6)
    got = {keys[q]: wq for q, wq in zip(idx, w)}
    tv = 0.5 * sum(abs(got.get(k, 0.0) - p) for k, p in exact.items())
    assert tv < 0.02
    uniq = [q for q in range(H) if u[q]]
    ratios = [math.exp(lw[q]) / exact[keys[q]] for q in uniq]
    np.testing.assert_allclose(ratios, ratios[0], rtol=1e-6)
    # the default (no table) is the table [ln(1 - P_D), 0, 0, ...]
    (al1, th1, lw1), _ = _sampler(orc, C, g, d, ps, pd, kappa, 50, seed=3)
    (al2, th2, lw2), _ = _sampler(orc, C, g, d, ps, pd, kappa, 50, seed=3,
                                 count_lp=np.array([math.log(1 - float(np.float32(pd))), 0.0]))
    np.testing.assert_array_equal(th1, th2)
    np.testing.assert_allclose(lw1, lw2, rtol=1e-15)

"""Seeded synthetic scenes shaped like BASELINE.json configs 0-4.

This module is the ONLY thing the product path and the oracle share: it makes
fp32 input arrays from numpy generators and holds none of the method's
arithmetic (no CTRV flow, no likelihood, no Philox).  Ground-truth objects move
by a plain explicit-Euler kinematic update (a generator convenience, not the
paper's CTRV model), detections are truth positions plus N(0, R) noise,
clutter is uniform over the scene (§Experiments: detections are sampled
around the true position with covariance sigma^2 I and left in sorted order).

Input recipe: every random quantity comes from a
numpy ``default_rng`` seeded by ``SeedSequence([seed, stream, index])`` so that
the particles of global track j depend only on (seed, j) -- a shard of the
tracks is generated identically at any world size.

The paper's own benchmark is a convoy built from a private GPS track
(not available); these scenes stand in for it.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np

# stream ids for SeedSequence([seed, stream, index])
_S_MEANS, _S_PART, _S_WEIGHT, _S_TRUTH, _S_DET, _S_CLUT, _S_BIRTH = range(7)


@dataclasses.dataclass(frozen=True)
class SceneConfig:
    name: str
    T: int            # surviving tracks
    B: int            # birth tracks per step (appended after survivors)
    P: int            # particles per track (multiple of 4)
    area: float       # square scene side [m]
    p_d: float        # detection probability used to draw detections
    clutter_lambda: float  # expected clutter count per step
    steps: int
    seed: int
    spread: tuple     # particle spread variances diag(x, y, v, psi, omega)
    weights: str      # "uniform" | "dirichlet"
    gamma: float
    kappa: float
    exact_M: Optional[int] = None  # cfg0: exactly T detections + (exact_M - T) clutter
    dt: float = 0.1
    sigma_a: float = 1.0
    sigma_w: float = 0.1
    R: tuple = (1.0, 0.0, 1.0)      # (Rxx, Rxy, Ryy), R = I2 m^2
    birth_cov: tuple = (25.0, 25.0, 4.0, 0.5, 0.05)

    @property
    def Tk(self) -> int:
        return self.T + self.B


# BASELINE.json configs (readings R4, R5, R20-R22 in DESIGN.md)
CONFIGS = {
    0: SceneConfig("cfg0-tiny", T=4, B=0, P=256, area=200.0, p_d=0.9, clutter_lambda=2,
                   steps=1, seed=0, spread=(1, 1, 0.5, 0.05, 0.02), weights="uniform",
                   gamma=1e-6, kappa=2.0 / 40000.0, exact_M=6),
    1: SceneConfig("cfg1-small", T=64, B=4, P=1024, area=200.0, p_d=0.9, clutter_lambda=20,
                   steps=1, seed=0, spread=(1, 1, 0.5, 0.05, 0.02), weights="dirichlet",
                   gamma=1e-6, kappa=2.0 / 40000.0),
    2: SceneConfig("cfg2-medium-seq", T=256, B=0, P=4096, area=1000.0, p_d=0.95,
                   clutter_lambda=50, steps=50, seed=1, spread=(1, 1, 0.5, 0.05, 0.02),
                   weights="uniform", gamma=1e-6, kappa=50.0 / 1e6),
    3: SceneConfig("cfg3-large", T=1024, B=16, P=8192, area=2000.0, p_d=0.9,
                   clutter_lambda=300, steps=1, seed=3, spread=(4, 4, 1, 0.1, 0.05),
                   weights="uniform", gamma=1e-8, kappa=300.0 / 4e6),
    4: SceneConfig("cfg4-sharded", T=4096, B=0, P=8192, area=4000.0, p_d=0.9,
                   clutter_lambda=1000, steps=20, seed=7, spread=(4, 4, 1, 0.1, 0.05),
                   weights="uniform", gamma=1e-8, kappa=1000.0 / 1.6e7),
}


def _rng(seed: int, stream: int, index: int = 0) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(seed), int(stream), int(index)]))


def _track_mean(cfg: SceneConfig, j: int) -> np.ndarray:
    """Truth mean of global track j: x,y~U(0,area), v~U(5,20), psi~U(-pi,pi), omega~N(0,0.1) (variance)."""
    r = _rng(cfg.seed, _S_MEANS, j)
    return np.array([r.uniform(0, cfg.area), r.uniform(0, cfg.area), r.uniform(5, 20),
                     r.uniform(-np.pi, np.pi), r.normal(0.0, np.sqrt(0.1))], np.float64)


def _birth_mean(cfg: SceneConfig, b: int) -> np.ndarray:
    r = _rng(cfg.seed, _S_BIRTH, b)
    return np.array([r.uniform(0, cfg.area), r.uniform(0, cfg.area), r.uniform(5, 20),
                     r.uniform(-np.pi, np.pi), 0.0], np.float64)


@dataclasses.dataclass
class Scene:
    cfg: SceneConfig
    # survivors (pre-predict state), rows = the requested global track range
    x: np.ndarray
    y: np.ndarray
    v: np.ndarray
    psi: np.ndarray
    omega: np.ndarray
    w: np.ndarray
    gid: np.ndarray          # int32 global ids of the rows above
    birth_mean: np.ndarray   # [B,5] fp32
    birth_chol: np.ndarray   # [B,15] fp32 packed lower triangle
    birth_gid: np.ndarray    # [B] int32
    Z: List[np.ndarray]      # per step [M_k,2] fp32
    theta: List[np.ndarray]  # per step [M_k] int32 (0 clutter, c>=1 global column)

    @property
    def P(self) -> int:
        return self.cfg.P


def track_particles(cfg: SceneConfig, j: int):
    """Particles of global track j: mean + N(0, diag(spread)), psi left unwrapped (as drawn)."""
    mu = _track_mean(cfg, j)
    r = _rng(cfg.seed, _S_PART, j)
    n = r.standard_normal((5, cfg.P))
    sd = np.sqrt(np.asarray(cfg.spread, np.float64))
    st = (mu[:, None] + sd[:, None] * n).astype(np.float32)
    if cfg.weights == "dirichlet":
        wr = _rng(cfg.seed, _S_WEIGHT, j)
        w = wr.dirichlet(np.ones(cfg.P)).astype(np.float32)
    else:
        w = np.full(cfg.P, 1.0 / cfg.P, np.float32)
    return st, w


def _truth_positions(cfg: SceneConfig, T_all: int, B: int, steps: int) -> np.ndarray:
    """Truth positions [steps, T_all + B, 2] by explicit Euler kinematics with noise."""
    means = np.stack([_track_mean(cfg, j) for j in range(T_all)] +
                     [_birth_mean(cfg, b) for b in range(B)]) if (T_all + B) else np.zeros((0, 5))
    r = _rng(cfg.seed, _S_TRUTH, 0)
    pos = np.zeros((steps, T_all + B, 2))
    s = means.copy()
    for k in range(steps):
        s[:, 0] += cfg.dt * s[:, 2] * np.cos(s[:, 3])
        s[:, 1] += cfg.dt * s[:, 2] * np.sin(s[:, 3])
        s[:, 3] += cfg.dt * s[:, 4]
        s[:, 2] += cfg.dt * cfg.sigma_a * r.standard_normal(len(s))
        s[:, 4] += cfg.dt * cfg.sigma_w * r.standard_normal(len(s))
        pos[k] = s[:, :2]
    return pos


def _detections(cfg: SceneConfig, truth_k: np.ndarray, k: int):
    """Z_k and truth-origin theta_k (column j+1 for object j, 0 for clutter), sorted by (x, y)."""
    n_obj = truth_k.shape[0]
    rd = _rng(cfg.seed, _S_DET, k)
    rc = _rng(cfg.seed, _S_CLUT, k)
    Rm = np.array([[cfg.R[0], cfg.R[1]], [cfg.R[1], cfg.R[2]]])
    Lr = np.linalg.cholesky(Rm)
    if cfg.exact_M is not None:
        det = np.ones(n_obj, bool)
        n_clut = cfg.exact_M - n_obj
    else:
        det = rd.random(n_obj) < cfg.p_d
        n_clut = rc.poisson(cfg.clutter_lambda)
    idx = np.nonzero(det)[0]
    zd = truth_k[idx] + rd.standard_normal((len(idx), 2)) @ Lr.T
    zc = rc.uniform(0, cfg.area, (n_clut, 2))
    Z = np.concatenate([zd, zc]).astype(np.float32)
    th = np.concatenate([idx + 1, np.zeros(n_clut, np.int64)]).astype(np.int32)
    order = np.lexsort((Z[:, 1], Z[:, 0]))
    return np.ascontiguousarray(Z[order]), np.ascontiguousarray(th[order])


def make_scene(cfg_id: int, rows: Optional[range] = None, steps: Optional[int] = None,
               **overrides) -> Scene:
    """Build config cfg_id.  rows = global survivor tracks to materialise (default all).
    Births (cfg.B) are global columns T..T+B-1 and are always described (mean/chol/gid)."""
    cfg = dataclasses.replace(CONFIGS[cfg_id], **overrides) if overrides else CONFIGS[cfg_id]
    rows = range(cfg.T) if rows is None else rows
    n_steps = cfg.steps if steps is None else steps
    P = cfg.P
    nr = len(rows)
    arrs = np.zeros((6, nr, P), np.float32)
    for a, j in enumerate(rows):
        st, w = track_particles(cfg, j)
        arrs[0:5, a] = st
        arrs[5, a] = w
    gid = np.asarray(list(rows), np.int32)
    bm = np.stack([_birth_mean(cfg, b) for b in range(cfg.B)]).astype(np.float32) \
        if cfg.B else np.zeros((0, 5), np.float32)
    bc = np.zeros((cfg.B, 15), np.float32)
    diag_idx = [0, 2, 5, 9, 14]
    for b in range(cfg.B):
        bc[b, diag_idx] = np.sqrt(np.asarray(cfg.birth_cov, np.float64))
    bgid = np.arange(cfg.T, cfg.T + cfg.B, dtype=np.int32)
    truth = _truth_positions(cfg, cfg.T, cfg.B, n_steps)
    Zs, ths = [], []
    for k in range(n_steps):
        Z, th = _detections(cfg, truth[k], k)
        Zs.append(Z)
        ths.append(th)
    return Scene(cfg, arrs[0], arrs[1], arrs[2], arrs[3], arrs[4], arrs[5], gid,
                 bm, bc, bgid, Zs, ths)


def random_cloud(T: int, P: int, seed: int, center_scale: float = 100.0,
                 spread: float = 1.0, dirichlet: bool = False):
    """Small generic fixture for tests: T tracks x P particles (x, y, v, psi, omega, w) fp32."""
    r = np.random.default_rng(seed)
    c = r.uniform(0, center_scale, (T, 2))
    x = (c[:, 0:1] + spread * r.standard_normal((T, P))).astype(np.float32)
    y = (c[:, 1:2] + spread * r.standard_normal((T, P))).astype(np.float32)
    v = r.uniform(0, 20, (T, P)).astype(np.float32)
    psi = r.uniform(-np.pi, np.pi, (T, P)).astype(np.float32)
    om = r.normal(0, 0.5, (T, P)).astype(np.float32)
    if dirichlet:
        w = r.dirichlet(np.ones(P), size=T).astype(np.float32)
    else:
        w = np.full((T, P), 1.0 / P, np.float32)
    return x, y, v, psi, om, w


# ------------------------------------------------------------------ hypothesis-machinery inputs
_S_HYP, _S_SYNC = 7, 8


def hypothesis_inputs(T: int, B: int, H_old: int, seed: int, p_s_survivor: float = 0.99,
                      p_s_birth: float = 0.1, p_in_parent: float = 0.9):
    """Parent hypotheses over the T_k = T + B columns of C_k:
    survivor j is in parent h with probability p_in_parent, births are in every parent
    (LMB birth is added to each hypothesis); parent log-weights = ln of a sorted
    Dirichlet(1) draw; prior survival p_s = p_s_survivor (survivors), p_s_birth (births).
    Returns (parent_mask u32 [H_old][ldt], parent_logw f64 [H_old], p_s f32 [T+B])."""
    Tk = T + B
    ldt = max(1, (Tk + 31) // 32)
    r = _rng(seed, _S_HYP, 0)
    member = np.zeros((H_old, Tk), bool)
    member[:, :T] = r.random((H_old, T)) < p_in_parent
    member[:, T:] = True
    mask = np.zeros((H_old, ldt), np.uint32)
    for j in range(Tk):
        mask[:, j // 32] |= (member[:, j].astype(np.uint32) << np.uint32(j % 32))
    w = np.sort(r.dirichlet(np.ones(H_old)))[::-1] if H_old else np.zeros(0)
    logw = np.log(np.maximum(w, 1e-300)).astype(np.float64)
    p_s = np.concatenate([np.full(T, p_s_survivor), np.full(B, p_s_birth)]).astype(np.float32)
    return mask, np.ascontiguousarray(logw), p_s


def synthetic_compat(T: int, M: int, seed: int, p_d: float = 0.9, mean_gated: float = 1.5):
    """A C_k-shaped sparse matrix without running the likelihood: each measurement row is
    gated to Poisson(mean_gated) distinct random tracks with entries p_d * 10^U(-8, 0.3).
    Returns (C_tracks fp32 [T][M], gate u32 [T][ceil(M/32)]) in glmb_compat's layout."""
    r = _rng(seed, _S_SYNC, 0)
    ldg = max(1, (M + 31) // 32)
    C = np.zeros((max(T, 0), M), np.float32)
    g = np.zeros((max(T, 0), ldg), np.uint32)
    for i in range(M):
        n = min(T, r.poisson(mean_gated))
        if n == 0:
            continue
        js = r.choice(T, size=n, replace=False)
        C[js, i] = (p_d * 10.0 ** r.uniform(-8, 0.3, n)).astype(np.float32)
        g[js, i // 32] |= np.uint32(1 << (i % 32))
    return C, g


# ------------------------------------------------------------------ the paper's convoy benchmark
_S_CONVOY = 9


@dataclasses.dataclass(frozen=True)
class ConvoyConfig:
    """P:182-186 §Experiments: N time-shifted copies of one ground track (delta steps apart),
    D detections per object per step ~ N(x*, sigma^2 I), no clutter (lambda = 0), dt = 0.1 s,
    548 steps (54.8 s), H_up = 100, tau = 1e-5, H_max in {5, ..., 100}.  The GPS track itself
    is private: a smooth synthetic figure-eight inside the 80 x 80 m area stands in (R35).
    Tracker settings the paper does not state (R35): P, the process noise, the birth model
    (one LMB birth per step at the track's entry point), P_S, P_D, kappa, gamma."""
    N: int = 20
    D: int = 5
    sigma: float = 0.25
    delta: int = 2
    K: int = 548
    dt: float = 0.1
    area: float = 80.0
    seed: int = 0
    P: int = 1024
    H_up: int = 100
    H_max: int = 100
    tau: float = 1e-5
    p_s: float = 0.99
    r_birth: float = 0.1
    p_d: float = 0.99
    kappa: float = 1e-4
    gamma: float = 1e-6
    sigma_a: float = 2.0
    sigma_w: float = 1.0
    birth_cov: tuple = (0.25, 0.25, 1.0, 0.1, 0.1)
    B: int = 1
    count_prior: bool = True   # measurement-count prior per object in the weight (R36)
    count_model: str = "binomial"   # "binomial" (Binomial(D/q, q): mean D, variance D(1-q)) | "poisson"
    count_q: float = 0.7

    @property
    def R(self):
        v = float(np.float32(self.sigma * self.sigma))
        return (v, 0.0, v)


TRACK_STEPS = 548   # the scenario lasts 54.8 s at 0.1 s per step


def ground_track(cfg: ConvoyConfig) -> np.ndarray:
    """[K, 4]: x, y, speed, heading of the synthetic ground track: one lap of the figure-eight
    x = c + 0.375 A sin(th), y = c + 0.25 A sin(2 th) in 54.8 s at constant speed (arc-length
    parameterised, ~4.6 m/s in the 80 x 80 m area), whatever the number of simulated steps K."""
    c, A = cfg.area / 2, cfg.area
    th = np.linspace(0.0, 2 * np.pi, 200001)
    x = c + 0.375 * A * np.sin(th)
    y = c + 0.25 * A * np.sin(2 * th)
    seg = np.hypot(np.diff(x), np.diff(y))
    s_arc = np.concatenate([[0.0], np.cumsum(seg)])
    v = s_arc[-1] / (TRACK_STEPS * cfg.dt)
    sk = (np.arange(cfg.K) * cfg.dt * v) % s_arc[-1]
    tk = np.interp(sk, s_arc, th)
    xk = c + 0.375 * A * np.sin(tk)
    yk = c + 0.25 * A * np.sin(2 * tk)
    hd = np.arctan2(0.5 * A * np.cos(2 * tk), 0.375 * A * np.cos(tk))
    return np.stack([xk, yk, np.full(cfg.K, v), hd], 1)


def convoy_scene(cfg: ConvoyConfig):
    """Returns (Z list [K] of fp32 [M_k, 2] sorted by (x, y), truth list [K] of [n_k, 2],
    birth_mean fp32 [B, 5], birth_chol fp32 [B, 15]).  Object n follows the track from step
    n*delta on (staggered entry, reading R19: x*_{n,k} = x*_{k - n delta})."""
    g = ground_track(cfg)
    r = _rng(cfg.seed, _S_CONVOY, 0)
    Zs, truth = [], []
    for k in range(cfg.K):
        n_on = [n for n in range(cfg.N) if k >= n * cfg.delta]
        pos = np.array([g[k - n * cfg.delta, :2] for n in n_on]).reshape(-1, 2)
        z = (np.repeat(pos, cfg.D, axis=0) + cfg.sigma * r.standard_normal((len(n_on) * cfg.D, 2)))
        z = z.astype(np.float32)
        order = np.lexsort((z[:, 1], z[:, 0]))
        Zs.append(np.ascontiguousarray(z[order]))
        truth.append(pos)
    bm = np.tile(np.array([g[0, 0], g[0, 1], g[0, 2], g[0, 3], 0.0], np.float32), (cfg.B, 1))
    bc = np.zeros((cfg.B, 15), np.float32)
    bc[:, [0, 2, 5, 9, 14]] = np.sqrt(np.asarray(cfg.birth_cov, np.float64))
    return Zs, truth, bm, bc

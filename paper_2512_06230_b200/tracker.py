"""The whole GLMB tracker loop on the GPU (§Approach,
the convoy benchmark of P:182-186 §Experiments).

One update per time step, every stage a libglmb.so kernel behind the C ABI:

    predict (survivors) -> birth -> compat -> death_prob -> compat_rows -> assoc_sample
    -> dedup -> prune -> assoc_pairs -> reweight_pairs -> resample -> map_estimate
    -> next_parents

The kept hypotheses' unique (track, measurement set) pairs become the next
step's tracks (rows of the new particle set), each kept hypothesis becomes a
parent over those rows plus the birth columns (R33).  Counts stay on the
device between stages; the host reads one int per step (the number of pairs,
which fixes the next step's track count and birth column) -- the only
synchronisation.  Python does argument marshalling and buffer bookkeeping only.
"""
from __future__ import annotations

import dataclasses
import time
from typing import List

import numpy as np
import torch

from . import _lib
from ._lib import Particles
from .hyp import HypothesisUpdate, ParticleUpdate, update_params
from .scenes import ConvoyConfig


@dataclasses.dataclass
class UpdateRecord:
    step: int
    M: int
    T_k: int
    n_parents: int
    n_kept: int
    n_pairs: int
    device_ms: float
    wall_ms: float


def count_log_prior(cfg: ConvoyConfig, M_max: int) -> np.ndarray:
    """lc(n), n = 0..n_max, for glmb_assoc_sample (reading R36): the set likelihood of n
    detections from one object is pi(n) n! prod L(z_i) for a count distribution pi; C already
    carries one P_D per measurement, so lc(n) = ln pi(n) + ln n! - n ln P_D.
    poisson:  pi = Poisson(D)            -> ln pi(n) + ln n! = -D + n ln D
    binomial: pi = Binomial(n_max, q), n_max = round(D / q) (mean ~D, variance D (1 - q))
              -> ln C(n_max, n) + n ln q + (n_max - n) ln(1 - q) + ln n!   (n > n_max: -1e4)"""
    from math import lgamma, log
    pd = float(np.float32(cfg.p_d))
    D = cfg.D
    if cfg.count_model == "poisson":
        n = np.arange(M_max + 1, dtype=np.float64)
        return -D + n * log(D) - n * log(pd)
    q = cfg.count_q
    nmax = int(round(D / q))
    lc = np.full(nmax + 2, -1e4)
    for n in range(nmax + 1):
        lc[n] = (lgamma(nmax + 1) - lgamma(n + 1) - lgamma(nmax - n + 1) + n * log(q)
                 + (nmax - n) * log(1.0 - q) + lgamma(n + 1) - n * log(pd))
    return lc


class ConvoyTracker:
    def __init__(self, cfg: ConvoyConfig, M_max: int, K_cap: int = 1024, device="cuda"):
        self.cfg = cfg
        dev = torch.device(device)
        self.dev = dev
        B, P = cfg.B, cfg.P
        self.K_cap, self.M_max = K_cap, M_max
        self.T_cap = K_cap + B
        rows = self.T_cap
        # two particle sets: [survivors | births]; the particle update writes the other one
        self.bufs = [Particles.empty(rows, P, device=dev), Particles.empty(rows, P, device=dev)]
        for b in self.bufs:
            b.data.zero_()
        self.cur = 0
        self.gid = torch.arange(rows, dtype=torch.int32, device=dev)
        # survival prior per column: P_S everywhere; each update sets its birth columns to r_b
        # and restores them after its kernels (enqueued before the host waits)
        self.p_s = torch.full((rows,), cfg.p_s, dtype=torch.float32, device=dev)
        self.ldc = max(32, (M_max + 31) // 32 * 32)
        self.ldg = max(1, (M_max + 31) // 32)
        self.C_clutter = torch.empty(max(M_max, 1), dtype=torch.float32, device=dev)
        self.C_tracks = torch.empty(rows, self.ldc, dtype=torch.float32, device=dev)
        self.gate = torch.empty(rows, self.ldg, dtype=torch.int32, device=dev)
        self.Z = torch.empty(max(M_max, 1), 2, dtype=torch.float32, device=dev)
        H = cfg.H_max
        self.hu = HypothesisUpdate(rows, M_max, H, cfg.H_up, H, device=dev)
        self.pu = ParticleUpdate(rows, M_max, H, P, K_cap=K_cap, device=dev, own_out=False)
        self.ldt = self.hu.ldt
        self.parent_mask = torch.zeros(H, self.ldt, dtype=torch.int32, device=dev)
        self.parent_logw = torch.zeros(H, dtype=torch.float64, device=dev)
        self.est = torch.empty(rows, 3, dtype=torch.float64, device=dev)
        self.count_lp = torch.from_numpy(count_log_prior(cfg, M_max)).to(dev) if cfg.count_prior else None
        self.birth_mean = None
        self.birth_chol = None
        self.n_surv = 0
        self.stream = torch.cuda.Stream(device=dev)
        # (n_pairs, n_kept, n_parents) live side by side: one 12-byte read-back per update
        self.counts = torch.zeros(3, dtype=torch.int32, device=dev)
        self.pu.n_pairs = self.counts[0:1]
        self.hu.n_kept = self.counts[1:2]
        self.n_parents = self.counts[2:3]
        self.counts_host = torch.zeros(3, dtype=torch.int32).pin_memory()
        self.Z_host = torch.zeros(max(M_max, 1), 2, dtype=torch.float32).pin_memory()
        self._ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        self._prm = [None, None]   # cached glmb_update argument blocks, one per particle buffer
        self.est_host = torch.zeros(rows, 3, dtype=torch.float64).pin_memory()
        # every buffer above was filled on the current stream; the tracker's kernels run on
        # self.stream (a non-blocking pool stream), so order it after those fills explicitly
        self.stream.wait_stream(torch.cuda.current_stream(dev))

    def reset(self, birth_mean: np.ndarray, birth_chol: np.ndarray):
        """Empty track set; one parent (the empty hypothesis, weight 1) over the birth columns."""
        cfg = self.cfg
        self.birth_mean = torch.from_numpy(np.ascontiguousarray(birth_mean, np.float32)).to(self.dev)
        self.birth_chol = torch.from_numpy(np.ascontiguousarray(birth_chol, np.float32)).to(self.dev)
        self.n_surv = 0
        self.cur = 0
        one = torch.ones(1, dtype=torch.float64, device=self.dev)
        n1 = torch.ones(1, dtype=torch.int32, device=self.dev)
        none = torch.full((1, 1), -1, dtype=torch.int32, device=self.dev)
        _lib.glmb_next_parents(n1, one, none, 0, cfg.B, 0, self.parent_mask[:1], self.parent_logw[:1],
                               self.n_parents, self.stream)

    STAGES = ("predict", "birth", "compat", "death_prob", "compat_rows", "assoc_sample", "dedup", "prune",
              "assoc_pairs", "reweight_pairs", "resample", "map_estimate")

    def update(self, k: int, Z: np.ndarray, profile: bool = False) -> UpdateRecord:
        """One tracker update.  profile=True records a CUDA event after every stage (self.last_events)."""
        cfg, s = self.cfg, self.stream
        M = Z.shape[0]
        assert M <= self.M_max
        t0 = time.perf_counter()
        e0, e1 = self._ev
        src = self.bufs[self.cur]
        dst = self.bufs[1 - self.cur]
        T, B = self.n_surv, cfg.B
        Tk = T + B
        evs = {}

        def mark(name):
            if profile:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(s)
                evs[name] = ev

        hu, pu = self.hu, self.pu
        # the hypothesis machinery works on T_k columns (capacity-sized buffers, views)
        hu.T = Tk
        pu.T = Tk
        self.Z_host[:M].numpy()[:] = Z      # pinned staging: the H2D copy is asynchronous
        with torch.cuda.stream(s):
            e0.record(s)
            self.Z[:M].copy_(self.Z_host[:M], non_blocking=True)
            Zk = self.Z[:M]
            self.p_s[T:Tk].fill_(cfg.r_birth)
            mark("start")
            if T:
                surv = src.rows(0, T)
                _lib.glmb_predict(surv, surv, self.gid[:T], cfg.dt, cfg.sigma_a, cfg.sigma_w, cfg.seed, k, s)
            mark("predict")
            _lib.glmb_birth(src.rows(T, Tk), self.gid[T:Tk], self.birth_mean, self.birth_chol, cfg.seed, k, s)
            mark("birth")
            trk = src.rows(0, Tk)
            _lib.glmb_compat(trk, Zk, cfg.R, cfg.p_d, cfg.kappa, cfg.gamma, self.C_clutter[:M],
                             self.C_tracks[:Tk], self.gate[:Tk], s)
            mark("compat")
            po = pu.pair_of.view(-1)[:cfg.H_max * Tk].view(cfg.H_max, Tk)   # packed [H][T_k]
            if profile:   # stage by stage, an event after each
                hu.run(self.C_tracks[:Tk], self.gate[:Tk], M, self.p_s[:Tk], self.parent_mask,
                       self.parent_logw, cfg.p_d, cfg.kappa, cfg.tau, cfg.seed, k, s, n_parents=self.n_parents,
                       count_lp=self.count_lp, mark=mark)
                pu.run(trk, Zk, cfg.R, hu.keep_idx, cfg.H_max, hu.alive, hu.theta, M, cfg.seed, k, s,
                       n_hyp_dev=hu.n_kept, out=dst.rows(0, self.K_cap), mark=mark)
                _lib.glmb_map_estimate(hu.n_kept, po[0], dst.rows(0, self.K_cap), self.est[:Tk], s)
                mark("map_estimate")
            else:         # one C call enqueues the whole chain (host overhead of one launch sequence)
                _lib.glmb_update(self._update_params(trk, Tk, M, k), s)
            self.counts_host.copy_(self.counts, non_blocking=True)   # (n_pairs, n_kept, n_parents)
            e1.record(s)
            self.p_s[T:Tk].fill_(cfg.p_s)   # these columns are survivors' rows next update
            # kept hypotheses -> parents over the new rows [0, K) and the next births at
            # [K, K + B), K read on the device (enqueued before the host waits for K)
            _lib.glmb_next_parents(hu.n_kept, hu.keep_w, po, self.K_cap, B, 0,
                                   self.parent_mask, self.parent_logw, self.n_parents, s,
                                   birth_col0_dev=pu.n_pairs)
        s.synchronize()
        self.last_events = evs
        K, n_kept, n_par = (int(v) for v in self.counts_host)
        if K > self.K_cap:
            raise RuntimeError(f"step {k}: {K} unique pairs exceed K_cap = {self.K_cap}")
        wall = (time.perf_counter() - t0) * 1e3
        self.n_surv = K
        self.cur = 1 - self.cur
        return UpdateRecord(k, M, Tk, n_par, n_kept, K, e0.elapsed_time(e1), wall)

    def _update_params(self, trk: Particles, Tk: int, M: int, k: int) -> "_lib.glmb_update_params":
        """The glmb_update argument block of this particle buffer, built once and then only
        its sizes and step updated (every buffer pointer is fixed)."""
        cfg, hu, pu = self.cfg, self.hu, self.pu
        prm = self._prm[self.cur]
        if prm is None:
            dst = self.bufs[1 - self.cur]
            prm = update_params(hu, pu, self.bufs[self.cur].rows(0, self.T_cap), self.C_tracks, self.gate, M,
                                self.Z, cfg.R, self.p_s, self.parent_mask, self.parent_logw, cfg.p_d, cfg.kappa,
                                cfg.tau, cfg.seed, k, n_parents=self.n_parents, count_lp=self.count_lp,
                                out=dst.rows(0, self.K_cap), est=self.est)
            self._prm[self.cur] = prm
        prm.T = Tk
        prm.M = M
        prm.K_cap = min(pu.K_cap, max(1, hu.h_max * Tk))
        prm.step = k
        prm.tracks.n_tracks = Tk
        return prm

    def estimate(self, T_k: int) -> np.ndarray:
        """MAP positions [n, 2] of the last update (host copy; evaluation only)."""
        e = self.est[:T_k].cpu().numpy()
        return e[e[:, 2] > 0, :2]


def run_convoy(cfg: ConvoyConfig, steps: int | None = None, K_cap: int = 1024, device="cuda",
               with_estimates: bool = True, stage_ms: dict | None = None):
    """Runs the tracker over the convoy scene; returns (records, estimates, truth).  With a dict
    as stage_ms, every update is profiled per stage (CUDA events) and the means are stored in it."""
    from .scenes import convoy_scene
    Zs, truth, bm, bc = convoy_scene(cfg)
    n = len(Zs) if steps is None else min(steps, len(Zs))
    M_max = max(len(z) for z in Zs[:n])
    tr = ConvoyTracker(cfg, M_max, K_cap=K_cap, device=device)
    tr.reset(bm, bc)
    recs: List[UpdateRecord] = []
    ests = []
    acc = {name: 0.0 for name in ConvoyTracker.STAGES}
    for k in range(n):
        rec = tr.update(k, Zs[k], profile=stage_ms is not None)
        recs.append(rec)
        if stage_ms is not None:
            prev = tr.last_events["start"]
            for name in ConvoyTracker.STAGES:
                acc[name] += prev.elapsed_time(tr.last_events[name])
                prev = tr.last_events[name]
        if with_estimates:
            ests.append(tr.estimate(rec.T_k))
    if stage_ms is not None:
        stage_ms.update({name: v / max(n, 1) for name, v in acc.items()})
    return recs, ests, truth[:n]


def convoy_metrics(ests, truth):
    """mean relative absolute cardinality error, and the mean distance of the
    Hungarian (minimum-distance) matching between estimated and true positions."""
    from scipy.optimize import linear_sum_assignment
    card, dist = [], []
    for e, t in zip(ests, truth):
        n = len(t)
        card.append(abs(len(e) - n) / max(n, 1))
        if len(e) and n:
            Dm = np.linalg.norm(e[:, None, :] - t[None, :, :], axis=2)
            r, c = linear_sum_assignment(Dm)
            dist.append(float(Dm[r, c].mean()))
    return float(np.mean(card)), float(np.mean(dist)) if dist else float("nan")

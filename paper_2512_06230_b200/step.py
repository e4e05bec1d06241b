"""Step driver: device-resident buffers for one (shard of a) scene and the
four C-ABI calls of one GLMB step (predict -> birth -> compat -> reweight).

A rank owns the contiguous block [lo, hi) of the T_k = T + B global columns
(survivors first, then births -- P:24 "superposition of these surviving
predicted and newborn tracks"); column c of C_k (c >= 1) is global track
c - 1.  All arithmetic runs in libglmb.so; this module only allocates torch
CUDA memory and passes pointers.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np
import torch

from . import _lib as L
from .scenes import Scene


@dataclasses.dataclass
class StepOutputs:
    C_clutter: torch.Tensor
    C_tracks: torch.Tensor   # [T_local, ldc]
    gate: torch.Tensor       # [T_local, ldg] int32 words (u32 bit pattern)
    log_norm: torch.Tensor   # [T_local]
    flags: torch.Tensor      # [T_local] int32


class GlmbStep:
    """Buffers + launch sequence for one rank.

    scene:  generated with rows = this rank's survivor rows (global ids in scene.gid).
    cols:   a contiguous block [lo, hi) of the T_k global columns (survivors, then births);
    births: or, with cols holding survivor columns only, this rank's births as birth indices
            [b0, b1) (global columns T + b) -- SURVEY 8(e)'s even split of the births
            (dist.ShardPlan).  The local rows are [survivors | births] either way.
    """

    def __init__(self, scene: Scene, cols: Optional[range] = None, device="cuda",
                 seed: Optional[int] = None, rows_alloc: Optional[int] = None,
                 births: Optional[range] = None):
        cfg = scene.cfg
        self.scene = scene
        self.cfg = cfg
        self.device = torch.device(device)
        Tk = cfg.T + cfg.B
        cols = range(0, Tk) if cols is None else cols
        lo, hi = cols.start, cols.stop
        if births is None:
            surv = range(lo, min(hi, cfg.T))
            births = range(max(lo, cfg.T) - cfg.T, max(hi, cfg.T) - cfg.T)
        else:
            if hi > cfg.T or births.start < 0 or births.stop > cfg.B:
                raise ValueError("with births given, cols must be survivor columns")
            surv = cols
        if list(scene.gid) != list(surv):
            raise ValueError("scene rows must equal this rank's survivor columns")
        self.surv_cols = surv
        self.birth_idx = births
        self.T_surv = len(surv)
        self.B_local = len(births)
        self.T_local = self.T_surv + self.B_local
        # global column (0-based track index) of every local row
        self.col_of_row = np.concatenate([np.arange(surv.start, surv.stop),
                                          cfg.T + np.arange(births.start, births.stop)]).astype(np.int64)
        # one reweight launch when the local rows are consecutive global columns, else two
        self.contiguous = (self.T_surv == 0 or self.B_local == 0
                           or (surv.stop == cfg.T and births.start == 0))
        self.col_offset = int(self.col_of_row[0]) if self.T_local else 0
        P = cfg.P
        self.P = P
        dev = self.device
        self.particles = L.Particles.empty(self.T_local, P, device=dev)
        if self.T_surv:
            init = np.stack([scene.x, scene.y, scene.v, scene.psi, scene.omega, scene.w])
            self.particles.data[:, :self.T_surv].copy_(torch.from_numpy(init))
        # double-buffered weights: reweight may write the other buffer while compat
        # reads the current one on another stream (glmb_reweight's w_out)
        self.w_bufs = [self.particles.data[5], torch.empty_like(self.particles.data[5])]
        self.w_cur = 0
        b_idx = list(births)
        gid = np.concatenate([np.asarray(scene.gid, np.int32),
                              scene.birth_gid[b_idx].astype(np.int32)])
        self.gid = torch.from_numpy(gid).to(dev)
        self.birth_mean = torch.from_numpy(np.ascontiguousarray(scene.birth_mean[b_idx])).to(dev)
        self.birth_chol = torch.from_numpy(np.ascontiguousarray(scene.birth_chol[b_idx])).to(dev)
        # measurements of every step resident in HBM (inputs of the timed region)
        self.M_max = max([len(z) for z in scene.Z] + [1])
        self.ldc = ((self.M_max + 31) // 32) * 32
        self.ldg = (self.M_max + 31) // 32
        self.Z = [torch.from_numpy(z).to(dev) for z in scene.Z]
        self.theta = [torch.from_numpy(t).to(dev) for t in scene.theta]
        # rows_alloc >= T_local pads the column block to the common all-gather size
        ra = self.T_local if rows_alloc is None else max(rows_alloc, self.T_local)
        self.rows_alloc = ra
        self.out = StepOutputs(
            C_clutter=torch.zeros(self.M_max, dtype=torch.float32, device=dev),
            C_tracks=torch.zeros(ra, self.ldc, dtype=torch.float32, device=dev),
            gate=torch.zeros(ra, self.ldg, dtype=torch.int32, device=dev),
            log_norm=torch.zeros(self.T_local, dtype=torch.float32, device=dev),
            flags=torch.zeros(self.T_local, dtype=torch.int32, device=dev))
        self.seed = cfg.seed if seed is None else seed
        self.R = cfg.R

    @property
    def cols(self) -> range:
        """The contiguous global column block of this rank (only when its rows are contiguous)."""
        if not self.contiguous:
            raise ValueError("this rank's columns are two blocks (survivors, births): use col_of_row")
        return range(self.col_offset, self.col_offset + self.T_local)

    # ---- the four stages (each is one C-ABI call) ----
    def survivors(self) -> L.Particles:
        return self.particles.rows(0, self.T_surv)

    def births(self) -> L.Particles:
        return self.particles.rows(self.T_surv, self.T_local)

    def predict(self, k: int, stream=None):
        s = self.survivors()
        L.glmb_predict(s, s, self.gid[:self.T_surv], self.cfg.dt, self.cfg.sigma_a,
                       self.cfg.sigma_w, self.seed, k, stream)

    def predict_to_spare(self, k: int, stream=None):
        """Out-of-place step start (software pipelining across steps): predict the survivors
        from the current state into a spare state buffer and draw the births there, then make
        the spare current (the weights are shared).  The old state stays readable by a compat
        still running on another stream; the spare must no longer be read by one (the caller
        orders that, e.g. with events)."""
        if not hasattr(self, "spare"):
            self.spare = torch.empty_like(self.particles.data)
        src = L.Particles(self.particles.data, self.P, self.w_bufs[self.w_cur])
        dst = L.Particles(self.spare, self.P, self.w_bufs[self.w_cur])
        if self.T_surv:
            L.glmb_predict(src.rows(0, self.T_surv), dst.rows(0, self.T_surv), self.gid[:self.T_surv],
                           self.cfg.dt, self.cfg.sigma_a, self.cfg.sigma_w, self.seed, k, stream)
        if self.B_local:
            L.glmb_birth(dst.rows(self.T_surv, self.T_local), self.gid[self.T_surv:], self.birth_mean,
                         self.birth_chol, self.seed, k, stream)
        self.spare = self.particles.data
        self.particles = dst

    def birth(self, k: int, stream=None):
        if self.B_local:
            L.glmb_birth(self.births(), self.gid[self.T_surv:], self.birth_mean, self.birth_chol,
                         self.seed, k, stream)

    def compat(self, k: int, stream=None, Z=None):
        zi = k % len(self.Z)
        o = self.out
        L.glmb_compat(self.particles, self.Z[zi] if Z is None else Z, self.R, self.cfg.p_d, self.cfg.kappa,
                      self.cfg.gamma, o.C_clutter, o.C_tracks, o.gate, stream)

    def reweight(self, k: int, stream=None, Z=None, theta=None, out_of_place: bool = False):
        """out_of_place: write the new weights into the spare buffer (the current weights
        stay readable by a concurrent compat) and make it current afterwards."""
        zi = k % len(self.Z)
        o = self.out
        w_out = self.w_bufs[1 - self.w_cur] if out_of_place else None
        Zk = self.Z[zi] if Z is None else Z
        thk = self.theta[zi] if theta is None else theta
        if self.contiguous:
            L.glmb_reweight(self.particles, Zk, self.R, thk, self.col_offset, o.log_norm, o.flags, stream,
                            w_out=w_out)
        else:   # survivors and births are two global column blocks: one launch per block
            for a, b, off in ((0, self.T_surv, self.surv_cols.start),
                              (self.T_surv, self.T_local, self.cfg.T + self.birth_idx.start)):
                L.glmb_reweight(self.particles.rows(a, b), Zk, self.R, thk, off, o.log_norm[a:b], o.flags[a:b],
                                stream, w_out=None if w_out is None else w_out[a:b])
        if out_of_place:
            self.w_cur = 1 - self.w_cur
            self.particles = L.Particles(self.particles.data, self.P, self.w_bufs[self.w_cur])

    def weights(self) -> torch.Tensor:
        return self.w_bufs[self.w_cur]

    def run(self, k: int, stream=None):
        """One whole step through the fused glmb_step entry point."""
        if not self.contiguous:
            raise ValueError("glmb_step takes one column offset: run the four stages instead")
        zi = k % len(self.Z)
        o = self.out
        prm = self.step_params(k)
        L.glmb_step(prm, self.Z[zi], self.theta[zi], o.C_clutter, o.C_tracks, o.gate, o.log_norm,
                    o.flags, stream)

    def step_params(self, k: int, out_of_place: bool = False) -> L.glmb_step_params:
        """out_of_place: the new weights go to the spare buffer (call swap_weights() after the
        step) -- lets glmb_step_host run reweight concurrently with compat."""
        c = self.cfg
        return L.make_step_params(self.particles, self.T_surv, self.gid, self.birth_mean,
                                  self.birth_chol, c.dt, c.sigma_a, c.sigma_w, self.seed, k,
                                  self.R, c.p_d, c.kappa, c.gamma, self.cols.start,
                                  w_out=self.w_bufs[1 - self.w_cur] if out_of_place else None)

    def swap_weights(self):
        """Make the spare weight buffer (written by an out-of-place step) the current one."""
        self.w_cur = 1 - self.w_cur
        self.particles = L.Particles(self.particles.data, self.P, self.w_bufs[self.w_cur])

    def evals(self, k: int) -> int:
        """Algorithmic particle-measurement likelihood evaluations of step k on this rank:
        M_k * T_k * P (compat, dense) + P * #{i : theta_i in this rank's columns} (reweight)."""
        zi = k % len(self.Z)
        M = len(self.scene.Z[zi])
        th = self.scene.theta[zi]
        n_assigned = int(np.isin(th - 1, self.col_of_row).sum())
        return M * self.T_local * self.P + self.P * n_assigned


class PipelinedSteps:
    """Software-pipelined GLMB steps on one rank (what bench.py times at N = 1): step k's
    predict + birth write the spare state buffer (GlmbStep.predict_to_spare) on a high-priority
    stream, so they run while step k-1's compat still reads the other buffer; reweight_k writes
    the spare weight buffer on `side` beside compat_k on `main`.  Event order: predict_k after
    compat_{k-2} and reweight_{k-2} (the readers of the buffer it overwrites); reweight_k after
    predict_k and compat_{k-1} (the reader of the weights it overwrites); compat_k after
    predict_k and reweight_{k-1} (its weights).  Every step does all of its work; the results
    are those of the sequential steps (tests/test_gpu_parity.py)."""

    def __init__(self, st: GlmbStep, main, side, pred=None):
        self.st, self.main, self.side = st, main, side
        self.pred = pred if pred is not None else torch.cuda.Stream(device=st.device, priority=-1)
        self.c = [None, None]    # compat events of steps k-1, k-2
        self.rw = [None, None]   # reweight events of steps k-1, k-2

    def start_after(self, event):
        self.pred.wait_event(event)
        self.side.wait_event(event)

    def step(self, k: int):
        st = self.st
        zi = k % len(st.Z)
        Zk, thk = st.Z[zi], st.theta[zi]
        c1, c2 = self.c
        r1, r2 = self.rw
        ev = lambda: torch.cuda.Event()
        with torch.cuda.stream(self.pred):
            for e in (c2, r2):
                if e is not None:
                    self.pred.wait_event(e)
            st.predict_to_spare(k, self.pred)
            ready = ev()
            ready.record(self.pred)
        p_now = st.particles          # compat reads these weights; reweight writes the spare
        self.side.wait_event(ready)
        if c1 is not None:
            self.side.wait_event(c1)
        with torch.cuda.stream(self.side):
            st.reweight(k, self.side, Z=Zk, theta=thk, out_of_place=True)
            rdone = ev()
            rdone.record(self.side)
        self.main.wait_event(ready)
        if r1 is not None:
            self.main.wait_event(r1)
        with torch.cuda.stream(self.main):
            o = st.out
            L.glmb_compat(p_now, Zk, st.R, st.cfg.p_d, st.cfg.kappa, st.cfg.gamma, o.C_clutter, o.C_tracks,
                          o.gate, self.main)
            cdone = ev()
            cdone.record(self.main)
        self.c = [cdone, c1]
        self.rw = [rdone, r1]

    def join(self):
        """Make `main` wait for every stream's last work (then one event on main ends the steps)."""
        if self.rw[0] is not None:
            self.main.wait_event(self.rw[0])

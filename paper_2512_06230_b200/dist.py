"""Track sharding over ranks (one process per GPU) and the one exchange step.

SURVEY.md §8(e): tracks (the columns of C_k) are independent -- column j of
C_k depends only on track j's particles and on all of Z_k ("the entire
construction of the joint compatibility matrix can be performed in
parallel"; "computed in parallel over hypotheses, measurements and
tracks").  So rank r owns a block of the T_k global columns and its particles
never move; the only communication per step is

  * Z_k and theta_k broadcast from rank 0 (the sensor side), packed in one
    buffer (one collective), and
  * an all-gather of the column blocks of C_k -- each row holds a column of C
    and, after it, that column's gate words, so one collective moves both --
    plus a small all-gather of the per-track log-normalisers and flags, so
    that every rank holds the full matrix the association sampler (f1)
    consumes.

Partition (``ShardPlan``): rank r owns ceil(T/W) consecutive survivor columns
and ceil(B/W) consecutive birth columns (births split evenly),
its local rows being [survivors | births]; every block is padded to the same
``per_rank`` rows so ``all_gather_into_tensor`` needs no per-rank counts.  The
gathered matrix is rank-major: global column c sits at row
``plan.row_of(c)``; with no births (config 4) or one rank, the first T_k rows
are C_k in global order.  Philox is keyed by the global track id and the
compat / reweight launch shapes depend on (M, P) only, so every gathered
entry is bit-identical to the single-GPU result.

This module holds no arithmetic of the method -- only the plan, buffers and
the collectives (NCCL on GPU; gloo with host-staged buffers in the CPU-side
and world-size-2 GPU tests).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist


@dataclasses.dataclass(frozen=True)
class ShardPlan:
    n_cols: int        # T_k = T + B global track columns: survivors 0..T-1, births T..T_k-1 (R11)
    world: int
    n_births: int = 0  # B, split evenly over the ranks

    @property
    def n_surv(self) -> int:
        return self.n_cols - self.n_births

    @property
    def per_surv(self) -> int:
        return -(-self.n_surv // self.world)

    @property
    def per_birth(self) -> int:
        return -(-self.n_births // self.world)

    @property
    def per_rank(self) -> int:
        return max(1, self.per_surv + self.per_birth)

    def surv(self, rank: int) -> range:
        lo = min(self.n_surv, rank * self.per_surv)
        return range(lo, min(self.n_surv, lo + self.per_surv))

    def births(self, rank: int) -> range:
        """Birth indices b of this rank (global column T + b)."""
        lo = min(self.n_births, rank * self.per_birth)
        return range(lo, min(self.n_births, lo + self.per_birth))

    def cols(self, rank: int):
        """Global columns of this rank's local rows, in local order ([survivors | births]).
        A range when they are consecutive (no births, or one rank), else a list."""
        s, b = self.surv(rank), self.births(rank)
        if len(b) == 0 or len(s) == 0 or (s.stop == self.n_surv and b.start == 0):
            lo = s.start if len(s) else self.n_surv + b.start
            return range(lo, lo + len(s) + len(b))
        return list(s) + [self.n_surv + x for x in b]

    def owner(self, col: int) -> int:
        if col < self.n_surv:
            return col // self.per_surv
        return (col - self.n_surv) // self.per_birth

    def row_of(self, col: int) -> int:
        """Row of global column `col` in the rank-major gathered buffer."""
        r = self.owner(col)
        if col < self.n_surv:
            return r * self.per_rank + col - self.surv(r).start
        return r * self.per_rank + len(self.surv(r)) + (col - self.n_surv) - self.births(r).start

    def global_rows(self) -> np.ndarray:
        """[T_k] gathered-buffer row of every global column (identity when contiguous)."""
        return np.array([self.row_of(c) for c in range(self.n_cols)], np.int64)


def broadcast_measurements(Z: torch.Tensor, theta: torch.Tensor, src: int = 0, group=None) -> None:
    """In-place broadcast of Z_k [M,2] fp32 and theta_k [M] int32 from `src` (two collectives;
    ShardedStep packs both into one)."""
    dist.broadcast(Z, src=src, group=group)
    dist.broadcast(theta, src=src, group=group)


def allgather_columns(local_block: torch.Tensor, gathered: torch.Tensor, group=None) -> torch.Tensor:
    """local_block [per_rank, ld] (rows past this rank's columns are padding) ->
    gathered [world * per_rank, ld]."""
    dist.all_gather_into_tensor(gathered, local_block.contiguous(), group=group)
    return gathered


class ShardedStep:
    """One rank's share of the GLMB step core, the public multi-GPU entry point:

        broadcast (Z_k, theta_k) -> predict -> birth -> compat (+ reweight) -> all-gather

    Buffers (all on this rank's GPU):
      meas      int32 [3 M_max]: Z_k (fp32 bits, [M][2]) then theta_k -- one broadcast
      block     fp32 [per][S]: row l = C column of local track l (ldc floats), then its gate
                words (ldg, as uint32 bits), S = ldc + ldg rounded to 32 -- compat writes it in
                place, one all-gather moves it
      gathered  fp32 [W * per][S]: the rank-major C_k + gate words of every rank
      ln_block  fp32 [2][per]: reweight's log-normalisers (row 0) and flags (row 1, uint32
                bits) of the local tracks; ln_all [W][2][per] gathered

    stage_on_host: collectives move host copies (gloo; the world-size-2 GPU test runs the
    real kernels of both ranks on one GPU this way, the ranks never waiting on each other's
    kernels).  fused: compat stores its columns straight into every rank's symmetric-memory
    copy of the gathered buffer over NVLink (glmb_compat_peers; symm.SymmetricColumns),
    replacing the C all-gather.
    Plumbing only: every step of the method runs in libglmb.so's kernels (step.GlmbStep).
    """

    def __init__(self, cfg_id: int, group=None, device=None, steps: Optional[int] = None,
                 stage_on_host: bool = False, fused: bool = False, scene=None):
        from . import _lib as L
        from .scenes import CONFIGS, make_scene
        from .step import GlmbStep
        self.L = L
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        cfg = CONFIGS[cfg_id]
        self.cfg = cfg
        self.plan = ShardPlan(cfg.T + cfg.B, self.world, cfg.B)
        r, plan = self.rank, self.plan
        self.scene = scene if scene is not None else make_scene(cfg_id, rows=plan.surv(r), steps=steps)
        self.st = GlmbStep(self.scene, cols=plan.surv(r), births=plan.births(r), device=self.dev,
                           rows_alloc=plan.per_rank)
        st = self.st
        per, W, dev = plan.per_rank, self.world, self.dev
        self.per = per
        self.M_max = st.M_max
        self.ldc, self.ldg = st.ldc, st.ldg
        self.S = self.ldc + (self.ldg + 31) // 32 * 32
        self.meas = torch.zeros(3 * self.M_max, dtype=torch.int32, device=dev)
        self.block = torch.zeros(per, self.S, dtype=torch.float32, device=dev)
        self.gathered = torch.zeros(W * per, self.S, dtype=torch.float32, device=dev)
        self.ln_block = torch.zeros(2, per, dtype=torch.float32, device=dev)
        self.ln_all = torch.zeros(W, 2, per, dtype=torch.float32, device=dev)
        st.out.log_norm = self.ln_block[0, :st.T_local]
        st.out.flags = self.ln_block[1, :st.T_local].view(torch.int32)
        self.stage_on_host = stage_on_host
        if stage_on_host:
            self.h_meas = torch.zeros(3 * self.M_max, dtype=torch.int32)
            self.h_block = torch.zeros(per, self.S, dtype=torch.float32)
            self.h_gathered = torch.zeros(W * per, self.S, dtype=torch.float32)
            self.h_ln = torch.zeros(2, per, dtype=torch.float32)
            self.h_ln_all = torch.zeros(W, 2, per, dtype=torch.float32)
        self.symm = None
        if fused:
            from .symm import SymmetricColumns
            self.symm = SymmetricColumns(per, self.S, self.ldc, dev, group=group)

    # ---- views
    def Z(self, M: int) -> torch.Tensor:
        return self.meas[:2 * M].view(torch.float32).view(M, 2)

    def theta(self, M: int) -> torch.Tensor:
        return self.meas[2 * self.M_max:2 * self.M_max + M]

    def local_C(self) -> torch.Tensor:
        return self.block[:, :self.ldc]

    def local_gate(self) -> torch.Tensor:
        return self.block.view(torch.int32)[:, self.ldc:self.ldc + self.ldg]

    def C_all(self, k: int = 0) -> torch.Tensor:
        """[W*per][ldc] (row stride S): the gathered C_k columns, rank-major."""
        g = self.gathered if self.symm is None else self.symm.buffer(k)
        return g[:, :self.ldc]

    def gate_all(self, k: int = 0) -> torch.Tensor:
        g = self.gathered if self.symm is None else self.symm.buffer(k)
        return g.view(torch.int32)[:, self.ldc:self.ldc + self.ldg]

    def log_norm_all(self) -> torch.Tensor:
        """[W*per] log-normalisers, rank-major rows like C_all."""
        return self.ln_all[:, 0].reshape(-1)

    def flags_all(self) -> torch.Tensor:
        return self.ln_all[:, 1].reshape(-1).view(torch.int32)

    # ---- the step
    def load_measurements(self, k: int, Z: Optional[torch.Tensor] = None, theta: Optional[torch.Tensor] = None,
                          stream=None):
        """Rank 0 (the sensor side) places step k's Z_k / theta_k into the broadcast buffer
        (from its scene, or from the given tensors -- e.g. pinned host tensors in the e2e leg),
        enqueued on `stream` (default: the current stream) -- pass the stream step() runs on."""
        sc = self.scene
        zi = k % len(sc.Z)
        M = len(sc.Z[zi]) if Z is None else Z.shape[0]
        if self.rank == 0:
            src_Z = self.st.Z[zi] if Z is None else Z
            src_t = self.st.theta[zi] if theta is None else theta
            with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream(self.dev)):
                self.Z(M).copy_(src_Z, non_blocking=True)
                self.theta(M).copy_(src_t, non_blocking=True)
        return M

    def _broadcast(self, M: int):
        if self.stage_on_host:
            self.h_meas.copy_(self.meas)
            dist.broadcast(self.h_meas, src=0, group=self.group)
            self.meas.copy_(self.h_meas)
        else:
            dist.broadcast(self.meas, src=0, group=self.group)

    def _gather(self):
        if self.stage_on_host:
            self.h_block.copy_(self.block)
            self.h_ln.copy_(self.ln_block)
            dist.all_gather_into_tensor(self.h_gathered, self.h_block, group=self.group)
            dist.all_gather_into_tensor(self.h_ln_all.view(-1), self.h_ln.view(-1), group=self.group)
            self.gathered.copy_(self.h_gathered)
            self.ln_all.copy_(self.h_ln_all)
        else:
            if self.symm is None:
                dist.all_gather_into_tensor(self.gathered, self.block, group=self.group)
            dist.all_gather_into_tensor(self.ln_all.view(-1), self.ln_block.view(-1), group=self.group)

    def step(self, k: int, M: int, stream=None, side=None):
        """One sharded step (the timed unit at N > 1).  Z_k / theta_k must be in `meas` on rank 0
        (load_measurements).  side: optional second stream -- reweight (into the spare weight
        buffer) then runs beside compat."""
        st, cfg, L = self.st, self.cfg, self.L
        stream = stream if stream is not None else torch.cuda.current_stream(self.dev)
        with torch.cuda.stream(stream):
            self._broadcast(M)
            Zk, thk = self.Z(M), self.theta(M)
            st.predict(k, stream)
            st.birth(k, stream)
            if side is not None:
                ready = torch.cuda.Event()
                ready.record(stream)
                side.wait_event(ready)
                p_now = st.particles
                with torch.cuda.stream(side):
                    st.reweight(k, side, Z=Zk, theta=thk, out_of_place=True)
                    done = torch.cuda.Event()
                    done.record(side)
            else:
                p_now = st.particles
            self._compat(p_now, Zk, k, stream)
            if side is not None:
                stream.wait_event(done)
            else:
                st.reweight(k, stream, Z=Zk, theta=thk)
            if self.symm is not None:
                self.symm.barrier(k, stream)
            self._gather()

    def _compat(self, trk, Zk, k, stream):
        st, cfg, L = self.st, self.cfg, self.L
        if self.symm is not None:
            self.symm.compat(trk, Zk, st.R, cfg.p_d, cfg.kappa, cfg.gamma, st.out.C_clutter, self.rank * self.per,
                             k, stream)
        else:
            L.glmb_compat(trk, Zk, st.R, cfg.p_d, cfg.kappa, cfg.gamma, st.out.C_clutter,
                          self.local_C()[:st.T_local], self.local_gate()[:st.T_local], stream)

    def evals(self, k: int) -> int:
        return self.st.evals(k)

    # ---- end to end: host measurements in, C_k's gated entries out (rank 0)
    def step_host_csr(self, k: int, Z_host: torch.Tensor, theta_host: torch.Tensor, stream=None, side=None,
                      first_copy: Optional[int] = None):
        """The sharded step with host I/O (the N > 1 end-to-end entry point): rank 0 copies the
        pinned host Z_k / theta_k into the broadcast buffer, every rank runs step(), and rank 0
        turns the gathered C_k into the CSR of its gated entries on the device
        (glmb_compat_rows over the W*per gathered rows; column c of the CSR = gathered row c,
        see ShardPlan.row_of) and reads back row_ptr, the entries (a speculative first copy of
        `first_copy`, the rest in a second exact copy) and the gathered log-normalisers and
        flags.  Synchronous.  Returns (nnz, h2d bytes, d2h bytes) on rank 0, (0, 0, 0) elsewhere."""
        L = self.L
        stream = stream if stream is not None else torch.cuda.current_stream(self.dev)
        M = Z_host.shape[0]
        n_rows = self.world * self.per
        if not hasattr(self, "_csr"):
            cap = max(1, n_rows * self.M_max)
            dev = self.dev
            pin = lambda t: t.pin_memory()
            self._csr = dict(
                rp=torch.empty(self.M_max + 1, dtype=torch.int32, device=dev),
                col=torch.empty(cap, dtype=torch.int32, device=dev),
                val=torch.empty(cap, dtype=torch.float32, device=dev),
                lv=torch.empty(cap, dtype=torch.float64, device=dev),
                rp_h=pin(torch.empty(self.M_max + 1, dtype=torch.int32)),
                col_h=pin(torch.empty(cap, dtype=torch.int32)),
                val_h=pin(torch.empty(cap, dtype=torch.float32)),
                ln_h=pin(torch.empty(self.world, 2, self.per, dtype=torch.float32)))
        b = self._csr
        first = 4 * self.M_max if first_copy is None else int(first_copy)
        first = min(first, b["col"].shape[0])
        with torch.cuda.stream(stream):
            if self.rank == 0:
                self.load_measurements(k, Z=Z_host, theta=theta_host, stream=stream)
            self.step(k, M, stream=stream, side=side)
            if self.rank != 0:
                stream.synchronize()
                return 0, 0, 0
            L.glmb_compat_rows(self.C_all(k), self.gate_all(k), M, b["rp"], b["col"], b["val"], b["lv"], stream)
            b["rp_h"][:M + 1].copy_(b["rp"][:M + 1], non_blocking=True)
            b["col_h"][:first].copy_(b["col"][:first], non_blocking=True)
            b["val_h"][:first].copy_(b["val"][:first], non_blocking=True)
            b["ln_h"].copy_(self.ln_all, non_blocking=True)
            stream.synchronize()
            nnz = int(b["rp_h"][M])
            if nnz > first:
                b["col_h"][first:nnz].copy_(b["col"][first:nnz], non_blocking=True)
                b["val_h"][first:nnz].copy_(b["val"][first:nnz], non_blocking=True)
                stream.synchronize()
        return nnz, M * 12, (M + 1) * 4 + max(first, nnz) * 8 + self.ln_all.numel() * 4

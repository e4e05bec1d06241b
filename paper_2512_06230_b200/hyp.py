"""Hypothesis update and particle loop on the GPU (§Approach).

``HypothesisUpdate`` owns the device buffers of one rank and issues, on one
stream, the five C-ABI calls that turn C_k into the pruned successor set:

    glmb_death_prob -> glmb_compat_rows -> glmb_assoc_sample -> glmb_dedup -> glmb_prune

``ParticleUpdate`` then closes the particle loop for the kept hypotheses:

    glmb_assoc_pairs -> glmb_reweight_pairs -> glmb_resample

Argument marshalling only: every step runs in libglmb.so's kernels.
"""
from __future__ import annotations

import torch

from . import _lib


class HypothesisUpdate:
    def __init__(self, T: int, M_max: int, H_old: int, H_up: int, h_max: int, device="cuda"):
        self.T, self.M_max, self.H_old, self.H_up, self.h_max = T, M_max, H_old, H_up, h_max
        dev = torch.device(device)
        n = H_old * H_up
        self.ldt = max(1, (T + 31) // 32)
        self.ldm = max(4, (M_max + 3) // 4 * 4)
        i32, f32, f64 = torch.int32, torch.float32, torch.float64
        self.d = torch.empty(max(T, 1), dtype=f32, device=dev)
        self.row_ptr = torch.empty(M_max + 1, dtype=i32, device=dev)
        cap = max(1, T * M_max)  # nnz <= T*M: never overflows, so no host round trip
        self.col = torch.empty(cap, dtype=i32, device=dev)
        self.val = torch.empty(cap, dtype=f32, device=dev)
        self.ln_val = torch.empty(cap, dtype=f64, device=dev)
        self.alive = torch.empty(max(n, 1), self.ldt, dtype=i32, device=dev)
        self.theta = torch.empty(max(n, 1), self.ldm, dtype=i32, device=dev)
        self.logw = torch.empty(max(n, 1), dtype=f64, device=dev)
        self.hash = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        self.unique = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        self.keys = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        self.keep_idx = torch.empty(max(h_max, 1), dtype=i32, device=dev)
        self.keep_w = torch.empty(max(h_max, 1), dtype=f64, device=dev)
        self.n_kept = torch.zeros(1, dtype=i32, device=dev)

    def run(self, C_tracks, gate, M, p_s, parent_mask, parent_logw, p_d, kappa, tau, seed, step,
            stream=None, mark=None, n_parents=None, count_lp=None):
        """n_parents: optional device int32 count of valid rows of parent_mask (<= H_old);
        count_lp: optional device fp64 measurement-count log prior per alive track."""
        """C_tracks [T, ldc] fp32 / gate [T, ldg] words as glmb_compat writes them (device);
        p_s [T] fp32; parent_mask [H_old, ldt] int32 words; parent_logw [H_old] fp64."""
        assert M <= self.M_max
        n = self.H_old * self.H_up
        mark = mark or (lambda name: None)   # optional stage hook (bench: CUDA events)
        _lib.glmb_death_prob(C_tracks, gate, M, p_d, kappa, p_s, self.d, stream)
        mark("death_prob")
        _lib.glmb_compat_rows(C_tracks, gate, M, self.row_ptr, self.col, self.val, self.ln_val, stream)
        mark("compat_rows")
        _lib.glmb_assoc_sample(self.H_up, parent_mask, parent_logw, self.d[:self.T], p_s, p_d, kappa,
                               self.row_ptr, self.col, self.val, self.ln_val, M, seed, step,
                               self.alive[:n], self.theta[:n], self.logw[:n], self.hash[:n], stream,
                               n_parents=n_parents, count_lp=count_lp)
        mark("assoc_sample")
        _lib.glmb_dedup(self.H_old, self.H_up, M, self.alive[:n], self.theta[:n], self.hash[:n],
                        self.unique[:n], stream, n_parents=n_parents)
        mark("dedup")
        _lib.glmb_prune(self.logw[:n], self.unique[:n], tau, self.h_max, self.keys[:n], self.keep_idx,
                        self.keep_w, self.n_kept, stream)
        mark("prune")


class ParticleUpdate:
    """Unique (track, measurement set) pairs of the kept hypotheses, their particle update and
    resampling into a new particle set with one row per pair."""

    def __init__(self, T: int, M_max: int, n_hyp_max: int, P: int, K_cap: int | None = None, device="cuda",
                 own_out: bool = True):
        """K_cap: rows of the new particle set (default min(n_hyp_max, 4) * T); the pair lists
        themselves are sized for the worst case n_hyp_max * T."""
        from ._lib import Particles
        dev = torch.device(device)
        self.T, self.M_max, self.n_hyp_max, self.P = T, M_max, n_hyp_max, P
        K = max(1, n_hyp_max * T)
        Kc = max(1, min(n_hyp_max, 4) * T) if K_cap is None else max(1, int(K_cap))
        i32 = torch.int32
        self.K_cap = Kc
        self.pair_track = torch.empty(K, dtype=i32, device=dev)
        self.pair_ptr = torch.empty(K + 1, dtype=i32, device=dev)
        self.pair_meas = torch.empty(max(1, n_hyp_max * M_max), dtype=i32, device=dev)
        self.pair_of = torch.empty(max(1, n_hyp_max), max(1, T), dtype=i32, device=dev)
        self.n_pairs = torch.zeros(1, dtype=i32, device=dev)
        nb = _lib.glmb_assoc_pairs_workspace_size(n_hyp_max, T, M_max)
        self.ws = torch.empty(max(16, nb), dtype=torch.uint8, device=dev)
        self.w_new = torch.empty(Kc, P, dtype=torch.float32, device=dev)
        self.log_norm = torch.empty(Kc, dtype=torch.float32, device=dev)
        self.flags = torch.empty(Kc, dtype=i32, device=dev)
        self.ess = torch.empty(Kc, dtype=torch.float32, device=dev)
        self.out = Particles.empty(Kc, P, device=dev) if own_out else None

    def run(self, src, Z, R, hyp_idx, n_hyp, alive, theta, M, seed, step, stream=None, n_hyp_dev=None,
            mark=None, out=None):
        """src: Particles of the T_k predicted tracks; hyp_idx [>= n_hyp] device int32 (e.g. the
        pruned keep_idx); alive / theta: the sampler's outputs; n_hyp_dev: optional device count
        (e.g. HypothesisUpdate.n_kept, with n_hyp = h_max) so nothing waits on the host.
        New set: rows < n_pairs of `out` (default self.out; any Particles with >= K_cap rows)."""
        assert n_hyp <= self.n_hyp_max and M <= self.M_max
        mark = mark or (lambda name: None)
        hi = hyp_idx[:n_hyp]
        _lib.glmb_assoc_pairs(hi, alive, theta, self.T, M, self.pair_track, self.pair_ptr, self.pair_meas,
                              self.pair_of, self.n_pairs, self.ws, stream, n_hyp_dev=n_hyp_dev)
        mark("assoc_pairs")
        K = min(self.K_cap, max(1, n_hyp * self.T))
        _lib.glmb_reweight_pairs(src, Z, R, K, self.n_pairs, self.pair_track, self.pair_ptr, self.pair_meas,
                                 self.w_new[:K], self.log_norm, self.flags, self.ess, stream)
        mark("reweight_pairs")
        _lib.glmb_resample(src, K, self.n_pairs, self.pair_track, self.w_new[:K], self.out if out is None else out,
                           seed, step, self.flags, stream)
        mark("resample")

    def n_pairs_checked(self) -> int:
        """Synchronises and returns K; raises if the pairs overflowed K_cap (rows past it were not updated)."""
        torch.cuda.synchronize()
        K = int(self.n_pairs.item())
        if K > self.K_cap:
            raise RuntimeError(f"{K} unique pairs exceed K_cap = {self.K_cap}")
        return K


def update_params(hu: HypothesisUpdate, pu: ParticleUpdate, tracks, C_tracks, gate, M, Z, R, p_s, parent_mask,
                  parent_logw, p_d, kappa, tau, seed, step, n_parents=None, count_lp=None, out=None,
                  est=None) -> _lib.glmb_update_params:
    """The glmb_update argument block over the buffers of hu / pu (T = hu.T columns)."""
    T = hu.T
    n = hu.H_old * hu.H_up
    K = min(pu.K_cap, max(1, hu.h_max * T))
    o = pu.out if out is None else out
    p = _lib._ptr
    return _lib.glmb_update_params(
        T, int(M), hu.H_old, hu.H_up, hu.h_max, K, p_d, kappa, R[0], R[1], R[2], float(tau),
        int(seed) & 0xFFFFFFFFFFFFFFFF, int(step), tracks.struct(), p(C_tracks), C_tracks.shape[1], p(gate),
        gate.shape[1], p(Z), p(p_s), p(parent_mask), parent_mask.shape[1], p(parent_logw), p(n_parents),
        p(count_lp), 0 if count_lp is None else count_lp.shape[0], p(hu.d), p(hu.row_ptr), p(hu.col),
        p(hu.val), p(hu.ln_val), hu.col.shape[0], p(hu.alive), p(hu.theta), hu.theta.shape[1], p(hu.logw),
        p(hu.hash), p(hu.unique), p(hu.keys), p(hu.keep_idx), p(hu.keep_w), p(hu.n_kept), p(pu.pair_track),
        p(pu.pair_ptr), p(pu.pair_meas), p(pu.pair_of), p(pu.n_pairs), p(pu.ws),
        pu.ws.numel() * pu.ws.element_size(), p(pu.w_new), pu.w_new.shape[1], p(pu.log_norm), p(pu.flags),
        p(pu.ess), o.struct(), p(est))

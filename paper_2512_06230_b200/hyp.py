"""Hypothesis update on the GPU (§Approach).

``HypothesisUpdate`` owns the device buffers of one rank and issues, on one
stream, the five C-ABI calls that turn C_k into the pruned successor set:

    glmb_death_prob -> glmb_compat_rows -> glmb_assoc_sample -> glmb_dedup -> glmb_prune

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
            stream=None):
        """C_tracks [T, ldc] fp32 / gate [T, ldg] words as glmb_compat writes them (device);
        p_s [T] fp32; parent_mask [H_old, ldt] int32 words; parent_logw [H_old] fp64."""
        assert M <= self.M_max
        n = self.H_old * self.H_up
        _lib.glmb_death_prob(C_tracks, gate, M, p_d, kappa, p_s, self.d, stream)
        _lib.glmb_compat_rows(C_tracks, gate, M, self.row_ptr, self.col, self.val, self.ln_val, stream)
        _lib.glmb_assoc_sample(self.H_up, parent_mask, parent_logw, self.d[:self.T], p_s, p_d, kappa,
                               self.row_ptr, self.col, self.val, self.ln_val, M, seed, step,
                               self.alive[:n], self.theta[:n], self.logw[:n], self.hash[:n], stream)
        _lib.glmb_dedup(self.H_old, self.H_up, M, self.alive[:n], self.theta[:n], self.hash[:n],
                        self.unique[:n], stream)
        _lib.glmb_prune(self.logw[:n], self.unique[:n], tau, self.h_max, self.keys[:n], self.keep_idx,
                        self.keep_w, self.n_kept, stream)

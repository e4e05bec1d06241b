"""Fused compat + all-gather over NVLink peer memory.

``SymmetricColumns`` allocates the gathered C_k [world*per][ldc] and gate words
[world*per][ldg] in torch symmetric memory (one allocation per rank, mapped into
every peer over NVLink), so ``glmb_compat_peers`` can store each finished column
straight into every rank's copy; a device-side barrier then orders the ranks.
Plumbing only: the stores happen in libglmb.so's compat kernel.  Construction
raises if symmetric memory is unavailable (the caller falls back to NCCL
all_gather_into_tensor).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib


class SymmetricColumns:
    def __init__(self, per: int, ldc: int, ldg: int, device, group=None):
        import torch.distributed._symmetric_memory as symm
        group = group if group is not None else dist.group.WORLD
        world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.per = per
        self.C = symm.empty(world * per, ldc, dtype=torch.float32, device=device)
        self.G = symm.empty(world * per, ldg, dtype=torch.int32, device=device)
        name = group.group_name
        self.hC = symm.rendezvous(self.C, name)
        self.hG = symm.rendezvous(self.G, name)
        self.peer_C = torch.tensor(list(self.hC.buffer_ptrs), dtype=torch.int64, device=device)
        self.peer_G = torch.tensor(list(self.hG.buffer_ptrs), dtype=torch.int64, device=device)
        self.ldc, self.ldg = ldc, ldg

    def compat(self, trk, Z, R, p_d, kappa, gamma, C_clutter, stream=None):
        """This rank's columns into every rank's C / gate (row = rank * per + local track)."""
        _lib.glmb_compat_peers(trk, Z, R, p_d, kappa, gamma, C_clutter, self.peer_C, self.peer_G,
                               self.rank * self.per, self.ldc, self.ldg, stream)

    def barrier(self, stream=None):
        """Device-side barrier across the ranks (after it, every rank's copy is complete)."""
        with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream()):
            self.hC.barrier(channel=0)

"""Fused compat + all-gather over NVLink peer memory.

``SymmetricColumns`` allocates the gathered C_k rows -- each row a column of C
(ldc floats) followed by its gate words, row stride S, as dist.ShardedStep lays
them out -- in torch symmetric memory (mapped into every peer over NVLink), so
``glmb_compat_peers`` stores each finished column straight into every rank's
copy; a device-side barrier then orders the ranks.

Double buffering: step k writes copy k % 2.  A consumer of step k's C_k on any
rank must be enqueued (on the step stream, or joined to it) before that rank's
step k + 1 barrier; the barrier of step k + 1 then proves every rank is done
with copy k % 2 before any rank's step k + 2 stores overwrite it, and step
k + 1's own stores go to the other copy -- so the stores of a fast rank never
race a slow rank's readers, with one barrier per step (no pre-store barrier).

Plumbing only: the stores happen in libglmb.so's compat kernel.  Construction
raises if symmetric memory is unavailable (the caller falls back to NCCL
all_gather_into_tensor).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib


class SymmetricColumns:
    def __init__(self, per: int, S: int, ldc: int, device, group=None):
        import torch.distributed._symmetric_memory as symm
        group = group if group is not None else dist.group.WORLD
        world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.per, self.S, self.ldc = per, S, ldc
        name = group.group_name
        self.bufs, self.handles, self.peers, self.peers_g = [], [], [], []
        for _ in range(2):
            b = symm.empty(world * per, S, dtype=torch.float32, device=device)
            b.zero_()
            h = symm.rendezvous(b, name)
            self.bufs.append(b)
            self.handles.append(h)
            self.peers.append(torch.tensor(list(h.buffer_ptrs), dtype=torch.int64, device=device))
            # gate words start ldc floats into each row
            self.peers_g.append(torch.tensor([q + 4 * ldc for q in h.buffer_ptrs], dtype=torch.int64,
                                             device=device))

    def buffer(self, k: int) -> torch.Tensor:
        """The gathered [W*per][S] rows written by step k."""
        return self.bufs[k % 2]

    def compat(self, trk, Z, R, p_d, kappa, gamma, C_clutter, row0: int, k: int, stream=None):
        """This rank's columns into row row0 + j of copy k % 2 on every rank: C in the first ldc
        floats of the row, the gate words after them (row stride S for both)."""
        _lib.glmb_compat_peers(trk, Z, R, p_d, kappa, gamma, C_clutter, self.peers[k % 2], self.peers_g[k % 2],
                               row0, self.S, self.S, stream)

    def barrier(self, k: int, stream=None):
        """Device-side barrier across the ranks (after it, copy k % 2 is complete everywhere)."""
        with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream()):
            self.handles[k % 2].barrier(channel=0)

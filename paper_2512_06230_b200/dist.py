"""Track sharding over ranks (one process per GPU) and the one exchange step.

SURVEY.md §8(e): tracks (the columns of C_k) are independent -- column j of
C_k depends only on track j's particles and on all of Z_k ("the entire
construction of the joint compatibility matrix can be performed in
parallel").  So rank r owns a contiguous block of the T_k global columns and
its particles never move; the only communication per step is

  * Z_k and theta_k broadcast from rank 0 (the sensor side), and
  * an all-gather of the column blocks of C_k (and of the gate words) so that
    every rank holds the full matrix the association sampler (NEXT, f1)
    consumes.

Blocks are ceil(T_k / W) columns, so every rank's block has the same size and
``all_gather_into_tensor`` needs no per-rank counts; the padding sits at the
tail of the last block(s), hence the first T_k rows of the gathered tensor are
C_k's track columns in global order.  This module holds no arithmetic of the
method -- only the plan and the collectives (NCCL on GPU, gloo in the CPU
tests).
"""
from __future__ import annotations

import dataclasses

import torch
import torch.distributed as dist


@dataclasses.dataclass(frozen=True)
class ShardPlan:
    n_cols: int   # T_k global track columns
    world: int

    @property
    def per_rank(self) -> int:
        return max(1, (self.n_cols + self.world - 1) // self.world)

    def cols(self, rank: int) -> range:
        lo = min(self.n_cols, rank * self.per_rank)
        return range(lo, min(self.n_cols, lo + self.per_rank))

    def owner(self, col: int) -> int:
        return col // self.per_rank


def broadcast_measurements(Z: torch.Tensor, theta: torch.Tensor, src: int = 0, group=None) -> None:
    """In-place broadcast of Z_k [M,2] fp32 and theta_k [M] int32 from `src`."""
    dist.broadcast(Z, src=src, group=group)
    dist.broadcast(theta, src=src, group=group)


def allgather_columns(local_block: torch.Tensor, gathered: torch.Tensor, group=None) -> torch.Tensor:
    """local_block [per_rank, ld] (rows past this rank's columns are padding) ->
    gathered [world * per_rank, ld]; returns gathered (first n_cols rows = global order)."""
    dist.all_gather_into_tensor(gathered, local_block.contiguous(), group=group)
    return gathered

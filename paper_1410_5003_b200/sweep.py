"""Angle sweep across processes: one process per GPU, each sweeping a
contiguous shard of the angle list through its own context (qps_sweep: the
alpha-free cache filled once per process, angles batched on the device).
Angles are independent, so the data path has no collective; the per-angle
results are gathered to every rank at the end (the sweep's output, not an
exchange step).  Replaces the reference's single-process loop over
assemble_system/solve_periodized per angle.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np

_KEYS = ("R", "T", "flux_error", "aU", "aD", "status")


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of n angles for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return n * rank // world, n * (rank + 1) // world


def _empty(K: int):
    nrb = 2 * K + 1
    return {"R": np.zeros(0), "T": np.zeros(0), "flux_error": np.zeros(0),
            "aU": np.zeros((0, nrb), np.complex128), "aD": np.zeros((0, nrb), np.complex128),
            "status": np.zeros(0, np.int32)}


def sharded_sweep(solver, thetas: Sequence[float], K: int, mode: int = 0, group=None):
    """Sweep `thetas` split across the ranks of `group` (torch.distributed,
    any backend; single process when not initialised).  Every rank returns the
    full result, in the order of `thetas`."""
    import torch.distributed as dist
    thetas = list(thetas)
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    else:
        rank, world = 0, 1
    lo, hi = shard_bounds(len(thetas), rank, world)
    part = solver.sweep(thetas[lo:hi], K, mode) if hi > lo else _empty(K)
    if world == 1:
        return part
    parts = [None] * world
    dist.all_gather_object(parts, part, group=group)
    return {k: np.concatenate([p[k] for p in parts]) for k in _KEYS}

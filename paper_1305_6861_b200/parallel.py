"""Domain decomposition over spins across GPUs — the reference's only strategy.

The reference cuts the spin set into contiguous blocks with ``np.linspace``
bounds (``partition_blocks``, engine.py:229-251), evolves them independently
and sums the block partials (engine.py:493-496) before dividing by the global
spin count (engine.py:507).  Across GPUs the same holds: one process per GPU
(``torch.distributed``), a contiguous rasterisation-order shard per rank, no
communication while integrating, and exactly one exchange — an fp64 sum of
the per-rank partial k-space to rank 0 (NCCL over NVLink on GPUs, gloo in the
CPU tests).  Final magnetisation needs no collective: per-rank shards
concatenate in rank order, which is the reference's block-order ``vstack``
(engine.py:497-504).
"""

from __future__ import annotations

from typing import Tuple

import numpy as np

from .engine import SpinBlock


def shard_bounds(n: int, world: int, rank: int) -> Tuple[int, int]:
    """[lo, hi) of rank's contiguous shard, np.linspace bounds as partition_blocks."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    b = np.linspace(0, n, world + 1).astype(int)
    return int(b[rank]), int(b[rank + 1])


def shard_block(block: SpinBlock, world: int, rank: int) -> SpinBlock:
    lo, hi = shard_bounds(block.n, world, rank)
    w = np.asarray(block.weight)
    return SpinBlock(
        index=rank, pos=block.pos[lo:hi], mx=block.mx[lo:hi], my=block.my[lo:hi], mz=block.mz[lo:hi],
        t1=block.t1[lo:hi], t2=block.t2[lo:hi], m0=block.m0[lo:hi], domega=block.domega[lo:hi],
        weight=w[..., lo:hi],
    )


def lattice_spacing(pos: np.ndarray, axis: int = 0) -> float:
    """Smallest positive spacing of the isochromat lattice along ``axis`` (0 if a single site)."""
    u = np.unique(np.asarray(pos)[:, axis]) if len(pos) else np.zeros(0)
    d = np.diff(u)
    d = d[d > 0]
    return float(d.min()) if d.size else 0.0


def weak_copy(block: SpinBlock, world: int, rank: int, spacing: float) -> SpinBlock:
    """Rank's spin set for weak scaling: the whole block, shifted by rank/world of the lattice spacing in x.

    The global object is ``world`` interleaved copies of the block's isochromat lattice (world x the
    isochromats per voxel along x); each isochromat of copy r keeps its site's tissue, off-resonance
    and receive weight.  Rank 0's copy is the block itself, so one rank is exactly the single-GPU
    workload, and each rank's work is fixed as the world grows.  The k-space is the sum over copies
    (``reduce_kspace``).
    """
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    pos = np.array(block.pos, dtype=np.float64, copy=True)
    if rank:
        pos[:, 0] += spacing * rank / world
    return SpinBlock(index=rank, pos=pos, mx=block.mx, my=block.my, mz=block.mz, t1=block.t1, t2=block.t2,
                     m0=block.m0, domega=block.domega, weight=block.weight)


def reduce_kspace(partial, dst: int = 0):
    """Sum a float64 partial k-space tensor over all ranks into ``dst`` (in place).

    ``partial`` is a torch tensor (CUDA for NCCL, CPU for gloo) holding the
    interleaved complex128 echoes of this rank.  Returns the tensor; on dst it
    holds the global sum.
    """
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.reduce(partial, dst=dst, op=dist.ReduceOp.SUM)
    return partial


def gather_final_state(local: np.ndarray, dst: int = 0):
    """Concatenate per-rank (n_r, 3) state shards in rank order on dst (None elsewhere)."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    objs = [None] * dist.get_world_size() if dist.get_rank() == dst else None
    dist.gather_object(local, objs, dst=dst)
    return np.concatenate(objs, axis=0) if dist.get_rank() == dst else None

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


def run_distributed(exp, compute=None, device=None):
    """``run(Experiment)`` with one process per GPU (torchrun + NCCL), the reference's worker pool
    (engine.py:465-595) with one GPU per worker.

    Every rank rasterises the same spin set (deterministic), takes its contiguous np.linspace shard
    (partition_blocks, engine.py:229-251), evolves it on its GPU, and the one exchange sums the
    partial k-space on rank 0 (``reduce_kspace``, NCCL over NVLink); the final-magnetisation shards
    concatenate in rank order (engine.py:497-504) and rank 0 divides by the global spin count
    (engine.py:507).  Rank 0 returns the RunResult, every other rank None.  ``busy_fraction`` holds
    each rank's busy time (engine.py:516-525).

    ``compute(tables, shard) -> (echoes, snapshots)`` replaces the GPU call (the CPU tests pass the
    float64 oracle); by default it is the engine on ``device`` (LOCAL_RANK).
    """
    import math
    import platform
    import time

    import torch
    import torch.distributed as dist

    from .engine import (EchoRecord, InvalidParameter, RunMetrics, RunResult, build_spin_arrays, get_engine,
                         precompute_sequence_tables)
    from .phantom import rasterize_arrays

    dist_on = dist.is_available() and dist.is_initialized()
    world = dist.get_world_size() if dist_on else 1
    rank = dist.get_rank() if dist_on else 0
    if exp.spacing is None:
        raise InvalidParameter("Experiment.spacing is required (the spacing analysis is out of scope)")
    wall_start = time.perf_counter()
    spacing = tuple(float(s) for s in exp.spacing)
    spins = rasterize_arrays(exp.phantom, spacing, cap=exp.spin_cap)
    if spins["m0"].size == 0:
        raise InvalidParameter("the phantom rasterized to zero spins")
    arrays = build_spin_arrays(spins, exp.system)
    tables = precompute_sequence_tables(exp.sequence, gamma=exp.system.gamma, snapshot_times=exp.snapshot_times)
    shard = shard_block(arrays, world, rank)
    if compute is None:
        eng = get_engine(device, exp.precision)

        def compute(t, b):
            return eng.compute(t, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)

    t0 = time.perf_counter()
    echoes, snaps = compute(tables, shard)
    busy = time.perf_counter() - t0
    backend = dist.get_backend() if dist_on else "gloo"
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    e = np.ascontiguousarray(echoes, dtype=np.complex128)
    part = torch.from_numpy(e.view(np.float64).reshape(-1).copy()).to(dev)
    reduce_kspace(part, dst=0)  # the one collective of the path
    finals = [gather_final_state(s if s is not None else np.zeros((0, 3)), dst=0) for s in snaps]
    busy_t = torch.tensor([busy], dtype=torch.float64, device=dev)
    gathered = [torch.zeros_like(busy_t) for _ in range(world)]
    if dist_on and world > 1:
        dist.all_gather(gathered, busy_t)
    else:
        gathered = [busy_t]
    if rank != 0:
        return None
    n_spins = arrays.n
    echo_sum = part.cpu().numpy().view(np.complex128).reshape(e.shape) / n_spins  # engine.py:507
    records = [EchoRecord(acq_index=i, values=echo_sum[..., i, : tables.acq_times[i].size],
                          timestamps=tables.acq_times[i]) for i in range(tables.n_acq)]
    wall = time.perf_counter() - wall_start
    metrics = RunMetrics(
        wall_time_s=wall, spin_count=n_spins, throughput=n_spins / wall if wall > 0 else math.inf, workers=world,
        blocks=world, busy_fraction={r: float(g.item()) / wall for r, g in enumerate(gathered)} if wall > 0 else {},
        hardware=f"{platform.machine()} {world} ranks ({backend}) sm_100a",
    )
    snapshots = [(t, f if f is not None and len(f) else np.zeros((0, 3))) for t, f in zip(tables.snapshot_times,
                                                                                         finals)]
    return RunResult(echoes=records, metrics=metrics, snapshots=snapshots, spin_count=n_spins, spacing=spacing)

"""CPU, world_size 2 (gloo): the multi-GPU decomposition over spins.

Each rank takes its contiguous shard (parallel.shard_block, the reference's
np.linspace partition, engine.py:229-251), evolves it (here with the float64
oracle standing in for the device, since this container has no GPU), and the
partial k-space is summed with the single collective of the path
(parallel.reduce_kspace -> dist.reduce); the final magnetisation shards are
concatenated in rank order (parallel.gather_final_state).  Rank 0's result
must equal the single-process result on the whole block — the reference's
linearity / block-partition invariance (test_engine.py:175-200).
"""

import os
import socket

import numpy as np
import pytest


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist

    from oracle import bloch_oracle as O
    from paper_1305_6861_b200 import configs
    from paper_1305_6861_b200.parallel import gather_final_state, reduce_kspace, shard_block

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = configs.make(0).subset(4)
    seq = w.sequence
    tables = O.precompute_tables(seq, snapshot_times=(seq.end_time,))
    shard = shard_block(w.block, world, rank)
    echoes, snaps = O.compute_block(tables, shard.pos, shard.mx, shard.my, shard.mz, shard.t1, shard.t2, shard.m0,
                                    shard.domega, shard.weight)
    t = torch.from_numpy(np.ascontiguousarray(echoes).view(np.float64).copy())
    reduce_kspace(t, dst=0)
    final = gather_final_state(snaps[0], dst=0)
    if rank == 0:
        np.savez(out_path, echoes=t.numpy().view(np.complex128).reshape(echoes.shape), final=final)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_reduce_matches_single_process(tmp_path):
    import torch.multiprocessing as mp

    from oracle import bloch_oracle as O
    from paper_1305_6861_b200 import configs

    out = str(tmp_path / "r0.npz")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    w = configs.make(0).subset(4)
    seq = w.sequence
    b = w.block
    ref_e, ref_s = O.compute_block(O.precompute_tables(seq, snapshot_times=(seq.end_time,)), b.pos, b.mx, b.my, b.mz,
                                   b.t1, b.t2, b.m0, b.domega, b.weight)
    assert O.rel_l2(ref_e, got["echoes"]) <= 1e-13
    assert np.array_equal(ref_s[0], got["final"])


def _weak_worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist

    from oracle import bloch_oracle as O
    from paper_1305_6861_b200 import configs
    from paper_1305_6861_b200.parallel import lattice_spacing, reduce_kspace, weak_copy

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = configs.make(0).subset(8)
    seq = w.sequence
    tables = O.precompute_tables(seq)
    mine = weak_copy(w.block, world, rank, lattice_spacing(configs.make(0).block.pos))
    echoes, _ = O.compute_block(tables, mine.pos, mine.mx, mine.my, mine.mz, mine.t1, mine.t2, mine.m0,
                                mine.domega, mine.weight)
    t = torch.from_numpy(np.ascontiguousarray(echoes).view(np.float64).copy())
    reduce_kspace(t, dst=0)
    if rank == 0:
        np.save(out_path, t.numpy().view(np.complex128).reshape(echoes.shape))
    dist.barrier()
    dist.destroy_process_group()


def test_weak_scaling_copies_sum_to_the_interleaved_object(tmp_path):
    """bench.py --scaling weak: rank r integrates the whole lattice shifted by r/world of its x spacing;
    the reduced k-space equals one process integrating all copies as one block."""
    import torch.multiprocessing as mp

    from oracle import bloch_oracle as O
    from paper_1305_6861_b200 import configs
    from paper_1305_6861_b200.parallel import lattice_spacing, weak_copy

    out = str(tmp_path / "weak.npy")
    mp.start_processes(_weak_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    w = configs.make(0).subset(8)
    h = lattice_spacing(configs.make(0).block.pos)
    assert h > 0
    c0, c1 = weak_copy(w.block, 2, 0, h), weak_copy(w.block, 2, 1, h)
    assert np.array_equal(c0.pos, w.block.pos)  # rank 0 is the single-GPU workload
    assert np.allclose(c1.pos[:, 0] - w.block.pos[:, 0], h / 2) and np.array_equal(c1.pos[:, 1:], w.block.pos[:, 1:])
    cat = lambda a, b: np.concatenate([a, b], axis=-1)
    both = {k: cat(getattr(c0, k), getattr(c1, k)) for k in ("mx", "my", "mz", "t1", "t2", "m0", "domega", "weight")}
    ref, _ = O.compute_block(O.precompute_tables(w.sequence), np.vstack([c0.pos, c1.pos]), both["mx"], both["my"],
                             both["mz"], both["t1"], both["t2"], both["m0"], both["domega"], both["weight"])
    assert O.rel_l2(ref, got) <= 1e-13


def _run_worker(rank, world, port, out_path):
    import pickle

    import torch.distributed as dist

    from oracle import bloch_oracle as O
    from paper_1305_6861_b200.parallel import run_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    exp = _small_experiment()

    def oracle_compute(tables, b):  # the float64 oracle stands in for the GPU (no device here)
        return O.compute_block(O.precompute_tables(exp.sequence, snapshot_times=exp.snapshot_times), b.pos, b.mx,
                               b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)

    res = run_distributed(exp, compute=oracle_compute)
    if rank == 0:
        with open(out_path, "wb") as fh:
            pickle.dump((res.echo_matrix(), res.snapshots[0][1], res.metrics.workers,
                         sorted(res.metrics.busy_fraction)), fh)
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


def _small_experiment():
    from paper_1305_6861_b200.engine import Experiment
    from paper_1305_6861_b200.phantom import Phantom, PhantomBox
    from paper_1305_6861_b200.sequence import build_spin_echo, readout_gradient

    seq = build_spin_echo(0.25, 16, te=0.03, tr=1.0, readout_grad=readout_gradient(0.25, 16, 0.008))
    ph = Phantom([PhantomBox(origin=(-0.05, -0.04, -5e-4), size=(0.1, 0.08, 1e-3), m0=1.0, t1=1.0, t2=0.2)])
    return Experiment(sequence=seq, phantom=ph, spacing=(0.008, 0.008, 0.002), snapshot_times=(seq.end_time,))


def test_run_distributed_two_ranks_matches_one_process(tmp_path):
    """parallel.run_distributed (one process per GPU): shards, one reduce, rank-order final M, ÷ N on
    rank 0, per-rank busy time — equal to the whole block in one process (engine.py:465-537)."""
    import pickle

    import torch.multiprocessing as mp

    from oracle import bloch_oracle as O
    from paper_1305_6861_b200.engine import build_spin_arrays
    from paper_1305_6861_b200.phantom import rasterize_arrays

    out = str(tmp_path / "run.pkl")
    mp.start_processes(_run_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    with open(out, "rb") as fh:
        echoes, final, workers, ranks = pickle.load(fh)
    exp = _small_experiment()
    a = build_spin_arrays(rasterize_arrays(exp.phantom, exp.spacing), exp.system)
    ref_e, ref_s = O.compute_block(O.precompute_tables(exp.sequence, snapshot_times=exp.snapshot_times), a.pos, a.mx,
                                   a.my, a.mz, a.t1, a.t2, a.m0, a.domega, a.weight)
    assert workers == 2 and ranks == [0, 1]
    assert O.rel_l2(ref_e / a.n, echoes) <= 1e-13
    assert np.array_equal(ref_s[0], final)

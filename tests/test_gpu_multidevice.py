"""GPU: the device-set context (bloch_create_multi) and run(Experiment(devices=...)).

One B200 is available here, so the device set lists device 0 two or three times: every shard runs on
its own sub-context and stream, and the one exchange (peer copy of each partial k-space to the first
device, rank-order fp64 sum) runs exactly as on distinct GPUs.  The shards follow the reference's
np.linspace bounds (engine.py:229-251) and the final magnetisation rows land in rank order
(engine.py:497-504)."""

import numpy as np
import pytest

from oracle import bloch_oracle as O
from paper_1305_6861_b200 import configs
from paper_1305_6861_b200.engine import BlochEngine, Experiment, get_engine, precompute_sequence_tables, run
from paper_1305_6861_b200.parallel import shard_bounds

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k", [2, 3])
@pytest.mark.parametrize("precision", [32, 64])
def test_device_set_matches_one_device(k, precision):
    w = configs.make(1).subset(97)  # ~7.2k spins
    b = w.block
    seq = w.sequence
    t = precompute_sequence_tables(seq, snapshot_times=(0.5 * seq.end_time, seq.end_time))
    one = get_engine(0, precision)
    e1, s1 = one.compute(t, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)
    multi = BlochEngine(precision=precision, devices=[0] * k)
    ek, sk = multi.compute(t, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)
    # per-spin fp64 state: the same operations whatever the shard
    for a, c in zip(s1, sk):
        assert O.rel_l2(a, c) <= 1e-12
    # the k-space: the same spins summed over a different tiling and a rank-order fp64 sum
    assert O.rel_l2(e1, ek) <= (1e-6 if precision == 32 else 1e-13)
    # the sum is exactly the rank-order sum of the shards' own partials
    parts = []
    for r in range(k):
        lo, hi = shard_bounds(b.n, k, r)
        e_r, _ = one.compute(t, b.pos[lo:hi], b.mx[lo:hi], b.my[lo:hi], b.mz[lo:hi], b.t1[lo:hi], b.t2[lo:hi],
                             b.m0[lo:hi], b.domega[lo:hi], np.asarray(b.weight)[lo:hi])
        parts.append(e_r)
    acc = parts[0].copy()
    for p in parts[1:]:
        acc = acc + p
    assert np.array_equal(acc, ek)
    times = multi.device_times()
    assert len(times) == k and all(v["device_ms"] > 0 for v in times.values())
    # repeated calls are bit-identical
    ek2, _ = multi.compute(t, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)
    assert np.array_equal(ek, ek2)
    multi.close()


def test_device_set_multicoil_and_rejects_device_inputs():
    w = configs.make(4).subset(400)  # 8 coils
    b = w.block
    t = precompute_sequence_tables(w.sequence)
    e1, _ = get_engine(0, 32).compute(t, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)
    multi = BlochEngine(precision=32, devices=[0, 0])
    e2, _ = multi.compute(t, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)
    assert e2.shape == e1.shape and O.rel_l2(e1, e2) <= 1e-6
    from paper_1305_6861_b200.errors import InvalidParameter

    with pytest.raises(InvalidParameter):
        multi.compute_device(t, {"pos": 1, "mx": 1, "my": 1, "mz": 1, "t1": 1, "t2": 1, "m0": 1, "domega": 1,
                                 "weight": 0}, 10, 1, 1)
    multi.close()


def test_run_with_a_device_set_reports_per_gpu_busy_time():
    from paper_1305_6861_b200.phantom import Phantom, PhantomBox
    from paper_1305_6861_b200.sequence import build_spin_echo, readout_gradient

    seq = build_spin_echo(0.25, 16, te=0.03, tr=1.0, readout_grad=readout_gradient(0.25, 16, 0.008))
    ph = Phantom([PhantomBox(origin=(-0.05, -0.04, -5e-4), size=(0.1, 0.08, 1e-3), m0=1.0, t1=1.0, t2=0.2)])
    one = run(Experiment(sequence=seq, phantom=ph, spacing=(0.004, 0.004, 0.002), precision=64))
    two = run(Experiment(sequence=seq, phantom=ph, spacing=(0.004, 0.004, 0.002), precision=64, devices=(0, 0)))
    assert two.metrics.workers == 2 and set(two.metrics.busy_fraction) == {0, 1}
    assert all(v > 0 for v in two.metrics.device_ms.values())
    assert O.rel_l2(one.echo_matrix(), two.echo_matrix()) <= 1e-13

"""The reference's engine tests (tests/test_engine.py) restated against this package.

CPU: table construction and memoisation (test_engine.py:73-112), the comparison metric
(:277-308) and the error mapping of a failing block (:214-222).  GPU: the same properties
through the CUDA engine — memoised vs recomputed tables, run() output shape (:168-173),
snapshots in rasterisation order (:225-235) and interval splitting (:257-274).
"""

import math

import numpy as np
import pytest

from paper_1305_6861_b200 import (
    ElementarySequence,
    Experiment,
    Phantom,
    PhantomBox,
    Sequence,
    WorkerPanic,
    build_spin_echo,
    build_tse,
    delta_e_stoer,
    flatten_tables,
    precompute_sequence_tables,
    rasterize,
    readout_gradient,
    run,
    simulate_spin,
)
from paper_1305_6861_b200 import _capi
from paper_1305_6861_b200.bloch import Magnetization, RelaxationParams
from paper_1305_6861_b200.phantom import SpinSample


def box_phantom(m0=1.0, t2=0.2):
    return Phantom([PhantomBox(origin=(-0.05, -0.04, -5e-4), size=(0.1, 0.08, 1e-3), m0=m0, t1=1.0, t2=t2)])


def small_experiment(**kw):
    seq = build_spin_echo(fov=0.25, n=16, te=0.03, tr=1.0, readout_grad=readout_gradient(0.25, 16, 0.008))
    d = dict(sequence=seq, phantom=box_phantom(), spacing=(0.008, 0.008, 0.002), workers=1)
    d.update(kw)
    return Experiment(**d)


# -- CPU -----------------------------------------------------------------------------------------------------------


def test_tables_one_entry_per_elementary_sequence():
    seq = build_tse(0.5, 32, 2, 0.03, 0.8, readout_gradient(0.5, 32, 0.01))
    tables = precompute_sequence_tables(seq)
    assert len(tables.entries) == len(seq.elements) and tables.n_acq == 32


def test_pulse_memo_shares_repeated_pulses():
    seq = build_tse(0.5, 16, 2, 0.03, 0.8, readout_gradient(0.5, 16, 0.01))
    assert precompute_sequence_tables(seq).pulse_memo_hits > 0


def test_memoized_tables_bit_identical_to_recomputation():
    seq = build_spin_echo(0.25, 8, 0.03, 0.5, readout_gradient(0.25, 8, 0.008))
    a = flatten_tables(precompute_sequence_tables(seq, memoize=True))
    b = flatten_tables(precompute_sequence_tables(seq, memoize=False))
    for k in a:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k


def test_delta_e_sentinel_scaled_and_zero():
    data = np.array([1.0 + 2.0j, 3.0 - 1.0j])
    assert delta_e_stoer(data, data) == -math.inf
    rng = np.random.default_rng(0)
    ref = rng.normal(size=256) + 1j * rng.normal(size=256)
    assert delta_e_stoer(ref, ref * (1.0 + 1e-6)) == pytest.approx(-120.0, abs=0.5)
    assert delta_e_stoer(np.array([1.0, 2.0, 3.0]), np.zeros(3)) == pytest.approx(0.0, abs=1e-12)


def test_device_failure_surfaces_block_index():
    """A CUDA failure status maps to WorkerPanic carrying the block index (engine.py:455-459, 575-577)."""
    with pytest.raises(WorkerPanic) as ei:
        _capi.check(_capi.BLOCH_E_CUDA, "bloch_compute_block", block_index=3)
    assert ei.value.block_index == 3


# -- GPU -----------------------------------------------------------------------------------------------------------


@pytest.mark.gpu
def test_memoized_vs_recomputed_on_gpu():
    seq = build_spin_echo(0.25, 8, 0.03, 0.5, readout_gradient(0.25, 8, 0.008))
    spin = SpinSample(position=(0.01, -0.005, 0.0), m=Magnetization(0, 0, 1), relax=RelaxationParams(1.0, 0.2, 1.0))
    a, _ = simulate_spin(spin, precompute_sequence_tables(seq, memoize=True), domega=35.0)
    b, _ = simulate_spin(spin, precompute_sequence_tables(seq, memoize=False), domega=35.0)
    assert np.array_equal(a, b)


@pytest.mark.gpu
def test_run_produces_expected_shape():
    res = run(small_experiment(blocks=8))
    assert len(res.echoes) == 16 and all(rec.values.size == 16 for rec in res.echoes)
    assert res.metrics.throughput > 0 and res.metrics.spin_count == res.spin_count


@pytest.mark.gpu
def test_snapshots_in_rasterization_order():
    exp = small_experiment(snapshot_times=(0.0, 0.0301), blocks=4, precision=64)
    res = run(exp)
    spins = rasterize(exp.phantom, exp.spacing)
    assert len(res.snapshots) == 2
    t0, snap0 = res.snapshots[0]
    assert t0 == 0.0 and snap0.shape == (len(spins), 3)
    np.testing.assert_allclose(snap0[:, 2], 0.0, atol=1e-12)  # right after the excitation pulse
    np.testing.assert_allclose(np.hypot(snap0[:, 0], snap0[:, 1]), 1.0, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", [64, 32])
def test_split_interval_trajectories_identical(precision):
    """Splitting the first elementary sequence in two (same pulse, same constant gradient) leaves the
    echoes unchanged (test_engine.py:257-274; split_elementary restated for constant gradients)."""
    seq = build_spin_echo(0.25, 8, 0.03, 0.5, readout_gradient(0.25, 8, 0.008))
    es = seq.elements[0]
    d1 = es.duration * 0.37
    first = ElementarySequence(pulse=es.pulse, gradient=es.gradient, duration=d1)
    second = ElementarySequence(gradient=es.gradient, duration=es.duration - d1)
    split = Sequence([first, second] + list(seq.elements[1:]), name="split")
    spin = SpinSample(position=(0.013, -0.007, 0.0), m=Magnetization(0, 0, 1), relax=RelaxationParams(1.0, 0.2, 1.0))
    a, _ = simulate_spin(spin, precompute_sequence_tables(seq), domega=12.0, precision=precision)
    b, _ = simulate_spin(spin, precompute_sequence_tables(split), domega=12.0, precision=precision)
    tol = 1e-12 if precision == 64 else 1e-6
    np.testing.assert_allclose(a, b, rtol=tol, atol=tol * np.abs(a).max())

"""CPU: host layer, C-ABI surface and the table compiler (no GPU needed).

* the library loads and exports every symbol include/bloch_b200.h declares;
* a compile-only context (BLOCH_HOST_ONLY) compiles every config and reports
  the reference table size E and ADC sample count;
* malformed tables are rejected with InvalidParameter (the reference's
  error type for bad arguments, engine.py:467-473), compute calls on a
  compile-only context raise, and there is no CPU fallback;
* the mirrored reference API behaves like the reference (partitioning,
  comparison metric, builders, error types).
"""

import math
import os
import re

import numpy as np
import pytest

from oracle import bloch_oracle as O
from paper_1305_6861_b200 import (
    AcquisitionSpec,
    DeviceError,
    ElementarySequence,
    Experiment,
    GradientWaveform,
    HardPulse,
    InvalidParameter,
    Sequence,
    build_tse,
    compare_results,
    configs,
    delta_e_stoer,
    partition_blocks,
    precompute_sequence_tables,
    readout_gradient,
    run,
)
from paper_1305_6861_b200 import _capi
from paper_1305_6861_b200.engine import BlochEngine, event_counts
from paper_1305_6861_b200.parallel import shard_bounds

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "bloch_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(bloch_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _capi.load()
    names = header_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(lib, name), f"{name} not exported"
        assert name in _capi.SIGNATURES, f"{name} not bound in _capi"
    assert lib.bloch_abi_version() == 1
    assert b"sm_100a" in lib.bloch_version()


def test_device_count_without_gpu_is_zero_or_more():
    assert _capi.device_count() >= 0


@pytest.fixture(scope="module")
def host_engine():
    return BlochEngine(device=-1)


@pytest.mark.parametrize("index", [0, 1, 2, 3, 4])
def test_compile_configs(host_engine, index):
    w = configs.make(index)
    tables = precompute_sequence_tables(w.sequence)
    host_engine.set_tables(tables)
    st = host_engine.program_stats()
    counts = event_counts(tables)
    assert st["events"] == counts["events"] == O.event_count(O.precompute_tables(w.sequence))
    assert st["samples"] == counts["adc"]
    assert st["window_samples"] + st["chirp_samples"] <= st["samples"]
    assert st["rot"] == counts["rot"]
    assert st["rot_classes"] <= 64
    # deferred-window view: every sample is either contracted or still summed by the integrator
    assert st["contracted_samples"] + st["integrator_samples"] == st["samples"]
    assert st["window_groups"] >= 1  # every config reads out in long uniform windows


@pytest.mark.parametrize("index,groups,integrator", [(0, 1, 0), (1, 1, 0), (2, 1, 0), (4, 1, 0)])
def test_window_groups_of_configs(host_engine, index, groups, integrator):
    """Spin-echo / TSE / stimulated-echo readouts: one group per readout class, nothing left to the
    integrator's per-warp sums (configs 0-2 and 4: one readout gradient)."""
    host_engine.set_tables(precompute_sequence_tables(configs.make(index).sequence))
    st = host_engine.program_stats()
    assert st["window_groups"] == groups
    assert st["integrator_samples"] == integrator
    assert st["contracted_samples"] == st["window_samples"]


def test_compile_detects_structure(host_engine):
    host_engine.set_tables(precompute_sequence_tables(configs.make(3).sequence))
    assert host_engine.program_stats()["chirp_samples"] > 2000  # trapezoid ramps under the ADC
    host_engine.set_tables(precompute_sequence_tables(configs.make(4).sequence))
    st = host_engine.program_stats()
    assert st["train_pairs"] == 3 * 256 * 128  # sinc sub-pulses
    # the three pulses of every line are the same sinc under the same slice gradient: one train class
    assert st["train_classes"] == 1 and st["train_class_ops"] == 3 * 128


def test_malformed_tables_rejected(host_engine):
    tables = precompute_sequence_tables(configs.make(0).sequence)
    tables.entries[3].ev_snap[:] = 5  # snapshot index beyond n_snap
    with pytest.raises(InvalidParameter):
        host_engine.set_tables(tables)
    tables = precompute_sequence_tables(configs.make(0).sequence)
    tables.entries[2].ev_dt[1] = -1.0
    with pytest.raises(InvalidParameter):
        host_engine.set_tables(tables)


def test_compute_on_host_only_context_raises(host_engine):
    tables = precompute_sequence_tables(configs.make(0).sequence)
    b = configs.make(0).block
    with pytest.raises(DeviceError):
        host_engine.compute(tables, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)


def test_no_cpu_fallback_without_device():
    if _capi.device_count() > 0:
        pytest.skip("a GPU is present")
    from paper_1305_6861_b200.errors import WorkerPanic

    with pytest.raises(WorkerPanic):
        BlochEngine(device=0)


def test_run_requires_spacing():
    w = configs.make(0)
    with pytest.raises(InvalidParameter):
        run(Experiment(sequence=w.sequence, phantom=None))
    with pytest.raises(InvalidParameter):
        run(Experiment(sequence=w.sequence, phantom=None, spacing=(1.0, 1.0, 1.0), workers=0))


def test_partition_blocks_cover_disjointly():  # test_engine.py:344-351
    b = configs.make(0).block
    blocks = partition_blocks(b, 7)
    assert sum(x.n for x in blocks) == b.n
    assert np.array_equal(np.vstack([x.pos for x in blocks]), b.pos)
    bounds = O.partition_bounds(b.n, 7)
    assert [x.n for x in blocks] == list(np.diff(bounds))


def test_shard_bounds_match_partition():
    for n in (0, 1, 7, 1000, 697708):
        for world in (1, 2, 3, 8):
            b = [shard_bounds(n, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[r][1] == b[r + 1][0] for r in range(world - 1))


def test_compare_results_counts_exceedances():  # test_engine.py:294-308
    ref = np.array([1.0, 1.0, 1.0, 1e-300])
    test = ref.copy()
    test[1] *= 1.0 + 1e-3
    cmp = compare_results(ref, test, rel_threshold=1e-6)
    assert cmp.exceedances == 1 and cmp.compared == 3
    assert delta_e_stoer(ref, ref) == -math.inf


def test_builders_reject_bad_input():
    with pytest.raises(InvalidParameter):
        readout_gradient(0.25, 1, 1e-3)
    with pytest.raises(InvalidParameter):
        build_tse(0.5, 10, 3, 0.03, 0.8, readout_gradient(0.5, 10, 0.01))
    with pytest.raises(InvalidParameter):
        ElementarySequence(duration=-1.0)
    with pytest.raises(InvalidParameter):
        ElementarySequence(duration=1e-3, gradient=GradientWaveform.trapezoid(gx=1e-3, ramp_s=1e-4, flat_s=1e-4))
    with pytest.raises(InvalidParameter):
        Sequence([])


def test_end_time_is_the_engine_clock():
    # Sequence.duration uses Python's compensated sum; the table compiler's running
    # t0 can differ by an ulp, and a snapshot at `duration` would then be dropped.
    seq = configs.make(0).sequence
    t = precompute_sequence_tables(seq, snapshot_times=(seq.end_time,))
    assert any((e.ev_snap >= 0).any() for e in t.entries)


def test_empty_and_single_sample_windows(host_engine):
    els = [ElementarySequence(pulse=HardPulse(math.pi / 2), duration=1e-3),
           ElementarySequence(duration=1e-3, acquisition=AcquisitionSpec(True, 1), kspace_row=0),
           ElementarySequence(duration=0.0)]
    tables = precompute_sequence_tables(Sequence(els))
    host_engine.set_tables(tables)
    st = host_engine.program_stats()
    assert st["samples"] == 1 and st["events"] == event_counts(tables)["events"]


def test_compiler_class_cap_with_absorbing_windows():
    """More reused (pre, window, post) runs than rotation-class slots: the windows beyond the cap must
    keep their neighbouring intervals separate (regression: 'absorbing window without a class')."""
    import ctypes

    from paper_1305_6861_b200 import build_cpmg, readout_gradient
    from paper_1305_6861_b200.engine import BlochEngine, precompute_sequence_tables

    seq = build_cpmg(fov=0.375, n=64, n_echoes=12, dte=0.02, tr=2.0, readout_grad=readout_gradient(0.375, 64, 0.012))
    eng = BlochEngine.__new__(BlochEngine)
    lib = _capi.load()
    eng._lib, eng.device, eng.precision, eng._tables_ref, eng._flat = lib, _capi.BLOCH_HOST_ONLY, 32, None, None
    h = ctypes.c_void_p()
    _capi.check(lib.bloch_create(_capi.BLOCH_HOST_ONLY, 32, ctypes.byref(h)), "bloch_create")
    eng._h = h
    try:
        eng.set_tables(precompute_sequence_tables(seq))
        st = eng.program_stats()
    finally:
        eng.close()
    assert st["rot_classes"] == 64 and st["window_samples"] == 64 * 12 * 64

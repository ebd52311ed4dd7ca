"""Seeded random sequences through the GPU engine vs the float64 oracle.

The program compiler (csrc/program.cpp) turns the event stream into windows,
chirps, RF trains, rotation/progression/chirp classes, fused intervals and
fused pulses; each pass has its own conditions.  This fuzzer builds random
sequences out of the structures that trigger them — repeated TR blocks with an
arithmetic phase-encode series (progressions), constant/trapezoid/sampled
readouts under the ADC (windows, chirps, generic samples), shaped pulses with
real and complex envelopes (RF trains, general and x-axis), hard pulses about
x/y/arbitrary axes (fused pulses), snapshots anywhere — and checks the k-space
and every snapshot against the oracle (oracle/bloch_oracle.py) in both
precision modes.  A separate CPU test compiles many more seeds on a host-only
context (no GPU) to catch compiler exceptions.
"""

import math

import numpy as np
import pytest

from oracle import bloch_oracle as O
from paper_1305_6861_b200.engine import get_engine
from paper_1305_6861_b200 import (
    GAMMA_PROTON,
    AcquisitionSpec,
    ElementarySequence,
    GradientWaveform,
    HardPulse,
    Sequence,
    SpinBlock,
    compute_block,
    expand_shaped_pulse,
    precompute_sequence_tables,
)


def random_gradient(rng, dur):
    kind = rng.integers(0, 4)
    amp = lambda: float(rng.uniform(-2e-3, 2e-3)) * (rng.random() < 0.7)  # noqa: E731
    if kind == 0:
        return GradientWaveform.none()
    if kind == 1:
        return GradientWaveform.constant(gx=amp(), gy=amp(), gz=amp())
    if kind == 2:
        ramp = dur * float(rng.uniform(0.05, 0.3))
        return GradientWaveform.trapezoid(gx=amp(), gy=amp(), ramp_s=ramp, flat_s=dur - 2 * ramp)
    m = int(rng.integers(2, 9))
    return GradientWaveform.from_samples(rng.uniform(-1e-3, 1e-3, size=(m, 3)), dur / m)


def random_es(rng, row):
    dur = float(rng.uniform(5e-5, 4e-3))
    pulse = None
    if rng.random() < 0.25:
        phi = [0.0, math.pi / 2, float(rng.uniform(0, 2 * math.pi))][int(rng.integers(0, 3))]
        pulse = HardPulse(float(rng.uniform(0.05, math.pi)), phi)
    acq = AcquisitionSpec(True, int(rng.integers(1, 80))) if rng.random() < 0.3 else AcquisitionSpec(False, 0)
    return ElementarySequence(pulse=pulse, gradient=random_gradient(rng, dur), duration=dur, acquisition=acq,
                              kspace_row=row if acq.enabled else None)


def random_sequence(seed):
    rng = np.random.default_rng(seed)
    els, row = [], 0
    # a TR block repeated with an arithmetic phase-encode series (progressions, window and interval classes)
    reps = int(rng.integers(1, 9))
    n_read = int(rng.integers(8, 70))
    read_dur = float(rng.uniform(2e-4, 2e-3))
    g_read = float(rng.uniform(-3e-3, 3e-3))
    trap = rng.random() < 0.4
    pe_step = float(rng.uniform(-4e-4, 4e-4))
    for r in range(reps):
        els.append(ElementarySequence(pulse=HardPulse(math.pi / 2, 0.0), duration=float(rng.uniform(1e-4, 1e-3))))
        els.append(ElementarySequence(gradient=GradientWaveform.constant(gy=(r - reps / 2) * pe_step, gx=-g_read / 2),
                                      duration=5e-4))
        if rng.random() < 0.5:
            els.append(ElementarySequence(pulse=HardPulse(math.pi, math.pi / 2), duration=2e-4))
        grad = (GradientWaveform.trapezoid(gx=g_read, ramp_s=read_dur * 0.2, flat_s=read_dur * 0.6) if trap
                else GradientWaveform.constant(gx=g_read))
        els.append(ElementarySequence(gradient=grad, duration=read_dur, acquisition=AcquisitionSpec(True, n_read),
                                      kspace_row=row))
        row += 1
        els.append(ElementarySequence(duration=float(rng.uniform(1e-3, 5e-3))))
    # a shaped pulse (RF train), real or complex envelope
    if rng.random() < 0.6:
        m = int(rng.integers(4, 40))
        env = np.sinc(np.linspace(-2, 2, m)) * 2e-6
        if rng.random() < 0.4:
            env = env * np.exp(1j * np.linspace(0, float(rng.uniform(0, 3)), m))
        els.extend(expand_shaped_pulse(env, 1e-5, GradientWaveform.constant(gz=float(rng.uniform(-5e-3, 5e-3)))))
    # free-form tail
    for _ in range(int(rng.integers(2, 12))):
        es = random_es(rng, row)
        if es.acquisition.enabled:
            row += 1
        els.append(es)
    return Sequence(els, name=f"fuzz{seed}")


def random_spins(seed, n=48):
    """Spins of seed: uniform 1+0j receive weight, a non-uniform single-coil weight, or 3 coils (seed % 3)."""
    rng = np.random.default_rng(seed + 1000)
    m0 = rng.uniform(0.2, 1.0, n)
    cplx = lambda *sh: rng.uniform(0.3, 1.0, sh) * np.exp(1j * rng.uniform(0, 2 * math.pi, sh))  # noqa: E731
    w = [np.full(n, 1 + 0j), cplx(n), cplx(3, n)][seed % 3]
    return SpinBlock(index=0, pos=rng.uniform(-0.05, 0.05, (n, 3)), mx=np.zeros(n), my=np.zeros(n), mz=m0.copy(),
                     t1=rng.uniform(0.3, 1.5, n), t2=rng.uniform(0.02, 0.3, n), m0=m0,
                     domega=rng.normal(0.0, 2 * math.pi * 30, n), weight=w)


def test_compiler_accepts_random_sequences():
    """Host-only compile of many random programs: no compiler exception, consistent statistics."""
    import ctypes

    from paper_1305_6861_b200 import _capi
    from paper_1305_6861_b200.engine import BlochEngine

    eng = BlochEngine.__new__(BlochEngine)
    lib = _capi.load()
    eng._lib, eng.device, eng.precision, eng._tables_ref, eng._flat = lib, _capi.BLOCH_HOST_ONLY, 32, None, None
    h = ctypes.c_void_p()
    _capi.check(lib.bloch_create(_capi.BLOCH_HOST_ONLY, 32, ctypes.byref(h)), "bloch_create")
    eng._h = h
    try:
        for seed in range(200):
            seq = random_sequence(seed)
            t = precompute_sequence_tables(seq, snapshot_times=(0.0, seq.end_time * 0.37, seq.end_time))
            eng.set_tables(t)
            st = eng.program_stats()
            assert st["events"] == O.event_count(t), seed
            assert st["samples"] == sum(x.size for x in t.acq_times), seed
    finally:
        eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(64))
def test_random_sequence_matches_oracle(seed):
    seq = random_sequence(seed)
    snaps_t = (0.0, seq.end_time * 0.37, seq.end_time)
    b = random_spins(seed)
    t = precompute_sequence_tables(seq, snapshot_times=snaps_t)
    ot = O.precompute_tables(seq, snapshot_times=snaps_t)
    ref_e, ref_s = O.compute_block(ot, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)
    for precision, tol_k, tol_m in ((64, 1e-10, 1e-11), (32, 1e-4, 1e-9)):
        e, s = compute_block(t, b, precision=precision)
        if np.linalg.norm(ref_e) > 0:
            assert O.rel_l2(ref_e, e) <= tol_k, (seed, precision, O.rel_l2(ref_e, e))
        for k, (a, r) in enumerate(zip(s, ref_s)):
            assert (a is None) == (r is None), (seed, k)
            if r is not None:
                assert O.rel_l2(r, a) <= tol_m, (seed, precision, k, O.rel_l2(r, a))


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("seed,coils,n", [(100, 1, 80_000), (101, 1, 320_000), (106, 1, 620_000), (102, 2, 80_000),
                                          (103, 4, 80_000), (104, 8, 80_000), (105, 8, 160_000), (107, 8, 20_000)])
def test_random_sequence_large_block(seed, coils, n):
    """Blocks large enough for the production kernel variants: the host picks spins per thread from the
    block size, the program and its planes (bloch_capi.cu pick_variant): 80k / 320k / 620k single-coil spins
    run 2 / 4-8 spins per thread, 20k / 80k / 160k eight-coil spins 1 / 2 / 4."""
    seq = random_sequence(seed)
    rng = np.random.default_rng(seed)
    m0 = rng.uniform(0.2, 1.0, n)
    w = (np.full(n, 1 + 0j) if coils == 1 else
         rng.uniform(0.3, 1.0, (coils, n)) * np.exp(1j * rng.uniform(0, 2 * math.pi, (coils, n))))
    b = SpinBlock(index=0, pos=rng.uniform(-0.05, 0.05, (n, 3)), mx=np.zeros(n), my=np.zeros(n), mz=m0.copy(),
                  t1=rng.uniform(0.3, 1.5, n), t2=rng.uniform(0.02, 0.3, n), m0=m0,
                  domega=rng.normal(0.0, 2 * math.pi * 30, n), weight=w)
    snaps_t = (seq.end_time,)
    t = precompute_sequence_tables(seq, snapshot_times=snaps_t)
    e, s = compute_block(t, b, precision=32)
    launch = get_engine(0, 32).last_launch()
    assert launch["precision"] == 32 and launch["spins_per_thread"] in (1, 2, 4, 8), launch
    ot = O.precompute_tables(seq, snapshot_times=snaps_t)
    ref_e, ref_s = O.compute_block(ot, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)
    assert O.rel_l2(ref_e, e) <= 1e-4, O.rel_l2(ref_e, e)
    assert O.rel_l2(ref_s[0], s[0]) <= 1e-9


def random_sequence_v2(seed):
    """Second generator: long (multi-pass) and very short windows, EPI-style alternating trapezoid readouts,
    repeated shaped pulses, zero-duration ES and pulses on acquiring ES."""
    rng = np.random.default_rng(10_000 + seed)
    els, row = [], 0
    els.append(ElementarySequence(pulse=HardPulse(float(rng.uniform(0.3, 1.6)), float(rng.uniform(0, 6.28))),
                                  duration=float(rng.uniform(1e-4, 2e-3))))
    n_lines = int(rng.integers(2, 7))
    n_read = int([rng.integers(2, 20), rng.integers(30, 90), rng.integers(250, 700)][int(rng.integers(0, 3))])
    dur = float(rng.uniform(3e-4, 3e-3))
    g = float(rng.uniform(5e-4, 3e-3))
    for line in range(n_lines):
        sign = 1.0 if line % 2 == 0 else -1.0
        grad = (GradientWaveform.trapezoid(gx=sign * g, ramp_s=0.15 * dur, flat_s=0.7 * dur) if rng.random() < 0.5
                else GradientWaveform.constant(gx=sign * g))
        els.append(ElementarySequence(gradient=grad, duration=dur, acquisition=AcquisitionSpec(True, n_read),
                                      kspace_row=row, kspace_reversed=bool(line % 2)))
        row += 1
        els.append(ElementarySequence(gradient=GradientWaveform.constant(gy=2e-4), duration=float(rng.uniform(2e-5, 1e-4))))
        if rng.random() < 0.3:
            els.append(ElementarySequence(duration=0.0))  # zero-duration ES
    if rng.random() < 0.6:  # the same shaped pulse twice (RF-train reuse)
        m = int(rng.integers(4, 24))
        env = np.hanning(m + 2)[1:-1] * float(rng.uniform(5e-7, 4e-6))
        for _ in range(2):
            els.extend(expand_shaped_pulse(env, 1e-5, GradientWaveform.constant(gz=float(rng.uniform(-4e-3, 4e-3)))))
            els.append(ElementarySequence(duration=float(rng.uniform(1e-4, 1e-3))))
    # a pulse on an acquiring ES, then a long plain window
    els.append(ElementarySequence(pulse=HardPulse(math.pi / 3, 0.7), gradient=GradientWaveform.constant(gy=-1e-3),
                                  duration=float(rng.uniform(2e-4, 1e-3)), acquisition=AcquisitionSpec(True, 40),
                                  kspace_row=row))
    row += 1
    els.append(ElementarySequence(gradient=GradientWaveform.constant(gx=float(rng.uniform(-1e-3, 1e-3))),
                                  duration=float(rng.uniform(1e-3, 4e-3)),
                                  acquisition=AcquisitionSpec(True, int(rng.integers(100, 600))), kspace_row=row))
    return Sequence(els, name=f"fuzz2_{seed}")


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(48))
def test_random_sequence_v2_matches_oracle(seed):
    seq = random_sequence_v2(seed)
    b = random_spins(seed)
    t_acq = precompute_sequence_tables(seq).acq_times
    # snapshots: one exactly on a sample instant, one mid-sequence, the end
    snaps_t = (float(t_acq[0][len(t_acq[0]) // 2]), seq.end_time * 0.61, seq.end_time)
    t = precompute_sequence_tables(seq, snapshot_times=snaps_t)
    ot = O.precompute_tables(seq, snapshot_times=snaps_t)
    ref_e, ref_s = O.compute_block(ot, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)
    for precision, tol_k, tol_m in ((64, 1e-10, 1e-11), (32, 1e-4, 1e-9)):
        e, s = compute_block(t, b, precision=precision)
        assert O.rel_l2(ref_e, e) <= tol_k, (seed, precision, O.rel_l2(ref_e, e))
        for k, (a, r) in enumerate(zip(s, ref_s)):
            assert (a is None) == (r is None), (seed, k)
            if r is not None:
                assert O.rel_l2(r, a) <= tol_m, (seed, precision, k, O.rel_l2(r, a))


def test_compiler_accepts_random_sequences_v2():
    import ctypes

    from paper_1305_6861_b200 import _capi
    from paper_1305_6861_b200.engine import BlochEngine

    eng = BlochEngine.__new__(BlochEngine)
    lib = _capi.load()
    eng._lib, eng.device, eng.precision, eng._tables_ref, eng._flat = lib, _capi.BLOCH_HOST_ONLY, 32, None, None
    h = ctypes.c_void_p()
    _capi.check(lib.bloch_create(_capi.BLOCH_HOST_ONLY, 32, ctypes.byref(h)), "bloch_create")
    eng._h = h
    try:
        for seed in range(200):
            seq = random_sequence_v2(seed)
            t = precompute_sequence_tables(seq, snapshot_times=(seq.end_time * 0.5,))
            eng.set_tables(t)
            assert eng.program_stats()["events"] == O.event_count(t), seed
    finally:
        eng.close()


def random_sequence_v3(seed):
    """Third generator: structures that the table compiler turns into shared per-spin tables — the same
    shaped pulse under the same gradient several times (train class: one composed affine propagator per
    spin) and alternating trapezoid readouts whose ramps mirror each other (chirp classes sharing a
    conjugated q plane), between hard pulses and plain windows."""
    rng = np.random.default_rng(20_000 + seed)
    m = int(rng.integers(4, 40))
    env = (np.hanning(m + 2)[1:-1] * float(rng.uniform(5e-7, 4e-6))).astype(complex)
    if seed % 2:  # a complex envelope (phase-modulated): general sub-pulse axes
        env = env * np.exp(1j * np.linspace(0.0, float(rng.uniform(0.5, 3.0)), m))
    gz = float(rng.uniform(-4e-3, 4e-3))
    g = float(rng.uniform(5e-4, 3e-3))
    dur = float(rng.uniform(3e-4, 2e-3))
    n_read = int(rng.integers(40, 160))
    els, row = [], 0
    for rep in range(int(rng.integers(2, 5))):
        els.extend(expand_shaped_pulse(env, 1e-5, GradientWaveform.constant(gz=gz)))
        els.append(ElementarySequence(duration=float(rng.uniform(2e-4, 1e-3))))
        for line in range(2):
            sign = 1.0 if line % 2 == 0 else -1.0
            els.append(ElementarySequence(gradient=GradientWaveform.trapezoid(gx=sign * g, ramp_s=0.2 * dur,
                                                                             flat_s=0.6 * dur),
                                          duration=dur, acquisition=AcquisitionSpec(True, n_read), kspace_row=row,
                                          kspace_reversed=bool(line)))
            row += 1
            els.append(ElementarySequence(gradient=GradientWaveform.constant(gy=3e-4), duration=4e-5))
        els.append(ElementarySequence(pulse=HardPulse(float(rng.uniform(0.3, 2.0)), float(rng.uniform(0, 6.28))),
                                      duration=float(rng.uniform(1e-4, 5e-4))))
    return Sequence(els, name=f"fuzz3_{seed}")


def _host_stats(seq):
    from paper_1305_6861_b200.engine import BlochEngine

    eng = BlochEngine(device=-1)
    try:
        eng.set_tables(precompute_sequence_tables(seq))
        return eng.program_stats()
    finally:
        eng.close()


def test_compiler_shares_trains_and_mirrored_ramps():
    for seed in range(8):
        st = _host_stats(random_sequence_v3(seed))
        assert st["train_classes"] == 1 and st["train_class_ops"] >= 2, (seed, st)
        assert st["chirp_classes"] >= 2 and st["chirp_samples"] > 0, (seed, st)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(16))
def test_shared_tables_match_oracle(seed):
    seq = random_sequence_v3(seed)
    b = random_spins(seed)
    snaps_t = (seq.end_time * 0.5, seq.end_time)
    t = precompute_sequence_tables(seq, snapshot_times=snaps_t)
    ot = O.precompute_tables(seq, snapshot_times=snaps_t)
    ref_e, ref_s = O.compute_block(ot, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)
    for precision, tol_k, tol_m in ((64, 1e-10, 1e-11), (32, 1e-4, 1e-9)):
        e, s = compute_block(t, b, precision=precision)
        assert O.rel_l2(ref_e, e) <= tol_k, (seed, precision, O.rel_l2(ref_e, e))
        for a, r in zip(s, ref_s):
            assert O.rel_l2(r, a) <= tol_m, (seed, precision, O.rel_l2(r, a))

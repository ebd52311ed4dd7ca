"""Parity cases shared by the golden generator (make_golden.py) and the tests.

Each case is a sequence built with the product's sequence model (field-for-field
the reference's, so make_golden.py converts it to reference objects), a spin
set, snapshot times, and the weight layout.  Small cases mirror the reference's
own engine tests (tests/test_engine.py:41-155, 225-269); the config cases are
BASELINE.json configs 0-4 (full size for config 0, deterministic rasterisation-
order subsets for 1-4).
"""

from __future__ import annotations

import math

import numpy as np

from paper_1305_6861_b200 import configs
from paper_1305_6861_b200.bloch import GAMMA_PROTON, HardPulse
from paper_1305_6861_b200.phantom import Phantom, PhantomBox
from paper_1305_6861_b200.sequence import (
    AcquisitionSpec,
    ElementarySequence,
    GradientWaveform,
    Sequence,
    build_cpmg,
    build_gradient_epi,
    build_spin_echo,
    build_tse,
    expand_shaped_pulse,
    readout_gradient,
)

# stride of the config subsets stored as goldens (and used by the GPU tests)
GOLDEN_STRIDE = {1: 14000, 2: 15000, 3: 15000, 4: 6000}


def box_phantom(m0=1.0, t2=0.2):  # test_engine.py:41-52
    return Phantom([PhantomBox(origin=(-0.05, -0.04, -5e-4), size=(0.1, 0.08, 1e-3), m0=m0, t1=1.0, t2=t2)])


def _spins(n, rng, spread=0.1, dw_sigma=50.0, complex_w=True, n_coils=0):
    pos = rng.uniform(-spread, spread, (n, 3))
    pos[:, 2] *= 0.05
    m0 = rng.uniform(0.2, 1.0, n)
    t1 = rng.uniform(0.3, 1.5, n)
    t2 = np.minimum(rng.uniform(0.02, 0.3, n), t1)
    dw = rng.normal(0.0, dw_sigma, n)
    if n_coils:
        w = rng.normal(size=(n_coils, n)) + 1j * rng.normal(size=(n_coils, n))
    elif complex_w:
        w = rng.normal(size=n) + 1j * rng.normal(size=n)
    else:
        w = np.full(n, 1.0 + 0.0j)
    # start off-equilibrium for half of the spins to exercise every state component
    mx = np.where(np.arange(n) % 2 == 0, 0.0, 0.3 * m0)
    my = np.where(np.arange(n) % 2 == 0, 0.0, -0.2 * m0)
    mz = np.where(np.arange(n) % 2 == 0, m0, 0.5 * m0)
    return dict(pos=pos, mx=mx, my=my, mz=mz, t1=t1, t2=t2, m0=m0, domega=dw, weight=w)


def fid_sequence(te=0.05):  # test_engine.py:105-112
    return Sequence([ElementarySequence(pulse=HardPulse(math.pi / 2, 0.0), duration=te),
                     ElementarySequence(duration=1e-3, acquisition=AcquisitionSpec(True, 5), kspace_row=0)],
                    name="fid")


def pair_sequence(k=500.0):  # test_engine.py:134-147
    return Sequence([ElementarySequence(pulse=HardPulse(math.pi / 2, -math.pi / 2), duration=0.0),
                     ElementarySequence(gradient=GradientWaveform.constant(gx=k / (GAMMA_PROTON * 0.01)),
                                        duration=0.01, acquisition=AcquisitionSpec(True, 9), kspace_row=0)],
                    name="pair")


def mixed_sequence():
    """Every event shape the compiler must handle: trapezoid + sampled gradients under
    ADC, single-sample ADC, zero-duration pulses, a discretised shaped pulse."""
    g = GAMMA_PROTON
    els = [ElementarySequence(pulse=HardPulse(math.pi / 3, 0.4), duration=0.0),
           ElementarySequence(pulse=HardPulse(math.pi / 2, 0.0), duration=2e-3,
                              gradient=GradientWaveform.constant(gx=2e-3, gz=1e-3))]
    els.append(ElementarySequence(gradient=GradientWaveform.trapezoid(gx=8e-3, gy=-2e-3, ramp_s=2e-4, flat_s=1.2e-3),
                                  duration=1.6e-3, acquisition=AcquisitionSpec(True, 33), kspace_row=0))
    samples = np.stack([np.linspace(0, 5e-3, 11), np.sin(np.linspace(0, 3, 11)) * 2e-3, np.zeros(11)], axis=1)
    els.append(ElementarySequence(gradient=GradientWaveform.from_samples(samples, 1e-4), duration=1e-3,
                                  acquisition=AcquisitionSpec(True, 17), kspace_row=1))
    env = np.sinc(np.linspace(-2, 2, 32)) * 1.5e-6 * np.exp(1j * np.linspace(0, 0.5, 32))
    env[5] = 0.0  # a zero sub-pulse carries no pulse
    els.extend(expand_shaped_pulse(env, 20e-6, GradientWaveform.constant(gz=4e-3), g))
    els.append(ElementarySequence(duration=3e-3, gradient=GradientWaveform.constant(gy=3e-3),
                                  acquisition=AcquisitionSpec(True, 1), kspace_row=2))
    els.append(ElementarySequence(pulse=HardPulse(math.pi, math.pi / 2), duration=1e-3))
    els.append(ElementarySequence(gradient=GradientWaveform.constant(gx=-5e-3), duration=2.4e-3,
                                  acquisition=AcquisitionSpec(True, 25), kspace_row=3))
    els.append(ElementarySequence(duration=0.05))
    return Sequence(els, name="mixed")


def small_cases():
    """name -> dict(sequence, spins, snapshot_times)."""
    rng = np.random.default_rng(20261019)
    out = {}
    fid_spin = dict(pos=np.zeros((1, 3)), mx=np.zeros(1), my=np.zeros(1), mz=np.ones(1), t1=np.ones(1),
                    t2=np.full(1, 0.2), m0=np.ones(1), domega=np.zeros(1), weight=np.full(1, 0.5 + 0j))
    out["fid"] = dict(sequence=fid_sequence(), spins=fid_spin, snapshot_times=(0.02,))
    pair = dict(pos=np.array([[0.004, 0, 0], [-0.004, 0, 0]]), mx=np.zeros(2), my=np.zeros(2), mz=np.ones(2),
                t1=np.full(2, np.inf), t2=np.full(2, np.inf), m0=np.ones(2), domega=np.zeros(2),
                weight=np.full(2, 1 + 0j))
    out["pair"] = dict(sequence=pair_sequence(), spins=pair, snapshot_times=())
    out["se16_box"] = dict(sequence=build_spin_echo(0.25, 16, 0.03, 1.0, readout_gradient(0.25, 16, 0.008)),
                           phantom=box_phantom(), spacing=(0.008, 0.008, 0.002), snapshot_times=(0.0, 0.0301))
    out["tse16"] = dict(sequence=build_tse(0.5, 16, 2, 0.03, 0.8, readout_gradient(0.5, 16, 0.01)),
                        spins=_spins(300, rng), snapshot_times=(0.4,))
    out["epi16"] = dict(sequence=build_gradient_epi(0.5, 16, 16, readout_gradient(0.5, 16, 1e-3)),
                        spins=_spins(300, rng, dw_sigma=200.0), snapshot_times=())
    out["cpmg8"] = dict(sequence=build_cpmg(0.375, 8, 4, 0.02, 1.0, readout_gradient(0.375, 8, 0.004)),
                        spins=_spins(200, rng, complex_w=False), snapshot_times=(0.5,))
    mixed = mixed_sequence()
    t_sample = 2e-3 + 1.6e-3 * 8 / 32  # exactly on an ADC instant of the trapezoid window
    out["mixed"] = dict(sequence=mixed, spins=_spins(250, rng, dw_sigma=300.0),
                        snapshot_times=(0.0, 1e-3, t_sample, 4.4e-3, mixed.end_time))
    out["mixed_coils"] = dict(sequence=mixed, spins=_spins(120, rng, dw_sigma=300.0, n_coils=3),
                              snapshot_times=(mixed.end_time,))
    out["tse_2coil"] = dict(sequence=build_tse(0.5, 16, 4, 0.03, 0.8, readout_gradient(0.5, 16, 0.01)),
                            spins=_spins(333, rng, n_coils=2), snapshot_times=(0.4,))
    return out


def config_case(index: int, stride=None):
    """Config `index`: full size for 0, the golden subset for 1-4 (or `stride`)."""
    w = configs.make(index)
    if index and (stride or GOLDEN_STRIDE[index]) > 1:
        w = w.subset(stride or GOLDEN_STRIDE[index])
    b = w.block
    spins = dict(pos=b.pos, mx=b.mx, my=b.my, mz=b.mz, t1=b.t1, t2=b.t2, m0=b.m0, domega=b.domega, weight=b.weight)
    return dict(sequence=w.sequence, spins=spins, snapshot_times=(w.sequence.end_time,), workload=w)

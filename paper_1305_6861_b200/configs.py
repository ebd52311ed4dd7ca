"""Seeded synthetic workloads — BASELINE.json ``configs`` 0-4.

No public dataset is involved: every input is generated here from
``numpy.random.Generator(PCG64(SeedSequence(cfg_index)))`` with child streams
spawned in the order geometry, tissue, off-resonance, RF jitter, coil maps
(SURVEY §8d).  Parameters BASELINE.json leaves open are marked † and recorded
in ``Workload.meta``:

* FOV 0.25 m †; ellipse centres U(-0.35, 0.35)·FOV †, semi-axes
  U(0.05, 0.35)·FOV †, angle U(0, pi) †; later ellipses override earlier ones
  (the head-phantom rule, phantom.py:167-169); per ellipse PD U[0,1],
  T1 U[0.3, 1.5] s, T2 U[0.04, 0.2] s (config 3: T2 U[0.02, 0.12] s).
  Background sites have PD = 0 and emit no spin (phantom.py:129-130), so the
  spin count is below the lattice size and the ÷N uses the emitted count.
* config 0: 64x64, 1 isochromat/pixel, spin echo 90°x / 180°y, TE 20 ms,
  TR 500 ms, 64x64 k-space, dwell 10 µs, Δω = 0, uniform receive.
* config 1: 256x256 px x 4x4 isochromats (1024² sites), Δω ~ N(0, (2π·20)²)
  per spin, TE 30 ms, TR 800 ms, 256x256 k-space, dwell 10 µs †.
* config 2: 512x512 px x 2x2 isochromats, TSE ETL 16, ESP 10 ms, 32 shots,
  refocusing 160° ± U(-5°, 5°) per echo, 512 samples, dwell 10 µs †,
  TR 2 s †, Δω a cubic 2-D polynomial scaled to peak ±2π·100 rad/s.
* config 3: 128x128 px x 8x8 isochromats, single-shot blipped EPI with
  trapezoidal readouts sampled every 4 µs on ramps and flat top
  (ramp 40 µs †, flat 500 µs †, blip 20 µs †), 128 lines, TE 40 ms at the
  k-space centre, T2 U[0.02, 0.12] s, Δω from 5 Gaussian bumps of ±2π·150 rad/s.
* config 4: 128x128x64 isochromats in a 3-D ellipsoid phantom; three
  slice-selective sinc pulses (TBW 4, 2.56 ms, 256 hard sub-pulses of 10 µs
  under a constant slice gradient, flips 90°/90°/90° †) centred at 0, 10 and
  25 ms; three 256-sample ADC windows per line † centred on the double
  (30 ms), stimulated (35 ms) and spin (40 ms) echoes; 128 phase-encode
  lines; TR 60 ms †; 8 receive coils with Gaussian |S| (σ = 0.4·FOV) centred
  on a ring of radius 0.5·FOV †, weight Sx - i·Sy (system.py:203-211).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, Optional

import numpy as np

from .bloch import GAMMA_PROTON, HardPulse
from .engine import SpinBlock
from .phantom import Phantom, PhantomBox, rasterize_arrays
from .sequence import (
    AcquisitionSpec,
    ElementarySequence,
    GradientWaveform,
    Sequence,
    build_spin_echo,
    build_tse,
    expand_shaped_pulse,
    readout_gradient,
)
from .system import CoilArray, GaussianCoil, complex_weight

FOV = 0.25
N_CONFIGS = 5


@dataclass
class Workload:
    index: int
    name: str
    sequence: Sequence
    block: SpinBlock
    meta: Dict = field(default_factory=dict)

    @property
    def n_spins(self) -> int:
        return self.block.n

    @property
    def n_coils(self) -> int:
        w = np.asarray(self.block.weight)
        return w.shape[0] if w.ndim == 2 else 1

    def subset(self, stride: int, offset: int = 0) -> "Workload":
        """Every stride-th spin in rasterisation order (deterministic parity subset)."""
        sl = slice(offset, None, stride)
        b = self.block
        w = np.asarray(b.weight)
        blk = SpinBlock(
            index=0, pos=b.pos[sl].copy(), mx=b.mx[sl].copy(), my=b.my[sl].copy(), mz=b.mz[sl].copy(),
            t1=b.t1[sl].copy(), t2=b.t2[sl].copy(), m0=b.m0[sl].copy(), domega=b.domega[sl].copy(),
            weight=w[..., sl].copy(),
        )
        meta = dict(self.meta, subset_stride=stride, subset_offset=offset)
        return Workload(self.index, self.name, self.sequence, blk, meta)


def _streams(index: int):
    ss = np.random.SeedSequence(index)
    geo, tissue, dw, rf, coil = ss.spawn(5)
    return (np.random.Generator(np.random.PCG64(s)) for s in (geo, tissue, dw, rf, coil))


class _Ellipses:
    """Vectorised label map of n seeded (2-D) ellipses or (3-D) ellipsoids."""

    def __init__(self, rng_geo, rng_tissue, n=10, dim=2, extent=(FOV, FOV, FOV), t2_range=(0.04, 0.2)):
        ext = np.asarray(extent[:dim], dtype=float)
        self.dim = dim
        self.c = rng_geo.uniform(-0.35, 0.35, (n, dim)) * ext
        self.ax = rng_geo.uniform(0.05, 0.35, (n, dim)) * ext
        self.ang = rng_geo.uniform(0.0, math.pi, n)
        self.pd = rng_tissue.uniform(0.0, 1.0, n)
        self.t1 = rng_tissue.uniform(0.3, 1.5, n)
        self.t2 = rng_tissue.uniform(t2_range[0], t2_range[1], n)

    def label(self, x, y, z):
        x = np.asarray(x, dtype=float)
        y = np.asarray(y, dtype=float)
        z = np.asarray(z, dtype=float)
        lab = np.full(x.shape, -1, dtype=np.int64)
        for k in range(self.pd.size):
            dx, dy = x - self.c[k, 0], y - self.c[k, 1]
            ca, sa = math.cos(self.ang[k]), math.sin(self.ang[k])
            u = (dx * ca + dy * sa) / self.ax[k, 0]
            v = (-dx * sa + dy * ca) / self.ax[k, 1]
            r = u * u + v * v
            if self.dim == 3:
                w = (z - self.c[k, 2]) / self.ax[k, 2]
                r = r + w * w
            lab = np.where(r <= 1.0, k, lab)  # later entries override earlier ones
        return lab

    def phantom(self, origin, size, bg_m0: float = 0.0) -> Phantom:
        def prop(table, background):
            def f(x, y, z):
                lab = self.label(x, y, z)
                return np.where(lab >= 0, table[np.maximum(lab, 0)], background)

            return f

        return Phantom([PhantomBox(origin=origin, size=size, m0=prop(self.pd, bg_m0), t1=prop(self.t1, 1.0),
                                   t2=prop(self.t2, 0.1))])


def _block(spins, domega, weight) -> SpinBlock:
    m0 = spins["m0"]
    return SpinBlock(
        index=0, pos=spins["pos"], mx=np.zeros_like(m0), my=np.zeros_like(m0), mz=m0.copy(),
        t1=spins["t1"], t2=spins["t2"], m0=m0, domega=np.asarray(domega, dtype=float), weight=weight,
    )


# --full-lattice: PD of the background tissue (T1 1 s, T2 0.1 s) †, so every lattice site emits a spin
FULL_LATTICE_BG_PD = 0.1


def _plane(pixels: int, iso: int, ell: _Ellipses, full_lattice: bool = False) -> Dict[str, np.ndarray]:
    spacing = FOV / (pixels * iso)
    ph = ell.phantom(origin=(-FOV / 2, -FOV / 2, -spacing / 2), size=(FOV, FOV, spacing),
                     bg_m0=FULL_LATTICE_BG_PD if full_lattice else 0.0)
    return rasterize_arrays(ph, (spacing, spacing, spacing), cap=4_000_000)


# ---------------------------------------------------------------------------


def config_sequence(index: int, rf=None) -> Sequence:
    """The sequence of config `index` (config 2 draws its refocusing jitter from the RF stream)."""
    if index in (0, 1):
        n, te, tr = (64, 0.020, 0.500) if index == 0 else (256, 0.030, 0.800)
        return build_spin_echo(FOV, n, te=te, tr=tr, readout_grad=readout_gradient(FOV, n, (n - 1) * 10e-6),
                               refocus_phi=math.pi / 2.0)
    if index == 2:
        if rf is None:
            rf = list(_streams(2))[3]
        n, tf = 512, 16
        jitter = rf.uniform(-5.0, 5.0, (n // tf, tf))
        return build_tse(FOV, n, tf, 0.010, tr=2.0, readout_grad=readout_gradient(FOV, n, (n - 1) * 10e-6),
                         refocus_alpha=lambda s, e: math.radians(160.0 + jitter[s, e]))
    if index == 3:
        return epi_trapezoid_sequence()
    if index == 4:
        return multipulse_3d_sequence()
    raise KeyError(index)


def _ring_coils(coil_rng, n_coils: int):
    """Gaussian coils on a ring of radius 0.5 FOV with a small seeded azimuth jitter."""
    ring = 0.5 * FOV
    jitter = coil_rng.uniform(-0.05, 0.05, n_coils)
    coils = []
    for c in range(n_coils):
        phi = 2.0 * math.pi * c / n_coils + jitter[c]
        coils.append(GaussianCoil(center=(ring * math.cos(phi), ring * math.sin(phi), 0.0), sigma=0.4 * FOV,
                                  phase=phi))
    return coils


def config0(full_lattice: bool = False) -> Workload:
    geo, tissue, _dw, _rf, _coil = _streams(0)
    ell = _Ellipses(geo, tissue)
    spins = _plane(64, 1, ell, full_lattice)
    seq = config_sequence(0)
    blk = _block(spins, np.zeros(spins["m0"].size), np.full(spins["m0"].size, 1.0 + 0.0j))
    return Workload(0, "cfg0_se64", seq, blk, {"fov": FOV, "grid": [64, 64], "iso": 1, "te": 0.02, "tr": 0.5,
                                                 "dwell": 10e-6})


def config1(full_lattice: bool = False) -> Workload:
    geo, tissue, dwr, _rf, _coil = _streams(1)
    ell = _Ellipses(geo, tissue)
    spins = _plane(256, 4, ell, full_lattice)
    seq = config_sequence(1)
    dw = dwr.normal(0.0, 2.0 * math.pi * 20.0, spins["m0"].size)
    blk = _block(spins, dw, np.full(spins["m0"].size, 1.0 + 0.0j))
    return Workload(1, "cfg1_se256_iso4", seq, blk, {"fov": FOV, "grid": [256, 256], "iso": 4, "te": 0.03,
                                                       "tr": 0.8, "dwell": 10e-6, "dw_sigma_hz": 20.0})


def config2(full_lattice: bool = False) -> Workload:
    geo, tissue, dwr, rf, _coil = _streams(2)
    ell = _Ellipses(geo, tissue)
    spins = _plane(512, 2, ell, full_lattice)
    n, tf = 512, 16
    seq = config_sequence(2, rf)
    # smooth cubic 2-D polynomial B0 map, peak +-2pi*100 rad/s over the lattice
    coef = dwr.normal(0.0, 1.0, 10)
    u = spins["pos"][:, 0] / (FOV / 2)
    v = spins["pos"][:, 1] / (FOV / 2)
    terms = [np.ones_like(u), u, v, u * u, u * v, v * v, u**3, u * u * v, u * v * v, v**3]
    poly = sum(c * t for c, t in zip(coef, terms))
    dw = poly * (2.0 * math.pi * 100.0 / max(np.max(np.abs(poly)), 1e-30))
    blk = _block(spins, dw, np.full(spins["m0"].size, 1.0 + 0.0j))
    return Workload(2, "cfg2_tse512_iso2", seq, blk, {"fov": FOV, "grid": [512, 512], "iso": 2, "etl": tf,
                                                        "esp": 0.01, "tr": 2.0, "dwell": 10e-6, "shots": n // tf,
                                                        "dw_peak_hz": 100.0})


def epi_trapezoid_sequence(n_lines=128, dwell=4e-6, ramp=40e-6, flat=500e-6, blip=20e-6, te=0.040,
                           prephase=0.5e-3, gamma=GAMMA_PROTON) -> Sequence:
    """Single-shot blipped EPI, trapezoidal readouts sampled on ramps and flat top."""
    dk = 2.0 * math.pi / FOV
    dur = 2.0 * ramp + flat
    n_samp = int(round(dur / dwell)) + 1
    g_read = (n_lines - 1) * dk / (gamma * flat)  # flat-top moment spans n_lines-1 k-steps
    m_line = gamma * g_read * (ramp + flat)
    period = dur + blip
    # centre of line n/2 (ky = +0.5 dk just past 0) at te
    t_train = te - (n_lines // 2) * period - dur / 2.0
    wait = t_train - prephase
    if wait <= 0.0:
        raise ValueError("EPI timing infeasible")
    ky0 = -(n_lines - 1) / 2.0 * dk
    els = [ElementarySequence(pulse=HardPulse(math.pi / 2.0, 0.0), duration=wait),
           ElementarySequence(gradient=GradientWaveform.constant(gx=-m_line / 2.0 / (gamma * prephase),
                                                                 gy=ky0 / (gamma * prephase)),
                              duration=prephase)]
    for line in range(n_lines):
        sign = 1.0 if line % 2 == 0 else -1.0
        els.append(ElementarySequence(gradient=GradientWaveform.trapezoid(gx=sign * g_read, ramp_s=ramp, flat_s=flat),
                                      duration=dur, acquisition=AcquisitionSpec(True, n_samp), kspace_row=line,
                                      kspace_reversed=line % 2 == 1))
        if line < n_lines - 1:
            els.append(ElementarySequence(gradient=GradientWaveform.constant(gy=dk / (gamma * blip)), duration=blip))
    return Sequence(els, name="epi_trapezoid", meta={"kind": "epi", "n": n_lines, "te": te, "dwell": dwell,
                                                      "ramp": ramp, "flat": flat, "blip": blip})


def config3(full_lattice: bool = False) -> Workload:
    geo, tissue, dwr, _rf, _coil = _streams(3)
    ell = _Ellipses(geo, tissue, t2_range=(0.02, 0.12))
    spins = _plane(128, 8, ell, full_lattice)
    seq = config_sequence(3)
    c = dwr.uniform(-0.4, 0.4, (5, 2)) * FOV
    sig = dwr.uniform(0.05, 0.15, 5) * FOV
    amp = np.where(dwr.uniform(0.0, 1.0, 5) < 0.5, -1.0, 1.0) * 2.0 * math.pi * 150.0
    x, y = spins["pos"][:, 0], spins["pos"][:, 1]
    dw = np.zeros_like(x)
    for k in range(5):
        dw += amp[k] * np.exp(-((x - c[k, 0]) ** 2 + (y - c[k, 1]) ** 2) / (2.0 * sig[k] ** 2))
    blk = _block(spins, dw, np.full(spins["m0"].size, 1.0 + 0.0j))
    return Workload(3, "cfg3_epi128_iso8", seq, blk, {"fov": FOV, "grid": [128, 128], "iso": 8, "te": 0.04,
                                                        "dwell": 4e-6, "bumps": 5, "bump_peak_hz": 150.0})


def sinc_envelope(flip: float, n: int = 256, tbw: float = 4.0, dt: float = 10e-6, gamma=GAMMA_PROTON) -> np.ndarray:
    """Real sinc B1 (tesla), time-bandwidth tbw, n samples of dt, small-tip area = flip."""
    t = (np.arange(n) + 0.5) / n - 0.5
    env = np.sinc(tbw * t)
    return env * (flip / (gamma * np.sum(env) * dt))


def multipulse_3d_sequence(n_lines=128, n_read=256, dwell=10e-6, flips=(math.pi / 2,) * 3,
                           centers=(0.0, 0.010, 0.025), windows=(0.030, 0.035, 0.040), slab=0.05, tr=0.060,
                           gamma=GAMMA_PROTON) -> Sequence:
    """Three slice-selective sinc pulses + three balanced ADC windows per line (config 4)."""
    dt, n_sub, tbw = 10e-6, 256, 4.0
    t_pulse = n_sub * dt
    gz = 2.0 * math.pi * (tbw / t_pulse) / (gamma * slab)
    g_read = readout_gradient(FOV, n_read, (n_read - 1) * dwell)
    t_win = (n_read - 1) * dwell
    m_read = gamma * g_read * t_win
    lobe = 0.5e-3
    dk = 2.0 * math.pi / FOV
    els = []
    for line in range(n_lines):
        ky = (line - (n_lines - 1) / 2.0) * dk
        t = -t_pulse / 2.0  # timeline relative to the first pulse centre
        for p, (flip, tc) in enumerate(zip(flips, centers)):
            start = tc - t_pulse / 2.0
            if start > t:
                els.append(ElementarySequence(duration=start - t))
            els.extend(expand_shaped_pulse(sinc_envelope(flip, n_sub, tbw, dt, gamma), dt,
                                           GradientWaveform.constant(gz=gz), gamma))
            t = tc + t_pulse / 2.0
            if p == 0:  # slice rephaser + phase encode
                els.append(ElementarySequence(
                    gradient=GradientWaveform.constant(gy=ky / (gamma * lobe), gz=-gz * (t_pulse / 2.0) / lobe),
                    duration=lobe))
                t += lobe
        for tw in windows:
            pre = tw - t_win / 2.0 - lobe
            if pre > t:
                els.append(ElementarySequence(duration=pre - t))
            els.append(ElementarySequence(gradient=GradientWaveform.constant(gx=-m_read / 2.0 / (gamma * lobe)),
                                          duration=lobe))
            els.append(ElementarySequence(gradient=GradientWaveform.constant(gx=g_read), duration=t_win,
                                          acquisition=AcquisitionSpec(True, n_read), kspace_row=line))
            els.append(ElementarySequence(gradient=GradientWaveform.constant(gx=-m_read / 2.0 / (gamma * lobe)),
                                          duration=lobe))
            t = tw + t_win / 2.0 + lobe
        end = tr - t_pulse / 2.0
        if end > t:
            els.append(ElementarySequence(duration=end - t))
    return Sequence(els, name="multipulse3d", meta={"kind": "3d-multipulse", "n_lines": n_lines, "tr": tr,
                                                     "flips": list(flips), "centers": list(centers),
                                                     "windows": list(windows)})


def config4(n_coils: int = 8, full_lattice: bool = False) -> Workload:
    geo, tissue, _dw, _rf, coil = _streams(4)
    ext = (FOV, FOV, FOV / 2)
    ell = _Ellipses(geo, tissue, dim=3, extent=ext)
    spacing = FOV / 128
    ph = ell.phantom(origin=(-FOV / 2, -FOV / 2, -FOV / 4), size=(FOV, FOV, FOV / 2),
                     bg_m0=FULL_LATTICE_BG_PD if full_lattice else 0.0)
    spins = rasterize_arrays(ph, (spacing, spacing, spacing), cap=4_000_000)
    seq = config_sequence(4)
    coils = _ring_coils(coil, n_coils)
    w = np.stack([complex_weight(cc, spins["pos"]) for cc in coils]) if spins["m0"].size else np.zeros((n_coils, 0))
    blk = _block(spins, np.zeros(spins["m0"].size), w)
    return Workload(4, "cfg4_3d_multipulse_8coil", seq, blk,
                    {"fov": FOV, "grid": [128, 128, 64], "coils": n_coils, "sigma_fov": 0.4, "ring_fov": 0.5,
                     "slab": 0.05, "tr": 0.06})


BUILDERS = {0: config0, 1: config1, 2: config2, 3: config3, 4: config4}


def make(index: int, full_lattice: bool = False) -> Workload:
    """Config `index`; ``full_lattice`` gives the background sites PD 0.1 (so configs 1-4 hold all
    1,048,576 lattice sites as spins, the count BASELINE.json states) and marks the name with ``_full``."""
    w = BUILDERS[int(index)](full_lattice=full_lattice)
    if full_lattice:
        w.name += "_full"
        w.meta["full_lattice_bg_pd"] = FULL_LATTICE_BG_PD
    return w


# ---------------------------------------------------------------------------
# the same workloads as device scenes (objects.DeviceScene)
# ---------------------------------------------------------------------------


@dataclass
class SceneWorkload:
    """A config whose spins are rasterised on the GPU (objects.rasterize_device)."""

    index: int
    name: str
    sequence: Sequence
    scene: object
    spacing: tuple
    extra_dw: Optional[object] = None  # n -> (n,) host array added per spin (random maps), or None
    cap: int = 4_000_000

    def rasterize(self, engine=None):
        from .objects import rasterize_device

        if self.extra_dw is None:
            return rasterize_device(self.scene, self.spacing, engine, cap=self.cap)
        # the count is only known after the lattice pass: rasterise, then add the per-spin map
        spins = rasterize_device(self.scene, self.spacing, engine, cap=self.cap)
        import torch

        spins.domega += torch.from_numpy(self.extra_dw(spins.n)).to(spins.domega.device)
        torch.cuda.current_stream(spins.domega.device).synchronize()
        return spins


def _label_box(ell: "_Ellipses", origin, size):
    from .objects import Ellipse, LabelBox

    shapes = []
    for k in range(ell.pd.size):
        shapes.append(Ellipse(center=tuple(ell.c[k]), axes=tuple(ell.ax[k]), angle=float(ell.ang[k]),
                              m0=float(ell.pd[k]), t1=float(ell.t1[k]), t2=float(ell.t2[k])))
    return LabelBox(origin=origin, size=size, m0=0.0, t1=1.0, t2=0.1, shapes=tuple(shapes))


def _plane_scene(pixels, iso, ell, **kw):
    from .objects import DeviceScene

    spacing = FOV / (pixels * iso)
    box = _label_box(ell, (-FOV / 2, -FOV / 2, -spacing / 2), (FOV, FOV, spacing))
    return DeviceScene([box], **kw), (spacing, spacing, spacing)


def scene(index: int) -> SceneWorkload:
    """Config `index` as a device scene: same seeded streams, same spins as make(index)."""
    from .objects import GaussianBumps, PolynomialField

    index = int(index)
    geo, tissue, dwr, rf, coil = _streams(index)
    if index == 0:
        ell = _Ellipses(geo, tissue)
        sc, sp = _plane_scene(64, 1, ell)
        return SceneWorkload(0, "cfg0_se64", config_sequence(0), sc, sp)
    if index == 1:
        ell = _Ellipses(geo, tissue)
        sc, sp = _plane_scene(256, 4, ell)
        return SceneWorkload(1, "cfg1_se256_iso4", config_sequence(1), sc, sp,
                             extra_dw=lambda n: dwr.normal(0.0, 2.0 * math.pi * 20.0, n))
    if index == 2:
        ell = _Ellipses(geo, tissue)
        seq = config_sequence(2, rf)
        coef = dwr.normal(0.0, 1.0, 10)
        expo = ((0, 0, 0), (1, 0, 0), (0, 1, 0), (2, 0, 0), (1, 1, 0), (0, 2, 0), (3, 0, 0), (2, 1, 0), (1, 2, 0),
                (0, 3, 0))
        poly = PolynomialField(coef=tuple(float(c) for c in coef), exponents=expo, length=FOV / 2,
                               peak=2.0 * math.pi * 100.0)
        sc, sp = _plane_scene(512, 2, ell, polynomial=poly)
        return SceneWorkload(2, "cfg2_tse512_iso2", seq, sc, sp)
    if index == 3:
        ell = _Ellipses(geo, tissue, t2_range=(0.02, 0.12))
        c = dwr.uniform(-0.4, 0.4, (5, 2)) * FOV
        sig = dwr.uniform(0.05, 0.15, 5) * FOV
        amp = np.where(dwr.uniform(0.0, 1.0, 5) < 0.5, -1.0, 1.0) * 2.0 * math.pi * 150.0
        bumps = GaussianBumps(centers=tuple(tuple(map(float, ck)) for ck in c), sigmas=tuple(map(float, sig)),
                              amps=tuple(map(float, amp)))
        sc, sp = _plane_scene(128, 8, ell, bumps=bumps)
        return SceneWorkload(3, "cfg3_epi128_iso8", config_sequence(3), sc, sp)
    if index == 4:
        from .objects import DeviceScene

        ext = (FOV, FOV, FOV / 2)
        ell = _Ellipses(geo, tissue, dim=3, extent=ext)
        spacing = FOV / 128
        box = _label_box(ell, (-FOV / 2, -FOV / 2, -FOV / 4), (FOV, FOV, FOV / 2))
        sc = DeviceScene([box], receive=CoilArray(_ring_coils(coil, 8)))
        return SceneWorkload(4, "cfg4_3d_multipulse_8coil", config_sequence(4), sc, (spacing,) * 3)
    raise KeyError(index)

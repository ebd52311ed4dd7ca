"""Rotating-frame constants and the hard-pulse operator (host side).

Sign conventions are the reference's (``mrsim/bloch.py:8-22``): a positive
angle turns the transverse magnetisation clockwise seen from +z, i.e.
``mx + 1j*my`` picks up ``exp(-1j*theta)``; a hard pulse (alpha, phi) tips
(0, 0, M0) to ``M0 * (-sin(phi)*sin(alpha), cos(phi)*sin(alpha), cos(alpha))``.
Only what the hot path needs lives here: the proton gyromagnetic ratio, the
pulse / relaxation value types, and the 3x3 pulse matrix the event tables
carry (``bloch.py:124-139``).
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np

# Gyromagnetic ratio of the proton, rad/(s*T) — bloch.py:41
GAMMA_PROTON = 2.0 * math.pi * 42.6e6


@dataclass(frozen=True)
class Magnetization:
    mx: float
    my: float
    mz: float

    def as_array(self) -> np.ndarray:
        return np.array([self.mx, self.my, self.mz], dtype=float)


def equilibrium(m0: float) -> Magnetization:
    return Magnetization(0.0, 0.0, float(m0))


@dataclass(frozen=True)
class RelaxationParams:
    """T1, T2 (s; ``math.inf`` disables) and equilibrium M0 (bloch.py:72-91)."""

    t1: float
    t2: float
    m0: float

    def __post_init__(self):
        if not (self.t1 > 0.0 and self.t2 > 0.0):
            raise ValueError(f"relaxation times must be positive, got t1={self.t1}, t2={self.t2}")
        if self.m0 < 0.0:
            raise ValueError(f"m0 must be non-negative, got {self.m0}")
        if self.t2 > self.t1:
            warnings.warn(f"t2={self.t2} s exceeds t1={self.t1} s (unphysical)", stacklevel=3)


@dataclass(frozen=True)
class HardPulse:
    """Instantaneous RF pulse: flip alpha about the transverse axis at azimuth phi."""

    alpha: float
    phi: float = 0.0

    @property
    def is_identity(self) -> bool:
        return self.alpha == 0.0


@dataclass(frozen=True)
class FrameContext:
    omega_hf: float
    gamma: float = GAMMA_PROTON


def hard_pulse_matrix(alpha: float, phi: float) -> np.ndarray:
    """Rotation by ``alpha`` about (cos phi, sin phi, 0), norm preserving.

    Axis-angle (Rodrigues) form R = cos(a) I + (1 - cos a) n n^T + sin(a) [n]x,
    transposed to the reference's sense (phi = 0 maps +z to +y), evaluated with
    the same products as bloch.py:131-139 so the tables match bit for bit.
    """
    ca, sa = np.cos(alpha), np.sin(alpha)
    cp, sp = np.cos(phi), np.sin(phi)
    one_m = 1.0 - ca
    return np.array(
        [
            [cp * cp + sp * sp * ca, sp * cp * one_m, -sp * sa],
            [sp * cp * one_m, sp * sp + cp * cp * ca, cp * sa],
            [sp * sa, -cp * sa, ca],
        ]
    )

"""Imaging-system model folded into the per-spin SoA before the kernel.

Mirrors the parts of ``mrsim.system`` the hot path consumes (system.py:105-225):
the per-spin rotating-frame off-resonance (``spin_off_resonance``, 123-132)
and the complex receive weight ``Sx - 1j*Sy`` (``complex_weight``, 203-211).
Extension: :class:`CoilArray`, a multi-coil receive model
whose weights form the ``(C, n)`` weight array of config 4.

Out of scope (host-side, not per event): the Legendre and loop Biot-Savart
models, grid loaders and the description grammar.  Inhomogeneity is given as
a vectorised callable ``delta_b0(x, y, z) -> tesla`` here.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from .bloch import GAMMA_PROTON, FrameContext


@dataclass(frozen=True)
class StaticField:
    b0: float
    inhomogeneity: Optional[Callable] = None  # vectorised delta_B0(x, y, z) in tesla

    def delta_b0(self, pos: np.ndarray) -> np.ndarray:
        pos = np.atleast_2d(pos)
        if self.inhomogeneity is None:
            return np.zeros(pos.shape[0])
        return np.asarray(self.inhomogeneity(pos[:, 0], pos[:, 1], pos[:, 2]), dtype=float)


@dataclass(frozen=True)
class UniformSensitivity:
    """Homogeneous transverse sensitivity (S, 0, 0) (system.py:140-147)."""

    s: float = 1.0

    def __call__(self, pos: np.ndarray) -> np.ndarray:
        pos = np.atleast_2d(pos)
        out = np.zeros((pos.shape[0], 3))
        out[:, 0] = self.s
        return out


@dataclass(frozen=True)
class GaussianCoil:
    """Transverse sensitivity |S| = exp(-|x - c|^2 / (2 sigma^2)) along azimuth ``phase``."""

    center: tuple
    sigma: float
    phase: float = 0.0

    def __call__(self, pos: np.ndarray) -> np.ndarray:
        pos = np.atleast_2d(pos)
        d2 = np.sum((pos - np.asarray(self.center, dtype=float)) ** 2, axis=1)
        mag = np.exp(-d2 / (2.0 * self.sigma**2))
        out = np.zeros((pos.shape[0], 3))
        out[:, 0] = mag * np.cos(self.phase)
        out[:, 1] = mag * np.sin(self.phase)
        return out


@dataclass(frozen=True)
class CoilArray:
    """C receive coils; the engine's weight array becomes (C, n)."""

    coils: List = field(default_factory=list)

    def __len__(self):
        return len(self.coils)


def complex_weight(sensitivity, pos: np.ndarray) -> np.ndarray:
    """Per-spin receive weight Sx - 1j*Sy (system.py:203-211), vectorised."""
    s = np.asarray(sensitivity(np.atleast_2d(pos)), dtype=float)
    return s[:, 0] - 1j * s[:, 1]


@dataclass(frozen=True)
class SystemModel:
    field: StaticField
    receive: object
    gamma: float = GAMMA_PROTON
    omega_hf: Optional[float] = None

    def frame(self) -> FrameContext:
        omega = self.omega_hf if self.omega_hf is not None else self.gamma * self.field.b0
        return FrameContext(omega_hf=omega, gamma=self.gamma)


def default_system(b0: float = 1.5) -> SystemModel:
    return SystemModel(field=StaticField(b0=b0), receive=UniformSensitivity())


def spin_off_resonance(system: SystemModel, pos: np.ndarray, object_dw: np.ndarray) -> np.ndarray:
    """(gamma*B0 - omega_hf) + gamma*delta_B0(x) + object offset (system.py:123-132; engine.py:201-210)."""
    ctx = system.frame()
    base = (ctx.gamma * system.field.b0 - ctx.omega_hf) + np.asarray(object_dw, dtype=float)
    if system.field.inhomogeneity is None:
        return base
    return (ctx.gamma * system.field.b0 - ctx.omega_hf) + ctx.gamma * system.field.delta_b0(pos) + np.asarray(
        object_dw, dtype=float
    )


def receive_weights(system: SystemModel, pos: np.ndarray) -> np.ndarray:
    """(n,) complex weights, or (C, n) for a :class:`CoilArray` (engine.py:211-214)."""
    rx = system.receive
    n = np.atleast_2d(pos).shape[0] if np.size(pos) else 0
    if isinstance(rx, UniformSensitivity):
        return np.full(n, complex(rx.s, 0.0))
    if isinstance(rx, CoilArray):
        return np.stack([complex_weight(c, pos) for c in rx.coils]) if n else np.zeros((len(rx), 0), complex)
    return complex_weight(rx, pos)

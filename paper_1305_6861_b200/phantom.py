"""Object model: boxes of tissue and their spin-lattice rasterization.

Same semantics as the reference's ``mrsim.phantom`` (phantom.py:29-142): each
box is sampled on a lattice centred in the box (``_lattice``, 91-95); spins are
ordered box, then z, y, x with x fastest (98-105, 125-127); sites whose M0
evaluates to zero emit no spin (129-130); every spin starts at (0, 0, M0)
(137).  :func:`rasterize_arrays` does this vectorised and returns the
structure-of-arrays the engine consumes directly (the reference's Python triple
loop costs ~15 µs per site); :func:`rasterize` keeps the
reference's list-of-``SpinSample`` return type.

Box properties may be constants or callables ``f(x, y, z)``; callables are
first tried on whole coordinate arrays and fall back to per-site evaluation.
The ten-ellipse head phantom (:func:`shepp_logan`, phantom.py:145-205) is
here, vectorised.  Out of scope: the object-file grammar.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Union

import numpy as np

from .bloch import Magnetization, RelaxationParams
from .errors import InvalidParameter, SpinBudgetExceeded

PropertyFn = Union[float, Callable[[float, float, float], float]]

DEFAULT_SPIN_CAP = 2_000_000  # phantom.py:26


@dataclass(frozen=True)
class PhantomBox:
    origin: tuple
    size: tuple
    m0: PropertyFn = 1.0
    t1: PropertyFn = 1.0
    t2: PropertyFn = 0.1
    delta_omega: PropertyFn = 0.0

    def __post_init__(self):
        if len(self.origin) != 3 or len(self.size) != 3:
            raise InvalidParameter("origin and size must be 3-vectors")
        if any(s <= 0.0 for s in self.size):
            raise InvalidParameter(f"box size components must be positive, got {self.size}")


@dataclass
class Phantom:
    boxes: List[PhantomBox] = field(default_factory=list)

    def __post_init__(self):
        if not self.boxes:
            raise InvalidParameter("a phantom needs at least one box")

    def bounding_box(self) -> tuple:
        lo = np.min([b.origin for b in self.boxes], axis=0)
        hi = np.max([np.add(b.origin, b.size) for b in self.boxes], axis=0)
        return lo, hi


@dataclass
class SpinSample:
    position: tuple
    m: Magnetization
    relax: RelaxationParams
    delta_omega: float = 0.0


def lattice(origin: float, size: float, spacing: float) -> np.ndarray:
    """1-D lattice with the given spacing, centred in [origin, origin+size] (phantom.py:91-95)."""
    n = max(1, int(math.floor(size / spacing + 1e-9)))
    offset = (size - (n - 1) * spacing) / 2.0
    return origin + offset + spacing * np.arange(n)


def _evaluate(prop: PropertyFn, x: np.ndarray, y: np.ndarray, z: np.ndarray) -> np.ndarray:
    if not callable(prop):
        return np.full(x.shape, float(prop))
    try:
        out = np.asarray(prop(x, y, z), dtype=float)
        if out.shape == x.shape:
            return out
        if out.ndim == 0:
            return np.full(x.shape, float(out))
    except Exception:  # scalar-only callable: evaluate per site like the reference
        pass
    return np.array([float(prop(float(a), float(b), float(c))) for a, b, c in zip(x, y, z)])


def _check_budget(phantom: Phantom, spacing, cap: int) -> tuple:
    spacing = tuple(float(s) for s in spacing)
    if len(spacing) != 3 or any(s <= 0.0 for s in spacing):
        raise InvalidParameter(f"spacing components must be positive, got {spacing}")
    total = 0
    for box in phantom.boxes:
        n = 1
        for axis in range(3):
            n *= max(1, int(math.floor(box.size[axis] / spacing[axis] + 1e-9)))
        total += n
    if total > cap:
        raise SpinBudgetExceeded(
            f"{total} lattice sites exceed the cap of {cap}; refine the spacing or raise the cap"
        )
    return spacing


def rasterize_arrays(phantom: Phantom, spacing, cap: int = DEFAULT_SPIN_CAP) -> Dict[str, np.ndarray]:
    """Rasterize to SoA arrays: pos (n,3), m0, t1, t2, delta_omega (n,), float64.

    Identical spins, values and order to the reference's ``rasterize``.
    """
    spacing = _check_budget(phantom, spacing, cap)
    parts = {k: [] for k in ("pos", "m0", "t1", "t2", "delta_omega")}
    for box in phantom.boxes:
        xs = lattice(box.origin[0], box.size[0], spacing[0])
        ys = lattice(box.origin[1], box.size[1], spacing[1])
        zs = lattice(box.origin[2], box.size[2], spacing[2])
        zg, yg, xg = np.meshgrid(zs, ys, xs, indexing="ij")  # x fastest
        x, y, z = xg.ravel(), yg.ravel(), zg.ravel()
        m0 = _evaluate(box.m0, x, y, z)
        keep = m0 != 0.0
        x, y, z, m0 = x[keep], y[keep], z[keep], m0[keep]
        parts["pos"].append(np.stack([x, y, z], axis=1))
        parts["m0"].append(m0)
        parts["t1"].append(_evaluate(box.t1, x, y, z))
        parts["t2"].append(_evaluate(box.t2, x, y, z))
        parts["delta_omega"].append(_evaluate(box.delta_omega, x, y, z))
    out = {k: np.concatenate(v) if v else np.zeros((0, 3) if k == "pos" else 0) for k, v in parts.items()}
    if np.any(out["m0"] < 0.0):
        raise ValueError("m0 must be non-negative")
    if np.any(~(out["t1"] > 0.0)) or np.any(~(out["t2"] > 0.0)):
        raise ValueError("relaxation times must be positive")
    return out


def rasterize(phantom: Phantom, spacing, cap: int = DEFAULT_SPIN_CAP) -> List[SpinSample]:
    """The reference's list-of-SpinSample form (phantom.py:98-142)."""
    a = rasterize_arrays(phantom, spacing, cap)
    return [
        SpinSample(
            position=(float(p[0]), float(p[1]), float(p[2])),
            m=Magnetization(0.0, 0.0, float(m0)),
            relax=RelaxationParams(t1=float(t1), t2=float(t2), m0=float(m0)),
            delta_omega=float(dw),
        )
        for p, m0, t1, t2, dw in zip(a["pos"], a["m0"], a["t1"], a["t2"], a["delta_omega"])
    ]


# ---------------------------------------------------------------------------
# ten-ellipse head phantom (phantom.py:145-205)
# ---------------------------------------------------------------------------

# The classic Shepp-Logan geometry in units of the half-width (centre x0, y0;
# semi-axes a, b; rotation in degrees) with the reference's per-region
# equilibrium magnetisation; later rows override earlier ones inside their
# footprint (phantom.py:167-182).
HEAD_ELLIPSES = np.array([
    # x0,     y0,      a,      b,      phi,   m0
    [0.0,     0.0,     0.69,   0.92,   0.0,   1.00],
    [0.0,    -0.0184,  0.6624, 0.874,  0.0,   0.51],
    [0.22,    0.0,     0.11,   0.31,  -18.0,  0.40],
    [-0.22,   0.0,     0.16,   0.41,   18.0,  0.40],
    [0.0,     0.35,    0.21,   0.25,   0.0,   0.60],
    [0.0,     0.1,     0.046,  0.046,  0.0,   0.80],
    [0.0,    -0.1,     0.046,  0.046,  0.0,   0.80],
    [-0.08,  -0.605,   0.046,  0.023,  0.0,   0.70],
    [0.0,    -0.605,   0.023,  0.023,  0.0,   0.70],
    [0.06,   -0.605,   0.023,  0.046,  0.0,   0.70],
])
SHEPP_LOGAN_T1 = 1.0
SHEPP_LOGAN_T2 = 0.2
# cos/sin of each rotation from the math library, as the reference's scalar test evaluates them
_HEAD_TRIG = [(math.cos(math.radians(p)), math.sin(math.radians(p))) for p in HEAD_ELLIPSES[:, 4]]


def shepp_logan_m0(x, y, scale: float = 1.0):
    """Equilibrium magnetisation of the head phantom at (x, y), 0 outside (phantom.py:185-191).

    Accepts scalars or arrays; the membership test is the reference's expression
    (phantom.py:158-164) evaluated elementwise in the same order, so the labels
    agree bit for bit."""
    xa = np.asarray(x, dtype=float) / scale
    ya = np.asarray(y, dtype=float) / scale
    value = np.zeros(np.broadcast(xa, ya).shape)
    for (x0, y0, a, b, _phi, m0), (c, s) in zip(HEAD_ELLIPSES, _HEAD_TRIG):
        dx, dy = xa - x0, ya - y0
        u = (dx * c + dy * s) / a
        v = (-dx * s + dy * c) / b
        value = np.where(u * u + v * v <= 1.0, m0, value)
    return float(value) if value.ndim == 0 else value


def shepp_logan(scale: float, thickness: float = 1e-3) -> Phantom:
    """Ten-ellipse head phantom scaled so the unit half-width maps to ``scale`` metres: one thin box
    with an ellipse-membership M0 (phantom.py:194-205)."""
    if scale <= 0.0:
        raise InvalidParameter(f"scale must be positive, got {scale}")
    box = PhantomBox(
        origin=(-scale, -scale, -thickness / 2.0),
        size=(2.0 * scale, 2.0 * scale, thickness),
        m0=lambda x, y, z: shepp_logan_m0(x, y, scale),
        t1=SHEPP_LOGAN_T1,
        t2=SHEPP_LOGAN_T2,
        delta_omega=0.0,
    )
    return Phantom([box])

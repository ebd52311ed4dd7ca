"""Device-side object model.

The reference builds every spin on the host: ``phantom.rasterize`` walks the
lattice in a Python triple loop (phantom.py:98-142, ~15 µs per site) and
``engine.build_spin_arrays`` folds off-resonance and receive weight per spin
(engine.py:192-226; system.py:123-132, 203-211).  Here a :class:`DeviceScene`
— boxes whose tissue is a constant overridden inside seeded ellipses /
ellipsoids (label maps), plus analytic off-resonance maps and receive coils —
is rasterised by ``bloch_rasterize`` straight into device memory in the
reference's spin order, and the integrator reads it in place
(:meth:`DeviceSpins.pointers` -> ``BlochEngine.compute_device``).

Lattice coordinates, labels, M0/T1/T2 and the spin order are bit-identical to
:func:`~.phantom.rasterize_arrays` on :meth:`DeviceScene.host_phantom`; the
analytic maps agree to the last few ulps (libm ``exp``/``pow`` differ from
CUDA's).  Scenes that need arbitrary Python callables stay on the host path.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence as TySequence, Tuple

import numpy as np

from . import _capi
from .errors import InvalidParameter, SpinBudgetExceeded
from .phantom import DEFAULT_SPIN_CAP, Phantom, PhantomBox
from .system import CoilArray, GaussianCoil, UniformSensitivity


@dataclass(frozen=True)
class Ellipse:
    """Tissue inside an ellipse (2-D: ``z`` ignored) or ellipsoid rotated by ``angle`` in x-y."""

    center: tuple
    axes: tuple
    angle: float = 0.0
    m0: float = 1.0
    t1: float = 1.0
    t2: float = 0.1
    delta_omega: float = 0.0

    @property
    def dim(self) -> int:
        return len(self.axes)


@dataclass(frozen=True)
class LabelBox:
    """A phantom box: background tissue overridden by its shapes, later shapes winning."""

    origin: tuple
    size: tuple
    m0: float = 0.0
    t1: float = 1.0
    t2: float = 0.1
    delta_omega: float = 0.0
    shapes: Tuple[Ellipse, ...] = ()


@dataclass(frozen=True)
class PolynomialField:
    """dw += scale * sum_k coef_k (x/L)^a (y/L)^b (z/L)^c; ``peak`` rescales to that max |value| over the spins."""

    coef: Tuple[float, ...]
    exponents: Tuple[Tuple[int, int, int], ...]
    length: float
    scale: float = 1.0
    peak: Optional[float] = None


@dataclass(frozen=True)
class GaussianBumps:
    """dw += sum_j amp_j exp(-|r - c_j|^2 / (2 sigma_j^2)); 2-D centres ignore z."""

    centers: Tuple[tuple, ...]
    sigmas: Tuple[float, ...]
    amps: Tuple[float, ...]


@dataclass
class DeviceScene:
    boxes: TySequence[LabelBox]
    const_dw: float = 0.0  # (gamma*B0 - omega_hf) of the system model (system.py:123-132)
    polynomial: Optional[PolynomialField] = None
    bumps: Optional[GaussianBumps] = None
    receive: object = field(default_factory=UniformSensitivity)

    def __post_init__(self):
        if not self.boxes:
            raise InvalidParameter("a scene needs at least one box")
        rx = self.receive
        if not isinstance(rx, (UniformSensitivity, GaussianCoil, CoilArray)):
            raise InvalidParameter(f"receive model {type(rx).__name__} has no device form")
        if isinstance(rx, CoilArray) and not all(isinstance(c, GaussianCoil) for c in rx.coils):
            raise InvalidParameter("device coil arrays take GaussianCoil members only")

    # -- host restatement (the parity partner of the device path) ---------------------------------------------
    def host_phantom(self) -> Phantom:
        """The same scene as a host :class:`Phantom` with vectorised label-map callables."""

        def prop(box, attr):
            shapes = box.shapes
            background = float(getattr(box, attr))
            if not shapes:
                return background
            values = np.array([float(getattr(s, attr)) for s in shapes])

            def f(x, y, z):
                lab = _host_label(shapes, np.asarray(x, float), np.asarray(y, float), np.asarray(z, float))
                return np.where(lab >= 0, values[np.maximum(lab, 0)], background)

            return f

        return Phantom([PhantomBox(origin=b.origin, size=b.size, m0=prop(b, "m0"), t1=prop(b, "t1"),
                                   t2=prop(b, "t2"), delta_omega=prop(b, "delta_omega")) for b in self.boxes])

    def host_field(self, pos: np.ndarray, tissue_dw: np.ndarray) -> np.ndarray:
        """Host evaluation of the off-resonance maps, in the device's summation order."""
        x, y, z = pos[:, 0], pos[:, 1], pos[:, 2]
        dw = np.asarray(tissue_dw, float) + self.const_dw
        poly_term = None
        if self.polynomial is not None:
            pf = self.polynomial
            u, v, w = x / pf.length, y / pf.length, z / pf.length
            p = np.zeros_like(x)
            for c, (a, b, e) in zip(pf.coef, pf.exponents):
                p = p + c * (u**a * v**b * w**e)
            if pf.peak is not None:
                poly_term = p * (pf.peak / max(float(np.max(np.abs(p))) if p.size else 0.0, 1e-30))
            else:
                dw = dw + p * pf.scale
        if self.bumps is not None:
            for c, s, a in zip(self.bumps.centers, self.bumps.sigmas, self.bumps.amps):
                d2 = (x - c[0]) ** 2 + (y - c[1]) ** 2
                if len(c) > 2:
                    d2 = d2 + (z - c[2]) ** 2
                dw = dw + a * np.exp(-d2 / (2.0 * s**2))
        if poly_term is not None:
            dw = dw + poly_term
        return dw

    def n_sites(self, spacing) -> int:
        return sum(int(np.prod(_lattice_counts(b, spacing))) for b in self.boxes)


def _host_label(shapes, x, y, z):
    lab = np.full(x.shape, -1, dtype=np.int64)
    for k, s in enumerate(shapes):
        ca, sa = math.cos(s.angle), math.sin(s.angle)
        dx, dy = x - s.center[0], y - s.center[1]
        u = (dx * ca + dy * sa) / s.axes[0]
        v = (-dx * sa + dy * ca) / s.axes[1]
        r = u * u + v * v
        if s.dim == 3:
            w = (z - s.center[2]) / s.axes[2]
            r = r + w * w
        lab = np.where(r <= 1.0, k, lab)
    return lab


def _lattice_counts(box, spacing):
    return [max(1, int(math.floor(box.size[a] / spacing[a] + 1e-9))) for a in range(3)]


@dataclass
class DeviceSpins:
    """Spins resident on one GPU (torch tensors), in the reference's SoA layout."""

    n: int
    n_coils: int
    pos: object
    mx: object
    my: object
    mz: object
    t1: object
    t2: object
    m0: object
    domega: object
    weight: object  # float64 (C, n, 2) interleaved complex, or None for the uniform 1+0j
    device: int = 0
    coil_array: bool = False  # receive model is a CoilArray: weights keep the coil axis even for one coil

    def pointers(self) -> dict:
        d = {k: getattr(self, k).data_ptr() for k in ("pos", "mx", "my", "mz", "t1", "t2", "m0", "domega")}
        d["weight"] = self.weight.data_ptr() if self.weight is not None else 0
        return d

    def to_host(self) -> dict:
        """numpy copies (pos, m0, t1, t2, delta_omega, mx, my, mz, weight) for checks and the host API."""
        w = self.weight.cpu().numpy() if self.weight is not None else np.ones((1, self.n, 2)) * [1.0, 0.0]
        wc = w[..., 0] + 1j * w[..., 1]
        out = {k: getattr(self, k).cpu().numpy() for k in ("pos", "mx", "my", "mz", "t1", "t2", "m0")}
        out["delta_omega"] = self.domega.cpu().numpy()
        out["weight"] = wc if (self.n_coils > 1 or self.coil_array) else wc[0]
        return out


def _coil_list(rx):
    if isinstance(rx, UniformSensitivity):
        return [], float(rx.s)
    coils = rx.coils if isinstance(rx, CoilArray) else [rx]
    return list(coils), 1.0


def rasterize_device(scene: DeviceScene, spacing, engine=None, cap: int = DEFAULT_SPIN_CAP,
                     extra_dw: Optional[np.ndarray] = None) -> DeviceSpins:
    """Rasterise `scene` on the engine's GPU (phantom.py:98-142 + engine.py:192-226 on the device).

    ``extra_dw`` (host, one value per emitted spin) is added on the device
    afterwards — for per-spin random maps that only exist as host arrays.
    """
    import torch

    from .engine import get_engine

    eng = engine if engine is not None else get_engine()
    spacing = tuple(float(s) for s in spacing)
    if len(spacing) != 3 or any(not s > 0.0 for s in spacing):
        raise InvalidParameter(f"spacing components must be positive, got {spacing}")
    sites = scene.n_sites(spacing)
    if sites > cap:
        raise SpinBudgetExceeded(f"{sites} lattice sites exceed the cap of {cap}; refine the spacing or raise the cap")
    shapes, boxes = [], []
    for b in scene.boxes:
        counts = _lattice_counts(b, spacing)
        bt = _capi.BoxT()
        for a in range(3):
            offset = (b.size[a] - (counts[a] - 1) * spacing[a]) / 2.0
            bt.base[a] = b.origin[a] + offset  # phantom._lattice: origin + offset + spacing * k
            bt.step[a] = spacing[a]
            bt.count[a] = counts[a]
        bt.m0, bt.t1, bt.t2, bt.dw = float(b.m0), float(b.t1), float(b.t2), float(b.delta_omega)
        bt.shape_begin, bt.shape_count = len(shapes), len(b.shapes)
        for s in b.shapes:
            st = _capi.ShapeT()
            for a in range(3):
                st.c[a] = float(s.center[a]) if a < len(s.center) else 0.0
                st.ax[a] = float(s.axes[a]) if a < s.dim else 0.0
            st.cos_a, st.sin_a = math.cos(s.angle), math.sin(s.angle)
            st.m0, st.t1, st.t2, st.dw = float(s.m0), float(s.t1), float(s.t2), float(s.delta_omega)
            shapes.append(st)
        boxes.append(bt)
    f = _capi.FieldT()
    f.const_dw = float(scene.const_dw)
    keep = []
    if scene.polynomial is not None:
        pf = scene.polynomial
        arr = np.ascontiguousarray([[c, *e] for c, e in zip(pf.coef, pf.exponents)], dtype=float)
        keep.append(arr)
        f.n_poly, f.poly, f.poly_len = arr.shape[0], _capi.dptr(arr), float(pf.length)
        f.poly_scale = float(pf.scale)
        f.poly_peak = float(pf.peak) if pf.peak is not None else 0.0
    if scene.bumps is not None:
        bb = scene.bumps
        arr = np.ascontiguousarray(
            [[c[0], c[1], c[2] if len(c) > 2 else math.nan, s, a] for c, s, a in zip(bb.centers, bb.sigmas, bb.amps)],
            dtype=float)
        keep.append(arr)
        f.n_bumps, f.bumps = arr.shape[0], _capi.dptr(arr)
    coils, uniform_s = _coil_list(scene.receive)
    coil_arr = (_capi.CoilT * max(len(coils), 1))()
    for i, c in enumerate(coils):
        for a in range(3):
            coil_arr[i].c[a] = float(c.center[a])
        coil_arr[i].sigma = float(c.sigma)
        coil_arr[i].cos_p, coil_arr[i].sin_p = math.cos(c.phase), math.sin(c.phase)
    n_coils = len(coils)
    ncw = max(n_coils, 1)
    dev = torch.device("cuda", eng.device)
    cap_n = max(sites, 1)
    buf = torch.empty(cap_n * (10 + 2 * ncw), dtype=torch.float64, device=dev)
    views, off = {}, 0
    for k, width in (("pos", 3), ("mx", 1), ("my", 1), ("mz", 1), ("t1", 1), ("t2", 1), ("m0", 1),
                     ("domega", 1), ("weight", 2 * ncw)):
        views[k] = buf[off: off + cap_n * width]
        off += cap_n * width
    box_arr = (_capi.BoxT * len(boxes))(*boxes)
    shape_arr = (_capi.ShapeT * max(len(shapes), 1))(*shapes)
    n_out = ctypes.c_int64(0)
    ptr = lambda t: ctypes.cast(ctypes.c_void_p(t.data_ptr()), ctypes.POINTER(ctypes.c_double))
    torch.cuda.current_stream(dev).synchronize()  # buffers allocated on torch's stream, written on the engine's
    _capi.check(
        eng._lib.bloch_rasterize(
            eng._h, box_arr, len(boxes), shape_arr, len(shapes), ctypes.byref(f), coil_arr, n_coils, uniform_s,
            cap_n, ptr(views["pos"]), ptr(views["mx"]), ptr(views["my"]), ptr(views["mz"]), ptr(views["t1"]),
            ptr(views["t2"]), ptr(views["m0"]), ptr(views["domega"]), ptr(views["weight"]), ctypes.byref(n_out),
        ),
        "bloch_rasterize",
    )
    n = int(n_out.value)
    if n == 0:
        raise InvalidParameter("the scene rasterized to zero spins")
    out = DeviceSpins(
        n=n, n_coils=ncw, pos=views["pos"][: 3 * n].view(n, 3), mx=views["mx"][:n], my=views["my"][:n],
        mz=views["mz"][:n], t1=views["t1"][:n], t2=views["t2"][:n], m0=views["m0"][:n],
        domega=views["domega"][:n], weight=views["weight"][: 2 * ncw * n].view(ncw, n, 2), device=eng.device,
        coil_array=isinstance(scene.receive, CoilArray),
    )
    if extra_dw is not None:
        extra = np.asarray(extra_dw, dtype=float)
        if extra.shape != (n,):
            raise InvalidParameter(f"extra_dw has shape {extra.shape}, the scene emitted {n} spins")
        out.domega += torch.from_numpy(extra).to(dev)
        torch.cuda.current_stream(dev).synchronize()  # the engine's stream reads domega next
    del keep
    return out

"""Host layer of the Bloch engine — the reference's ``mrsim.engine`` API over the GPU.

The seam is the reference's own: ``compute_block(tables, block)``
(engine.py:259-310) with identical argument meaning and return types, fed by
``precompute_sequence_tables`` (engine.py:83-164) and ``build_spin_arrays``
(engine.py:192-226) and folded by ``run`` (engine.py:465-537).  The per-event
arithmetic runs in ``libbloch_b200.so`` (sm_100a) through the C-ABI in
``include/bloch_b200.h``; there is no CPU fallback — without the library or a
device every compute call raises.

Because the function is a drop-in, the reference package itself can be driven
by the GPU: ``mrsim.engine.compute_block = paper_1305_6861_b200.compute_block``
 — ``compute_block`` accepts the reference's own
``OperatorTables`` / ``SpinBlock`` objects (duck-typed) as well as the mirror
classes defined here.
"""

from __future__ import annotations

import ctypes
import dataclasses
import math
import os
import platform
import time
import weakref
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import _capi
from .bloch import GAMMA_PROTON, hard_pulse_matrix
from .errors import InvalidParameter
from .phantom import DEFAULT_SPIN_CAP, Phantom, rasterize_arrays
from .sequence import Sequence
from .system import SystemModel, UniformSensitivity, default_system, receive_weights, spin_off_resonance

# ---------------------------------------------------------------------------
# event tables (master side) — engine.py:51-164
# ---------------------------------------------------------------------------


@dataclass
class EsTable:
    """Operator data of one elementary sequence (engine.py:51-70)."""

    pulse_mat: Optional[np.ndarray]
    duration: float
    moments: np.ndarray
    ev_dt: np.ndarray
    ev_dmom: np.ndarray
    ev_sample: np.ndarray
    ev_snap: np.ndarray
    acq: int = -1
    n_samples: int = 0


@dataclass(eq=False)
class OperatorTables:
    entries: List[EsTable]
    n_acq: int
    acq_times: List[np.ndarray]
    snapshot_times: Tuple[float, ...]
    pulse_memo_hits: int
    gamma: float


def precompute_sequence_tables(
    sequence: Sequence, gamma: float = GAMMA_PROTON, snapshot_times=(), memoize: bool = True
) -> OperatorTables:
    """Per-ES operator tables, event for event those of engine.py:83-164.

    Events partition each ES at its ADC and snapshot instants (a snapshot sorts
    before a sample at the same instant, engine.py:119); event i carries the
    interval ``ev_dt[i]`` and moment increment ``ev_dmom[i]`` leading up to it;
    a tail event closes the ES when the last instant misses the end or the
    accumulated moment differs from the total in any bit (engine.py:135-140).
    The increments are formed with ``np.diff`` — the same subtractions as the
    reference loop, so the tables are bit-identical.
    """
    snapshot_times = tuple(sorted(snapshot_times))
    entries: List[EsTable] = []
    acq_times: List[np.ndarray] = []
    memo: Dict[Tuple[float, float], np.ndarray] = {}
    hits = 0
    t0 = 0.0
    acq = 0
    zero3 = np.zeros((1, 3))
    for es in sequence.elements:
        mat = None
        if es.pulse is not None and es.pulse.alpha != 0.0:
            key = (es.pulse.alpha, es.pulse.phi)
            if memoize and key in memo:
                mat = memo[key]
                hits += 1
            else:
                mat = hard_pulse_matrix(es.pulse.alpha, es.pulse.phi)
                if memoize:
                    memo[key] = mat
        t1 = t0 + es.duration
        s_ts = es.acquisition.sample_times(es.duration)
        snaps = [
            (float(t_abs - t0), si)
            for si, t_abs in enumerate(snapshot_times)
            if t0 < t_abs <= t1 or (t_abs == 0.0 == t0)
        ]
        if not snaps and s_ts.size == 0:  # no instants: the tail event alone (engine.py:135-140)
            total = es.gradient.moments(es.duration, gamma)
            if 0.0 < es.duration or np.any(total != 0.0):
                ev_dt, ev_dmom = np.array([es.duration - 0.0]), (total - np.zeros(3)).reshape(1, 3)
            else:
                ev_dt, ev_dmom = np.zeros(0), np.zeros((0, 3))
            entries.append(EsTable(pulse_mat=mat, duration=es.duration, moments=np.asarray(total, dtype=float),
                                   ev_dt=ev_dt, ev_dmom=ev_dmom, ev_sample=np.zeros(ev_dt.size, dtype=bool),
                                   ev_snap=np.full(ev_dt.size, -1, dtype=int)))
            t0 = t1
            continue
        if snaps:
            events = [(float(t), True, -1) for t in s_ts] + [(t, False, si) for t, si in snaps]
            events.sort(key=lambda e: (e[0], e[1]))
            ts = np.array([e[0] for e in events])
            is_sample = np.array([e[1] for e in events], dtype=bool)
            snap_idx = np.array([e[2] for e in events], dtype=int)
        else:
            ts = np.asarray(s_ts, dtype=float)
            is_sample = np.ones(ts.size, dtype=bool)
            snap_idx = np.full(ts.size, -1, dtype=int)
        partial = es.gradient.partial_moments(ts, es.duration, gamma) if ts.size else np.zeros((0, 3))
        total = es.gradient.moments(es.duration, gamma)
        ev_dt = np.diff(ts, prepend=0.0)
        ev_dmom = np.diff(partial, axis=0, prepend=zero3) if ts.size else np.zeros((0, 3))
        prev_t = float(ts[-1]) if ts.size else 0.0
        prev_m = partial[-1] if ts.size else np.zeros(3)
        if prev_t < es.duration or np.any(prev_m != total):
            ev_dt = np.append(ev_dt, es.duration - prev_t)
            ev_dmom = np.vstack([ev_dmom, (total - prev_m)[None, :]])
            is_sample = np.append(is_sample, False)
            snap_idx = np.append(snap_idx, -1)
        entry = EsTable(
            pulse_mat=mat,
            duration=es.duration,
            moments=np.asarray(total, dtype=float),
            ev_dt=np.asarray(ev_dt, dtype=float),
            ev_dmom=np.asarray(ev_dmom, dtype=float).reshape(-1, 3),
            ev_sample=np.asarray(is_sample, dtype=bool),
            ev_snap=np.asarray(snap_idx, dtype=int),
        )
        if es.acquisition.enabled:
            entry.acq = acq
            entry.n_samples = es.acquisition.n_samples
            acq_times.append(t0 + s_ts)
            acq += 1
        entries.append(entry)
        t0 = t1
    return OperatorTables(
        entries=entries, n_acq=acq, acq_times=acq_times, snapshot_times=snapshot_times,
        pulse_memo_hits=hits, gamma=gamma,
    )


def event_counts(tables) -> Dict[str, int]:
    """Reference table size E and per-class counts.

    E = #ES with a pulse matrix + #events; classes: rot, prec_relax (dt != 0),
    prec (dt == 0, moment != 0), noop, adc (sampled events)."""
    out = {"rot": 0, "prec_relax": 0, "prec": 0, "noop": 0, "adc": 0}
    for e in tables.entries:
        out["rot"] += int(e.pulse_mat is not None)
        if e.ev_dt.size:
            dt = np.asarray(e.ev_dt)
            moving = np.any(np.asarray(e.ev_dmom) != 0.0, axis=1)
            out["prec_relax"] += int(np.sum(dt != 0.0))
            out["prec"] += int(np.sum((dt == 0.0) & moving))
            out["noop"] += int(np.sum((dt == 0.0) & ~moving))
            out["adc"] += int(np.sum(e.ev_sample))
    out["events"] = out["rot"] + out["prec_relax"] + out["prec"] + out["noop"]
    return out


def flatten_tables(tables) -> Dict[str, np.ndarray]:
    """Flatten OperatorTables (product or reference object) into the C-ABI arrays."""
    entries = tables.entries
    n_es = len(entries)
    counts = np.fromiter((e.ev_dt.size for e in entries), dtype=np.int64, count=n_es)
    offset = np.zeros(n_es + 1, dtype=np.int64)
    np.cumsum(counts, out=offset[1:])
    has_pulse = np.fromiter((e.pulse_mat is not None for e in entries), dtype=np.uint8, count=n_es)
    mats = np.zeros((n_es, 9))
    for i, e in enumerate(entries):
        if e.pulse_mat is not None:
            mats[i] = np.asarray(e.pulse_mat, dtype=float).reshape(9)
    acq = np.fromiter((e.acq for e in entries), dtype=np.int32, count=n_es)
    E = int(offset[-1])
    if E:
        ev_dt = np.ascontiguousarray(np.concatenate([e.ev_dt for e in entries]), dtype=np.float64)
        ev_dmom = np.ascontiguousarray(
            np.concatenate([np.asarray(e.ev_dmom, dtype=float).reshape(-1, 3) for e in entries]), dtype=np.float64
        )
        ev_sample = np.ascontiguousarray(np.concatenate([e.ev_sample for e in entries]), dtype=np.uint8)
        ev_snap = np.ascontiguousarray(np.concatenate([e.ev_snap for e in entries]), dtype=np.int32)
    else:
        ev_dt, ev_dmom = np.zeros(0), np.zeros((0, 3))
        ev_sample, ev_snap = np.zeros(0, np.uint8), np.zeros(0, np.int32)
    max_ns = max((e.n_samples for e in entries), default=0)
    return dict(
        n_es=n_es, offset=offset, has_pulse=has_pulse, mats=np.ascontiguousarray(mats), acq=acq,
        ev_dt=ev_dt, ev_dmom=ev_dmom, ev_sample=ev_sample, ev_snap=ev_snap,
        n_acq=int(tables.n_acq), max_ns=int(max_ns), n_snap=len(tables.snapshot_times),
    )


# ---------------------------------------------------------------------------
# spin blocks — engine.py:172-251
# ---------------------------------------------------------------------------


@dataclass
class SpinBlock:
    """Contiguous slice of the spin set (engine.py:172-189).

    ``weight`` is complex (n,) — or (C, n) for C receive coils (extension)."""

    index: int
    pos: np.ndarray
    mx: np.ndarray
    my: np.ndarray
    mz: np.ndarray
    t1: np.ndarray
    t2: np.ndarray
    m0: np.ndarray
    domega: np.ndarray
    weight: np.ndarray

    @property
    def n(self) -> int:
        return self.mx.size


def build_spin_arrays(spins, system: SystemModel) -> SpinBlock:
    """Pack spins into SoA arrays, folding in off-resonance and receive weight (engine.py:192-226).

    ``spins`` is the dict returned by :func:`~.phantom.rasterize_arrays` or a
    list of ``SpinSample`` (the reference's form).
    """
    if isinstance(spins, dict):
        pos = np.asarray(spins["pos"], dtype=float).reshape(-1, 3)
        m0 = np.asarray(spins["m0"], dtype=float)
        t1 = np.asarray(spins["t1"], dtype=float)
        t2 = np.asarray(spins["t2"], dtype=float)
        obj_dw = np.asarray(spins["delta_omega"], dtype=float)
        mx, my, mz = np.zeros_like(m0), np.zeros_like(m0), m0.copy()
    else:
        n = len(spins)
        pos = np.array([s.position for s in spins], dtype=float).reshape(n, 3)
        m0 = np.array([s.relax.m0 for s in spins], dtype=float)
        t1 = np.array([s.relax.t1 for s in spins], dtype=float)
        t2 = np.array([s.relax.t2 for s in spins], dtype=float)
        obj_dw = np.array([s.delta_omega for s in spins], dtype=float)
        mx = np.array([s.m.mx for s in spins], dtype=float)
        my = np.array([s.m.my for s in spins], dtype=float)
        mz = np.array([s.m.mz for s in spins], dtype=float)
    return SpinBlock(
        index=0, pos=pos, mx=mx, my=my, mz=mz, t1=t1, t2=t2, m0=m0,
        domega=spin_off_resonance(system, pos, obj_dw), weight=receive_weights(system, pos),
    )


def partition_blocks(arrays: SpinBlock, n_blocks: int) -> List[SpinBlock]:
    """At most n_blocks contiguous disjoint blocks, np.linspace bounds (engine.py:229-251)."""
    n = arrays.n
    n_blocks = max(1, min(n_blocks, n)) if n else 1
    bounds = np.linspace(0, n, n_blocks + 1).astype(int)
    w = np.asarray(arrays.weight)
    out = []
    for b in range(n_blocks):
        lo, hi = bounds[b], bounds[b + 1]
        out.append(
            SpinBlock(
                index=b, pos=arrays.pos[lo:hi].copy(), mx=arrays.mx[lo:hi].copy(), my=arrays.my[lo:hi].copy(),
                mz=arrays.mz[lo:hi].copy(), t1=arrays.t1[lo:hi].copy(), t2=arrays.t2[lo:hi].copy(),
                m0=arrays.m0[lo:hi].copy(), domega=arrays.domega[lo:hi].copy(),
                weight=(w[..., lo:hi].copy()),
            )
        )
    return out


# ---------------------------------------------------------------------------
# the device engine (C-ABI context)
# ---------------------------------------------------------------------------


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


MAX_COILS = 8  # receive coils per device call (bloch_compute_block); more run as groups (BlochEngine.compute)


class BlochEngine:
    """One libbloch_b200 context: a CUDA device (or a device set), a state precision, the uploaded tables.

    ``devices=[d0, d1, ...]`` opens a device-set context (bloch_create_multi): ``compute`` shards the
    block over the devices with the reference's np.linspace bounds (engine.py:229-251), runs the shards
    concurrently and sums the partial k-spaces on ``d0`` in rank order — the reference's worker pool
    (engine.py:540-595) with one GPU per worker."""

    def __init__(self, device: int = 0, precision: int = 32, devices: Optional[List[int]] = None):
        lib = _capi.load()
        self._lib = lib
        self.precision = int(precision)
        h = ctypes.c_void_p()
        if devices is not None and len(devices) > 1:
            self.devices = [int(d) for d in devices]
            arr = (ctypes.c_int32 * len(self.devices))(*self.devices)
            _capi.check(lib.bloch_create_multi(arr, len(self.devices), self.precision, ctypes.byref(h)),
                        "bloch_create_multi")
        else:
            self.devices = [int(devices[0]) if devices else int(device)]
            _capi.check(lib.bloch_create(self.devices[0], self.precision, ctypes.byref(h)), "bloch_create")
        self.device = self.devices[0]
        self._h = h
        self._tables_ref = None
        self._flat = None

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.bloch_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- tables --------------------------------------------------------------
    def set_tables(self, tables) -> Dict[str, np.ndarray]:
        if self._tables_ref is not None and self._tables_ref() is tables:
            return self._flat
        f = flatten_tables(tables)
        i32 = ctypes.POINTER(ctypes.c_int32)
        u8 = ctypes.POINTER(ctypes.c_uint8)
        _capi.check(
            self._lib.bloch_set_tables(
                self._h, f["n_es"], f["offset"].ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                f["has_pulse"].ctypes.data_as(u8), _capi.dptr(f["mats"]), f["acq"].ctypes.data_as(i32),
                _capi.dptr(f["ev_dt"]), _capi.dptr(f["ev_dmom"]), f["ev_sample"].ctypes.data_as(u8),
                f["ev_snap"].ctypes.data_as(i32), f["n_acq"], f["max_ns"], f["n_snap"],
            ),
            "bloch_set_tables",
        )
        try:
            self._tables_ref = weakref.ref(tables)
        except TypeError:
            self._tables_ref = None
        self._flat = f
        return f

    def program_stats(self) -> Dict[str, int]:
        vals = [ctypes.c_int64() for _ in range(8)]
        _capi.check(self._lib.bloch_program_stats(self._h, *[ctypes.byref(v) for v in vals]), "bloch_program_stats")
        keys = ("events", "samples", "rot", "interval", "window_ops", "window_samples", "chirp_samples",
                "train_pairs")
        out = {k: v.value for k, v in zip(keys, vals)}
        lay = [ctypes.c_int64() for _ in range(4)]
        _capi.check(self._lib.bloch_program_layout(self._h, *[ctypes.byref(v) for v in lay]), "bloch_program_layout")
        out.update(zip(("ops", "rot_classes", "relax_classes", "onthefly_intervals"), (v.value for v in lay)))
        cls = [ctypes.c_int64() for _ in range(5)]
        _capi.check(self._lib.bloch_program_classes(self._h, *[ctypes.byref(v) for v in cls]), "bloch_program_classes")
        out.update(zip(("prog_classes", "chirp_classes", "train_classes", "train_class_ops", "planes"),
                       (v.value for v in cls)))
        g, cs, rs = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
        _capi.check(self._lib.bloch_program_groups(self._h, ctypes.byref(g), ctypes.byref(cs), ctypes.byref(rs)),
                    "bloch_program_groups")
        out.update(window_groups=g.value, contracted_samples=cs.value, integrator_samples=rs.value)
        return out

    def program_ops(self, deferred: bool = False) -> Dict[str, np.ndarray]:
        """The compiled op stream (bloch_program_ops): kind, count, rot, prg, pre and planes (n, 4) per op."""
        n = ctypes.c_int32()
        _capi.check(self._lib.bloch_program_ops(self._h, int(deferred), 0, ctypes.byref(n), *([None] * 6)),
                    "bloch_program_ops")
        k = n.value
        out = {name: np.zeros(k, dtype=np.int32) for name in ("kind", "count", "rot", "prg", "pre")}
        out["pl"] = np.zeros((k, 4), dtype=np.int32)
        p32 = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        _capi.check(self._lib.bloch_program_ops(self._h, int(deferred), k, ctypes.byref(n), p32(out["kind"]),
                                                p32(out["count"]), p32(out["rot"]), p32(out["prg"]), p32(out["pre"]),
                                                p32(out["pl"])), "bloch_program_ops")
        return out

    def last_timing(self) -> Dict[str, float]:
        k, d, n = ctypes.c_float(), ctypes.c_float(), ctypes.c_int32()
        _capi.check(self._lib.bloch_last_timing(self._h, ctypes.byref(k), ctypes.byref(d), ctypes.byref(n)), "timing")
        return {"kernel_ms": k.value, "device_ms": d.value, "launches": n.value}

    def device_times(self) -> Dict[int, Dict[str, float]]:
        """Per-device integrator / whole-call device time (ms) of the last synchronous call, rank order
        (bloch_last_device_times): the reference's per-worker busy time (engine.py:516-525)."""
        k = len(self.devices)
        km, dm = (ctypes.c_float * k)(), (ctypes.c_float * k)()
        _capi.check(self._lib.bloch_last_device_times(self._h, k, km, dm), "bloch_last_device_times")
        return {r: {"device": self.devices[r], "kernel_ms": km[r], "device_ms": dm[r]} for r in range(k)}

    def last_launch(self) -> Dict[str, int]:
        """Shape of the last integrator launch: precision bits, spins per thread, coil-group width,
        grid (CTAs) and threads per CTA (bloch_last_launch)."""
        v = [ctypes.c_int32() for _ in range(5)]
        _capi.check(self._lib.bloch_last_launch(self._h, *[ctypes.byref(x) for x in v]), "bloch_last_launch")
        return dict(zip(("precision", "spins_per_thread", "coils", "grid", "threads"), (x.value for x in v)))

    def last_segments(self) -> int:
        """Program segments of the last call (bloch_last_segments): 1 unless the partial rows of one
        launch would exceed BLOCH_PARTIAL_BUDGET_MB."""
        v = ctypes.c_int32()
        _capi.check(self._lib.bloch_last_segments(self._h, ctypes.byref(v)), "bloch_last_segments")
        return v.value

    def set_contraction(self, enable: bool) -> None:
        """Window contraction on the tensor cores (bloch_set_contraction; fp32 mode, one coil): the long
        tabulated ADC windows of a rotation class form one product over spins instead of per-warp sums
        (replaces engine.py:303-305 for those windows).  On by default."""
        _capi.check(self._lib.bloch_set_contraction(self._h, 1 if enable else 0), "bloch_set_contraction")

    def set_resident(self, enable: bool) -> None:
        """Resident-table integrator (bloch_set_resident): the class tables of a CTA's spins held in shared
        memory for the whole launch (the relax cache of engine.py:292-299, generalised, on chip).  On by
        default; off keeps the integrator that reads the tables through L2 at every op."""
        _capi.check(self._lib.bloch_set_resident(self._h, 1 if enable else 0), "bloch_set_resident")

    def last_resident(self) -> Dict[str, int]:
        """Whether the last call ran the resident-table integrator and the table bytes per spin of the
        program's resident plan (bloch_last_resident)."""
        a, b = ctypes.c_int32(), ctypes.c_int32()
        _capi.check(self._lib.bloch_last_resident(self._h, ctypes.byref(a), ctypes.byref(b)), "bloch_last_resident")
        return {"resident": a.value, "bytes_per_spin": b.value}

    def last_phases(self) -> Dict[str, float]:
        """Integrator vs window-contraction device time (ms) of the last call, the window groups
        contracted and the samples they produced (bloch_last_phases)."""
        a, b, g, k = ctypes.c_float(), ctypes.c_float(), ctypes.c_int32(), ctypes.c_int64()
        _capi.check(self._lib.bloch_last_phases(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(g),
                                                ctypes.byref(k)), "bloch_last_phases")
        return {"integrate_ms": a.value, "contract_ms": b.value, "groups": g.value, "contracted_samples": k.value}

    def set_stream(self, stream_ptr: int) -> None:
        """Run on an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); 0 = own stream."""
        _capi.check(self._lib.bloch_set_stream(self._h, ctypes.c_void_p(int(stream_ptr) or None)), "bloch_set_stream")

    # -- compute -------------------------------------------------------------
    def compute_device(self, tables, spins: Dict[str, int], n: int, n_coils: int, out_echoes: int,
                       out_snaps: int = 0, sync: bool = False, present: Optional[np.ndarray] = None) -> None:
        """compute_block on device-resident float64 arrays (raw CUDA pointers).

        ``spins`` maps pos/mx/my/mz/t1/t2/m0/domega/weight to device pointers
        (weight 0 = uniform 1+0j); outputs are device pointers.  Asynchronous on
        the engine's stream unless ``sync``.  ``present`` (uint8, one per
        snapshot time) receives which snapshots were taken.
        """
        f = self.set_tables(tables)
        ptr = lambda key: ctypes.cast(ctypes.c_void_p(int(spins[key])), ctypes.POINTER(ctypes.c_double)) \
            if spins.get(key) else None
        flags = _capi.BLOCH_IN_DEVICE | _capi.BLOCH_OUT_DEVICE | (0 if sync else _capi.BLOCH_NO_SYNC)
        st = self._lib.bloch_compute_block(
            self._h, int(n), ptr("pos"), ptr("mx"), ptr("my"), ptr("mz"), ptr("t1"), ptr("t2"), ptr("m0"),
            ptr("domega"), ptr("weight"), int(n_coils),
            ctypes.cast(ctypes.c_void_p(int(out_echoes)), ctypes.POINTER(ctypes.c_double)) if out_echoes else None,
            ctypes.cast(ctypes.c_void_p(int(out_snaps)), ctypes.POINTER(ctypes.c_double)) if out_snaps else None,
            present.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)) if present is not None else None, flags,
        )
        _capi.check(st, "bloch_compute_block")
        del f

    def compute(self, tables, pos, mx, my, mz, t1, t2, m0, domega, weight, block_index=0,
                out_echoes: Optional[np.ndarray] = None, out_snaps: Optional[np.ndarray] = None):
        """compute_block on host numpy arrays; returns (echoes, snapshots).

        ``out_echoes`` (complex128 (C, n_acq, max_ns)) and ``out_snaps`` (float64
        (n_snap, n, 3)) may be preallocated (e.g. pinned) buffers.  More than
        ``MAX_COILS`` receive coils run as consecutive groups of coils (the spin
        state is recomputed per group; the snapshots come from the first)."""
        w = np.asarray(weight)
        if w.ndim == 2 and w.shape[0] > MAX_COILS:
            f = self.set_tables(tables)
            eshape = (w.shape[0], f["n_acq"], f["max_ns"])
            if out_echoes is None:
                out_echoes = np.zeros(eshape, dtype=np.complex128)
            elif out_echoes.shape != eshape or out_echoes.dtype != np.complex128:
                raise InvalidParameter(f"out_echoes must be complex128 {eshape}")
            snaps = None
            for g0 in range(0, w.shape[0], MAX_COILS):
                e, s = self._submit(tables, pos, mx, my, mz, t1, t2, m0, domega, w[g0:g0 + MAX_COILS], block_index,
                                    None, out_snaps if g0 == 0 else None, sync=True).wait()
                out_echoes[g0:g0 + MAX_COILS] = e
                if g0 == 0:
                    snaps = s
            return out_echoes, snaps
        return self._submit(tables, pos, mx, my, mz, t1, t2, m0, domega, weight, block_index, out_echoes,
                            out_snaps, sync=True).wait()

    def submit(self, tables, pos, mx, my, mz, t1, t2, m0, domega, weight, block_index=0,
               out_echoes: Optional[np.ndarray] = None, out_snaps: Optional[np.ndarray] = None) -> "Pending":
        """compute without waiting: returns a :class:`Pending` whose ``wait()`` gives (echoes, snapshots).

        The host inputs and the (pinned) output buffers must stay untouched until ``wait()``.  With
        two engines (:class:`Pipeline`) the uploads of one block overlap the kernels of the other."""
        return self._submit(tables, pos, mx, my, mz, t1, t2, m0, domega, weight, block_index, out_echoes,
                            out_snaps, sync=False)

    def _submit(self, tables, pos, mx, my, mz, t1, t2, m0, domega, weight, block_index, out_echoes, out_snaps,
                sync):
        f = self.set_tables(tables)
        n = int(np.asarray(mx).size)
        pos = _f64(np.asarray(pos, dtype=float).reshape(n, 3))
        arrs = [_f64(a) for a in (mx, my, mz, t1, t2, m0, domega)]
        w = np.asarray(weight)
        multi = w.ndim == 2
        n_coils = w.shape[0] if multi else 1
        if w.shape[-1] != n:
            raise InvalidParameter(f"weight has {w.shape[-1]} spins, block has {n}")
        wc = np.ascontiguousarray(w, dtype=np.complex128).reshape(n_coils, n)
        eshape = (n_coils, f["n_acq"], f["max_ns"])
        if out_echoes is not None:
            if out_echoes.shape != eshape or out_echoes.dtype != np.complex128 or not out_echoes.flags.c_contiguous:
                raise InvalidParameter(f"out_echoes must be C-contiguous complex128 {eshape}")
            echoes = out_echoes
        else:
            echoes = np.zeros(eshape, dtype=np.complex128)
        n_snap = f["n_snap"]
        if n_snap and out_snaps is not None:
            if out_snaps.shape != (n_snap, n, 3) or out_snaps.dtype != np.float64:
                raise InvalidParameter(f"out_snaps must be float64 {(n_snap, n, 3)}")
            snaps = out_snaps
        else:
            snaps = np.zeros((n_snap, n, 3)) if n_snap else None
        present = np.zeros(max(n_snap, 1), dtype=np.uint8)
        # the uniform receive weight 1+0j (the reference's default system) travels as NULL: no
        # upload, and the kernel skips the weighting (bloch_b200.h: weight NULL = uniform 1+0j)
        wptr = None if (n_coils == 1 and n and _unit_weight(wc)) else _capi.dptr(wc.view(np.float64))
        st = self._lib.bloch_compute_block(
            self._h, n, _capi.dptr(pos), *[_capi.dptr(a) for a in arrs],
            wptr, n_coils, _capi.dptr(echoes.view(np.float64)),
            _capi.dptr(snaps) if snaps is not None else None,
            present.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), 0 if sync else _capi.BLOCH_NO_SYNC,
        )
        _capi.check(st, "bloch_compute_block", block_index)
        return Pending(self, echoes if multi else echoes[0], snaps, present, n_snap, keep=(pos, arrs, wc),
                       done=sync, block_index=block_index)


class Pending:
    """A submitted compute_block (BlochEngine.submit); wait() synchronises and returns its outputs."""

    def __init__(self, eng, echoes, snaps, present, n_snap, keep, done, block_index=0):
        self._eng, self._echoes, self._snaps, self._present = eng, echoes, snaps, present
        self._n_snap, self._keep, self._done, self._block = n_snap, keep, done, block_index

    def wait(self):
        if not self._done:
            _capi.check(self._eng._lib.bloch_synchronize(self._eng._h), "bloch_synchronize", self._block)
            self._done = True
            self._keep = None
        snaps = [self._snaps[i] if self._present[i] else None for i in range(self._n_snap)]
        return self._echoes, snaps


class Pipeline:
    """Double-buffered host-to-host compute_block: ``depth`` engine contexts (own stream, own device
    buffers) take successive blocks in turn, so the uploads and downloads of one block overlap the
    kernels of the other.  ``submit`` waits only for the block that last used the same context."""

    def __init__(self, device: Optional[int] = None, precision: Optional[int] = None, depth: int = 2):
        import torch

        dev = default_device() if device is None else int(device)
        prec = int(os.environ.get("BLOCH_PRECISION", "32")) if precision is None else int(precision)
        self.engines = [BlochEngine(dev, prec) for _ in range(depth)]
        self._pending: List[Optional[Pending]] = [None] * depth
        self._k = 0
        # the integrators run in submission order: context i waits on context i-1's kernel
        with torch.cuda.device(dev):
            self._events = [torch.cuda.Event() for _ in range(depth)]
            for ev in self._events:  # torch creates the CUDA event lazily: record once (it then counts as done)
                ev.record()
            torch.cuda.synchronize(dev)
        for i, e in enumerate(self.engines):
            _capi.check(e._lib.bloch_set_kernel_gate(e._h, ctypes.c_void_p(self._events[i - 1].cuda_event),
                                                     ctypes.c_void_p(self._events[i].cuda_event)),
                        "bloch_set_kernel_gate")

    def submit(self, tables, *arrays, out_echoes=None, out_snaps=None, block_index=0) -> Pending:
        i = self._k % len(self.engines)
        self._k += 1
        if self._pending[i] is not None:
            self._pending[i].wait()
        self._pending[i] = self.engines[i].submit(tables, *arrays, block_index=block_index, out_echoes=out_echoes,
                                                  out_snaps=out_snaps)
        return self._pending[i]

    def drain(self) -> None:
        for p in self._pending:
            if p is not None:
                p.wait()

    def close(self) -> None:
        self.drain()
        for e in self.engines:
            e.close()


def _unit_weight(wc: np.ndarray, chunk: int = 1 << 15) -> bool:
    """All weights exactly 1+0j.  Bit-compared in cache-sized chunks (early exit): the check
    must cost less than the 16 B/spin upload it saves."""
    u = np.ascontiguousarray(wc).reshape(-1).view(np.uint64)
    one = np.uint64(0x3FF0000000000000)
    pattern = np.empty(min(2 * chunk, u.size), dtype=np.uint64)
    pattern[0::2], pattern[1::2] = one, 0
    for i in range(0, u.size, 2 * chunk):
        seg = u[i: i + 2 * chunk]
        if not np.array_equal(seg, pattern[: seg.size]):
            return False
    return True


_ENGINES: Dict[Tuple, BlochEngine] = {}


def default_device() -> int:
    return int(os.environ.get("LOCAL_RANK", "0"))


def get_engine(device: Optional[int] = None, precision: Optional[int] = None,
               devices: Optional[List[int]] = None) -> BlochEngine:
    """Process-wide engine per (device or device set, precision); precision from BLOCH_PRECISION (32)."""
    prec = int(os.environ.get("BLOCH_PRECISION", "32")) if precision is None else int(precision)
    if devices is not None and len(devices) > 1:
        key = (tuple(int(d) for d in devices), prec)
    else:
        dev = int(devices[0]) if devices else (default_device() if device is None else int(device))
        key = (dev, prec)
    eng = _ENGINES.get(key)
    if eng is None:
        eng = BlochEngine(precision=prec, devices=list(key[0]) if isinstance(key[0], tuple) else [key[0]])
        _ENGINES[key] = eng
    return eng


# ---------------------------------------------------------------------------
# the kernel seam — engine.py:259-335
# ---------------------------------------------------------------------------


def compute_block(tables, block, *, device: Optional[int] = None, precision: Optional[int] = None):
    """Evolve one block through the whole sequence on the GPU (engine.py:259-310).

    Returns ``(echo_partials, snapshots)``: complex128 (n_acq, max_ns) — or
    (C, n_acq, max_ns) for a (C, n) weight — of receive-weighted transverse
    sums over the block, and one (n, 3) array (or None) per snapshot time.
    The block is not mutated.
    """
    eng = get_engine(device, precision)
    return eng.compute(
        tables, block.pos, block.mx, block.my, block.mz, block.t1, block.t2, block.m0, block.domega,
        block.weight, block_index=getattr(block, "index", 0),
    )


def simulate_spin(spin, tables, domega: float = 0.0, weight: complex = 1.0 + 0.0j, **kw):
    """Single-spin wrapper (engine.py:313-335)."""
    block = SpinBlock(
        index=0, pos=np.array([spin.position], dtype=float), mx=np.array([spin.m.mx]),
        my=np.array([spin.m.my]), mz=np.array([spin.m.mz]), t1=np.array([spin.relax.t1]),
        t2=np.array([spin.relax.t2]), m0=np.array([spin.relax.m0]), domega=np.array([float(domega)]),
        weight=np.array([complex(weight)]),
    )
    return compute_block(tables, block, **kw)


# ---------------------------------------------------------------------------
# run orchestration — engine.py:343-537
# ---------------------------------------------------------------------------


@dataclass
class EchoRecord:
    acq_index: int
    values: np.ndarray
    timestamps: np.ndarray


@dataclass
class RunMetrics:
    wall_time_s: float
    spin_count: int
    throughput: float  # spins per second of wall time
    workers: int
    blocks: int
    busy_fraction: Dict[int, float]
    hardware: str
    kernel_ms: float = 0.0
    events_per_spin: int = 0
    device_ms: Dict[int, float] = field(default_factory=dict)  # per GPU (rank order), whole-call device time


@dataclass
class RunResult:
    echoes: List[EchoRecord]
    metrics: RunMetrics
    snapshots: List[Tuple[float, np.ndarray]]
    spin_count: int
    spacing: Tuple[float, float, float]
    spacing_report: Optional[object] = None

    def echo_matrix(self) -> np.ndarray:
        return np.array([rec.values for rec in self.echoes])


@dataclass
class Experiment:
    sequence: Sequence
    phantom: Phantom
    system: SystemModel = field(default_factory=default_system)
    spacing: Optional[Tuple[float, float, float]] = None
    workers: int = 1  # accepted for API parity; one host process drives the device
    deterministic: bool = True  # the device fold is always in a fixed order
    blocks: Optional[int] = None
    snapshot_times: Tuple[float, ...] = ()
    spin_cap: int = DEFAULT_SPIN_CAP
    precision: int = 32
    device: Optional[int] = None
    devices: Optional[Tuple[int, ...]] = None  # > 1: a device set, the spins sharded over the GPUs


def _busy(eng, wall: float) -> Dict[int, float]:
    """busy_fraction per worker (engine.py:516-525): each GPU's device time over the wall time."""
    if wall <= 0:
        return {}
    return {r: t["device_ms"] / 1e3 / wall for r, t in eng.device_times().items()}


def run(exp: Experiment) -> RunResult:
    """Execute one experiment on the GPU (engine.py:465-537).

    Differences from the reference, all outside the hot path: ``spacing`` must
    be given (the spin-spacing analysis of mrsim.discretize is out of scope,
    SURVEY §2), and the spin set runs as one device block — the device result
    does not depend on the block partition (fixed per-CTA tiling, ordered fold).
    """
    if exp.workers < 1:
        raise InvalidParameter(f"workers must be >= 1, got {exp.workers}")
    if exp.spacing is None:
        raise InvalidParameter(
            "Experiment.spacing is required: the spacing analysis (mrsim.discretize) is out of "
            "scope for the GPU engine"
        )
    wall_start = time.perf_counter()
    spacing = tuple(float(s) for s in exp.spacing)
    from .objects import DeviceScene

    if isinstance(exp.phantom, DeviceScene):
        return _run_device_scene(exp, spacing, wall_start)
    spins = rasterize_arrays(exp.phantom, spacing, cap=exp.spin_cap)
    if spins["m0"].size == 0:
        raise InvalidParameter("the phantom rasterized to zero spins")
    arrays = build_spin_arrays(spins, exp.system)
    tables = precompute_sequence_tables(exp.sequence, gamma=exp.system.gamma, snapshot_times=exp.snapshot_times)
    eng = get_engine(exp.device, exp.precision, devices=list(exp.devices) if exp.devices else None)
    t_k = time.perf_counter()
    echo_sum, snaps = eng.compute(
        tables, arrays.pos, arrays.mx, arrays.my, arrays.mz, arrays.t1, arrays.t2, arrays.m0, arrays.domega,
        arrays.weight,
    )
    busy = time.perf_counter() - t_k
    n_spins = arrays.n
    records = []
    if tables.n_acq:
        echo_sum = echo_sum / n_spins  # engine.py:507
        for i in range(tables.n_acq):
            records.append(
                EchoRecord(acq_index=i, values=echo_sum[..., i, : tables.acq_times[i].size],
                           timestamps=tables.acq_times[i])
            )
    wall = time.perf_counter() - wall_start
    timing = eng.last_timing()
    metrics = RunMetrics(
        wall_time_s=wall, spin_count=n_spins, throughput=n_spins / wall if wall > 0 else math.inf,
        workers=len(eng.devices), blocks=len(eng.devices), busy_fraction=_busy(eng, wall),
        hardware=f"{platform.machine()} cuda:{','.join(map(str, eng.devices))} sm_100a", kernel_ms=timing["kernel_ms"],
        events_per_spin=eng.program_stats()["events"], device_ms={r: t["device_ms"] for r, t in
                                                                   eng.device_times().items()},
    )
    snapshots = [
        (t, snaps[i] if snaps[i] is not None else np.zeros((0, 3))) for i, t in enumerate(tables.snapshot_times)
    ]
    return RunResult(echoes=records, metrics=metrics, snapshots=snapshots, spin_count=n_spins, spacing=spacing)


def _run_device_scene(exp: Experiment, spacing, wall_start: float) -> RunResult:
    """run() for a DeviceScene: spins are rasterised on the GPU and never visit the host."""
    import torch

    from .objects import rasterize_device

    sysm = exp.system
    if sysm.field.inhomogeneity is not None:
        raise InvalidParameter("a DeviceScene carries its own off-resonance maps; the system inhomogeneity "
                               "callable has no device form")
    tables = precompute_sequence_tables(exp.sequence, gamma=sysm.gamma, snapshot_times=exp.snapshot_times)
    eng = get_engine(exp.device, exp.precision)
    ctx = sysm.frame()
    scene = exp.phantom
    base = ctx.gamma * sysm.field.b0 - ctx.omega_hf
    if base != 0.0:
        scene = dataclasses.replace(scene, const_dw=scene.const_dw + base)
    spins = rasterize_device(scene, spacing, eng, cap=exp.spin_cap)
    f = eng.set_tables(tables)
    dev = spins.pos.device
    echo = torch.zeros((spins.n_coils, f["n_acq"], f["max_ns"]), dtype=torch.complex128, device=dev)
    snaps = torch.zeros((f["n_snap"], spins.n, 3), dtype=torch.float64, device=dev) if f["n_snap"] else None
    present = np.zeros(max(f["n_snap"], 1), dtype=np.uint8)
    torch.cuda.current_stream(dev).synchronize()
    t_k = time.perf_counter()
    ptrs = spins.pointers()
    if spins.n_coils == 1 and isinstance(scene.receive, UniformSensitivity) and scene.receive.s == 1.0:
        ptrs["weight"] = 0
    eng.compute_device(tables, ptrs, spins.n, spins.n_coils, echo.data_ptr(),
                       snaps.data_ptr() if snaps is not None else 0, sync=True, present=present)
    busy = time.perf_counter() - t_k
    echo_sum = echo.cpu().numpy()
    if spins.n_coils == 1 and not spins.coil_array:  # a CoilArray keeps its coil axis, as on the host path
        echo_sum = echo_sum[0]
    n_spins = spins.n
    records = []
    if tables.n_acq:
        echo_sum = echo_sum / n_spins  # engine.py:507
        for i in range(tables.n_acq):
            records.append(EchoRecord(acq_index=i, values=echo_sum[..., i, : tables.acq_times[i].size],
                                      timestamps=tables.acq_times[i]))
    snap_host = snaps.cpu().numpy() if snaps is not None else None
    wall = time.perf_counter() - wall_start
    timing = eng.last_timing()
    metrics = RunMetrics(
        wall_time_s=wall, spin_count=n_spins, throughput=n_spins / wall if wall > 0 else math.inf,
        workers=1, blocks=1, busy_fraction=_busy(eng, wall),
        hardware=f"{platform.machine()} cuda:{eng.device} sm_100a", kernel_ms=timing["kernel_ms"],
        events_per_spin=eng.program_stats()["events"], device_ms={0: timing["device_ms"]},
    )
    snapshots = [(t, snap_host[i] if present[i] else np.zeros((0, 3))) for i, t in enumerate(tables.snapshot_times)]
    return RunResult(echoes=records, metrics=metrics, snapshots=snapshots, spin_count=n_spins, spacing=spacing)


# ---------------------------------------------------------------------------
# result comparison — engine.py:603-656
# ---------------------------------------------------------------------------


def delta_e_stoer(ref, test) -> float:
    """10*log10(sum|ref-test|^2 / sum|ref|^2); -inf when identical (engine.py:603-616)."""
    ref = np.asarray(ref).ravel()
    test = np.asarray(test).ravel()
    if ref.shape != test.shape:
        raise InvalidParameter(f"shape mismatch: {ref.shape} vs {test.shape}")
    num = float(np.sum(np.abs(ref - test) ** 2))
    den = float(np.sum(np.abs(ref) ** 2))
    if den == 0.0:
        return -math.inf if num == 0.0 else math.inf
    if num == 0.0:
        return -math.inf
    return 10.0 * math.log10(num / den)


@dataclass(frozen=True)
class ComparisonResult:
    delta_e_db: float
    exceedances: int
    compared: int
    rel_threshold: float


def compare_results(ref, test, rel_threshold: float = 1e-6) -> ComparisonResult:
    """ΔE_stör plus per-component relative exceedances, eps-scale pairs unrated (engine.py:627-656)."""
    ref = np.asarray(ref)
    test = np.asarray(test)
    if ref.shape != test.shape:
        raise InvalidParameter(f"shape mismatch: {ref.shape} vs {test.shape}")
    if np.iscomplexobj(ref) or np.iscomplexobj(test):
        ref = np.concatenate([np.real(ref).ravel(), np.imag(ref).ravel()])
        test = np.concatenate([np.real(test).ravel(), np.imag(test).ravel()])
    else:
        ref = ref.ravel().astype(float)
        test = test.ravel().astype(float)
    scale = float(np.max(np.abs(ref))) if ref.size else 0.0
    eps_scale = np.finfo(float).eps * max(scale, 1e-300)
    rated = ~((np.abs(ref) < eps_scale) & (np.abs(test) < eps_scale))
    rel = np.zeros_like(ref)
    denom = np.abs(ref[rated])
    denom = np.where(denom > 0.0, denom, eps_scale)
    rel[rated] = np.abs(ref[rated] - test[rated]) / denom
    return ComparisonResult(
        delta_e_db=delta_e_stoer(ref, test), exceedances=int(np.sum(rel > rel_threshold)),
        compared=int(np.sum(rated)), rel_threshold=rel_threshold,
    )

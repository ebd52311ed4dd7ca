"""float64 numpy restatement of the reference hot path — TEST INFRASTRUCTURE ONLY.

Restates, operation for operation, the reference algorithm so that on the same
inputs the results are bit-identical to the reference on the same machine
(pinned by ``tests/test_oracle_golden.py`` against vectors produced by the
reference itself, ``tests/golden/make_golden.py``).

Reference files (``/root/reference/pkg/src/mrsim/``):

* ``engine.py:83-164``   precompute_sequence_tables  → :func:`precompute_tables`
* ``engine.py:259-310``  compute_block               → :func:`compute_block`
* ``engine.py:229-251``  partition_blocks            → :func:`partition_bounds`
* ``engine.py:493-515``  fold + normalisation         → :func:`fold_partials`
* ``engine.py:603-616``  delta_e_stoer               → :func:`delta_e_stoer`
* ``sequence.py:92-125`` GradientWaveform.moments / partial_moments
* ``sequence.py:139-144`` AcquisitionSpec.sample_times
* ``bloch.py:124-139``   hard_pulse_matrix

Sequence objects are duck-typed: anything with ``.elements`` whose items carry
``pulse`` (``alpha``, ``phi``) or None, ``gradient`` (``shape``, ``gx``, ``gy``,
``gz``, ``ramp_s``, ``flat_s``, ``samples``, ``sample_dt``), ``duration`` and
``acquisition`` (``enabled``, ``n_samples``) works — the reference's own
classes and the product's mirror classes alike.

Extension beyond the reference (documented, used for config 4): ``weight`` may
be a ``(C, n)`` complex array (C receive coils); the echoes then carry a
leading coil axis.  The reference supports one weight per spin
(``engine.py:185``); per coil the arithmetic here is exactly the reference's.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import numpy as np

GAMMA_PROTON = 2.0 * math.pi * 42.6e6  # bloch.py:41


# ---------------------------------------------------------------------------
# helpers the master precompute calls
# ---------------------------------------------------------------------------


def hard_pulse_matrix(alpha: float, phi: float) -> np.ndarray:
    """Rotation by alpha about (cos phi, sin phi, 0) — bloch.py:124-139."""
    ca, sa = np.cos(alpha), np.sin(alpha)
    cp, sp = np.cos(phi), np.sin(phi)
    return np.array(
        [
            [cp * cp + sp * sp * ca, sp * cp * (1.0 - ca), -sp * sa],
            [sp * cp * (1.0 - ca), sp * sp + cp * cp * ca, cp * sa],
            [sp * sa, -cp * sa, ca],
        ]
    )


def sample_times(acq, duration: float) -> np.ndarray:
    """ADC instants i*dur/(n-1), endpoints inclusive — sequence.py:139-144."""
    if not acq.enabled:
        return np.empty(0)
    if acq.n_samples == 1:
        return np.array([0.0])
    return np.arange(acq.n_samples) * (duration / (acq.n_samples - 1))


def _amplitudes(g) -> np.ndarray:
    return np.array([g.gx, g.gy, g.gz])  # sequence.py:89-90


def total_moment(g, duration: float, gamma: float) -> np.ndarray:
    """gamma * integral of G over the interval — sequence.py:92-99."""
    if g.shape == "constant":
        return gamma * _amplitudes(g) * duration
    if g.shape == "trapezoid":
        return gamma * _amplitudes(g) * (g.ramp_s + g.flat_s)
    arr = np.asarray(g.samples, dtype=float)
    return gamma * np.trapezoid(arr, dx=g.sample_dt, axis=0)


def partial_moments(g, ts, duration: float, gamma: float) -> np.ndarray:
    """Cumulative moments at times ts, shape (len(ts), 3) — sequence.py:101-125."""
    ts = np.asarray(ts, dtype=float)
    if g.shape == "constant":
        return gamma * np.outer(ts, _amplitudes(g))
    if g.shape == "trapezoid":
        r, f = g.ramp_s, g.flat_s
        up = np.clip(ts, 0.0, r)
        flat = np.clip(ts - r, 0.0, f)
        down = np.clip(ts - r - f, 0.0, r)
        unit = up**2 / (2.0 * r) if r > 0.0 else np.zeros_like(ts)
        unit = unit + flat
        if r > 0.0:
            unit = unit + down - down**2 / (2.0 * r)
        return gamma * np.outer(unit, _amplitudes(g))
    arr = np.asarray(g.samples, dtype=float)
    grid = np.arange(arr.shape[0]) * g.sample_dt
    cum = np.concatenate(
        [np.zeros((1, 3)), np.cumsum((arr[1:] + arr[:-1]) / 2.0 * g.sample_dt, axis=0)]
    )
    out = np.empty((ts.size, 3))
    for ax in range(3):
        out[:, ax] = np.interp(ts, grid, cum[:, ax])
    return gamma * out


# ---------------------------------------------------------------------------
# event tables (master side) — engine.py:51-164
# ---------------------------------------------------------------------------


@dataclass
class OracleEsTable:
    """Same fields as engine.EsTable (engine.py:51-70)."""

    pulse_mat: Optional[np.ndarray]
    duration: float
    moments: np.ndarray
    ev_dt: np.ndarray
    ev_dmom: np.ndarray
    ev_sample: np.ndarray
    ev_snap: np.ndarray
    acq: int = -1
    n_samples: int = 0


@dataclass
class OracleTables:
    """Same fields as engine.OperatorTables (engine.py:73-80)."""

    entries: List[OracleEsTable]
    n_acq: int
    acq_times: List[np.ndarray]
    snapshot_times: Tuple[float, ...]
    pulse_memo_hits: int
    gamma: float


def precompute_tables(
    sequence, gamma: float = GAMMA_PROTON, snapshot_times=(), memoize: bool = True
) -> OracleTables:
    """Restatement of engine.precompute_sequence_tables (engine.py:83-164).

    Per elementary sequence: the memoised 3x3 pulse matrix (104-112), the ADC
    and snapshot instants sorted so a snapshot precedes a sample at equal t
    (114-119), per-event dt and moment increments (121-134), and the tail
    event when the last instant misses the end *or* the accumulated moment
    differs from the total by any bit (135-140).  ``repetitions`` is ignored,
    as in the reference (102).
    """
    snapshot_times = tuple(sorted(snapshot_times))
    entries: List[OracleEsTable] = []
    acq_times: List[np.ndarray] = []
    memo: Dict[Tuple[float, float], np.ndarray] = {}
    hits = 0
    t0 = 0.0
    acq = 0
    for es in sequence.elements:
        mat = None
        pulse = es.pulse
        if pulse is not None and not (pulse.alpha == 0.0):  # bloch.py:106-108
            key = (pulse.alpha, pulse.phi)
            if memoize and key in memo:
                mat = memo[key]
                hits += 1
            else:
                mat = hard_pulse_matrix(pulse.alpha, pulse.phi)
                if memoize:
                    memo[key] = mat
        t1 = t0 + es.duration
        s_ts = sample_times(es.acquisition, es.duration)
        events = [(float(t), True, -1) for t in s_ts]
        for si, t_abs in enumerate(snapshot_times):
            if t0 < t_abs <= t1 or (t_abs == 0.0 == t0):
                events.append((float(t_abs - t0), False, si))
        events.sort(key=lambda e: (e[0], e[1]))
        ts = np.array([e[0] for e in events])
        partial = (
            partial_moments(es.gradient, ts, es.duration, gamma) if ts.size else np.zeros((0, 3))
        )
        total = total_moment(es.gradient, es.duration, gamma)
        ev_dt, ev_dmom, ev_sample, ev_snap = [], [], [], []
        prev_t, prev_m = 0.0, np.zeros(3)
        for i, (t, is_sample, snap) in enumerate(events):
            ev_dt.append(t - prev_t)
            ev_dmom.append(partial[i] - prev_m)
            ev_sample.append(is_sample)
            ev_snap.append(snap)
            prev_t, prev_m = t, partial[i]
        if prev_t < es.duration or np.any(prev_m != total):
            ev_dt.append(es.duration - prev_t)
            ev_dmom.append(total - prev_m)
            ev_sample.append(False)
            ev_snap.append(-1)
        entry = OracleEsTable(
            pulse_mat=mat,
            duration=es.duration,
            moments=np.asarray(total, dtype=float),
            ev_dt=np.array(ev_dt, dtype=float),
            ev_dmom=np.array(ev_dmom, dtype=float) if ev_dmom else np.zeros((0, 3)),
            ev_sample=np.array(ev_sample, dtype=bool),
            ev_snap=np.array(ev_snap, dtype=int),
        )
        if es.acquisition.enabled:
            entry.acq = acq
            entry.n_samples = es.acquisition.n_samples
            acq_times.append(t0 + s_ts)
            acq += 1
        entries.append(entry)
        t0 = t1
    return OracleTables(
        entries=entries,
        n_acq=acq,
        acq_times=acq_times,
        snapshot_times=snapshot_times,
        pulse_memo_hits=hits,
        gamma=gamma,
    )


def event_count(tables) -> int:
    """E = #(ES with a pulse matrix) + #table events (SURVEY §8d metric)."""
    return sum(int(e.pulse_mat is not None) + int(e.ev_dt.size) for e in tables.entries)


def event_class_counts(tables) -> Dict[str, int]:
    """Per-class event counts for the algorithmic roofline."""
    n_rot = n_pr = n_p = n_noop = n_adc = 0
    for e in tables.entries:
        n_rot += int(e.pulse_mat is not None)
        dt = e.ev_dt
        moving = np.any(e.ev_dmom != 0.0, axis=1) if e.ev_dmom.size else np.zeros(0, bool)
        n_pr += int(np.sum(dt != 0.0))
        n_p += int(np.sum((dt == 0.0) & moving))
        n_noop += int(np.sum((dt == 0.0) & ~moving))
        n_adc += int(np.sum(e.ev_sample))
    return {"rot": n_rot, "prec_relax": n_pr, "prec": n_p, "noop": n_noop, "adc": n_adc}


# ---------------------------------------------------------------------------
# the kernel (worker side) — engine.py:259-310
# ---------------------------------------------------------------------------


def compute_block(tables, pos, mx, my, mz, t1, t2, m0, domega, weight):
    """Restatement of engine.compute_block (engine.py:259-310).

    Arguments are the SpinBlock fields (engine.py:172-189) as float64 arrays
    (``pos`` (n, 3)); ``weight`` is complex (n,) or (C, n).  Returns
    ``(echoes, snapshots)``: echoes complex128 (n_acq, max_ns) — or
    (C, n_acq, max_ns) for a (C, n) weight — and one (n, 3) array (or None)
    per snapshot time.  The input state is not mutated (engine.py:267).
    """
    mx, my, mz = np.array(mx, dtype=float), np.array(my, dtype=float), np.array(mz, dtype=float)
    pos = np.asarray(pos, dtype=float).reshape(-1, 3)
    domega = np.asarray(domega, dtype=float)
    w = np.asarray(weight)
    multi = w.ndim == 2
    ws = [w[c] for c in range(w.shape[0])] if multi else [w]
    inv_t1, inv_t2 = 1.0 / np.asarray(t1, dtype=float), 1.0 / np.asarray(t2, dtype=float)
    m0 = np.asarray(m0, dtype=float)
    relax_cache: Dict[float, Tuple[np.ndarray, np.ndarray, np.ndarray]] = {}
    n_samples = max((e.n_samples for e in tables.entries), default=0)
    echoes = np.zeros((len(ws), tables.n_acq, n_samples), dtype=complex)
    snapshots: Dict[int, np.ndarray] = {}
    for entry in tables.entries:
        if entry.pulse_mat is not None:  # engine.py:277-283
            r = entry.pulse_mat
            mx, my, mz = (
                r[0, 0] * mx + r[0, 1] * my + r[0, 2] * mz,
                r[1, 0] * mx + r[1, 1] * my + r[1, 2] * mz,
                r[2, 0] * mx + r[2, 1] * my + r[2, 2] * mz,
            )
        sample_idx = 0
        for i in range(entry.ev_dt.size):  # engine.py:285-308
            dt = entry.ev_dt[i]
            dmom = entry.ev_dmom[i]
            if dt != 0.0 or dmom.any():
                theta = pos @ dmom + domega * dt
                c, s = np.cos(theta), np.sin(theta)
                mx, my = c * mx + s * my, -s * mx + c * my  # clockwise, bloch.py:10-17
                if dt != 0.0:
                    cached = relax_cache.get(dt)
                    if cached is None:
                        e1 = np.exp(-dt * inv_t1)
                        e2 = np.exp(-dt * inv_t2)
                        cached = (e1, e2, m0 * (1.0 - e1))
                        relax_cache[dt] = cached
                    e1, e2, regrow = cached
                    mx *= e2
                    my *= e2
                    mz = mz * e1 + regrow
            if entry.ev_sample[i]:
                for c_i, wc in enumerate(ws):
                    echoes[c_i, entry.acq, sample_idx] = np.dot(wc, mx) + 1j * np.dot(wc, my)
                sample_idx += 1
            snap = entry.ev_snap[i]
            if snap >= 0:
                snapshots[snap] = np.column_stack([mx, my, mz])
    snap_list = [snapshots.get(i) for i in range(len(tables.snapshot_times))]
    return (echoes if multi else echoes[0]), snap_list


# ---------------------------------------------------------------------------
# partition + reduction — engine.py:229-251, 493-515
# ---------------------------------------------------------------------------


def partition_bounds(n: int, n_blocks: int) -> np.ndarray:
    """Contiguous block bounds exactly as partition_blocks (engine.py:229-251)."""
    n_blocks = max(1, min(n_blocks, n)) if n else 1
    return np.linspace(0, n, n_blocks + 1).astype(int)


def fold_partials(partials, n_spins: int, tables):
    """Ordered fold of block partials, ÷ N, per-acq truncation (engine.py:493-515).

    Returns a list of (values, timestamps) per acquisition (EchoRecord fields).
    """
    echo_sum = None
    for echoes in partials:
        echo_sum = echoes if echo_sum is None else echo_sum + echoes
    records = []
    if echo_sum is not None and tables.n_acq:
        echo_sum = echo_sum / n_spins
        for i in range(tables.n_acq):
            size = tables.acq_times[i].size
            records.append((echo_sum[..., i, :size], tables.acq_times[i]))
    return records


def delta_e_stoer(ref, test) -> float:
    """Difference energy over reference energy in dB (engine.py:603-616)."""
    ref = np.asarray(ref).ravel()
    test = np.asarray(test).ravel()
    if ref.shape != test.shape:
        raise ValueError(f"shape mismatch: {ref.shape} vs {test.shape}")
    num = float(np.sum(np.abs(ref - test) ** 2))
    den = float(np.sum(np.abs(ref) ** 2))
    if den == 0.0:
        return -math.inf if num == 0.0 else math.inf
    if num == 0.0:
        return -math.inf
    return 10.0 * math.log10(num / den)


def rel_l2(ref, test) -> float:
    """Relative L2 error ||test - ref|| / ||ref|| (the BASELINE.json parity metric)."""
    ref = np.asarray(ref).ravel()
    test = np.asarray(test).ravel()
    den = float(np.linalg.norm(ref))
    num = float(np.linalg.norm(test - ref))
    if den == 0.0:
        return 0.0 if num == 0.0 else math.inf
    return num / den

"""B200 backend for the reference's spin kernel — the binding a maintainer would add to ``mrsim``.

This module is the reference-side stub of INTEGRATION.md §2 as a runnable file: plain ctypes over
``libbloch_b200.so`` (include/bloch_b200.h), no dependency on the ``paper_1305_6861_b200`` Python
package.  It replaces exactly one function, ``mrsim.engine.compute_block(tables, block)``
(engine.py:259-310): same arguments (the reference's ``OperatorTables`` / ``SpinBlock``), same
return value ``(echoes complex128 (n_acq, max_ns), [snapshot (n, 3) | None, ...])``, and the
reference's exception types (``InvalidParameter``, ``WorkerPanic(block_index, msg)``,
engine.py:455-459, errors.py:57-62).

    import mrsim.engine, mrsim_b200
    mrsim.engine.compute_block = mrsim_b200.compute_block_b200     # or install()

Environment: ``MRSIM_B200_LIB`` (path of libbloch_b200.so), ``MRSIM_B200_PRECISION`` (32 default,
64 for the reference's 1e-12 unit tests), ``LOCAL_RANK`` (device).  Each process (the reference's
forked/forkserver pool workers included) opens its own context on first use.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_DEFAULT_LIB = os.path.join(os.path.dirname(_HERE), "paper_1305_6861_b200", "libbloch_b200.so")

_PD = ctypes.POINTER(ctypes.c_double)
_PI32 = ctypes.POINTER(ctypes.c_int32)
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PU8 = ctypes.POINTER(ctypes.c_uint8)

_state = {"lib": None, "ctx": None, "tables": None, "calls": 0}


def _lib():
    lib = _state["lib"]
    if lib is None:
        lib = ctypes.CDLL(os.environ.get("MRSIM_B200_LIB", _DEFAULT_LIB))
        lib.bloch_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
        lib.bloch_set_tables.argtypes = [ctypes.c_void_p, ctypes.c_int32, _PI64, _PU8, _PD, _PI32, _PD, _PD, _PU8,
                                         _PI32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
        lib.bloch_compute_block.argtypes = ([ctypes.c_void_p, ctypes.c_int64] + [_PD] * 9 +
                                            [ctypes.c_int32, _PD, _PD, _PU8, ctypes.c_uint32])
        lib.bloch_last_error.restype = ctypes.c_char_p
        _state["lib"] = lib
    return lib


def _check(status, block_index):
    from mrsim.errors import InvalidParameter, WorkerPanic

    if status == 0:
        return
    msg = (_lib().bloch_last_error() or b"").decode()
    if status == -1:
        raise InvalidParameter(msg)
    raise WorkerPanic(block_index, msg)


def _context(block_index):
    if _state["ctx"] is None:
        ctx = ctypes.c_void_p()
        prec = int(os.environ.get("MRSIM_B200_PRECISION", "32"))
        _check(_lib().bloch_create(int(os.environ.get("LOCAL_RANK", "0")), prec, ctypes.byref(ctx)), block_index)
        _state["ctx"] = ctx
    return _state["ctx"]


def _upload(ctx, tables, block_index):
    if _state["tables"] is tables:  # once per OperatorTables object (kept alive: identity is safe)
        return
    e = tables.entries
    off = np.zeros(len(e) + 1, dtype=np.int64)
    np.cumsum([x.ev_dt.size for x in e], out=off[1:])
    has = np.array([x.pulse_mat is not None for x in e], dtype=np.uint8)
    mats = np.ascontiguousarray(
        np.stack([np.ravel(x.pulse_mat) if x.pulse_mat is not None else np.zeros(9) for x in e]) if e
        else np.zeros((0, 9)), dtype=np.float64)
    acq = np.array([x.acq for x in e], dtype=np.int32)
    cat = lambda key, shape, dt: (np.ascontiguousarray(np.concatenate([np.asarray(getattr(x, key)).reshape(shape)
                                                                       for x in e]), dtype=dt)
                                  if off[-1] else np.zeros((0,) + shape[1:], dtype=dt))
    dt_ = cat("ev_dt", (-1,), np.float64)
    dm = cat("ev_dmom", (-1, 3), np.float64)
    smp = cat("ev_sample", (-1,), np.uint8)
    snp = cat("ev_snap", (-1,), np.int32)
    max_ns = max((x.n_samples for x in e), default=0)
    _check(_lib().bloch_set_tables(ctx, len(e), off.ctypes.data_as(_PI64), has.ctypes.data_as(_PU8),
                                   mats.ctypes.data_as(_PD), acq.ctypes.data_as(_PI32), dt_.ctypes.data_as(_PD),
                                   dm.ctypes.data_as(_PD), smp.ctypes.data_as(_PU8), snp.ctypes.data_as(_PI32),
                                   int(tables.n_acq), int(max_ns), len(tables.snapshot_times)), block_index)
    _state["tables"] = tables


def compute_block_b200(tables, block):
    """``mrsim.engine.compute_block`` on the B200 (engine.py:259-310); the block is not mutated."""
    ctx = _context(block.index)
    _upload(ctx, tables, block.index)
    n = int(np.asarray(block.mx).size)
    max_ns = max((x.n_samples for x in tables.entries), default=0)
    n_snap = len(tables.snapshot_times)
    echoes = np.zeros((tables.n_acq, max_ns), dtype=np.complex128)
    snaps = np.zeros((n_snap, n, 3))
    present = np.zeros(max(1, n_snap), dtype=np.uint8)
    keep = [np.ascontiguousarray(a, dtype=np.float64) for a in (block.pos, block.mx, block.my, block.mz, block.t1,
                                                                  block.t2, block.m0, block.domega)]
    w = np.ascontiguousarray(block.weight, dtype=np.complex128)
    ptr = lambda a: a.ctypes.data_as(_PD)
    _check(_lib().bloch_compute_block(ctx, n, *[ptr(a) for a in keep], ptr(w.view(np.float64)), 1,
                                      ptr(echoes.view(np.float64)), ptr(snaps), present.ctypes.data_as(_PU8), 0),
           block.index)
    _state["calls"] += 1
    return echoes, [snaps[i] if present[i] else None for i in range(n_snap)]


def calls() -> int:
    """compute_block_b200 calls made in this process."""
    return _state["calls"]


def install(engine_module=None):
    """Swap the reference's kernel: ``mrsim.engine.compute_block = compute_block_b200``."""
    if engine_module is None:
        import mrsim.engine as engine_module
    engine_module.compute_block = compute_block_b200
    return engine_module

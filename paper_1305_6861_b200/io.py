"""Wire formats of the simulation outputs.

Byte-compatible with ``mrsim.io`` (io.py:17-140) — pinned by
``tests/test_recon_io.py`` against files the reference itself wrote
(``tests/golden/wire/``).  Every format is one ASCII header line followed by
a little-endian payload:

==========  ===============================  ==================================
format      header                           payload
==========  ===============================  ==================================
echo        ``MRSIM1 n_acq n_samples``       f64 (re, im) pairs, acquisition-major;
                                             plus ``<path>.manifest.json``
snapshot    ``n_spins t_s``                  f64 (Mx, My, Mz) per spin
raw grid    ``nx ny dtype=c128|f64``         row-major [y, x], x fastest
PGM (P5)    ``P5\\nnx ny\\n255``             u8 magnitude after a linear window
==========  ===============================  ==================================
"""

from __future__ import annotations

import json
import time
from typing import Optional, Tuple

import numpy as np

from .errors import InvalidParameter, ParseError

ECHO_MAGIC = "MRSIM1"
_GRID_TYPES = {"c128": "<c16", "f64": "<f8"}


def _put(path: str, header: str, payload: np.ndarray) -> None:
    with open(path, "wb") as fh:
        fh.write(header.encode("ascii"))
        fh.write(payload.tobytes())


def _get(path: str, dtype: str):
    """(header tokens, payload as a flat `dtype` array)."""
    with open(path, "rb") as fh:
        tokens = fh.readline().decode("ascii").split()
        return tokens, np.frombuffer(fh.read(), dtype=dtype)


def _need(path: str, data: np.ndarray, count: int, what: str = "floats") -> None:
    if data.size != count:
        raise ParseError(f"{path}: expected {count} {what}, found {data.size}")


def _json_default(obj):
    if isinstance(obj, np.ndarray):
        return obj.tolist()
    if isinstance(obj, (np.floating, np.integer)):
        return obj.item()
    return str(obj)


# -- echo file + manifest (io.py:20-64) ---------------------------------------------------------------------------


def write_echo_file(path: str, matrix, manifest: Optional[dict] = None) -> None:
    m = np.asarray(matrix, dtype=complex)
    if m.ndim != 2:
        raise InvalidParameter(f"echo matrix must be 2-D, got shape {m.shape}")
    n_acq, n_samples = m.shape
    # complex128 in memory already is (re, im) f64 pairs: view instead of interleaving by hand
    _put(path, f"{ECHO_MAGIC} {n_acq} {n_samples}\n", np.ascontiguousarray(m).view(np.float64).astype("<f8"))
    meta = dict(manifest or {})
    meta.setdefault("written_at", time.strftime("%Y-%m-%dT%H:%M:%S%z"))
    meta.update(n_acq=n_acq, n_samples=n_samples)
    with open(path + ".manifest.json", "w", encoding="utf-8") as fh:
        fh.write(json.dumps(meta, indent=2, default=_json_default) + "\n")


def read_echo_file(path: str) -> np.ndarray:
    tok, data = _get(path, "<f8")
    if len(tok) != 3 or tok[0] != ECHO_MAGIC:
        raise ParseError(f"{path} is not an echo file (bad header {tok!r})")
    n_acq, n_samples = int(tok[1]), int(tok[2])
    _need(path, data, 2 * n_acq * n_samples)
    pairs = data.reshape(n_acq, n_samples, 2)
    return pairs[..., 0] + 1j * pairs[..., 1]


def read_manifest(path: str) -> dict:
    with open(path + ".manifest.json", "r", encoding="utf-8") as fh:
        return json.load(fh)


# -- magnetisation snapshots (io.py:67-87) ------------------------------------------------------------------------


def write_snapshot_file(path: str, t: float, magnetization) -> None:
    m = np.asarray(magnetization, dtype=float)
    if m.ndim != 2 or m.shape[1] != 3:
        raise InvalidParameter(f"snapshot must be (n, 3), got {m.shape}")
    _put(path, f"{m.shape[0]} {t!r}\n", m.astype("<f8"))


def read_snapshot_file(path: str) -> Tuple[float, np.ndarray]:
    tok, data = _get(path, "<f8")
    if len(tok) != 2:
        raise ParseError(f"{path} is not a snapshot file")
    n = int(tok[0])
    _need(path, data, 3 * n)
    return float(tok[1]), data.reshape(n, 3)


# -- raw grids and previews (io.py:90-140) ------------------------------------------------------------------------


def write_raw_grid(path: str, grid) -> None:
    g = np.asarray(grid)
    if g.ndim != 2:
        raise InvalidParameter(f"raw grid must be 2-D, got shape {g.shape}")
    kind = "c128" if np.iscomplexobj(g) else "f64"
    _put(path, f"{g.shape[1]} {g.shape[0]} dtype={kind}\n", np.ascontiguousarray(g).astype(_GRID_TYPES[kind]))


def read_raw_grid(path: str) -> np.ndarray:
    with open(path, "rb") as fh:
        tok = fh.readline().decode("ascii").split()
        if len(tok) != 3 or not tok[2].startswith("dtype="):
            raise ParseError(f"{path} is not a raw grid file")
        kind = tok[2][len("dtype="):]
        if kind not in _GRID_TYPES:
            raise ParseError(f"{path}: unknown dtype {kind}")
        data = np.frombuffer(fh.read(), dtype=_GRID_TYPES[kind])
    nx, ny = int(tok[0]), int(tok[1])
    _need(path, data, nx * ny, "values")
    return data.reshape(ny, nx)


def write_pgm(path: str, image, window: Optional[Tuple[float, float]] = None) -> None:
    img = np.asarray(image, dtype=float)
    if img.ndim != 2:
        raise InvalidParameter(f"image must be 2-D, got shape {img.shape}")
    lo, hi = (img.min(), img.max()) if window is None else window
    lo, hi = float(lo), float(hi)
    level = np.clip((img - lo) / (hi - lo), 0.0, 1.0) if hi > lo else np.zeros_like(img)
    _put(path, f"P5\n{img.shape[1]} {img.shape[0]}\n255\n", np.round(level * 255.0).astype(np.uint8))

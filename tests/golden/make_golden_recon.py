"""Golden vectors for reconstruction and the wire formats, made by the REFERENCE.

    python tests/golden/make_golden_recon.py [--ref /root/reference/pkg/src]

Runs ``mrsim.recon`` (assemble_kspace, reconstruct, forward_dft, cpmg_fit) on
seeded inputs and records the outputs in ``tests/golden/recon.npz``; writes
echo / snapshot / raw-grid / PGM files with ``mrsim.io`` into
``tests/golden/wire/`` so the tests can check byte compatibility.  Build
container only — the tests read the committed outputs, never the reference.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def recon_cases():
    """(name, echoes, trajectory, n_rows, fov) seeded inputs covering the table modes."""
    rng = np.random.default_rng(1305)

    def cplx(*shape):
        return rng.normal(size=shape) + 1j * rng.normal(size=shape)

    se16 = np.load(os.path.join(HERE, "se16_box.npz"))
    se_echo = se16["echo_full"].reshape(tuple(se16["echo_shape"]))
    se_echo = se_echo.reshape(-1, se_echo.shape[-1])
    return [
        ("se_sim16", se_echo, [(0, i, False) for i in range(se_echo.shape[0])], None, 0.2),
        ("epi12x10", cplx(12, 10), [(0, i, i % 2 == 1) for i in range(12)], 12, 0.3),
        ("odd15x9", cplx(15, 9), [(0, i, False) for i in range(15)], 15, 0.25),
        ("tse_seq8", cplx(8, 8), [(0, (i // 4) * 4 + i % 4, False) for i in range(8)], 8, None),
        ("volumes6x4", cplx(6, 4), [(e % 3, e // 3, False) for e in range(6)], 2, 0.5),
        ("missing_rows", cplx(3, 6), [(0, 0, False), (0, 3, True), (0, 5, False)], 7, 0.4),
    ]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    from mrsim import io as rio
    from mrsim import recon as rr

    out = {}
    for name, echoes, table, n_rows, fov in recon_cases():
        mats = rr.assemble_kspace(echoes, table, n_rows=n_rows, fov=fov)
        out[f"{name}__echoes"] = np.asarray(echoes, complex)
        out[f"{name}__table"] = np.array(table, dtype=np.int64).reshape(-1, 3)
        out[f"{name}__n_rows"] = np.int64(-1 if n_rows is None else n_rows)
        out[f"{name}__fov"] = np.float64(np.nan if fov is None else fov)
        out[f"{name}__n_vol"] = np.int64(len(mats))
        for i, k in enumerate(mats):
            img = rr.reconstruct(k)
            out[f"{name}__k{i}"] = k.data
            out[f"{name}__filled{i}"] = k.row_filled
            out[f"{name}__axes{i}"] = np.array([k.k0[0], k.k0[1], k.dk[0], k.dk[1]])
            out[f"{name}__vol{i}"] = np.int64(k.volume)
            out[f"{name}__img{i}"] = img.complex_image
            out[f"{name}__pix{i}"] = np.array(img.pixel_size)
    rng = np.random.default_rng(77)
    img = rng.normal(size=(8, 12)) + 1j * rng.normal(size=(8, 12))
    k0y, dky = rr.standard_axes(0.3, 8)
    k0x, dkx = rr.standard_axes(0.3, 12)
    fk = rr.forward_dft(rr.ImageVolume(img, (1.0, 1.0)), k0=(k0y, k0x), dk=(dky, dkx))
    out["fwd__img"] = img
    out["fwd__axes"] = np.array([k0y, k0x, dky, dkx])
    out["fwd__k"] = fk.data
    t = np.arange(1, 13) * 0.02
    series = [0.8 * np.exp(-t / 0.2), 0.5 * np.exp(-t / 0.12) * (1 + 0.01 * np.random.default_rng(4).normal(size=12))]
    out["fit__t"] = t
    out["fit__y"] = np.array(series)
    out["fit__res"] = np.array([[f.rho, f.t2, f.residual_norm] for f in (rr.cpmg_fit(t, y) for y in series)])
    np.savez_compressed(os.path.join(HERE, "recon.npz"), **out)

    wire = os.path.join(HERE, "wire")
    os.makedirs(wire, exist_ok=True)
    rng = np.random.default_rng(5)
    echo = rng.normal(size=(3, 5)) + 1j * rng.normal(size=(3, 5))
    rio.write_echo_file(os.path.join(wire, "echo.mrsim"), echo,
                        {"written_at": "fixed", "sequence": "golden", "arr": np.arange(3), "n": np.int64(7)})
    snap = rng.normal(size=(4, 3))
    rio.write_snapshot_file(os.path.join(wire, "snap.mrsim"), 0.0125, snap)
    grid_c = rng.normal(size=(3, 4)) + 1j * rng.normal(size=(3, 4))
    grid_f = rng.normal(size=(2, 5))
    rio.write_raw_grid(os.path.join(wire, "grid_c128.raw"), grid_c)
    rio.write_raw_grid(os.path.join(wire, "grid_f64.raw"), grid_f)
    pgm_img = np.abs(rng.normal(size=(6, 7)))
    rio.write_pgm(os.path.join(wire, "auto.pgm"), pgm_img)
    rio.write_pgm(os.path.join(wire, "window.pgm"), pgm_img, window=(0.2, 1.1))
    rio.write_pgm(os.path.join(wire, "flat.pgm"), np.ones((2, 3)))
    np.savez(os.path.join(wire, "inputs.npz"), echo=echo, snap=snap, grid_c=grid_c, grid_f=grid_f, pgm_img=pgm_img)
    with open(os.path.join(wire, "README"), "w") as fh:
        fh.write("Written by mrsim.io via tests/golden/make_golden_recon.py; inputs in inputs.npz.\n")
    print(json.dumps({k: list(np.shape(v)) for k, v in out.items() if k.endswith("__img0")}))


if __name__ == "__main__":
    main()

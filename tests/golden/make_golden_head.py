"""Golden vectors for the ten-ellipse head phantom, made by the REFERENCE.

    python tests/golden/make_golden_head.py [--ref /root/reference/pkg/src]

Evaluates ``mrsim.phantom.shepp_logan_m0`` on a seeded point cloud and on a
grid that grazes the ellipse boundaries, and rasterises ``shepp_logan(0.255)``
at acceptance criterion 6's spacing (test_acceptance.py:341-354).  Writes
``tests/golden/head.npz``.  Build container only — the tests read the
committed file, never the reference.
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    from mrsim.phantom import rasterize, shepp_logan, shepp_logan_m0

    rng = np.random.default_rng(6)
    scale = 0.255
    pts = rng.uniform(-1.05 * scale, 1.05 * scale, (20000, 2))
    g = np.linspace(-scale, scale, 257)
    gx, gy = np.meshgrid(g, g)
    grid = np.stack([gx.ravel(), gy.ravel()], axis=1)
    allp = np.vstack([pts, grid])
    m0 = np.array([shepp_logan_m0(float(x), float(y), scale) for x, y in allp])
    fov, n = 0.5, 64
    spacing = (fov / n * 0.999, fov / n * 0.999, 1.0)
    spins = rasterize(shepp_logan(scale), spacing)
    pos = np.array([s.position for s in spins])
    sm0 = np.array([s.m.mz for s in spins])
    np.savez_compressed(os.path.join(HERE, "head.npz"), points=allp, m0=m0, scale=scale,
                        spacing=np.array(spacing), spin_pos=pos, spin_m0=sm0)
    print(f"head.npz: {len(allp)} points, {len(spins)} spins")


if __name__ == "__main__":
    main()

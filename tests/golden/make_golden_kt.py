"""Golden echoes from the reference's independent k-t engine (build container only).

    python tests/golden/make_golden_kt.py [--ref /root/reference/pkg/src]

Acceptance criterion 2 of the reference (tests/test_acceptance.py:127-184) checks the spin engine
against the configuration-population (k-t) engine, a different algorithm, on seeded random
sequences in a homogeneous field.  This script runs the reference's own pieces for that check —
rasterize (phantom.py:98-142) of an Affine-M0 box, lattice_spectrum and simulate_kt
(ktspace.py:301-369, 490-505) — on the criterion's seeded sequences and stores the sequence
parameters, the spins and the k-t echoes in ``tests/golden/kt_random.npz``.  The GPU test
rebuilds the same sequences and spins with this package and compares.
"""

from __future__ import annotations

import argparse
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    from mrsim import phantom as rp
    from mrsim.bloch import GAMMA_PROTON, HardPulse, RelaxationParams
    from mrsim.ktspace import lattice_spectrum, simulate_kt
    from mrsim.sequence import AcquisitionSpec, ElementarySequence, GradientWaveform, Sequence

    rng = np.random.default_rng(7041)
    unit, t1, t2 = 80.0, 0.5, 0.3
    box = rp.PhantomBox(origin=(-0.05, -5e-4, -5e-4), size=(0.1, 1e-3, 1e-3), m0=rp.Affine(1.0, gx=5.0),
                        t1=t1, t2=t2)
    spacing = (0.002, 0.01, 0.01)
    spins = rp.rasterize(rp.Phantom([box]), spacing)
    pos = np.array([s.position for s in spins])
    m0 = np.array([s.relax.m0 for s in spins])
    spectrum = lattice_spectrum([s.position for s in spins], [s.relax.m0 / len(spins) for s in spins])
    out = {"pos": pos, "m0": m0, "t1": np.float64(t1), "t2": np.float64(t2), "n_seq": np.int64(5)}
    for q_i in range(5):
        rows = []  # alpha, phi, q, dt per pulse element
        elements = []
        for _ in range(int(rng.integers(3, 7)) - 1):
            dt = rng.uniform(0.002, 0.02)
            q = int(rng.integers(-3, 4))
            alpha, phi = rng.uniform(0.1, math.pi), rng.uniform(0, 2 * math.pi)
            rows.append((alpha, phi, q, dt))
            elements.append(ElementarySequence(pulse=HardPulse(alpha, phi),
                                               gradient=GradientWaveform.constant(gx=q * unit / (GAMMA_PROTON * dt)),
                                               duration=dt))
        ro = 0.01
        elements.append(ElementarySequence(gradient=GradientWaveform.constant(gx=4 * unit / (GAMMA_PROTON * ro)),
                                           duration=ro, acquisition=AcquisitionSpec(True, 33), kspace_row=0))
        kt = simulate_kt(Sequence(elements, name="random"), RelaxationParams(t1, t2, 1.0), object_spectrum=spectrum)
        out[f"seq{q_i}_rows"] = np.array(rows, dtype=float)
        out[f"seq{q_i}_kt"] = np.concatenate(kt.echoes)
    np.savez_compressed(os.path.join(HERE, "kt_random.npz"), **out)
    print(f"{len(spins)} spins, 5 sequences -> kt_random.npz")


if __name__ == "__main__":
    main()

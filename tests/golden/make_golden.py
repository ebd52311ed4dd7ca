"""Generate golden vectors by running the REFERENCE itself (build container only).

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

Imports ``mrsim`` from the read-only reference checkout, converts every case
of ``tests/golden/cases.py`` to the reference's own objects, and records what
the reference computes:

* ``precompute_sequence_tables`` (engine.py:83-164) -> flattened tables
* ``rasterize`` (phantom.py:98-142) for phantom cases -> spin arrays
* ``compute_block`` (engine.py:259-310) -> echoes + snapshots (one reference
  pass per receive coil for multi-coil cases: the reference takes one weight
  per spin, engine.py:185)

The .npz files are committed; the tests never import the reference.  Large
config cases store the first/last acquisitions in full plus per-acquisition
checksums (sum and energy) to keep the fixtures small.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import cases  # noqa: E402
from paper_1305_6861_b200.engine import flatten_tables  # noqa: E402

FULL_ACQ_LIMIT = 4096  # store every acquisition when the k-space has at most this many samples x coils


def projection_vector(n):
    """Seeded complex projection: a per-acquisition checksum without cancellation bias."""
    rng = np.random.default_rng(12345)
    return rng.normal(size=n) + 1j * rng.normal(size=n)


def to_ref_sequence(seq, ref):
    els = []
    for es in seq.elements:
        p = None if es.pulse is None else ref.bloch.HardPulse(es.pulse.alpha, es.pulse.phi)
        g = es.gradient
        rg = ref.sequence.GradientWaveform(g.shape, g.gx, g.gy, g.gz, ramp_s=g.ramp_s, flat_s=g.flat_s,
                                           samples=g.samples, sample_dt=g.sample_dt)
        acq = ref.sequence.AcquisitionSpec(es.acquisition.enabled, es.acquisition.n_samples)
        els.append(ref.sequence.ElementarySequence(pulse=p, gradient=rg, duration=es.duration, acquisition=acq,
                                                   kspace_row=es.kspace_row, kspace_volume=es.kspace_volume,
                                                   kspace_reversed=es.kspace_reversed))
    return ref.sequence.Sequence(els, name=seq.name)


def to_ref_phantom(ph, ref):
    return ref.phantom.Phantom([ref.phantom.PhantomBox(origin=b.origin, size=b.size, m0=b.m0, t1=b.t1, t2=b.t2,
                                                       delta_omega=b.delta_omega) for b in ph.boxes])


def run_case(name, case, ref, out_dir):
    t0 = time.time()
    rseq = to_ref_sequence(case["sequence"], ref)
    tables = ref.engine.precompute_sequence_tables(rseq, snapshot_times=case["snapshot_times"])
    rec = {}
    if "phantom" in case:
        spins = ref.phantom.rasterize(to_ref_phantom(case["phantom"], ref), case["spacing"])
        arr = ref.engine.build_spin_arrays(spins, ref.system.default_system())
        sp = dict(pos=arr.pos, mx=arr.mx, my=arr.my, mz=arr.mz, t1=arr.t1, t2=arr.t2, m0=arr.m0,
                  domega=arr.domega, weight=arr.weight)
    else:
        sp = case["spins"]
    w = np.asarray(sp["weight"])
    weights = [w[c] for c in range(w.shape[0])] if w.ndim == 2 else [w]
    echoes, snaps = [], None
    for wc in weights:
        blk = ref.engine.SpinBlock(index=0, pos=np.asarray(sp["pos"], float), mx=np.asarray(sp["mx"], float),
                                   my=np.asarray(sp["my"], float), mz=np.asarray(sp["mz"], float),
                                   t1=np.asarray(sp["t1"], float), t2=np.asarray(sp["t2"], float),
                                   m0=np.asarray(sp["m0"], float), domega=np.asarray(sp["domega"], float),
                                   weight=np.asarray(wc, complex))
        e, s = ref.engine.compute_block(tables, blk)
        echoes.append(e)
        snaps = s
    echoes = np.stack(echoes) if w.ndim == 2 else echoes[0]
    flat = flatten_tables(tables)
    for k, v in flat.items():
        rec["tab_" + k] = np.asarray(v)
    for k, v in sp.items():
        rec["spin_" + k] = np.asarray(v)
    ek = echoes.reshape(-1, echoes.shape[-2], echoes.shape[-1]) if echoes.ndim == 3 else echoes[None]
    n_acq = ek.shape[1]
    rec["echo_shape"] = np.array(echoes.shape)
    rec["echo_sum"] = ek.sum(axis=-1)
    rec["echo_proj"] = ek @ projection_vector(ek.shape[-1])
    rec["echo_energy"] = (np.abs(ek) ** 2).sum(axis=-1)
    if ek.size <= FULL_ACQ_LIMIT * 4 or n_acq <= 8:
        rec["echo_full"] = echoes
    else:
        rec["echo_head"] = ek[:, :4]
        rec["echo_tail"] = ek[:, -4:]
    for i, s in enumerate(snaps):
        rec[f"snap_{i}"] = np.zeros((0, 3)) if s is None else s
        rec[f"snap_{i}_present"] = np.array(s is not None)
    rec["n_snap"] = np.array(len(snaps))
    rec["snapshot_times"] = np.array(case["snapshot_times"], dtype=float)
    rec["pulse_memo_hits"] = np.array(tables.pulse_memo_hits)
    np.savez_compressed(os.path.join(out_dir, f"{name}.npz"), **rec)
    print(f"{name:12s} n={len(sp['mx']):6d} echoes {echoes.shape} {time.time() - t0:.1f}s", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--only", nargs="*")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    import mrsim  # noqa: F401
    import mrsim.bloch
    import mrsim.engine
    import mrsim.phantom
    import mrsim.sequence
    import mrsim.system

    class Ref:
        bloch = mrsim.bloch
        engine = mrsim.engine
        phantom = mrsim.phantom
        sequence = mrsim.sequence
        system = mrsim.system

    all_cases = dict(cases.small_cases())
    for i in range(5):
        all_cases[f"cfg{i}"] = None
    for name, case in all_cases.items():
        if args.only and name not in args.only:
            continue
        if case is None:
            case = cases.config_case(int(name[3:]))
        run_case(name, case, Ref, HERE)


if __name__ == "__main__":
    main()

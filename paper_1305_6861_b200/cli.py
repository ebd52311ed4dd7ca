"""Command-line front end (mirrors ``mrsim.cli`` cli.py:44-237).

Subcommands keep the reference's names, output files and printed keys:

* ``simulate`` — runs a workload through the GPU engine and writes
  ``echoes.mrsim`` (+ ``.manifest.json``) and ``snapshot_NNN.mrsim`` into
  ``--out`` (cli.py:44-99).  The reference reads sequence/object/system
  description files; their text grammars are out of scope here,
  so the workload is one of the seeded benchmark configurations
  (``--config 0..4``, optionally thinned with ``--subset``).
* ``compare`` — ΔE_stör and exceedance count of two echo files (cli.py:102-110).
* ``recon`` — k-space assembly + centred iFFT on the GPU, PGM + raw grid
  output (cli.py:113-135).
* ``fit-t2`` — exponential fit of a two-column (t, I) series (cli.py:150-161).

Errors print ``error: ...`` to stderr and exit with status 2 (cli.py:227-233).
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

from . import io as mrio
from .errors import InvalidParameter, MrSimError


def _parse_times(text):
    return tuple(float(v) for v in text.split(",")) if text else ()


def _simulate_device_scene(args) -> int:
    """simulate with the spins rasterised on the GPU (objects.DeviceScene -> run(Experiment))."""
    from . import configs
    from .engine import Experiment, run

    if args.subset > 1:
        raise InvalidParameter("--device-raster rasterises the whole lattice (no --subset)")
    sw = configs.scene(args.config)
    if sw.extra_dw is not None:
        raise InvalidParameter(f"config {args.config} has a per-spin random off-resonance map; use the host path")
    res = run(Experiment(sequence=sw.sequence, phantom=sw.scene, spacing=sw.spacing, device=args.device,
                         precision=args.precision, snapshot_times=_parse_times(args.snapshot), spin_cap=sw.cap))
    echoes = res.echo_matrix()
    if echoes.ndim == 3:  # (n_acq, C, ns) -> coil-major
        echoes = np.moveaxis(echoes, 1, 0)
    else:
        echoes = echoes[None]
    os.makedirs(args.out, exist_ok=True)
    seq = sw.sequence
    manifest = {
        "sequence": seq.name, "workload": sw.name, "config": int(args.config), "rasterised_on": "device",
        "spin_count": int(res.spin_count), "spacing_m": list(res.spacing), "workers": 1, "blocks": 1,
        "deterministic": True, "precision": int(args.precision), "wall_time_s": res.metrics.wall_time_s,
        "throughput_spins_per_s": res.metrics.throughput, "busy_fraction": res.metrics.busy_fraction,
        "hardware": res.metrics.hardware, "kernel_ms": res.metrics.kernel_ms,
        "events_per_spin": res.metrics.events_per_spin, "n_coils": int(echoes.shape[0]),
        "acquisition_t0_s": [float(r.timestamps[0]) if r.timestamps.size else 0.0 for r in res.echoes],
        "sample_dt_s": [float(r.timestamps[1] - r.timestamps[0]) if r.timestamps.size > 1 else 0.0
                        for r in res.echoes],
        "trajectory": [list(t) for t in seq.trajectory_table()],
    }
    echo_path = os.path.join(args.out, "echoes.mrsim")
    if echoes.shape[0] > 1:
        manifest["coil_files"] = [f"echoes_coil{c:02d}.mrsim" for c in range(echoes.shape[0])]
        for c in range(echoes.shape[0]):
            mrio.write_echo_file(os.path.join(args.out, manifest["coil_files"][c]), echoes[c], manifest)
    mrio.write_echo_file(echo_path, echoes[0], manifest)
    for i, (t, arr) in enumerate(res.snapshots):
        mrio.write_snapshot_file(os.path.join(args.out, f"snapshot_{i:03d}.mrsim"), t, arr)
    print(f"simulated {res.spin_count} spins (rasterised on cuda), {len(res.echoes)} acquisitions -> {echo_path}")
    print(f"wall {res.metrics.wall_time_s:.3f} s, kernel {res.metrics.kernel_ms:.3f} ms")
    return 0


def _cmd_simulate(args) -> int:
    from . import configs
    from .engine import get_engine, precompute_sequence_tables

    if args.device_raster:
        return _simulate_device_scene(args)
    wl = configs.make(args.config)
    if args.subset > 1:
        wl = wl.subset(args.subset)
    b = wl.block
    seq = wl.sequence
    tables = precompute_sequence_tables(seq, snapshot_times=_parse_times(args.snapshot))
    wall0 = time.perf_counter()
    eng = get_engine(args.device, args.precision)
    t_k = time.perf_counter()
    echoes, snaps = eng.compute(tables, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)
    busy = time.perf_counter() - t_k
    wall = time.perf_counter() - wall0
    n = b.n
    timing = eng.last_timing()
    stats = eng.program_stats()
    echoes = echoes / n  # engine.py:507
    if echoes.ndim == 2:  # single receive weight: (n_acq, max_ns)
        echoes = echoes[None]
    n_coils = echoes.shape[0]
    ns = [t.size for t in tables.acq_times]
    os.makedirs(args.out, exist_ok=True)
    updates = float(n) * stats["events"]
    manifest = {
        "sequence": seq.name,
        "workload": wl.name,
        "config": int(args.config),
        "subset_stride": int(args.subset),
        "spin_count": int(n),
        "spacing_m": wl.meta.get("spacing"),
        "workers": 1,
        "blocks": 1,
        "deterministic": True,
        "precision": int(args.precision),
        "wall_time_s": wall,
        "throughput_spins_per_s": n / wall if wall > 0 else None,
        "busy_fraction": {"0": busy / wall if wall > 0 else None},
        "hardware": f"cuda:{eng.device} sm_100a",
        "kernel_ms": timing["kernel_ms"],
        "events_per_spin": stats["events"],
        "updates_per_s_kernel": updates / (timing["kernel_ms"] * 1e-3) if timing["kernel_ms"] > 0 else None,
        "n_coils": int(n_coils),
        "n_samples": ns,
        "acquisition_t0_s": [float(t[0]) if t.size else 0.0 for t in tables.acq_times],
        "sample_dt_s": [float(t[1] - t[0]) if t.size > 1 else 0.0 for t in tables.acq_times],
        "trajectory": [list(t) for t in seq.trajectory_table()],
    }
    echo_path = os.path.join(args.out, "echoes.mrsim")
    if n_coils > 1:
        manifest["coil_files"] = [f"echoes_coil{c:02d}.mrsim" for c in range(n_coils)]
        for c in range(n_coils):
            mrio.write_echo_file(os.path.join(args.out, manifest["coil_files"][c]), echoes[c], manifest)
    mrio.write_echo_file(echo_path, echoes[0], manifest)
    for i, t in enumerate(tables.snapshot_times):
        arr = snaps[i] if snaps is not None else np.zeros((0, 3))
        mrio.write_snapshot_file(os.path.join(args.out, f"snapshot_{i:03d}.mrsim"), t, arr)
    print(f"simulated {n} spins, {tables.n_acq} acquisitions -> {echo_path}")
    print(f"wall {wall:.3f} s, kernel {timing['kernel_ms']:.3f} ms, throughput {n / wall:.1f} spins/s "
          f"on cuda:{eng.device}")
    return 0


def _cmd_compare(args) -> int:
    from .engine import compare_results

    ref = mrio.read_echo_file(args.ref)
    test = mrio.read_echo_file(args.test)
    cmp = compare_results(ref, test, rel_threshold=args.rel_threshold)
    print(f"delta_e_stoer_db={cmp.delta_e_db!r}")
    print(f"exceedances={cmp.exceedances}")
    print(f"compared={cmp.compared}")
    print(f"rel_threshold={cmp.rel_threshold!r}")
    return 0


def _read_table(path):
    table = []
    with open(path, "r", encoding="utf-8") as fh:
        for line in fh:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            parts = line.replace(",", " ").split()
            if len(parts) != 3:
                raise InvalidParameter(f"trajectory line {line!r} needs volume row reversed")
            table.append((int(parts[0]), int(parts[1]), parts[2].lower() in ("1", "true")))
    return table


def _cmd_recon(args) -> int:
    from .recon import assemble_kspace, export_image, reconstruct, trajectory_table

    echoes = mrio.read_echo_file(args.echoes)
    if args.trajectory.startswith("table:"):
        table = _read_table(args.trajectory[len("table:"):])
    else:
        table = trajectory_table(args.trajectory, echoes.shape[0], turbo_factor=args.turbo_factor)
    mats = assemble_kspace(echoes, table, n_rows=args.size[1], fov=args.fov)
    base, ext = os.path.splitext(args.out)
    outputs = []
    for k in mats:
        img = reconstruct(k, device=args.device)
        path = args.out if len(mats) == 1 else f"{base}_vol{k.volume:03d}{ext}"
        export_image(img, path)
        outputs.append(path)
    print("\n".join(outputs))
    return 0


def _cmd_fit_t2(args) -> int:
    from .recon import cpmg_fit

    try:
        data = np.loadtxt(args.series, ndmin=2)
    except ValueError as exc:
        raise InvalidParameter(f"cannot read series {args.series}: {exc}") from exc
    if data.shape[1] != 2:
        raise InvalidParameter("series file needs two columns: t_s intensity")
    fit = cpmg_fit(data[:, 0], data[:, 1])
    print(f"rho={fit.rho!r}")
    print(f"t2_s={fit.t2!r}")
    print(f"residual_norm={fit.residual_norm!r}")
    print(f"iterations={fit.iterations}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_1305_6861_b200", description="B200 Bloch event-stream simulator")
    sub = p.add_subparsers(dest="command", required=True)

    sim = sub.add_parser("simulate", help="run a spin-level simulation on the GPU")
    sim.add_argument("--config", type=int, default=0, choices=range(5), help="seeded workload (BASELINE configs)")
    sim.add_argument("--subset", type=int, default=1, help="keep every N-th spin")
    sim.add_argument("--precision", type=int, default=32, choices=(32, 64))
    sim.add_argument("--device", type=int, default=None)
    sim.add_argument("--snapshot", default=None, metavar="T1,T2,...")
    sim.add_argument("--device-raster", action="store_true",
                     help="rasterise the config's phantom on the GPU (objects.DeviceScene) instead of on the host")
    sim.add_argument("--out", required=True)
    sim.set_defaults(func=_cmd_simulate)

    cmp = sub.add_parser("compare", help="compare two echo files")
    cmp.add_argument("--ref", required=True)
    cmp.add_argument("--test", required=True)
    cmp.add_argument("--rel-threshold", type=float, default=1e-6)
    cmp.set_defaults(func=_cmd_compare)

    rec = sub.add_parser("recon", help="assemble k-space and reconstruct")
    rec.add_argument("--echoes", required=True)
    rec.add_argument("--trajectory", required=True, help="se | epi | tse-seq | table:PATH")
    rec.add_argument("--size", type=int, nargs=2, required=True, metavar=("NX", "NY"))
    rec.add_argument("--fov", type=float, default=None)
    rec.add_argument("--turbo-factor", type=int, default=2)
    rec.add_argument("--device", default="cuda", help="torch device for the transform")
    rec.add_argument("--out", default="image.pgm")
    rec.set_defaults(func=_cmd_recon)

    fit = sub.add_parser("fit-t2", help="exponential fit of an intensity series")
    fit.add_argument("--series", required=True)
    fit.set_defaults(func=_cmd_fit_t2)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (MrSimError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())

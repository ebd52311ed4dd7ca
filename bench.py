#!/usr/bin/env python
"""bench.py — isochromat-event updates/s of the sm_100a Bloch engine (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--scaling strong|weak]
                    [--impl ours|reference] [--full-lattice]

One process per GPU.  ``--gpus N > 1`` without a torchrun environment re-launches
itself under ``python -m torch.distributed.run --nproc-per-node N`` (127.0.0.1);
under torchrun (WORLD_SIZE set) it must equal the world size.

A step is one pass of the hot path over the workload: every spin of config C
(default 2, "2D turbo spin echo" — the largest configuration by work, 1.98e11
isochromat-event updates) through the whole event stream, the reduction of the
ADC sums to the k-space and, for N > 1, the one NCCL reduce to rank 0.  The
default is STRONG scaling: the config's own spins are sharded over the ranks
with the reference's np.linspace bounds (partition_blocks, engine.py:229-251).

* ``value``: N_spins * E / T with inputs resident in HBM, T = device time of the
  K timed steps (CUDA events on the launching stream, L2 flushed between steps
  by writing 256 MiB, max over ranks).  E is the reference table size (pulses +
  events).
* ``e2e``: the same metric through the public host API (BlochEngine / Pipeline
  -> C-ABI bloch_compute_block, pinned host buffers): every step copies the
  spin arrays host->device and the k-space and final magnetisation
  device->host.  This is the headline against the reference arm.
* ``roofline``: the dominant kernel of the step.  With the window contraction
  (fp32 mode) a step is two kernels: the integrator (the spin state through
  the event stream; the long ADC windows only store their entry magnetisation
  U) and the contraction (every window group's samples as one bf16x3 product
  on tcgen05).  ``roofline`` is whichever of the two takes the larger share
  of the step (``roofline.kernel`` names it); both are always present as
  ``roofline_integrator`` and ``roofline_contraction``.  The integrator is
  charged against HBM (algorithmic bytes: staged spins, each class table once,
  U, final state; ``traffic`` = ncu DRAM bytes of this build,
  profiles/ncu_counters.json) with its issue-slot fraction — with the class
  tables resident in shared memory (resident_integrate_kernel) it is bound by
  instruction issue, not by memory; the contraction against the measured bf16
  tensor peak (MEASURED_PEAKS.json): 3 passes x 4 real MAC per complex term.
  Without the contraction (fp64 mode, or windows it does not take) the
  integrator's own tensor-core windows are charged against the measured
  mma.sync rate (512 MAC/clk/SM).  The SURVEY §8d FP32/MUFU model stays as
  ``model_frac`` (the reference's per-event arithmetic, which the closed
  forms do not execute, so it exceeds 1).
* ``per_config``: value / kernel ms / fracs of configs 0-4 (device-resident,
  same world and sharding) — the other configurations on the same box.
* ``strong_scaling_projection`` (N = 1): device time of the 1/2, 1/4, 1/8
  shards on this GPU, i.e. the per-rank work of a strong-scaled run.
* ``cpu_baseline`` / ``--impl reference``: the reference's compute_block on
  every host core — the unmodified reference from baseline/_ref through its own
  _run_pool when it is installed (single-coil configs), else the oracle port —
  on a bounded spin sample through the full event stream.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "isochromat-event updates/s"
L2_NOTE = "flushed between timed steps (256 MiB write)"
MMA_MAC_PER_CLK_SM = 512  # mma.sync m16n8k8 tf32, measured (profiles/r1_mma_microbench.txt)


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="N > 1: strong = the config's spins sharded over the ranks (default); weak = every rank "
                         "integrates a full config-sized spin set (world interleaved copies of the lattice)")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", type=int, default=32, choices=[32, 64])
    ap.add_argument("--full-lattice", action="store_true",
                    help="background tissue on every lattice site: all 1,048,576 sites of configs 1-4 emit a spin")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--no-projection", action="store_true")
    ap.add_argument("--cpu-spins-per-core", type=int, default=2048)
    ap.add_argument("--dry", action="store_true",
                    help="plumbing check without a GPU: gloo ranks, shards, one reduce, max-over-ranks timing")
    ap.add_argument("--quiet", action="store_true")
    return ap.parse_args(argv)


def log(msg, quiet=False):
    if not quiet:
        print(msg, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md "clocks" recipe)
# ---------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None
        self.marks = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        threading.Thread(target=self._read, daemon=True).start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append((time.perf_counter(), parts))

    def mark(self):
        self.marks.append(time.perf_counter())

    def stop(self):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        lo, hi = (self.marks[0], self.marks[-1]) if len(self.marks) >= 2 else (0, 1e30)
        inside = [p for t, p in self.samples if lo <= t <= hi] or [p for _, p in self.samples]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for p in inside for i in range(4) if p[3 + i].lower().startswith("active")})

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [v for v in (num(p[0]) for p in inside) if v is not None]
        mx = [v for v in (num(p[1]) for p in inside) if v is not None]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside)}


# ---------------------------------------------------------------------------
# workload description shared by both arms (identical `config` objects)
# ---------------------------------------------------------------------------


def make_workload(args):
    from paper_1305_6861_b200 import configs

    return configs.make(args.config, full_lattice=args.full_lattice)


def config_dict(w, world, E, counts, scaling, full_lattice):
    return {"workload": w.name, "config_index": w.index, "spins_total": w.n_spins, "events_per_spin": E,
            "coils": w.n_coils, "event_classes": counts, "full_lattice": bool(full_lattice),
            "sharding": ("single GPU" if world == 1 else
                         "strong: np.linspace spin shards of the config (partition_blocks, engine.py:229-251), one "
                         "NCCL reduce of the fp64 k-space" if scaling == "strong" else
                         "weak: every rank a full config-sized spin set (world interleaved lattice copies, "
                         "parallel.weak_copy), one NCCL reduce of the fp64 k-space"),
            "l2": L2_NOTE, "parallelism": f"spin-shards x{world}"}


# ---------------------------------------------------------------------------
# the CPU reference path (all host cores)
# ---------------------------------------------------------------------------


def _reference_engine():
    """The unmodified reference (baseline/_ref, installed by tools/install_reference.sh), or None."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "mrsim")):
        return None
    if path not in sys.path:
        sys.path.append(path)
    try:
        import mrsim.engine as ref_engine  # noqa: F401
    except Exception:
        return None
    return ref_engine


def cpu_sample(workload, E, spins_per_core, steps=1, warmup=0, quiet=False):
    """Time the reference's compute_block on a bounded spin sample with every host core."""
    cores = os.cpu_count() or 1
    n_sample = min(workload.n_spins, cores * spins_per_core)
    stride = max(1, workload.n_spins // n_sample)
    sub = workload.subset(stride).block
    idx = slice(0, n_sample)
    arrays = dict(pos=sub.pos[idx], mx=sub.mx[idx], my=sub.my[idx], mz=sub.mz[idx], t1=sub.t1[idx], t2=sub.t2[idx],
                  m0=sub.m0[idx], domega=sub.domega[idx], weight=np.asarray(sub.weight)[..., idx])
    n = int(arrays["mx"].size)
    ref = _reference_engine() if workload.n_coils == 1 else None
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(k, "1")
    if ref is not None:
        # the reference itself: its precompute, SpinBlock, partition_blocks and process pool (engine.py:540-595)
        from types import SimpleNamespace

        tables = ref.precompute_sequence_tables(workload.sequence)
        block = ref.SpinBlock(index=0, pos=np.ascontiguousarray(arrays["pos"]), mx=arrays["mx"].copy(),
                              my=arrays["my"].copy(), mz=arrays["mz"].copy(), t1=arrays["t1"].copy(),
                              t2=arrays["t2"].copy(), m0=arrays["m0"].copy(), domega=arrays["domega"].copy(),
                              weight=np.asarray(arrays["weight"], dtype=np.complex128).reshape(-1).copy())
        exp = SimpleNamespace(workers=cores, deterministic=True)

        def one():
            try:
                from threadpoolctl import threadpool_limits

                lim = threadpool_limits(1)
            except Exception:
                lim = None
            t0 = time.perf_counter()
            blocks = ref.partition_blocks(block, 4 * cores)
            ref._run_pool(exp, tables, blocks, {})
            wall = time.perf_counter() - t0
            if lim is not None:
                lim.restore_original_limits()
            return wall

        kind, what = "reference", (f"mrsim.engine._run_pool (baseline/_ref, unmodified) with {cores} workers, "
                                   f"4 blocks/worker, deterministic, 1 BLAS thread each")
    else:
        from oracle import cpu_pool
        from oracle.bloch_oracle import precompute_tables

        tables = precompute_tables(workload.sequence)

        def one():
            return cpu_pool.run_pool(tables, arrays, workers=cores)[2]

        kind, what = "port", (f"oracle/bloch_oracle.compute_block on a {cores}-process pool (engine._run_pool "
                              f"restated, 4 blocks/worker, 1 BLAS thread each)")
    walls = []
    for i in range(warmup + steps):
        wall = one()
        log(f"[cpu] step {i}: {n} spins x {E} events in {wall:.2f}s ({kind})", quiet)
        if i >= warmup:
            walls.append(wall)
    mean = sum(walls) / len(walls)
    return {"value": n * E / mean, "unit": METRIC, "cores": cores, "kind": kind,
            "sample": f"{n} spins (every {stride}th in rasterisation order) x {E} events of config {workload.index}, "
                      f"{what}, mean of {len(walls)}",
            "seconds_per_step": mean}


def reference_arm(args):
    from paper_1305_6861_b200.engine import event_counts, precompute_sequence_tables

    w = make_workload(args)
    counts = event_counts(precompute_sequence_tables(w.sequence))
    E = counts["events"]
    cb = cpu_sample(w, E, args.cpu_spins_per_core, steps=args.steps, warmup=args.warmup, quiet=args.quiet)
    line = {
        "metric": METRIC, "value": cb["value"], "unit": METRIC, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["seconds_per_step"] * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json config recipe)",
        "config": config_dict(w, args.gpus, E, counts, args.scaling, args.full_lattice),
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# one process per GPU: spawn / plumbing check
# ---------------------------------------------------------------------------


def _free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn(args_argv, n):
    """Re-launch this script with n ranks under torch.distributed.run; rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__), *args_argv]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def dry_run(args, world, rank):
    """The multi-rank plumbing without a GPU: shards, one gloo reduce, max-over-ranks time, the JSON line."""
    import torch
    import torch.distributed as dist

    from paper_1305_6861_b200 import configs
    from paper_1305_6861_b200.engine import event_counts, precompute_sequence_tables
    from paper_1305_6861_b200.parallel import reduce_kspace, shard_block

    if world > 1:
        dist.init_process_group("gloo")
    w = configs.make(args.config, full_lattice=args.full_lattice)
    counts = event_counts(precompute_sequence_tables(w.sequence))
    E = counts["events"]
    shard = shard_block(w.block, world, rank) if args.scaling == "strong" else w.block
    k = torch.zeros(4, dtype=torch.float64)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        k.fill_(float(shard.n))
        reduce_kspace(k, dst=0)
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    n_total = w.n_spins if args.scaling == "strong" else world * w.n_spins
    if rank == 0:
        assert args.scaling != "strong" or int(k[0].item()) == w.n_spins, "shards do not cover the config"
        print(json.dumps({"metric": METRIC, "value": n_total * E * args.steps / max(t.item(), 1e-9), "unit": METRIC,
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "dry": True,
                          "scaling": args.scaling, "spins_reduced": int(k[0].item()),
                          "config": config_dict(w, world, E, counts, args.scaling, args.full_lattice)}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# GPU measurement
# ---------------------------------------------------------------------------


def _peaks():
    f_max, hbm, bf16 = 1965.0, None, None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            mp = json.load(fh)
        f_max = float(mp.get("sm_max_mhz", f_max))
        hbm = float(mp.get("hbm_gbs")) if mp.get("hbm_gbs") else None
        bf16 = float(mp.get("bf16_tflops")) if mp.get("bf16_tflops") else None
    except Exception:
        pass
    # B200_PROFILING.md fallbacks when the driver-written file is absent
    return f_max, hbm or 6500.0, bf16 or 1650.0


def _lib_sha():
    """Identity of the kernel build the counters in profiles/ncu_counters.json must match: the hash of the
    kernel sources (nvcc output is not bit-reproducible), or of the file for an explicit BLOCH_LIB."""
    import hashlib

    path = os.environ.get("BLOCH_LIB")
    try:
        if path:
            with open(path, "rb") as fh:
                return hashlib.sha256(fh.read()).hexdigest()[:16]
        from paper_1305_6861_b200.build import source_hash

        return source_hash()
    except OSError:
        return None


def _ncu_counters(config_index, lib_sha, kernel=""):
    """Per-launch ncu counters of the integrator (kernel="") or the contraction (kernel="_contract") for this
    build (profiles/ncu_counters.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_counters.json")) as fh:
            d = json.load(fh)
    except Exception:
        return None
    rec = d.get(f"config{config_index}{kernel}")
    if not rec or (lib_sha and rec.get("lib_sha16") not in (None, lib_sha)):
        return None
    return rec


def roofline(counts, pstats, n_local, C, t_kernel_s, n_sm, f_max_mhz, config_index, lib_sha, precision, hbm_peak,
             t_integ_s=None, t_contract_s=None, bf16_peak=None, resident=False):
    """Floors of the step's kernels: the integrator against HBM (algorithmic bytes) and its issue slots (ncu
    counters of this build), the window contraction against the measured bf16 tensor peak, the §8d model."""
    f = f_max_mhz * 1e6
    contracted = pstats.get("contracted_samples", 0) if (t_contract_s or 0) > 0 else 0
    t_integ = t_integ_s if t_integ_s else t_kernel_s
    w_fp32 = n_local * (9 * counts["rot"] + 12 * counts["prec_relax"] + 9 * counts["prec"] + 4 * C * counts["adc"])
    w_mufu = n_local * 2 * (counts["prec_relax"] + counts["prec"])
    t_model = max(w_fp32 / (n_sm * 128 * f), w_mufu / (n_sm * 16 * f))
    rec = _ncu_counters(config_index, lib_sha)
    t_issue = rec["inst_executed"] / (n_sm * 4 * f) if rec and rec.get("inst_executed") else None
    traffic = (rec.get("dram_read") or 0) + (rec.get("dram_write") or 0) if rec else None
    # integrator algorithmic bytes: SpinConst (64 B) + initial state (24 B) + every plane once (16 B) + the U words of
    # the contracted windows (8 B per window) + final state (24 B) per spin
    n_windows = pstats.get("window_ops", 0) if contracted else 0
    alg = n_local * (64 + 24 + 16 * pstats.get("planes", 0) + 8 * n_windows + 24)
    # the integrator's own tensor-core windows (no contraction): 8 tf32-rate MAC per spin-sample-coil on mma.sync
    w_mma = n_local * pstats["window_samples"] * C * 8 if (precision == 32 and not contracted) else 0
    t_tensor = w_mma / (n_sm * MMA_MAC_PER_CLK_SM * f)
    out = {
        "kernel": "resident_integrate_kernel" if resident else "integrate_kernel",
        "bound": "hbm",
        "achieved": alg / t_integ / 1e9,
        "peak": hbm_peak,
        "unit": "GB/s",
        "frac": (alg / t_integ / 1e9 / hbm_peak) if hbm_peak else None,
        "traffic": traffic,
        "algorithmic_bytes": alg,
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)",
        "traffic_source": (f"ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, profiles/ncu_counters.json "
                           f"({rec.get('source', '')})") if traffic else "no ncu counters for this build/config",
        "issue_frac": t_issue / t_integ if t_issue else None,
        "tensor_frac": t_tensor / t_integ if w_mma else None,
        "tensor_note": (f"mma.sync tf32 m16n8k8, {MMA_MAC_PER_CLK_SM} MAC/clk/SM measured x {n_sm} SM x "
                        f"{f_max_mhz:.0f} MHz; 8 tf32-rate MAC per spin-sample-coil") if w_mma else None,
        "model_frac": t_model / t_kernel_s,
        "model": "SURVEY §8d: T* = max(W_fp32 / (SM 128 f), W_mufu / (SM 16 f)), W_fp32 = N(9 rot + 12 prec_relax + "
                 "9 prec + 4C adc), W_mufu = 2N(prec_relax + prec) — the reference's per-event arithmetic; the "
                 "engine's closed forms do less, so model_frac > 1",
        "kernel_ms": t_integ * 1e3,
        "step_kernel_ms": t_kernel_s * 1e3,
        "issue_floor_ms": t_issue * 1e3 if t_issue else None,
        "model_ms": t_model * 1e3,
    }
    contraction = None
    if contracted and t_contract_s:
        macs = 3 * 4 * n_local * contracted * C  # bf16 hi*hi + hi*lo + lo*hi, 4 real MAC per complex term
        crec = _ncu_counters(config_index, lib_sha, "_contract")
        contraction = {
            "traffic": ((crec.get("dram_read") or 0) + (crec.get("dram_write") or 0)) if crec else None,
            "hmma_active_pct": crec.get("hmma_active_pct") if crec else None,
            "kernel": "contract_kernel (+ prep, fold)",
            "bound": "tensor",
            "achieved": 2 * macs / t_contract_s / 1e12,
            "peak": bf16_peak,
            "unit": "TFLOP/s",
            "frac": (2 * macs / t_contract_s / 1e12 / bf16_peak) if bf16_peak else None,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (cuBLAS bf16 8192^3, burst)",
            "work": "3 bf16 passes x 4 real MAC per (spin, contracted sample, coil)",
            "kernel_ms": t_contract_s * 1e3,
        }
    return out, contraction


class Runner:
    """One engine + stream on this rank; device-resident steps of a (sharded) workload."""

    def __init__(self, local_rank, precision, world, rank, scaling):
        import torch

        from paper_1305_6861_b200.engine import get_engine

        self.torch = torch
        self.dev = torch.device("cuda", local_rank)
        self.stream = torch.cuda.Stream(self.dev)
        torch.cuda.set_stream(self.stream)
        self.eng = get_engine(local_rank, precision)
        self.eng.set_stream(self.stream.cuda_stream)
        self.world, self.rank, self.scaling = world, rank, scaling
        self.flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=self.dev)  # 256 MiB > 126 MB L2

    def shard(self, w):
        from paper_1305_6861_b200.parallel import lattice_spacing, shard_block, weak_copy

        if self.world == 1:
            return w.block, w.n_spins
        if self.scaling == "weak":
            return weak_copy(w.block, self.world, self.rank, lattice_spacing(w.block.pos)), self.world * w.n_spins
        return shard_block(w.block, self.world, self.rank), w.n_spins

    def prepare(self, w, shard):
        from paper_1305_6861_b200.engine import _unit_weight, precompute_sequence_tables

        torch = self.torch
        C, n = w.n_coils, shard.n
        seq = w.sequence
        tables = precompute_sequence_tables(seq, snapshot_times=(seq.end_time,))  # final M is part of the output

        def dev64(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.dev)

        wt = np.ascontiguousarray(np.asarray(shard.weight, dtype=np.complex128).reshape(C, n)).view(np.float64)
        d = {"pos": dev64(shard.pos), "mx": dev64(shard.mx), "my": dev64(shard.my), "mz": dev64(shard.mz),
             "t1": dev64(shard.t1), "t2": dev64(shard.t2), "m0": dev64(shard.m0), "domega": dev64(shard.domega),
             "weight": dev64(wt)}
        ptrs = {k: v.data_ptr() for k, v in d.items()}
        unit_w = C == 1 and _unit_weight(wt.view(np.complex128))
        if unit_w:  # the uniform 1+0j receive weight travels as NULL, as BlochEngine.compute sends it
            ptrs["weight"] = 0
        f = self.eng.set_tables(tables)
        echo = torch.zeros(C * f["n_acq"] * f["max_ns"] * 2, dtype=torch.float64, device=self.dev)
        snap = torch.empty(max(1, n) * 3, dtype=torch.float64, device=self.dev)
        return dict(tables=tables, d=d, ptrs=ptrs, echo=echo, snap=snap, n=n, C=C, wt=wt, unit_w=unit_w, f=f)

    def timed(self, p, steps, warmup, clocks=None):
        """K device-resident steps (compute + reduce), L2 flushed before each; per-step device time."""
        import torch.distributed as dist

        from paper_1305_6861_b200.parallel import reduce_kspace

        torch = self.torch

        def step():
            self.eng.compute_device(p["tables"], p["ptrs"], p["n"], p["C"], p["echo"].data_ptr(),
                                    p["snap"].data_ptr())
            if self.world > 1:
                reduce_kspace(p["echo"], dst=0)

        for _ in range(warmup):
            self.flush.fill_(1.0)
            step()
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()
        if clocks is not None:
            clocks.start()
            time.sleep(0.3)
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()
        if clocks is not None:
            clocks.mark()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        kernel_ms, launches, integ_ms, contract_ms = [], 0, [], []
        for k in range(steps):
            self.flush.fill_(float(k))  # untimed: evict the L2 between steps
            ev[k][0].record(self.stream)
            step()
            ev[k][1].record(self.stream)
            t = self.eng.last_timing()  # waits for this step's work
            ph = self.eng.last_phases()
            kernel_ms.append(t["kernel_ms"])
            integ_ms.append(ph["integrate_ms"])
            contract_ms.append(ph["contract_ms"])
            launches += t["launches"]
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()
        if clocks is not None:
            clocks.mark()
            clocks.stop()
        step_ms = [a.elapsed_time(b) for a, b in ev]
        tot = torch.tensor([sum(step_ms), sum(kernel_ms), sum(integ_ms), sum(contract_ms)], dtype=torch.float64,
                           device=self.dev)
        if self.world > 1:
            dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        self.last_phase_s = (tot[2].item() / 1e3, tot[3].item() / 1e3)
        return tot[0].item() / 1e3, tot[1].item() / 1e3, launches


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    args = parse_args(argv)
    env_world = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return 0
        return reference_arm(args)
    if env_world is None and args.gpus > 1:
        return spawn(argv, args.gpus)
    world = int(env_world or "1")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.dry:
        return dry_run(args, world, rank)

    import torch
    import torch.distributed as dist

    from paper_1305_6861_b200 import configs
    from paper_1305_6861_b200.engine import event_counts, precompute_sequence_tables

    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    run = Runner(local_rank, args.precision, world, rank, args.scaling)
    dev = run.dev
    f_max, hbm_peak, bf16_peak = _peaks()
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    lib_sha = _lib_sha()

    t_setup = time.perf_counter()
    w = make_workload(args)
    counts = event_counts(precompute_sequence_tables(w.sequence))
    E = counts["events"]
    shard, n_total = run.shard(w)
    p = run.prepare(w, shard)
    pstats = run.eng.program_stats()
    n_local, C = p["n"], p["C"]
    log(f"[rank {rank}] config {w.index} {w.name}: {n_total} spins ({n_local} local, {args.scaling}) x {E} events, "
        f"setup {time.perf_counter() - t_setup:.1f}s", args.quiet)

    clocks = ClockSampler(local_rank)
    t_total_s, t_kernel_s, launches = run.timed(p, args.steps, args.warmup, clocks)
    t_integ, t_contract = (x / args.steps for x in run.last_phase_s)
    value = n_total * E * args.steps / t_total_s
    launch_shape = run.eng.last_launch()
    launch_shape.update(run.eng.last_resident())
    t_kernel = t_kernel_s / args.steps

    # ---- end to end through the public host API (pinned host buffers) ------------------
    from paper_1305_6861_b200.parallel import reduce_kspace

    e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).pin_memory().numpy()
    h = {k: pin(getattr(shard, k)) for k in ("pos", "mx", "my", "mz", "t1", "t2", "m0", "domega")}
    hw = torch.from_numpy(p["wt"].copy()).pin_memory().numpy().view(np.complex128).reshape(C, n_local)
    if C == 1:
        hw = hw[0]
    f = p["f"]
    n_acq, max_ns = f["n_acq"], f["max_ns"]
    tables = p["tables"]
    red = torch.zeros(C * n_acq * max_ns * 2, dtype=torch.float64, device=dev)
    if world == 1:
        # one GPU: the engine's double-buffered Pipeline (two contexts, own streams and device buffers),
        # so step k+1's uploads and step k's downloads overlap the kernels; every step still moves its
        # own inputs host->device and its k-space + final M device->host inside the timed region
        from paper_1305_6861_b200.engine import Pipeline

        pipe = Pipeline(local_rank, args.precision, depth=2)
        slots = []
        for _ in range(2):
            oe = torch.zeros(C * n_acq * max_ns * 2, dtype=torch.float64).pin_memory().numpy()
            os_ = torch.zeros(n_local * 3, dtype=torch.float64).pin_memory().numpy().reshape(1, n_local, 3)
            slots.append((oe.view(np.complex128).reshape(C, n_acq, max_ns), os_))

        def e2e_run(n_steps):
            for k in range(n_steps):
                oe, os_ = slots[k % 2]
                pipe.submit(tables, h["pos"], h["mx"], h["my"], h["mz"], h["t1"], h["t2"], h["m0"], h["domega"], hw,
                            out_echoes=oe, out_snaps=os_)
            pipe.drain()

        e2e_run(2)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_run(e2e_steps)
        torch.cuda.synchronize()
        out_e, out_s = slots[0]
        e2e_path = "Pipeline (2 engine contexts) -> bloch_compute_block, pinned host buffers, uploads/downloads overlapped"
    else:
        out_e = torch.zeros(C * n_acq * max_ns * 2, dtype=torch.float64).pin_memory().numpy().view(np.complex128)
        out_e = out_e.reshape(C, n_acq, max_ns)
        out_s = torch.zeros(n_local * 3, dtype=torch.float64).pin_memory().numpy().reshape(1, n_local, 3)

        def e2e_step():
            run.eng.compute(tables, h["pos"], h["mx"], h["my"], h["mz"], h["t1"], h["t2"], h["m0"], h["domega"], hw,
                            out_echoes=out_e, out_snaps=out_s)
            red.copy_(torch.from_numpy(out_e.view(np.float64).reshape(-1)), non_blocking=False)
            reduce_kspace(red, dst=0)
            torch.cuda.synchronize()

        e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_path = "BlochEngine.compute -> bloch_compute_block (pinned host buffers) + NCCL reduce per step"
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = n_total * E * e2e_steps / e2e_s.item()
    h2d = sum(a.nbytes for a in h.values()) + (0 if p["unit_w"] else p["wt"].nbytes)
    d2h = out_e.nbytes + out_s.nbytes

    roof, roof_c = roofline(counts, pstats, n_local, C, t_kernel, n_sm, f_max, w.index, lib_sha, args.precision,
                            hbm_peak, t_integ, t_contract, bf16_peak, resident=bool(launch_shape.get("resident")))
    # the dominant kernel of the step carries the headline roofline
    dominant = roof_c if (roof_c and t_contract > t_integ) else roof
    line = {
        "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_total_s * 1e3 / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None,
        "dtype": ("f64 spin state/phase; ADC sums: bf16x3-split products with f32 accumulation on tcgen05 "
                  "(window contraction), f64 fold" if args.precision == 32 else "f64"),
        "data": "synthetic (seeded, BASELINE.json config recipe)",
        "config": config_dict(w, world, E, counts, args.scaling, args.full_lattice),
        "spins_per_rank": n_local,
        "program": pstats,
        "roofline": dict(dominant, share_of_step=(max(t_contract, t_integ) / t_kernel) if t_kernel else None),
        "roofline_integrator": roof,
        "roofline_contraction": roof_c,
        "phases_ms": {"integrate": t_integ * 1e3, "contract": t_contract * 1e3},
        "integrator_launch": launch_shape,
        "e2e": {"value": e2e_value, "unit": METRIC, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "steps": e2e_steps, "path": e2e_path},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "kernel_ms_per_step": t_kernel * 1e3,
        "lib_sha16": lib_sha,
    }
    del p
    if world == 1:
        pipe.close()

    # ---- the other configurations, same world and sharding --------------------------------
    if not args.no_per_config:
        per = {}
        for c in range(configs.N_CONFIGS):
            wc = w if c == args.config else configs.make(c, full_lattice=args.full_lattice)
            cc = event_counts(precompute_sequence_tables(wc.sequence))
            sh, nt = run.shard(wc)
            pc = run.prepare(wc, sh)
            ps = run.eng.program_stats()
            st = max(3, min(args.steps, 10))
            tt, tk, _ = run.timed(pc, st, 2)
            ti, tc = (x / st for x in run.last_phase_s)
            rc, rcc = roofline(cc, ps, pc["n"], pc["C"], tk / st, n_sm, f_max, c, lib_sha, args.precision, hbm_peak,
                               ti, tc, bf16_peak, resident=bool(run.eng.last_resident()["resident"]))
            per[f"config{c}"] = {"workload": wc.name, "spins_total": nt, "events_per_spin": cc["events"],
                                 "value": nt * cc["events"] * st / tt, "ms_per_step": tt * 1e3 / st,
                                 "kernel_ms": tk * 1e3 / st, "integrate_ms": ti * 1e3, "contract_ms": tc * 1e3,
                                 "frac": rc["frac"], "issue_frac": rc["issue_frac"],
                                 "contraction_frac": rcc["frac"] if rcc else None, "model_frac": rc["model_frac"],
                                 "spins_per_thread": run.eng.last_launch()["spins_per_thread"],
                                 "resident": run.eng.last_resident()["resident"]}
            del pc
        line["per_config"] = per

    # ---- strong scaling: the per-rank work of N = 2, 4, 8 on this GPU -----------------------
    if world == 1 and not args.no_projection:
        from paper_1305_6861_b200.parallel import shard_block

        proj = {}
        t1 = t_total_s / args.steps
        for nr in (2, 4, 8):
            sh = shard_block(w.block, nr, 0)  # the largest shard (np.linspace bounds)
            pc = run.prepare(w, sh)
            st = max(3, min(args.steps, 10))
            tt, tk, _ = run.timed(pc, st, 2)
            proj[str(nr)] = {"shard_spins": sh.n, "ms_per_step": tt * 1e3 / st, "kernel_ms": tk * 1e3 / st,
                             "efficiency_est": t1 / (nr * tt / st), "spins_per_thread":
                             run.eng.last_launch()["spins_per_thread"],
                             "integrate_ms": run.last_phase_s[0] * 1e3 / st, "contract_ms": run.last_phase_s[1] * 1e3 / st}
            del pc
        line["strong_scaling_projection"] = {
            "note": "one B200: device time of rank 0's np.linspace shard (the largest) per step vs this line's "
                    "ms_per_step; excludes the NCCL reduce of the fp64 k-space (config 2: 4 MiB)",
            **proj}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_sample(w, E, args.cpu_spins_per_core, quiet=args.quiet)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

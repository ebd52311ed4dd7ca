#!/usr/bin/env python
"""bench.py — isochromat-event updates/s of the sm_100a Bloch engine (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU, NCCL)

A step is one pass of the hot path over the workload: every spin of config C
(default 1 — "2D spin echo at scale", the configuration BASELINE.json's metric
is quoted on) through the whole event stream, plus the fp64 fold of the
partial k-space (and, for N > 1, the one NCCL reduce to rank 0).

* ``value``: N_spins * E / T with inputs resident in HBM, T = device time of
  the K timed steps (CUDA events on the launching stream, L2 flushed between
  steps by writing 256 MiB, max over ranks).  E is the reference table size
  (pulses + events).
* ``e2e``: the same metric through the public host API
  (``BlochEngine.compute`` -> C-ABI ``bloch_compute_block`` with pinned host
  buffers): every step copies the spin arrays host->device and the k-space and
  final magnetisation device->host.  This is the headline against the
  reference arm.
* ``roofline``: FP32/MUFU model of SURVEY §8d (the path is not a dense
  contraction): achieved = model ops / integrator-kernel time, peak = SMs x
  128 FP32 lanes x f_max; ``frac`` = roofline time / measured kernel time.
* ``cpu_baseline``: the oracle port of the reference's ``compute_block`` on
  every host core (rank 0, N = 1), a bounded spin sample through the full
  event stream.
* ``--impl reference``: that CPU path alone, as the reference arm.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="N > 1: weak = every rank integrates a full config-sized spin set (world interleaved "
                         "copies of the lattice, parallel.weak_copy); strong = the config's spins sharded")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", type=int, default=32, choices=[32, 64])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-spins-per-core", type=int, default=2048)
    ap.add_argument("--quiet", action="store_true")
    return ap.parse_args()


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
# the CPU reference path (oracle port of compute_block, all host cores)
# ---------------------------------------------------------------------------


def cpu_sample(workload, tables, E, spins_per_core, steps=1, warmup=0, quiet=False):
    """Time the oracle port of the reference's compute_block on a spin sample (bounded CPU work)."""
    from oracle import cpu_pool

    cores = os.cpu_count() or 1
    n_sample = min(workload.n_spins, cores * spins_per_core)
    stride = max(1, workload.n_spins // n_sample)
    sub = workload.subset(stride).block
    idx = slice(0, n_sample)
    arrays = dict(pos=sub.pos[idx], mx=sub.mx[idx], my=sub.my[idx], mz=sub.mz[idx], t1=sub.t1[idx], t2=sub.t2[idx],
                  m0=sub.m0[idx], domega=sub.domega[idx], weight=np.asarray(sub.weight)[..., idx])
    n = int(arrays["mx"].size)
    walls = []
    for i in range(warmup + steps):
        _, _, wall = cpu_pool.run_pool(tables, arrays, workers=cores)
        log(f"[cpu] step {i}: {n} spins x {E} events in {wall:.2f}s", quiet)
        if i >= warmup:
            walls.append(wall)
    mean = sum(walls) / len(walls)
    return {
        "value": n * E / mean,
        "unit": "isochromat-event updates/s",
        "cores": cores,
        "kind": "port",
        "sample": f"{n} spins (every {stride}th in rasterisation order) x {E} events of config "
                  f"{workload.index}, oracle/bloch_oracle.compute_block on a {cores}-process pool "
                  f"(engine._run_pool restated, 4 blocks/worker, 1 BLAS thread each), mean of {len(walls)}",
        "seconds_per_step": mean,
    }


# ---------------------------------------------------------------------------


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    from paper_1305_6861_b200 import configs
    from paper_1305_6861_b200.engine import event_counts, precompute_sequence_tables

    metric = "isochromat-event updates/s"

    if args.impl == "reference":
        if rank != 0:
            return 0
        w = configs.make(args.config)
        tables = precompute_sequence_tables(w.sequence)
        E = event_counts(tables)["events"]
        cb = cpu_sample(w, tables, E, args.cpu_spins_per_core, steps=args.steps,
                        warmup=args.warmup, quiet=args.quiet)
        line = {
            "metric": metric, "value": cb["value"], "unit": cb["unit"], "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["seconds_per_step"] * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE.json config recipe)",
            "config": {"workload": w.name, "config_index": w.index, "spins_total": w.n_spins, "events_per_spin": E,
                       "coils": w.n_coils},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist

    from paper_1305_6861_b200.engine import _unit_weight, get_engine
    from paper_1305_6861_b200.parallel import lattice_spacing, reduce_kspace, shard_block, weak_copy

    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # one explicit stream shared by torch (flush, events, NCCL ordering) and the library
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    t_setup = time.perf_counter()
    w = configs.make(args.config)
    seq = w.sequence
    tables_plain = precompute_sequence_tables(seq)
    counts = event_counts(tables_plain)
    E = counts["events"]
    tables = precompute_sequence_tables(seq, snapshot_times=(seq.end_time,))  # final M is part of the output
    weak = args.scaling == "weak"
    if weak:
        shard = weak_copy(w.block, world, rank, lattice_spacing(w.block.pos)) if world > 1 else w.block
    else:
        shard = shard_block(w.block, world, rank)
    n_local, C = shard.n, w.n_coils
    n_total = world * n_local if weak else w.n_spins
    log(f"[rank {rank}] config {w.index} {w.name}: {n_total} spins ({n_local} local, {args.scaling}) x {E} events, "
        f"setup {time.perf_counter() - t_setup:.1f}s", args.quiet)

    eng = get_engine(local_rank, args.precision)
    eng.set_stream(stream.cuda_stream)
    eng.set_tables(tables)
    pstats = eng.program_stats()

    def dev64(a):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)

    wt = np.ascontiguousarray(np.asarray(shard.weight, dtype=np.complex128).reshape(C, n_local)).view(np.float64)
    d = {"pos": dev64(shard.pos), "mx": dev64(shard.mx), "my": dev64(shard.my), "mz": dev64(shard.mz),
         "t1": dev64(shard.t1), "t2": dev64(shard.t2), "m0": dev64(shard.m0), "domega": dev64(shard.domega),
         "weight": dev64(wt)}
    ptrs = {k: v.data_ptr() for k, v in d.items()}
    unit_w = C == 1 and _unit_weight(wt.view(np.complex128))
    if unit_w:  # the uniform 1+0j receive weight travels as NULL, as BlochEngine.compute sends it
        ptrs["weight"] = 0
    n_acq = tables.n_acq
    max_ns = max(e.n_samples for e in tables.entries)
    echo = torch.zeros(C * n_acq * max_ns * 2, dtype=torch.float64, device=dev)
    snap = torch.empty(max(1, n_local) * 3, dtype=torch.float64, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2

    def step():
        eng.compute_device(tables, ptrs, n_local, C, echo.data_ptr(), snap.data_ptr())
        if world > 1:
            reduce_kspace(echo, dst=0)

    for _ in range(args.warmup):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks.mark()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kernel_ms, launches = [], 0
    for k in range(args.steps):
        flush.fill_(float(k))  # untimed: evict the L2 between steps
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
        t = eng.last_timing()  # waits for this step's work
        kernel_ms.append(t["kernel_ms"])
        launches += t["launches"]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks.mark()
    clocks.stop()
    launch_shape = eng.last_launch()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = torch.tensor([sum(step_ms), sum(kernel_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    t_total_s, t_kernel_s = total_ms[0].item() / 1e3, total_ms[1].item() / 1e3
    value = n_total * E * args.steps / t_total_s

    # ---- end to end through the public host API (pinned host buffers) ------------------
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).pin_memory().numpy()
    h = {"pos": pin(shard.pos), "mx": pin(shard.mx), "my": pin(shard.my), "mz": pin(shard.mz), "t1": pin(shard.t1),
         "t2": pin(shard.t2), "m0": pin(shard.m0), "domega": pin(shard.domega)}
    hw = torch.from_numpy(wt.copy()).pin_memory().numpy().view(np.complex128).reshape(C, n_local)
    if C == 1:
        hw = hw[0]
    out_e = torch.zeros(C * n_acq * max_ns * 2, dtype=torch.float64).pin_memory().numpy().view(np.complex128)
    out_e = out_e.reshape(C, n_acq, max_ns)
    out_s = torch.zeros(1 * n_local * 3, dtype=torch.float64).pin_memory().numpy().reshape(1, n_local, 3)
    red = torch.zeros(C * n_acq * max_ns * 2, dtype=torch.float64, device=dev)

    def e2e_step():
        e, s = eng.compute(tables, h["pos"], h["mx"], h["my"], h["mz"], h["t1"], h["t2"], h["m0"], h["domega"], hw,
                           out_echoes=out_e, out_snaps=out_s)
        if world > 1:
            red.copy_(torch.from_numpy(out_e.view(np.float64).reshape(-1)), non_blocking=False)
            reduce_kspace(red, dst=0)
            torch.cuda.synchronize()
        return e, s

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
        e2e_path = "Pipeline (2 engine contexts) -> bloch_compute_block, pinned host buffers, uploads/downloads overlapped"
    else:
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
    h2d = sum(a.nbytes for a in h.values()) + (0 if unit_w else wt.nbytes)
    d2h = out_e.nbytes + out_s.nbytes

    # ---- roofline (FP32 / MUFU model) --------------------------------------
    props = torch.cuda.get_device_properties(dev)
    n_sm = props.multi_processor_count
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    f_max = 1965.0
    try:
        with open(peaks_path) as fh:
            f_max = float(json.load(fh).get("sm_max_mhz", f_max))
    except Exception:
        pass
    w_fp32 = n_local * (9 * counts["rot"] + 12 * counts["prec_relax"] + 9 * counts["prec"] + 4 * C * counts["adc"])
    w_mufu = n_local * 2 * (counts["prec_relax"] + counts["prec"])
    p_fp32 = n_sm * 128 * f_max * 1e6
    p_mufu = n_sm * 16 * f_max * 1e6
    t_star = max(w_fp32 / p_fp32, w_mufu / p_mufu)
    t_kernel = t_kernel_s / args.steps
    model_ops = max(w_fp32, 8 * w_mufu)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh).get(f"config{args.config}")
    except Exception:
        pass
    # the contract's measured denominators (MEASURED_PEAKS.json), beside the SURVEY §8d model:
    # HBM traffic of the integrator (ncu capture) and the tensor pipe's actual work in the ADC
    # windows: per spin-sample-coil one tf32 m16n8k8 pass (4 real MAC at the measured 512 MAC/clk/SM)
    # and one bf16 m16n8k16 pass for both cross terms (8 real MAC at 1024 MAC/clk/SM), i.e. 8
    # tf32-rate MAC equivalents (profiles/r1_mma_microbench.txt).
    hbm_peak = bf16_peak = None
    try:
        with open(peaks_path) as fh:
            mp = json.load(fh)
        hbm_peak, bf16_peak = float(mp["hbm_gbs"]), float(mp["bf16_tflops"])
    except Exception:
        pass
    w_mma = n_local * pstats["window_samples"] * C * 8 if args.precision == 32 else 0
    p_mma = n_sm * 512 * f_max * 1e6
    measured = {
        "hbm": {"achieved_gbs": traffic / t_kernel / 1e9 if traffic else None, "peak_gbs": hbm_peak,
                "frac": traffic / t_kernel / 1e9 / hbm_peak if traffic and hbm_peak else None,
                "source": "peak of measured (MEASURED_PEAKS.json hbm_gbs)"},
        "tensor_mma_tf32": {"achieved_tflops": 2 * w_mma / t_kernel / 1e12, "peak_tflops": 2 * p_mma / 1e12,
                            "frac": w_mma / p_mma / t_kernel,
                            "source": "tf32-rate MAC equivalents (tf32 hi*hi + bf16 k16 cross terms) over the "
                                      "measured mma.sync m16n8k8 tf32 peak, 512 MAC/clk/SM "
                                      "(profiles/r1_mma_microbench.txt); bf16 GEMM peak of measured "
                                      f"{bf16_peak} TFLOP/s is tcgen05 bf16 and does not apply"},
    }
    roofline = {
        "bound": "fp32+mufu",
        "achieved": model_ops / t_kernel / 1e12,
        "peak": p_fp32 / 1e12,
        "unit": "TFLOP/s",
        "frac": t_star / t_kernel,
        "traffic": traffic,
        "model": "ops = max(W_fp32, 8*W_mufu); W_fp32 = N(9 rot + 12 prec_relax + 9 prec + 4C adc), "
                 "W_mufu = 2N(prec_relax + prec); FP32 op = 1 lane-instruction (FFMA/FMUL/FADD); "
                 f"peak = {n_sm} SM x 128 lanes x {f_max:.0f} MHz (nominal; FFMA measured 125.3/128, profiles/)",
        "kernel_ms": t_kernel * 1e3,
        "roofline_ms": t_star * 1e3,
        "updates_per_s_at_roofline": n_local * E / t_star,
        "measured_peaks": measured,
    }

    line = {
        "metric": metric, "value": value, "unit": metric, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_total_s * 1e3 / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None,
        "dtype": ("f64 spin state/phase/fold; f32 ADC sums (tf32 hi*hi + bf16 cross terms on the tensor cores)"
                  if args.precision == 32 else "f64"),
        "data": "synthetic (seeded, BASELINE.json config recipe)",
        "config": {"workload": w.name, "config_index": w.index, "spins_total": n_total, "spins_per_rank": n_local,
                   "sharding": ("weak: every rank a full config-sized spin set (world interleaved copies of the "
                                "lattice, shifted by rank/world of its x spacing; parallel.weak_copy), one NCCL "
                                "reduce of the k-space" if weak else "strong: np.linspace spin shards of the config")
                               if world > 1 else "single GPU",
                   "events_per_spin": E, "coils": C, "event_classes": counts, "program": pstats,
                   "l2": "flushed between timed steps (256 MiB write)", "parallelism": f"spin-shards x{world}"},
        "roofline": roofline,
        "integrator_launch": launch_shape,
        "e2e": {"value": e2e_value, "unit": metric, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "steps": e2e_steps, "path": e2e_path},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "kernel_ms_per_step": t_kernel * 1e3,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_sample(w, tables_plain, E, args.cpu_spins_per_core, quiet=args.quiet)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

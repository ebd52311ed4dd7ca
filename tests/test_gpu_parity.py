"""GPU parity: libbloch_b200 through the C-ABI vs the reference's own outputs.

Every case replays a golden record produced by the reference itself
(tests/golden/make_golden.py): the same spin arrays and the same sequence go
through ``paper_1305_6861_b200.compute_block`` (ctypes -> bloch_compute_block
-> sm_100a kernels) and the echoes / snapshots are compared with the
BASELINE.json tolerances:

* fp32 state (default engine): k-space rel L2 <= 1e-4, final magnetisation
  rel L2 <= 1e-5;
* fp64 state engine: rel L2 <= 1e-11 (the reference unit tests' regime).
"""

import math

import numpy as np
import pytest

import cases
from conftest import load_golden
from make_golden import projection_vector
from oracle.bloch_oracle import rel_l2
from paper_1305_6861_b200 import SpinBlock, compute_block, precompute_sequence_tables

pytestmark = pytest.mark.gpu

SMALL = ["fid", "pair", "se16_box", "tse16", "epi16", "cpmg8", "mixed", "mixed_coils", "tse_2coil"]
CONFIGS = ["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"]

KSPACE_TOL = {32: 1e-4, 64: 1e-11}
STATE_TOL = {32: 1e-5, 64: 1e-11}


def _sequence_of(name):
    if name.startswith("cfg"):
        from paper_1305_6861_b200 import configs

        return configs.make(int(name[3:])).sequence
    return cases.small_cases()[name]["sequence"]


_SEQ_CACHE = {}


def _tables(name, rec):
    if name not in _SEQ_CACHE:
        _SEQ_CACHE[name] = precompute_sequence_tables(
            _sequence_of(name), snapshot_times=tuple(rec["snapshot_times"].tolist())
        )
    return _SEQ_CACHE[name]


def _block(rec):
    return SpinBlock(index=0, pos=rec["spin_pos"], mx=rec["spin_mx"], my=rec["spin_my"], mz=rec["spin_mz"],
                     t1=rec["spin_t1"], t2=rec["spin_t2"], m0=rec["spin_m0"], domega=rec["spin_domega"],
                     weight=rec["spin_weight"])


def echo_error(rec, echoes):
    """rel L2 of the GPU echoes vs the golden (full array, or head/tail + per-acq checksums)."""
    if "echo_full" in rec:
        return rel_l2(rec["echo_full"], echoes)
    shape = tuple(rec["echo_shape"])
    ek = np.asarray(echoes).reshape((-1,) + shape[-2:])
    errs = [rel_l2(rec["echo_head"], ek[:, :4]), rel_l2(rec["echo_tail"], ek[:, -4:]),
            rel_l2(rec["echo_proj"], ek @ projection_vector(ek.shape[-1]))]
    return max(errs)


def snapshot_errors(rec, snaps):
    out = []
    for i in range(int(rec["n_snap"])):
        present = bool(rec[f"snap_{i}_present"])
        assert (snaps[i] is not None) == present, f"snapshot {i} presence"
        if present:
            out.append(rel_l2(rec[f"snap_{i}"], snaps[i]))
    return out


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("name", SMALL + CONFIGS)
def test_gpu_matches_reference_golden(name, precision):
    rec = load_golden(name)
    tables = _tables(name, rec)
    echoes, snaps = compute_block(tables, _block(rec), precision=precision)
    assert echoes.shape == tuple(rec["echo_shape"])
    err = echo_error(rec, echoes)
    assert err <= KSPACE_TOL[precision], f"{name} fp{precision} k-space rel L2 {err:.3e}"
    for i, e in enumerate(snapshot_errors(rec, snaps)):
        assert e <= STATE_TOL[precision], f"{name} fp{precision} snapshot {i} rel L2 {e:.3e}"


# --- reference engine tests restated against the GPU path (tests/test_engine.py) ---


def test_fid_amplitude():  # test_engine.py:115-122
    rec = load_golden("fid")
    echoes, _ = compute_block(_tables("fid", rec), _block(rec), precision=64)
    assert abs(echoes[0, 0]) == pytest.approx(0.5 * math.exp(-0.05 / 0.2), rel=1e-12)
    echoes32, _ = compute_block(_tables("fid", rec), _block(rec), precision=32)
    assert abs(echoes32[0, 0]) == pytest.approx(0.5 * math.exp(-0.05 / 0.2), rel=1e-6)


def test_zero_m0_contributes_nothing():  # test_engine.py:125-131
    rec = load_golden("fid")
    blk = _block(rec)
    blk.mz = np.zeros(1)
    blk.m0 = np.zeros(1)
    for prec in (32, 64):
        echoes, _ = compute_block(_tables("fid", rec), blk, precision=prec)
        assert np.all(echoes == 0)


def test_opposite_positions_sum_to_real_signal():  # test_engine.py:134-155
    rec = load_golden("pair")
    echoes, _ = compute_block(_tables("pair", rec), _block(rec), precision=64)
    np.testing.assert_allclose(echoes.imag, 0.0, atol=1e-14)
    assert np.max(np.abs(echoes.real)) > 0.1


def test_empty_block():
    rec = load_golden("tse16")
    blk = _block(rec)
    empty = SpinBlock(index=0, pos=np.zeros((0, 3)), mx=np.zeros(0), my=np.zeros(0), mz=np.zeros(0),
                      t1=np.zeros(0), t2=np.zeros(0), m0=np.zeros(0), domega=np.zeros(0),
                      weight=np.zeros(0, complex))
    echoes, snaps = compute_block(_tables("tse16", rec), empty)
    assert echoes.shape == tuple(rec["echo_shape"]) and np.all(echoes == 0)
    assert all(s is None or s.shape == (0, 3) for s in snaps)
    del blk


def test_scaling_m0_by_two_is_exact():  # test_engine.py:203-206 (power-of-two scaling commutes with rounding)
    rec = load_golden("se16_box")
    t = _tables("se16_box", rec)
    a, _ = compute_block(t, _block(rec))
    blk = _block(rec)
    blk.m0 = blk.m0 * 2.0
    blk.mz = blk.mz * 2.0
    b, _ = compute_block(t, blk)
    assert np.array_equal(a * 2.0, b)


def test_deterministic_repeat_bit_identical():  # test_engine.py:181-184
    rec = load_golden("cfg1")
    t = _tables("cfg1", rec)
    a, sa = compute_block(t, _block(rec))
    b, sb = compute_block(t, _block(rec))
    assert np.array_equal(a, b) and np.array_equal(sa[0], sb[0])


def test_block_partition_linearity():  # test_engine.py:175-179, 191-200
    rec = load_golden("tse16")
    t = _tables("tse16", rec)
    full, _ = compute_block(t, _block(rec))
    blk = _block(rec)
    parts = []
    for lo, hi in ((0, 77), (77, 300)):
        sub = SpinBlock(index=0, pos=blk.pos[lo:hi], mx=blk.mx[lo:hi], my=blk.my[lo:hi], mz=blk.mz[lo:hi],
                        t1=blk.t1[lo:hi], t2=blk.t2[lo:hi], m0=blk.m0[lo:hi], domega=blk.domega[lo:hi],
                        weight=blk.weight[lo:hi])
        parts.append(compute_block(t, sub)[0])
    assert rel_l2(full, parts[0] + parts[1]) <= 1e-6


@pytest.mark.gpu
def test_graph_replay_of_repeated_device_calls():
    """Repeated device-resident calls replay a captured CUDA graph: the results stay bit-identical to
    the first (uncaptured) call; a different output pointer or new tables re-enqueue (no stale graph)."""
    import torch

    from paper_1305_6861_b200 import configs
    from paper_1305_6861_b200.engine import BlochEngine

    eng = BlochEngine(0, 32)
    w = configs.make(0)
    b = w.block
    dev = torch.device("cuda", 0)
    d = {k: torch.from_numpy(np.ascontiguousarray(getattr(b, k), dtype=np.float64)).to(dev)
         for k in ("pos", "mx", "my", "mz", "t1", "t2", "m0", "domega")}
    ptrs = {k: v.data_ptr() for k, v in d.items()}
    ptrs["weight"] = 0

    def call(tables, out):
        f = eng.set_tables(tables)
        eng.compute_device(tables, ptrs, b.n, 1, out.data_ptr(), sync=True)
        return out.cpu().numpy().copy(), f

    t1 = precompute_sequence_tables(w.sequence)
    f = eng.set_tables(t1)
    outs = [torch.zeros(f["n_acq"] * f["max_ns"] * 2, dtype=torch.float64, device=dev) for _ in range(2)]
    first, _ = call(t1, outs[0])
    for _ in range(4):  # call 2 is captured, calls 3.. replay the graph
        again, _ = call(t1, outs[0])
        assert np.array_equal(first, again)
        assert eng.last_timing()["kernel_ms"] > 0
    other, _ = call(t1, outs[1])  # new output pointer: a fresh enqueue into the other buffer
    assert np.array_equal(first, other)
    seq2 = configs.config_sequence(0)
    seq2 = type(seq2)(list(seq2.elements)[: len(seq2.elements) // 2], name="half")
    t2 = precompute_sequence_tables(seq2)
    f2 = eng.set_tables(t2)
    out2 = torch.zeros(f2["n_acq"] * f2["max_ns"] * 2, dtype=torch.float64, device=dev)
    half, _ = call(t2, out2)
    ref, _ = eng.compute(t2, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)
    np.testing.assert_array_equal(half.view(np.complex128).reshape(np.asarray(ref).shape), ref)
    eng.close()


@pytest.mark.gpu
def test_graph_not_replayed_after_buffer_reallocation():
    """A, A (captured), A (replayed), then B with more spins (the context's scratch buffers grow, i.e. are
    freed and reallocated), then A again: the graph recorded before the reallocation holds dead pointers
    and must not be replayed; A's result stays bit-identical throughout."""
    import torch

    from paper_1305_6861_b200 import configs
    from paper_1305_6861_b200.engine import BlochEngine

    eng = BlochEngine(0, 32)
    w = configs.make(0)
    big = configs.make(1).subset(40)  # ~17k spins: larger than config 0's 2,444
    dev = torch.device("cuda", 0)

    def dev_ptrs(b):
        d = {k: torch.from_numpy(np.ascontiguousarray(getattr(b, k), dtype=np.float64)).to(dev)
             for k in ("pos", "mx", "my", "mz", "t1", "t2", "m0", "domega")}
        p = {k: v.data_ptr() for k, v in d.items()}
        p["weight"] = 0
        return d, p

    t = precompute_sequence_tables(w.sequence)
    f = eng.set_tables(t)
    out = torch.zeros(f["n_acq"] * f["max_ns"] * 2, dtype=torch.float64, device=dev)
    da, pa = dev_ptrs(w.block)
    db, pb = dev_ptrs(big.block)

    def call(p, n):
        eng.compute_device(t, p, n, 1, out.data_ptr(), sync=True)
        return out.cpu().numpy().copy()

    first = call(pa, w.block.n)
    for _ in range(2):  # second call captured, third replayed
        assert np.array_equal(call(pa, w.block.n), first)
    call(pb, big.block.n)  # B: every per-spin scratch buffer grows
    for _ in range(3):  # A again: re-enqueued, re-captured, replayed — never the stale graph
        assert np.array_equal(call(pa, w.block.n), first)
    eng.close()


@pytest.mark.gpu
def test_pipeline_matches_synchronous_compute():
    """Double-buffered Pipeline submissions give the same k-space and final M as synchronous calls."""
    import torch

    from paper_1305_6861_b200 import configs
    from paper_1305_6861_b200.engine import Pipeline, get_engine

    w = configs.make(0)
    b = w.block
    t = precompute_sequence_tables(w.sequence, snapshot_times=(w.sequence.end_time,))
    ref_e, ref_s = get_engine(0, 32).compute(t, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)
    pipe = Pipeline(0, 32, depth=2)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    outs = [(pin(np.zeros((1,) + ref_e.shape, complex)), pin(np.zeros((1, b.n, 3)))) for _ in range(2)]
    pend = [pipe.submit(t, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight, out_echoes=outs[k % 2][0],
                        out_snaps=outs[k % 2][1]) for k in range(5)]
    for p in pend[-2:]:
        e, s = p.wait()
        assert np.array_equal(e, ref_e) and np.array_equal(s[0], ref_s[0])
    pipe.close()


@pytest.mark.parametrize("precision", [32, 64])
def test_more_coils_than_one_call_takes(precision):
    """12 receive coils (> MAX_COILS = 8 per device call): BlochEngine.compute runs coil groups; every
    coil's k-space matches the oracle (one weighted sum per coil, engine.py:303-305 per weight)."""
    from oracle import bloch_oracle as O

    rec = load_golden("mixed")
    b = _block(rec)
    rng = np.random.default_rng(12)
    w = rng.uniform(0.3, 1.0, (12, b.n)) * np.exp(1j * rng.uniform(0, 2 * math.pi, (12, b.n)))
    seq = _sequence_of("mixed")
    snaps_t = tuple(rec["snapshot_times"].tolist())
    t = precompute_sequence_tables(seq, snapshot_times=snaps_t)
    e, s = compute_block(t, SpinBlock(index=0, pos=b.pos, mx=b.mx, my=b.my, mz=b.mz, t1=b.t1, t2=b.t2, m0=b.m0,
                                      domega=b.domega, weight=w), precision=precision)
    ot = O.precompute_tables(seq, snapshot_times=snaps_t)
    ref_e, ref_s = O.compute_block(ot, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, w)
    assert e.shape == ref_e.shape == (12,) + ref_e.shape[1:]
    for c in range(12):
        assert rel_l2(ref_e[c], e[c]) <= KSPACE_TOL[precision], c
    for a, r in zip(s, ref_s):
        if r is not None:
            assert rel_l2(r, a) <= STATE_TOL[precision]


# --- the window contraction (contract.h) and the integrator's own window sums, both against the goldens ---


@pytest.mark.parametrize("name", SMALL + CONFIGS)
def test_gpu_window_sums_without_contraction(name):
    """fp32 mode with the contraction switched off: every window summed by the integrator's warps."""
    from paper_1305_6861_b200.engine import get_engine

    rec = load_golden(name)
    eng = get_engine(0, 32)
    eng.set_contraction(False)
    try:
        echoes, snaps = compute_block(_tables(name, rec), _block(rec), precision=32)
        assert eng.last_phases()["groups"] == 0
    finally:
        eng.set_contraction(True)
    err = echo_error(rec, echoes)
    assert err <= KSPACE_TOL[32], f"{name} k-space rel L2 {err:.3e}"
    for i, e in enumerate(snapshot_errors(rec, snaps)):
        assert e <= STATE_TOL[32], f"{name} snapshot {i} rel L2 {e:.3e}"


# --- the resident-table integrator (resident.h) and the integrator that reads the tables through L2 ---

RESIDENT = ["cfg0", "cfg1", "cfg2", "cfg3", "cfg4", "epi16"]  # must run resident; the small cases: whatever their plan says


@pytest.mark.parametrize("name", SMALL + CONFIGS)
def test_gpu_resident_on_and_off_match_goldens(name):
    """Fully deferred fp32 programs run resident_integrate_kernel (class tables in shared memory); with it
    switched off the same programs run integrate_kernel's deferred variant.  Both against the goldens, and
    against each other much tighter (same fp64 state arithmetic, same U words up to the fp32 u)."""
    from paper_1305_6861_b200.engine import get_engine

    rec = load_golden(name)
    eng = get_engine(0, 32)
    out = {}
    for on in (True, False):
        eng.set_resident(on)
        try:
            echoes, snaps = compute_block(_tables(name, rec), _block(rec), precision=32)
            used = eng.last_resident()["resident"]
        finally:
            eng.set_resident(True)
        if not on:
            assert used == 0
        elif name in RESIDENT:
            assert used == 1, (name, eng.last_resident())
        err = echo_error(rec, echoes)
        assert err <= KSPACE_TOL[32], f"{name} resident={on} k-space rel L2 {err:.3e}"
        for i, e in enumerate(snapshot_errors(rec, snaps)):
            assert e <= STATE_TOL[32], f"{name} resident={on} snapshot {i} rel L2 {e:.3e}"
        out[on] = (np.asarray(echoes), snaps)
    assert rel_l2(out[False][0], out[True][0]) <= 2e-6
    for a, b in zip(out[False][1], out[True][1]):
        if a is not None:
            assert rel_l2(a, b) <= 1e-12


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "se16_box", "tse16", "epi16", "tse_2coil"])
def test_gpu_contraction_runs_and_matches(name):
    """The long tabulated windows of these programs go through the tensor-core contraction."""
    from paper_1305_6861_b200.engine import get_engine

    rec = load_golden(name)
    eng = get_engine(0, 32)
    echoes, _ = compute_block(_tables(name, rec), _block(rec), precision=32)
    ph = eng.last_phases()
    assert ph["groups"] >= 1 and ph["contracted_samples"] > 0, ph
    assert echo_error(rec, echoes) <= KSPACE_TOL[32]


_SHORT_CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests"); sys.path.insert(0, sys.argv[1] + "/tests/golden")
from test_gpu_parity import _tables, _block, echo_error, snapshot_errors
from conftest import load_golden
from paper_1305_6861_b200 import compute_block
from paper_1305_6861_b200.engine import get_engine
name = sys.argv[2]
rec = load_golden(name)
e, s = compute_block(_tables(name, rec), _block(rec), precision=32)
eng = get_engine(0, 32)
print(json.dumps({"err": echo_error(rec, e), "snap": max(snapshot_errors(rec, s) or [0.0]),
                  "groups": eng.program_stats()["window_groups"], "rest": eng.program_stats()["integrator_samples"],
                  "resident": eng.last_resident()["resident"], "spins_per_thread": eng.last_launch()["spins_per_thread"]}))
"""


def _run_child(name, **env_extra):
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _SHORT_CHILD, root, name], capture_output=True, text=True,
                       env=dict(os.environ, **env_extra), timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("name", ["cfg0", "cfg1", "cfg2", "cfg4", "tse16", "tse_2coil"])
def test_gpu_resident_two_spins_per_thread(name):
    """The two-spins-per-thread instance of resident_integrate_kernel (full-size blocks pick it; forced here on
    the golden subsets with BLOCH_RESIDENT_SPINS=2), against the reference goldens."""
    d = _run_child(name, BLOCH_RESIDENT_SPINS="2")
    assert d["err"] <= KSPACE_TOL[32] and d["snap"] <= STATE_TOL[32], d
    if name.startswith("cfg"):
        assert d["resident"] == 1 and d["spins_per_thread"] == 2, d


@pytest.mark.parametrize("name", ["epi16", "mixed", "cfg3"])
def test_gpu_resident_short_runs(name):
    """BLOCH_DEFER_SHORT=1 makes the EPI programs fully deferred (OP_UCHIRP, one-sample OP_UWIN): they then
    run the resident-table integrator."""
    d = _run_child(name, BLOCH_DEFER_SHORT="1")
    assert d["err"] <= KSPACE_TOL[32] and d["snap"] <= STATE_TOL[32], d
    if name == "epi16":
        assert d["resident"] == 1, d


@pytest.mark.parametrize("name", ["epi16", "mixed", "mixed_coils", "cfg3"])
def test_gpu_short_run_contraction(name):
    """BLOCH_DEFER_SHORT=1: tabulated chirps (trapezoid ramps, u r0^(k+1) q^(k(k+1)/2)) and single-sample
    events contracted as well, against the reference goldens."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, BLOCH_DEFER_SHORT="1")
    r = subprocess.run([sys.executable, "-c", _SHORT_CHILD, root, name], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["err"] <= KSPACE_TOL[32] and d["snap"] <= STATE_TOL[32], d
    if name == "epi16":
        assert d["rest"] == 0, d  # every sample contracted
    if name == "cfg3":  # runs in groups smaller than kMinDeferGroup (program.h) stay in the integrator
        assert d["rest"] < 16, d

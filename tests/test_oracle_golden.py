"""CPU: pin the oracle (and the product's host-side table builder) to the reference's own outputs.

Golden records were produced by running the reference package itself
(tests/golden/make_golden.py).  Here, without importing the reference:

* the oracle's table restatement equals the reference tables bit for bit;
* the product's ``precompute_sequence_tables`` equals them bit for bit;
* the product's vectorised ``rasterize_arrays`` equals the reference's
  ``rasterize`` + ``build_spin_arrays`` output bit for bit;
* the oracle's ``compute_block`` reproduces the reference echoes and
  snapshots (same numpy arithmetic, rel 1e-12 to allow a different BLAS
  kernel for ``pos @ dmom`` on another CPU).
"""

import numpy as np
import pytest

import cases
from conftest import load_golden
from make_golden import projection_vector
from oracle import bloch_oracle as O
from paper_1305_6861_b200 import configs, flatten_tables, precompute_sequence_tables
from paper_1305_6861_b200.phantom import rasterize_arrays

SMALL = ["fid", "pair", "se16_box", "tse16", "epi16", "cpmg8", "mixed", "mixed_coils", "tse_2coil"]
CONFIGS = ["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"]


def _sequence(name):
    if name.startswith("cfg"):
        return configs.make(int(name[3:])).sequence
    return cases.small_cases()[name]["sequence"]


def _assert_tables_equal(rec, tables):
    flat = flatten_tables(tables)
    for k, v in flat.items():
        ref = rec["tab_" + k]
        assert np.array_equal(np.asarray(v), ref), f"table field {k} differs"


@pytest.mark.parametrize("name", SMALL + CONFIGS)
def test_oracle_tables_match_reference(name):
    rec = load_golden(name)
    seq = _sequence(name)
    snaps = tuple(rec["snapshot_times"].tolist())
    _assert_tables_equal(rec, O.precompute_tables(seq, snapshot_times=snaps))
    tabs = O.precompute_tables(seq, snapshot_times=snaps)
    assert tabs.pulse_memo_hits == int(rec["pulse_memo_hits"])


@pytest.mark.parametrize("name", SMALL + CONFIGS)
def test_product_tables_match_reference(name):
    rec = load_golden(name)
    tables = precompute_sequence_tables(_sequence(name), snapshot_times=tuple(rec["snapshot_times"].tolist()))
    _assert_tables_equal(rec, tables)
    assert tables.pulse_memo_hits == int(rec["pulse_memo_hits"])


def test_rasterize_matches_reference():  # phantom.py:98-142 + engine.py:192-226
    rec = load_golden("se16_box")
    case = cases.small_cases()["se16_box"]
    a = rasterize_arrays(case["phantom"], case["spacing"])
    assert np.array_equal(a["pos"], rec["spin_pos"])
    assert np.array_equal(a["m0"], rec["spin_m0"])
    assert np.array_equal(a["t1"], rec["spin_t1"])
    assert np.array_equal(a["t2"], rec["spin_t2"])


def _oracle_run(name, rec):
    tables = O.precompute_tables(_sequence(name), snapshot_times=tuple(rec["snapshot_times"].tolist()))
    return O.compute_block(tables, rec["spin_pos"], rec["spin_mx"], rec["spin_my"], rec["spin_mz"], rec["spin_t1"],
                           rec["spin_t2"], rec["spin_m0"], rec["spin_domega"], rec["spin_weight"])


def _check_echoes(rec, echoes, tol):
    assert echoes.shape == tuple(rec["echo_shape"])
    if "echo_full" in rec:
        assert O.rel_l2(rec["echo_full"], echoes) <= tol
        return
    ek = echoes.reshape((-1,) + echoes.shape[-2:])
    assert O.rel_l2(rec["echo_head"], ek[:, :4]) <= tol
    assert O.rel_l2(rec["echo_tail"], ek[:, -4:]) <= tol
    assert O.rel_l2(rec["echo_proj"], ek @ projection_vector(ek.shape[-1])) <= tol
    assert O.rel_l2(rec["echo_energy"], (np.abs(ek) ** 2).sum(axis=-1)) <= tol


@pytest.mark.parametrize("name", SMALL + ["cfg0", "cfg1", "cfg3"])
def test_oracle_compute_block_matches_reference(name):
    rec = load_golden(name)
    echoes, snaps = _oracle_run(name, rec)
    _check_echoes(rec, echoes, 1e-12)
    for i in range(int(rec["n_snap"])):
        if bool(rec[f"snap_{i}_present"]):
            assert O.rel_l2(rec[f"snap_{i}"], snaps[i]) <= 1e-12
        else:
            assert snaps[i] is None


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg2", "cfg4"])
def test_oracle_compute_block_matches_reference_long(name):
    rec = load_golden(name)
    echoes, snaps = _oracle_run(name, rec)
    _check_echoes(rec, echoes, 1e-12)
    assert O.rel_l2(rec["snap_0"], snaps[0]) <= 1e-12


def test_event_counts_match_survey():  # E = 4,480 / 67,072 / 264,768
    want = {0: 4480, 1: 67072, 2: 264768}
    for i, e in want.items():
        assert O.event_count(O.precompute_tables(configs.make(i).sequence)) == e


def test_delta_e_stoer_and_rel_l2():  # engine.py:603-616; test_engine.py:277-291
    rng = np.random.default_rng(0)
    ref = rng.normal(size=256) + 1j * rng.normal(size=256)
    assert O.delta_e_stoer(ref, ref) == -np.inf
    assert O.delta_e_stoer(ref, ref * (1 + 1e-6)) == pytest.approx(-120.0, abs=0.5)
    assert O.delta_e_stoer(np.array([1.0, 2.0, 3.0]), np.zeros(3)) == pytest.approx(0.0, abs=1e-12)
    assert O.rel_l2(ref, ref * (1 + 1e-4)) == pytest.approx(1e-4, rel=1e-6)


def test_oracle_vs_kt_engine():
    """The float64 oracle against the reference's independent k-t engine (golden kt_random.npz,
    criterion 2 of the reference's acceptance tests): a second, algorithmically different pin."""
    import math
    import os

    from paper_1305_6861_b200 import (GAMMA_PROTON, AcquisitionSpec, ElementarySequence, GradientWaveform,
                                      HardPulse, Sequence)

    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "kt_random.npz"))
    pos, m0 = g["pos"], g["m0"]
    n = m0.size
    worst = 0.0
    for i in range(int(g["n_seq"])):
        els = [ElementarySequence(pulse=HardPulse(a, p), gradient=GradientWaveform.constant(gx=q * 80.0 / (GAMMA_PROTON * dt)),
                                  duration=dt) for a, p, q, dt in g[f"seq{i}_rows"]]
        els.append(ElementarySequence(gradient=GradientWaveform.constant(gx=4 * 80.0 / (GAMMA_PROTON * 0.01)),
                                      duration=0.01, acquisition=AcquisitionSpec(True, 33), kspace_row=0))
        tabs = O.precompute_tables(Sequence(els, name="random"))
        e, _ = O.compute_block(tabs, pos, np.zeros(n), np.zeros(n), m0.copy(), np.full(n, float(g["t1"])),
                               np.full(n, float(g["t2"])), m0.copy(), np.zeros(n), np.full(n, 1 + 0j))
        spin = np.asarray(e).ravel()[: g[f"seq{i}_kt"].size] / n
        worst = max(worst, np.linalg.norm(spin - g[f"seq{i}_kt"]) / np.linalg.norm(spin))
    assert worst <= 1e-6 and math.isfinite(worst)


@pytest.mark.parametrize("index", [1, 3])
def test_full_size_golden_pinned_by_oracle(index):
    """The full-size goldens (make_golden_full.py: every spin of the config through the reference's own
    process pool) agree with the oracle on a sample of their stored final-magnetisation rows, run here
    through the whole event stream, and carry the config's spin count (the GPU test's reference)."""
    import os

    path = os.path.join(os.path.dirname(__file__), "golden", f"full_cfg{index}.npz")
    if not os.path.exists(path):
        pytest.skip("full-size golden not generated")
    g = dict(np.load(path))
    w = configs.make(index)
    b = w.block
    assert int(g["n_spins"]) == b.n
    stride = int(g["m_stride"])
    rows = np.arange(0, g["m_sub"].shape[0], max(1, g["m_sub"].shape[0] // 24))[:24]
    idx = rows * stride
    t = O.precompute_tables(w.sequence, snapshot_times=(float(g["snapshot_time"]),))
    _, s = O.compute_block(t, b.pos[idx], b.mx[idx], b.my[idx], b.mz[idx], b.t1[idx], b.t2[idx], b.m0[idx],
                           b.domega[idx], np.asarray(b.weight)[idx])
    np.testing.assert_allclose(s[0], g["m_sub"][rows], rtol=0, atol=1e-12)
    assert np.isclose(g["m_sum"].sum(), g["m_sub"].sum() * stride, rtol=0.2)  # the checksum is of the whole array

"""Reconstruction, wire formats and CLI.

Pinned against what the reference itself computed / wrote
(tests/golden/make_golden_recon.py -> recon.npz, wire/), plus restatements of
the reference's own recon and CLI tests (tests/test_recon.py, tests/test_cli.py).
CPU tests run the torch transform on the host; the gpu-marked ones run it on
cuda:0 and drive `simulate` through the CUDA engine.
"""

import json
import math
import os

import numpy as np
import pytest

from paper_1305_6861_b200 import io as mrio
from paper_1305_6861_b200.cli import main
from paper_1305_6861_b200.errors import FitDiverged, InvalidParameter, ParseError, TrajectoryMismatch
from paper_1305_6861_b200.recon import (
    ImageVolume,
    KSpaceMatrix,
    assemble_kspace,
    cpmg_fit,
    export_image,
    forward_dft,
    reconstruct,
    standard_axes,
    trajectory_table,
)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
WIRE = os.path.join(GOLD, "wire")
CASES = ["se_sim16", "epi12x10", "odd15x9", "tse_seq8", "volumes6x4", "missing_rows"]


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(os.path.join(GOLD, "recon.npz")))


def _case(g, name):
    table = [(int(v), int(r), bool(x)) for v, r, x in g[f"{name}__table"]]
    n_rows = int(g[f"{name}__n_rows"])
    fov = float(g[f"{name}__fov"])
    return g[f"{name}__echoes"], table, (None if n_rows < 0 else n_rows), (None if math.isnan(fov) else fov)


def _check_case(g, name, device):
    echoes, table, n_rows, fov = _case(g, name)
    mats = assemble_kspace(echoes, table, n_rows=n_rows, fov=fov)
    assert len(mats) == int(g[f"{name}__n_vol"])
    for i, k in enumerate(mats):
        assert np.array_equal(k.data, g[f"{name}__k{i}"])  # assembly is pure data movement: bit-exact
        assert np.array_equal(k.row_filled, g[f"{name}__filled{i}"])
        assert k.volume == int(g[f"{name}__vol{i}"])
        np.testing.assert_allclose([*k.k0, *k.dk], g[f"{name}__axes{i}"], rtol=0, atol=0)
        img = reconstruct(k, device=device)
        ref = g[f"{name}__img{i}"]
        scale = max(np.abs(ref).max(), 1e-300)
        np.testing.assert_allclose(img.complex_image, ref, rtol=0, atol=1e-12 * scale)
        np.testing.assert_allclose(img.pixel_size, g[f"{name}__pix{i}"], rtol=1e-15)


@pytest.mark.parametrize("name", CASES)
def test_recon_matches_reference_cpu(gold, name):
    _check_case(gold, name, "cpu")


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_recon_matches_reference_gpu(gold, name):
    _check_case(gold, name, "cuda")


def test_forward_dft_matches_reference(gold):
    a = gold["fwd__axes"]
    k = forward_dft(ImageVolume(gold["fwd__img"], (1.0, 1.0)), k0=(a[0], a[1]), dk=(a[2], a[3]), device="cpu")
    np.testing.assert_allclose(k.data, gold["fwd__k"], rtol=0, atol=1e-12 * np.abs(gold["fwd__k"]).max())


def test_cpmg_fit_matches_reference(gold):
    for y, (rho, t2, rn) in zip(gold["fit__y"], gold["fit__res"]):
        f = cpmg_fit(gold["fit__t"], y)
        assert f.rho == pytest.approx(rho, rel=1e-9) and f.t2 == pytest.approx(t2, rel=1e-9)
        assert f.residual_norm == pytest.approx(rn, rel=1e-6, abs=1e-14)


# -- restated reference recon tests (tests/test_recon.py) ----------------------------------------------------------


def _kspace(data, fov=0.5):
    ny, nx = data.shape
    ky0, dky = standard_axes(fov, ny)
    kx0, dkx = standard_axes(fov, nx)
    return KSpaceMatrix(np.asarray(data, complex), np.ones(ny, bool), (ky0, kx0), (dky, dkx))


def test_trajectory_tables():
    assert [r for _, r, _ in trajectory_table("tse-seq", 8, turbo_factor=2)] == list(range(8))
    assert [rv for _, _, rv in trajectory_table("epi", 4)] == [False, True, False, True]
    with pytest.raises(InvalidParameter):
        trajectory_table("spiral", 4)


def test_assembly_errors_and_missing_rows():
    with pytest.raises(TrajectoryMismatch):
        assemble_kspace(np.ones((2, 4), complex), [(0, 1, False), (0, 1, False)], n_rows=4)
    with pytest.raises(TrajectoryMismatch):
        assemble_kspace(np.ones((3, 4), complex), [(0, 0, False)], n_rows=4)
    with pytest.raises(TrajectoryMismatch):
        assemble_kspace(np.ones((1, 4), complex), [(0, 4, False)], n_rows=4)
    k = assemble_kspace(np.ones((2, 4), complex), [(0, 0, False), (0, 2, False)], n_rows=4)[0]
    assert list(k.row_filled) == [True, False, True, False]


def test_delta_flat_magnitude_and_half_sample_ramp():
    n = 16
    d = np.zeros((n, n), complex)
    d[n // 2, n // 2] = 1.0
    img = reconstruct(_kspace(d), device="cpu")
    np.testing.assert_allclose(img.magnitude, img.magnitude[0, 0], rtol=1e-12)
    dphi = np.angle(img.complex_image[8, 9] / img.complex_image[8, 8])
    assert dphi == pytest.approx((2 * math.pi / 0.5) / 2.0 * img.pixel_size[1], rel=1e-9)


def test_round_trip_and_parseval():
    rng = np.random.default_rng(2)
    n = 24
    data = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    ky0, dky = standard_axes(0.4, n)
    k = forward_dft(ImageVolume(data, (1.0, 1.0)), k0=(ky0, ky0), dk=(dky, dky), device="cpu")
    np.testing.assert_allclose(reconstruct(k, device="cpu").complex_image, data, rtol=1e-10, atol=1e-12)
    img = reconstruct(_kspace(data), device="cpu")
    assert np.sum(np.abs(img.complex_image) ** 2) == pytest.approx(np.sum(np.abs(data) ** 2) / n ** 2, rel=1e-10)


def test_real_object_has_flat_phase():
    n = 32
    image = np.zeros((n, n))
    image[10:22, 8:24] = 1.0
    a = standard_axes(0.5, n)
    k = forward_dft(ImageVolume(image.astype(complex), (0.5 / n, 0.5 / n)), k0=(a[0], a[0]), dk=(a[1], a[1]),
                    device="cpu")
    img = reconstruct(k, device="cpu")
    np.testing.assert_allclose(img.phase[image > 0.5], 0.0, atol=1e-10)


def test_cpmg_fit_divergence():
    t = np.arange(1, 13) * 0.02
    with pytest.raises(FitDiverged):
        cpmg_fit(t, np.full(12, 0.7))
    with pytest.raises(FitDiverged):
        cpmg_fit(t, np.zeros(12))


# -- wire formats: byte compatibility with files the reference wrote -----------------------------------------------


@pytest.fixture(scope="module")
def wire_inputs():
    return dict(np.load(os.path.join(WIRE, "inputs.npz")))


def _bytes(path):
    with open(path, "rb") as fh:
        return fh.read()


def test_echo_file_bytes(tmp_path, wire_inputs):
    ref_path = os.path.join(WIRE, "echo.mrsim")
    assert np.array_equal(mrio.read_echo_file(ref_path), wire_inputs["echo"])
    p = str(tmp_path / "echo.mrsim")
    mrio.write_echo_file(p, wire_inputs["echo"],
                         {"written_at": "fixed", "sequence": "golden", "arr": np.arange(3), "n": np.int64(7)})
    assert _bytes(p) == _bytes(ref_path)
    assert _bytes(p + ".manifest.json") == _bytes(ref_path + ".manifest.json")
    assert mrio.read_manifest(p)["n_acq"] == 3


def test_snapshot_grid_pgm_bytes(tmp_path, wire_inputs):
    t, arr = mrio.read_snapshot_file(os.path.join(WIRE, "snap.mrsim"))
    assert t == 0.0125 and np.array_equal(arr, wire_inputs["snap"])
    for name, data in (("grid_c128.raw", wire_inputs["grid_c"]), ("grid_f64.raw", wire_inputs["grid_f"])):
        assert np.array_equal(mrio.read_raw_grid(os.path.join(WIRE, name)), data)
        p = str(tmp_path / name)
        mrio.write_raw_grid(p, data)
        assert _bytes(p) == _bytes(os.path.join(WIRE, name))
    p = str(tmp_path / "s.mrsim")
    mrio.write_snapshot_file(p, 0.0125, wire_inputs["snap"])
    assert _bytes(p) == _bytes(os.path.join(WIRE, "snap.mrsim"))
    for name, img, window in (("auto.pgm", wire_inputs["pgm_img"], None),
                              ("window.pgm", wire_inputs["pgm_img"], (0.2, 1.1)),
                              ("flat.pgm", np.ones((2, 3)), None)):
        p = str(tmp_path / name)
        mrio.write_pgm(p, img, window=window)
        assert _bytes(p) == _bytes(os.path.join(WIRE, name)), name


def test_wire_format_errors(tmp_path):
    bad = tmp_path / "bad.mrsim"
    bad.write_bytes(b"MRSIM2 1 1\n" + b"\0" * 16)
    with pytest.raises(ParseError):
        mrio.read_echo_file(str(bad))
    bad.write_bytes(b"MRSIM1 2 2\n" + b"\0" * 16)
    with pytest.raises(ParseError):
        mrio.read_echo_file(str(bad))
    bad.write_bytes(b"2 2 dtype=c64\n")
    with pytest.raises(ParseError):
        mrio.read_raw_grid(str(bad))
    with pytest.raises(InvalidParameter):
        mrio.write_echo_file(str(bad), np.zeros(3))
    with pytest.raises(InvalidParameter):
        mrio.write_snapshot_file(str(bad), 0.0, np.zeros((3, 2)))


# -- CLI (reference tests/test_cli.py) -------------------------------------------------------------------------------


def test_cli_compare_identical(capsys):
    path = os.path.join(WIRE, "echo.mrsim")
    assert main(["compare", "--ref", path, "--test", path]) == 0
    out = capsys.readouterr().out
    assert "exceedances=0" in out and "delta_e_stoer_db=-inf" in out


def test_cli_recon_and_fit(tmp_path, capsys, gold):
    echoes = gold["se_sim16__echoes"]
    ep = str(tmp_path / "e.mrsim")
    mrio.write_echo_file(ep, echoes)
    out = str(tmp_path / "img.pgm")
    assert main(["recon", "--echoes", ep, "--trajectory", "se", "--size", "16", "16", "--fov", "0.2",
                 "--device", "cpu", "--out", out]) == 0
    grid = mrio.read_raw_grid(out + ".raw")
    np.testing.assert_allclose(grid, gold["se_sim16__img0"], rtol=0, atol=1e-12 * np.abs(grid).max())
    series = tmp_path / "series.txt"
    t = np.arange(1, 13) * 0.02
    np.savetxt(series, np.column_stack([t, 0.5 * np.exp(-t / 0.12)]))
    capsys.readouterr()
    assert main(["fit-t2", "--series", str(series)]) == 0
    t2 = float([l for l in capsys.readouterr().out.splitlines() if l.startswith("t2_s=")][0].split("=")[1])
    assert t2 == pytest.approx(0.12, rel=1e-6)
    bad = tmp_path / "bad.txt"
    bad.write_text("[box]\nm0 = 1\n")
    assert main(["fit-t2", "--series", str(bad)]) == 2
    assert "error:" in capsys.readouterr().err


def test_export_image(tmp_path):
    img = ImageVolume(np.arange(12).reshape(3, 4) * (1 + 1j), (1.0, 1.0))
    p = export_image(img, str(tmp_path / "x.pgm"))
    assert np.array_equal(mrio.read_raw_grid(p + ".raw"), img.complex_image)


@pytest.mark.gpu
def test_cli_simulate_matches_oracle(tmp_path, capsys):
    """simulate (CUDA engine) -> echoes.mrsim + manifest + snapshot; the file's k-space matches the oracle."""
    from oracle import bloch_oracle as orc
    from paper_1305_6861_b200 import configs

    out = tmp_path / "run"
    assert main(["simulate", "--config", "0", "--subset", "8", "--snapshot", "0.0,0.02", "--out", str(out)]) == 0
    echoes = mrio.read_echo_file(str(out / "echoes.mrsim"))
    man = mrio.read_manifest(str(out / "echoes.mrsim"))
    wl = configs.make(0).subset(8)
    assert man["spin_count"] == wl.n_spins and man["n_acq"] == echoes.shape[0]
    assert len(man["trajectory"]) == echoes.shape[0] and man["kernel_ms"] > 0
    b = wl.block
    tabs = orc.precompute_tables(wl.sequence, snapshot_times=(0.0, 0.02))
    ref_e, ref_s = orc.compute_block(tabs, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)
    ref_e = np.asarray(ref_e).reshape(echoes.shape) / wl.n_spins
    assert orc.rel_l2(echoes, ref_e) <= 1e-4
    t, arr = mrio.read_snapshot_file(str(out / "snapshot_001.mrsim"))
    assert t == 0.02 and arr.shape == (wl.n_spins, 3)
    assert main(["recon", "--echoes", str(out / "echoes.mrsim"), "--trajectory", "se", "--size",
                 str(echoes.shape[1]), str(echoes.shape[0]), "--out", str(tmp_path / "img.pgm")]) == 0
    assert (tmp_path / "img.pgm.raw").exists()


@pytest.mark.gpu
def test_cli_simulate_device_raster_matches_host_path(tmp_path):
    """simulate --device-raster (spins rasterised on the GPU) writes the same k-space as the host path."""
    a, b = tmp_path / "host", tmp_path / "dev"
    assert main(["simulate", "--config", "0", "--precision", "64", "--out", str(a)]) == 0
    assert main(["simulate", "--config", "0", "--precision", "64", "--device-raster", "--out", str(b)]) == 0
    ea, eb = mrio.read_echo_file(str(a / "echoes.mrsim")), mrio.read_echo_file(str(b / "echoes.mrsim"))
    assert mrio.read_manifest(str(b / "echoes.mrsim"))["rasterised_on"] == "device"
    np.testing.assert_allclose(eb, ea, rtol=0, atol=1e-12 * np.abs(ea).max())

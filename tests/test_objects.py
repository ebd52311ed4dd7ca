"""Device-side object model: bloch_rasterize vs the host rasteriser.

CPU: the scene descriptions reproduce the seeded workloads on the host
(phantom.rasterize semantics, phantom.py:98-142), and the ctypes structs match
the C header's layout.  GPU: the device lattice, labels, tissue and spin order
are bit-identical to the host; analytic maps agree to a few ulps; computing
from device-resident spins gives the same k-space as the host-array path.
"""

import ctypes
import math
import os
import subprocess
import time

import numpy as np
import pytest

from paper_1305_6861_b200 import _capi, configs
from paper_1305_6861_b200.errors import InvalidParameter, SpinBudgetExceeded
from paper_1305_6861_b200.objects import DeviceScene, Ellipse, GaussianBumps, LabelBox, PolynomialField
from paper_1305_6861_b200.phantom import rasterize_arrays

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "bloch_b200.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(bloch_box_t), '
                   'sizeof(bloch_shape_t), sizeof(bloch_field_t), sizeof(bloch_coil_t), '
                   'offsetof(bloch_box_t, shape_begin), offsetof(bloch_field_t, poly_peak), '
                   'offsetof(bloch_field_t, bumps));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [ctypes.sizeof(_capi.BoxT), ctypes.sizeof(_capi.ShapeT), ctypes.sizeof(_capi.FieldT),
            ctypes.sizeof(_capi.CoilT), _capi.BoxT.shape_begin.offset, _capi.FieldT.poly_peak.offset,
            _capi.FieldT.bumps.offset]
    assert got == want


@pytest.mark.parametrize("index", [0, 2, 3])
def test_scene_reproduces_workload_on_host(index):
    """The scene's host restatement rasterises to exactly the workload's spins (small configs; cfg2/3 stride)."""
    wl = configs.make(index)
    sw = configs.scene(index)
    spins = rasterize_arrays(sw.scene.host_phantom(), sw.spacing, cap=sw.cap)
    b = wl.block
    assert spins["m0"].size == b.n
    for k, ref in (("pos", b.pos), ("m0", b.m0), ("t1", b.t1), ("t2", b.t2)):
        assert np.array_equal(spins[k], ref), k
    dw = sw.scene.host_field(spins["pos"], spins["delta_omega"])
    scale = max(np.abs(b.domega).max(), 1.0)
    np.testing.assert_allclose(dw, b.domega, rtol=0, atol=1e-12 * scale)


def test_scene_validation():
    with pytest.raises(InvalidParameter):
        DeviceScene([])
    with pytest.raises(InvalidParameter):
        DeviceScene([LabelBox((0, 0, 0), (1, 1, 1))], receive=object())


# -- GPU ----------------------------------------------------------------------------------------------------------


def _compare_spins(dev, b, tol_dw=1e-12, tol_w=1e-13):
    h = dev.to_host()
    assert dev.n == b.n
    for k, ref in (("pos", b.pos), ("m0", b.m0), ("t1", b.t1), ("t2", b.t2), ("mx", b.mx), ("my", b.my),
                   ("mz", b.mz)):
        assert np.array_equal(h[k], ref), k
    scale = max(np.abs(b.domega).max(), 1.0)
    np.testing.assert_allclose(h["delta_omega"], b.domega, rtol=0, atol=tol_dw * scale)
    w = np.asarray(b.weight)
    np.testing.assert_allclose(h["weight"], w, rtol=0, atol=tol_w * max(np.abs(w).max(), 1.0))


@pytest.mark.gpu
@pytest.mark.parametrize("index", [0, 1, 2, 3, 4])
def test_device_rasterize_matches_host(index):
    import torch

    from paper_1305_6861_b200.engine import get_engine

    eng = get_engine(0, 32)
    sw = configs.scene(index)
    t0 = time.perf_counter()
    dev = sw.rasterize(eng)
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    wl = configs.make(index)
    t_host = time.perf_counter() - t0
    _compare_spins(dev, wl.block)
    print(f"cfg{index}: {dev.n} spins, device rasterise {t_dev * 1e3:.1f} ms, host build {t_host * 1e3:.0f} ms")


@pytest.mark.gpu
@pytest.mark.parametrize("index", [0, 4])
def test_compute_from_device_spins(index):
    """Device-resident spins through compute_device == host arrays through compute (same engine)."""
    import torch

    from paper_1305_6861_b200.engine import get_engine, precompute_sequence_tables

    eng = get_engine(0, 32)
    wl = configs.make(index).subset(4) if index == 4 else configs.make(index)
    sw = configs.scene(index)
    dev = sw.rasterize(eng)
    tables = precompute_sequence_tables(sw.sequence)
    b = configs.make(index).block
    ref, _ = eng.compute(tables, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight)
    f = eng.set_tables(tables)
    out = torch.zeros((dev.n_coils, f["n_acq"], f["max_ns"]), dtype=torch.complex128, device=dev.pos.device)
    torch.cuda.synchronize()
    eng.compute_device(tables, dev.pointers(), dev.n, dev.n_coils, out.data_ptr(), sync=True)
    got = out.cpu().numpy()
    ref = np.asarray(ref).reshape(got.shape)
    if index == 0:
        assert np.array_equal(got, ref)  # identical inputs, deterministic kernel
    else:
        assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)
    del wl


@pytest.mark.gpu
def test_run_with_device_scene_matches_host_run():
    from paper_1305_6861_b200.engine import Experiment, run

    sw = configs.scene(0)
    r_dev = run(Experiment(sequence=sw.sequence, phantom=sw.scene, spacing=sw.spacing, snapshot_times=(0.01,)))
    r_host = run(Experiment(sequence=sw.sequence, phantom=sw.scene.host_phantom(), spacing=sw.spacing,
                            snapshot_times=(0.01,)))
    assert r_dev.spin_count == r_host.spin_count
    assert np.array_equal(r_dev.echo_matrix(), r_host.echo_matrix())
    assert np.array_equal(r_dev.snapshots[0][1], r_host.snapshots[0][1])


@pytest.mark.gpu
def test_device_rasterize_errors_and_general_scene():
    from paper_1305_6861_b200.engine import get_engine
    from paper_1305_6861_b200.objects import rasterize_device
    from paper_1305_6861_b200.system import CoilArray, GaussianCoil

    eng = get_engine(0, 32)
    box = LabelBox((-0.01, -0.01, -0.01), (0.02, 0.02, 0.02), m0=0.0,
                   shapes=(Ellipse((0.0, 0.0), (0.008, 0.005), angle=0.3, m0=1.0, t1=0.8, t2=0.0),))
    with pytest.raises(InvalidParameter):
        rasterize_device(DeviceScene([box]), (0.001,) * 3, eng)
    ok = LabelBox((-0.01, -0.01, -0.01), (0.02, 0.02, 0.02), m0=0.5, t1=1.2, t2=0.09, delta_omega=3.0,
                  shapes=(Ellipse((0.0, 0.0, 0.0), (0.008, 0.005, 0.004), angle=0.3, m0=1.0, t1=0.8, t2=0.05,
                                  delta_omega=-7.0),
                          Ellipse((0.003, 0.0), (0.002, 0.002), m0=0.0)))
    with pytest.raises(SpinBudgetExceeded):
        rasterize_device(DeviceScene([ok]), (0.0001,) * 3, eng, cap=1000)
    # two boxes, constant + polynomial (scale mode) + 3-D bumps, two coils: device vs the host restatement
    box2 = LabelBox((0.02, -0.005, -0.004), (0.01, 0.01, 0.008), m0=0.7, t1=0.9, t2=0.07)
    sc = DeviceScene([ok, box2], const_dw=1.5,
                     polynomial=PolynomialField((0.5, -1.0, 2.0), ((0, 0, 0), (1, 2, 0), (0, 1, 3)), 0.02,
                                                scale=40.0),
                     bumps=GaussianBumps(((0.0, 0.0, 0.0), (0.01, 0.0)), (0.004, 0.006), (30.0, -20.0)),
                     receive=CoilArray([GaussianCoil((0.05, 0.0, 0.0), 0.03, 0.2),
                                        GaussianCoil((0.0, 0.05, 0.01), 0.04, 1.7)]))
    spacing = (0.0011, 0.0009, 0.001)
    dev = rasterize_device(sc, spacing, eng).to_host()
    host = rasterize_arrays(sc.host_phantom(), spacing)
    for k in ("pos", "m0", "t1", "t2"):
        assert np.array_equal(dev[k], host[k]), k
    np.testing.assert_allclose(dev["delta_omega"], sc.host_field(host["pos"], host["delta_omega"]), rtol=1e-13,
                               atol=1e-12)
    from paper_1305_6861_b200.system import receive_weights

    np.testing.assert_allclose(dev["weight"], receive_weights(type("S", (), {"receive": sc.receive})(),
                                                              host["pos"]), rtol=0, atol=1e-14)
    assert math.isclose(float(np.sum(dev["m0"])), float(np.sum(host["m0"])), rel_tol=0, abs_tol=0)


def _random_scene(seed):
    from paper_1305_6861_b200.system import CoilArray, GaussianCoil, UniformSensitivity

    rng = np.random.default_rng(seed)
    boxes = []
    for _ in range(int(rng.integers(1, 4))):
        origin = tuple(rng.uniform(-0.05, 0.03, 3))
        size = tuple(rng.uniform(0.005, 0.04, 3))
        shapes = []
        for _ in range(int(rng.integers(0, 6))):
            dim = int(rng.integers(2, 4))
            c = tuple(np.add(origin, rng.uniform(0, 1, 3) * size)[:dim])
            ax = tuple(rng.uniform(0.002, 0.02, dim))
            shapes.append(Ellipse(c, ax, angle=float(rng.uniform(0, math.pi)), m0=float(rng.choice([0.0, rng.uniform(0.1, 1)])),
                                  t1=float(rng.uniform(0.3, 2)), t2=float(rng.uniform(0.02, 0.3)),
                                  delta_omega=float(rng.normal(0, 50))))
        boxes.append(LabelBox(origin, size, m0=float(rng.choice([0.0, 0.5])), t1=1.0, t2=0.1,
                              delta_omega=float(rng.normal(0, 10)), shapes=tuple(shapes)))
    poly = None
    if rng.random() < 0.5:
        k = int(rng.integers(1, 6))
        poly = PolynomialField(tuple(rng.normal(0, 1, k)), tuple(tuple(int(v) for v in rng.integers(0, 3, 3)) for _ in range(k)),
                               0.05, scale=float(rng.uniform(1, 50)), peak=(None if rng.random() < 0.5 else 300.0))
    bumps = None
    if rng.random() < 0.5:
        k = int(rng.integers(1, 4))
        bumps = GaussianBumps(tuple(tuple(rng.uniform(-0.05, 0.05, int(rng.integers(2, 4)))) for _ in range(k)),
                              tuple(rng.uniform(0.005, 0.03, k)), tuple(rng.normal(0, 100, k)))
    rx = [UniformSensitivity(), CoilArray([GaussianCoil(tuple(rng.uniform(-0.1, 0.1, 3)), 0.05, float(rng.uniform(0, 6)))
                                           for _ in range(int(rng.integers(1, 5)))])][int(rng.integers(0, 2))]
    spacing = tuple(rng.uniform(0.0015, 0.004, 3))
    return DeviceScene(boxes, const_dw=float(rng.normal(0, 5)), polynomial=poly, bumps=bumps, receive=rx), spacing


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(24))
def test_device_rasterize_random_scenes(seed):
    from paper_1305_6861_b200.engine import get_engine
    from paper_1305_6861_b200.objects import rasterize_device
    from paper_1305_6861_b200.system import receive_weights

    scene, spacing = _random_scene(seed)
    host = rasterize_arrays(scene.host_phantom(), spacing)
    if host["m0"].size == 0:
        with pytest.raises(InvalidParameter):
            rasterize_device(scene, spacing, get_engine(0, 32))
        return
    dev = rasterize_device(scene, spacing, get_engine(0, 32)).to_host()
    for k in ("pos", "m0", "t1", "t2"):
        assert np.array_equal(dev[k], host[k]), (seed, k)
    dw = scene.host_field(host["pos"], host["delta_omega"])
    np.testing.assert_allclose(dev["delta_omega"], dw, rtol=1e-12, atol=1e-9)
    w = receive_weights(type("S", (), {"receive": scene.receive})(), host["pos"])
    np.testing.assert_allclose(dev["weight"], w, rtol=0, atol=1e-13)

"""CPU: the ten-ellipse head phantom (phantom.py:145-205) against vectors made by the reference
(tests/golden/make_golden_head.py): M0 labels on 86k points, including a grid that grazes the
ellipse boundaries, and the rasterised spins of acceptance criterion 6 — bit for bit."""

import numpy as np
import pytest

from conftest import load_golden
from paper_1305_6861_b200 import shepp_logan, shepp_logan_m0
from paper_1305_6861_b200.errors import InvalidParameter
from paper_1305_6861_b200.phantom import rasterize, rasterize_arrays


def test_m0_labels_bit_identical():
    g = load_golden("head")
    pts = g["points"]
    got = shepp_logan_m0(pts[:, 0], pts[:, 1], float(g["scale"]))
    assert np.array_equal(got, g["m0"])
    # scalar form, as the reference calls it
    assert shepp_logan_m0(float(pts[7, 0]), float(pts[7, 1]), float(g["scale"])) == g["m0"][7]


def test_rasterised_head_matches_reference():
    g = load_golden("head")
    spins = rasterize_arrays(shepp_logan(float(g["scale"])), tuple(g["spacing"]))
    assert spins["pos"].shape[0] == g["spin_pos"].shape[0] == 2129
    assert np.array_equal(spins["pos"], g["spin_pos"])
    assert np.array_equal(spins["m0"], g["spin_m0"])
    assert np.all(spins["t1"] == 1.0) and np.all(spins["t2"] == 0.2)
    listed = rasterize(shepp_logan(float(g["scale"])), tuple(g["spacing"]))
    assert len(listed) == 2129


def test_scale_must_be_positive():
    with pytest.raises(InvalidParameter):
        shepp_logan(0.0)

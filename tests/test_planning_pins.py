"""Pins of the planning oracle (oracle/planning.py) against what the paper,
SPEC worked examples and independent routines fix (-m "not gpu")."""
import math

import numpy as np
import pytest

from oracle import planning as P
from paper_2409_18122_b200 import workloads as W


# ----------------------------------------------------------------- N4 ledger

def test_ledger_closed_form_and_retention():
    prev = np.array([[0.0, 1.0, 5.0], [0.0, 2.0, 5.0], [0.0, 3.0, 5.0]], np.float32)
    cur = prev.copy()
    cur[:, 0] = [3.0, 4.0, 12.0]          # |(3, 4, 12)| = 13 exactly
    cur[2, 1] = 3.5                        # moved 0.5 along z
    w_prev = np.array([7.0, 7.0, 0.25], np.float32)
    w = P.ledger_update(prev, cur, w_prev)
    assert w[0] == 13.0
    assert w[1] == np.float32(0.5)
    assert w[2] == np.float32(0.25)       # unchanged mean: retains its previous value


def test_ledger_matches_numpy_norm():
    rng = np.random.default_rng(3)
    prev = rng.normal(0, 10, (3, 500)).astype(np.float32)
    cur = prev + rng.normal(0, 0.1, (3, 500)).astype(np.float32) * (rng.random(500) < 0.7)
    w_prev = rng.random(500).astype(np.float32)
    w = P.ledger_update(prev, cur, w_prev)
    ref = np.linalg.norm(cur.astype(np.float64) - prev.astype(np.float64), axis=0).astype(np.float32)
    moved = np.any(cur != prev, axis=0)
    assert np.array_equal(w[moved], ref[moved])
    assert np.array_equal(w[~moved], w_prev[~moved])
    assert np.all(w >= 0)


# ----------------------------------------------------------------- N2 region utility

def test_region_utility_spec_examples():
    # cell with displacements {0.1, 0.3} -> 0.2; cell with a single Gaussian at 0 -> 0; empty -> 0
    means = np.array([[0.5, 1.0, 3.0], [0.5, 1.0, 0.5], [0.5, 1.0, 0.5]], np.float32)
    w = np.array([0.1, 0.3, 0.0], np.float32)
    om, cnt = P.region_utility(means, w, None, (0.0, 0.0, 0.0), 2.5, (2, 1, 1))
    assert om[0] == pytest.approx(0.2, rel=1e-7) and cnt[0] == 2
    assert om[1] == 0.0 and cnt[1] == 1
    om, cnt = P.region_utility(means, w, None, (0.0, 0.0, 0.0), 2.5, (3, 1, 1))
    assert cnt[2] == 0 and om[2] == 0.0


def test_region_utility_matches_bincount_and_filters():
    rng = np.random.default_rng(4)
    n = 3000
    means = rng.uniform(-6, 6, (3, n)).astype(np.float32)
    w = rng.random(n).astype(np.float32)
    flags = (rng.random(n) < 0.2).astype(np.uint8) * P.FLAG_NO_GAIN
    origin, size, dims = (-5.0, -5.0, -5.0), 2.5, (4, 4, 4)     # the box [-5, 5]^3: some Gaussians outside
    om, cnt = P.region_utility(means, w, flags, origin, size, dims)
    # independent route: vectorised cell index + bincount
    ijk = np.floor((means.astype(np.float64) - np.array(origin)[:, None]) / size).astype(int)
    ok = np.all((ijk >= 0) & (ijk < np.array(dims)[:, None]), axis=0) & (flags == 0)
    flat = (ijk[2] * dims[1] + ijk[1]) * dims[0] + ijk[0]
    c = np.bincount(flat[ok], minlength=64)
    s = np.bincount(flat[ok], weights=w[ok].astype(np.float64), minlength=64)
    assert np.array_equal(cnt, c)
    ref = np.where(c > 0, s / np.maximum(c, 1), 0.0)
    assert np.allclose(om, ref, rtol=1e-12, atol=0)
    assert cnt.sum() < n and cnt.sum() == ok.sum()


def test_region_boundaries_belong_to_upper_cell():
    means = np.array([[2.5, 2.4999998], [0.0, 0.0], [0.0, 0.0]], np.float32)
    om, cnt = P.region_utility(means, np.array([1.0, 3.0], np.float32), None, (0, 0, 0), 2.5, (2, 1, 1))
    assert list(cnt) == [1, 1] and list(om) == [3.0, 1.0]


# ----------------------------------------------------------------- N2 view placement

def test_view_distance_spec_example_and_min_fov():
    cam90 = W.Camera(640, 480, 320.0, 320.0, 320.0, 240.0, 0.1, 10.0)   # hfov = 90 deg, vfov < 90
    h, v = P.fov(cam90)
    assert h == pytest.approx(math.pi / 2, rel=1e-14)
    assert v == pytest.approx(2 * math.atan(240 / 320), rel=1e-14)
    sq = W.Camera(640, 640, 320.0, 320.0, 320.0, 320.0, 0.1, 10.0)        # square: both 90 deg
    assert P.view_distance(2.5, sq) == pytest.approx(1.25, rel=1e-14)     # tan 45 = 1
    assert P.view_distance(2.5, cam90) == pytest.approx(1.25 / (240 / 320), rel=1e-12)   # vfov is the min
    # off-centre principal point: the field of view is the angle [0, W] subtends
    off = W.Camera(640, 640, 320.0, 320.0, 0.0, 320.0, 0.1, 10.0)
    assert P.fov(off)[0] == pytest.approx(math.atan(2.0), rel=1e-14)


def test_view_ring_geometry_and_visibility():
    from oracle import oracle as O
    cam = W.Camera(640, 480, 500.0, 500.0, 320.0, 240.0, 0.2, 15.0)
    cen = np.array([[3.0, -2.0, 0.5], [10.0, 4.0, 0.5]])
    x, y, z, yaw = P.view_ring(cen, 2.5, cam, 8, 0.5)
    d = P.view_distance(2.5, cam)
    assert x.shape == (16,)
    for r in range(2):
        for j in range(8):
            k = r * 8 + j
            assert math.hypot(x[k] - cen[r, 0], y[k] - cen[r, 1]) == pytest.approx(d, rel=1e-6)
            assert math.atan2(y[k] - cen[r, 1], x[k] - cen[r, 0]) % (2 * math.pi) == pytest.approx(
                2 * math.pi * j / 8, abs=1e-6)
            # facing the centroid: it lies on the optical axis (visible, lateral slack symmetric)
            sg, _ = O.visibility_slacks(cen[r], (x[k], y[k], z[k], yaw[k]), cam)
            assert np.all(sg >= 0)
            assert sg[2] == pytest.approx(sg[3], rel=1e-5)


# ----------------------------------------------------------------- N2 cost-benefit

def test_cost_benefit_spec_examples():
    assert P.cost_benefit([1.0], [0.0]) == (0, 1.0)                       # e^0 = 1
    b, s = P.cost_benefit([1.0, 2.0], [1.0, 2.0])                          # 0.3679 vs 0.2707
    assert b == 0 and s == pytest.approx(math.exp(-1), rel=1e-15)
    assert 2.0 / math.exp(2.0) == pytest.approx(0.2707, abs=1e-4)
    # ties: smaller d wins, then smaller index
    b, _ = P.cost_benefit([math.e, 1.0], [1.0, 0.0])
    assert b == 1
    b, _ = P.cost_benefit([1.0, 1.0, 1.0], [0.5, 0.5, 0.5])
    assert b == 0
    assert P.cost_benefit([], []) == (-1, -math.inf)

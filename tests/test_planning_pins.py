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


# ----------------------------------------------------------------- N3 motion-primitive tree

class _Params:
    def __init__(self, **kw):
        d = dict(n_v=3, n_omega=5, v_max=0.6, omega_max=0.9, dt=1.0, lambda_t=1.0, samples=5, max_depth=8,
                 goal_radius=0.5, lattice_xy=0.1, lattice_deg=10.0, beam=4096, n_traj=10, z=0.5)
        d.update(kw)
        self.__dict__.update(d)


def test_controls_paper_grid():
    c = P.controls(3, 5, 0.6, 0.9)                       # N_v = 3, v_max = 0.6, N_w = 5, w_max = 0.9
    assert len(c) == 15
    vs = sorted({v for v, _ in c})
    ws = sorted({w for _, w in c})
    assert vs == pytest.approx([0.0, 0.3, 0.6], abs=1e-7)
    assert ws == pytest.approx([-0.9, -0.45, 0.0, 0.45, 0.9], abs=1e-7)
    assert P.controls(1, 1, 0.6, 0.9) == [(float(np.float32(0.6)), 0.0)]


def test_unicycle_closed_form_spec_examples():
    assert P.unicycle_at(0, 0, 0, 1.0, 0.0, 1.0) == pytest.approx((1.0, 0.0, 0.0))
    x, y, th = P.unicycle_at(0, 0, 0, 1.0, math.pi / 2, 1.0)
    assert (x, y, th) == pytest.approx((2 / math.pi, 2 / math.pi, math.pi / 2), rel=1e-15)
    assert P.unicycle_at(1.5, -2.0, 0.3, 0.0, 0.0, 1.0) == (1.5, -2.0, 0.3)


def test_tree_open_map_straight_goal_cost():
    """empty map, goal 3 m ahead -> the selected candidate reaches the goal with cost
    within 10 % of 3 m / v_max (lambda_t + v_max^2)."""
    res = P.plan_tree(lambda pts: np.zeros(len(pts), bool), (0.0, 0.0, 0.0), (3.0, 0.0), _Params(beam=256))
    assert res["reached"]
    best = res["nodes"][res["cands"][0]]
    assert (best[0] - 3.0) ** 2 + best[1] ** 2 <= 0.25
    bound = 3.0 / 0.6 * (1.0 + 0.36)
    assert best[3] <= 1.1 * bound
    costs = [res["nodes"][i][3] for i in res["cands"]]
    assert costs == sorted(costs) and len(costs) == 10


def test_tree_equals_exhaustive_enumeration():
    """without the lattice and with an unbounded beam, the cheapest candidate equals the
    minimum over the exhaustively enumerated control sequences (stopping at the goal region)."""
    import itertools
    p = _Params(max_depth=3, lattice_xy=0.0, beam=10 ** 6, goal_radius=0.3)
    goal = (1.0, 0.4)
    free = lambda pts: np.zeros(len(pts), bool)
    res = P.plan_tree(free, (0.0, 0.0, 0.2), goal, p)
    ctl = P.controls(3, 5, 0.6, 0.9)
    best = math.inf
    for seq in itertools.chain.from_iterable(itertools.product(range(15), repeat=d) for d in (1, 2, 3)):
        x, y, th, g = 0.0, 0.0, float(np.float32(0.2)), 0.0
        for k, pi in enumerate(seq):
            v, w = ctl[pi]
            x, y, th = P.unicycle_at(x, y, th, v, w, 1.0)
            th = P.wrap_pi(th)
            g += (1.0 + v * v + w * w) * 1.0
            if (x - 1.0) ** 2 + (y - float(np.float32(0.4))) ** 2 <= float(np.float32(0.3)) ** 2:
                if k == len(seq) - 1:
                    best = min(best, g)
                break
    assert res["reached"] and res["nodes"][res["cands"][0]][3] == pytest.approx(best, rel=1e-12)


def _primitive_samples(par, child, ctl, S=5):
    """The sample states of the control leading from node par to node child (found by its end state)."""
    for v, w in ctl:
        e = P.unicycle_at(par[0], par[1], par[2], v, w, 1.0)
        if abs(e[0] - child[0]) < 1e-12 and abs(e[1] - child[1]) < 1e-12:
            return [P.unicycle_at(par[0], par[1], par[2], v, w, j / (S - 1)) for j in range(1, S)]
    raise AssertionError("no control reproduces the child")


def test_tree_wall_samples_avoid_obstacle_and_fallback():
    wall = lambda pts: (np.abs(pts[:, 0] - 1.5) < 0.3) & (np.abs(pts[:, 1]) < 1.0)
    res = P.plan_tree(wall, (0.0, 0.0, 0.0), (3.0, 0.0), _Params(max_depth=6, beam=512))
    assert res["reached"]
    ctl = P.controls(3, 5, 0.6, 0.9)
    nodes = res["nodes"]
    for i in res["cands"]:      # re-check every sample of every primitive of every candidate
        while nodes[i][4] >= 0:
            smp = _primitive_samples(nodes[nodes[i][4]], nodes[i], ctl)
            assert not np.any(wall(np.array([[x, y, 0.5] for x, y, _ in smp], np.float32)))
            i = nodes[i][4]
    # a goal behind a closed wall: nothing reaches it -> the nodes closest to the goal
    closed = lambda pts: pts[:, 0] > 0.7
    r2 = P.plan_tree(closed, (0.0, 0.0, 0.0), (3.0, 0.0), _Params(max_depth=2))
    assert not r2["reached"] and len(r2["cands"]) == 10
    hs = [math.hypot(3.0 - r2["nodes"][i][0], r2["nodes"][i][1]) for i in r2["cands"]]
    assert hs == sorted(hs)


def test_double_integrator_matches_ode_and_heading():
    """The double-integrator sampler's oracle against an ODE integration of p'' = a, and its heading
    against the velocity direction; zero velocity has heading 0 (atan2(0, 0))."""
    from scipy.integrate import solve_ivp
    start, v0, a, dt, T = (5.0, -1.0, 0.5, 0.0), (1.0, 0.25), (-0.5, 0.75), 0.1, 40
    x, y, z, yaw = P.double_integrator(start, v0, a, dt, T)
    f = lambda v: float(np.float32(v))
    sol = solve_ivp(lambda t, s: [s[2], s[3], f(a[0]), f(a[1])], (0, T * f(dt)),
                    [f(start[0]), f(start[1]), f(v0[0]), f(v0[1])], t_eval=(np.arange(T) + 1) * f(dt),
                    rtol=1e-12, atol=1e-12)
    assert np.allclose(x, sol.y[0], atol=1e-9) and np.allclose(y, sol.y[1], atol=1e-9)
    assert np.allclose(yaw, np.arctan2(sol.y[3], sol.y[2]), atol=1e-9)
    assert np.all(z == f(start[2]))
    # braking to rest at t = 1 s exactly: heading 0 there, and reversing after
    x, y, z, yaw = P.double_integrator((0, 0, 0, 0), (1.0, 0.0), (-1.0, 0.0), 0.5, 4)
    assert yaw[1] == 0.0 and abs(yaw[2]) == math.pi and x[1] == 0.5

"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test pins oracle arithmetic to something other than itself: printed/hand
values (tests/golden/*.json, each with its citation), closed forms, invariants,
independent library routines (scipy Rotation, numpy inverse covariance, numpy
pinhole projection, an ODE integrator) and brute force on tiny inputs.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.integrate import solve_ivp
from scipy.spatial.transform import Rotation

from oracle import oracle as O
from paper_2409_18122_b200 import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------- collision (O2)

@pytest.mark.parametrize("case", _gold("collision_cases.json")["cases"], ids=lambda c: c["name"])
def test_collision_golden(case):
    q = O.collision_q(case["mu"], case["quat"], case["s"], case["r_robot"], case["lambda_g"], case["p"])
    assert q == pytest.approx(case["q"], rel=1e-12)
    assert (q < 1.0) == case["collide"]


def _scipy_q(mu, quat, s, r, lam, p):
    """Independent route: Mahalanobis distance d^T Sigma'^{-1} d with Sigma' = R diag(a^2) R^T,
    R from scipy (scalar-last quaternion), inverse by numpy.linalg.inv."""
    R = Rotation.from_quat([quat[1], quat[2], quat[3], quat[0]]).as_matrix()
    a = lam * np.asarray(s, float) + r
    cov = R @ np.diag(a ** 2) @ R.T
    d = np.asarray(p, float) - np.asarray(mu, float)
    return float(d @ np.linalg.inv(cov) @ d)


def test_collision_matches_inverse_covariance_route():
    rng = np.random.default_rng(11)
    for _ in range(300):
        mu = rng.uniform(-20, 20, 3)
        q = rng.standard_normal(4)
        q /= np.linalg.norm(q)
        s = np.exp(rng.uniform(np.log(0.005), np.log(0.5), 3))
        r = rng.uniform(0.2, 0.6)
        p = mu + rng.normal(0, 1.0, 3)
        ours = O.collision_q(mu, q, s, r, 3.0, p)
        ref = _scipy_q(mu, q, s, r, 3.0, p)
        assert ours == pytest.approx(ref, rel=1e-9)


def test_collision_unnormalised_quaternion_is_normalised():
    q = np.array([0.3, -0.2, 0.9, 0.1])
    a = O.collision_q([0, 0, 0], q, [0.1, 0.2, 0.3], 0.3, 3.0, [0.2, 0.3, -0.1])
    b = O.collision_q([0, 0, 0], 7.5 * q, [0.1, 0.2, 0.3], 0.3, 3.0, [0.2, 0.3, -0.1])
    assert a == pytest.approx(b, rel=1e-13)


def test_isotropic_reduces_to_sphere_distance():
    """isotropic -> ||d|| < r_robot + lambda_g r, for any rotation."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        r = rng.uniform(0.01, 0.3)
        q = rng.standard_normal(4)
        p = rng.normal(0, 1, 3)
        mu = rng.normal(0, 1, 3)
        gamma = 0.3 + 3.0 * r
        qq = O.collision_q(mu, q, [r, r, r], 0.3, 3.0, p)
        assert qq == pytest.approx(np.sum((p - mu) ** 2) / gamma ** 2, rel=1e-12)
        assert (qq < 1) == (np.linalg.norm(p - mu) < gamma)


def test_rotation_invariance():
    rng = np.random.default_rng(5)
    for _ in range(100):
        q = rng.standard_normal(4)
        q /= np.linalg.norm(q)
        s = rng.uniform(0.02, 0.3, 3)
        d = rng.normal(0, 0.5, 3)
        g = rng.standard_normal(4)
        g /= np.linalg.norm(g)
        Rg = Rotation.from_quat([g[1], g[2], g[3], g[0]])
        # compose rotation: new orientation = Rg * R(q), new point = Rg d
        Rq = Rotation.from_quat([q[1], q[2], q[3], q[0]])
        xyzw = (Rg * Rq).as_quat()
        q2 = [xyzw[3], xyzw[0], xyzw[1], xyzw[2]]
        a = O.collision_q([0, 0, 0], q, s, 0.3, 3.0, d)
        b = O.collision_q([0, 0, 0], q2, s, 0.3, 3.0, Rg.apply(d))
        assert a == pytest.approx(b, rel=1e-10)


def test_threshold_points_are_in_band():
    """p = mu + R (a * u), |u| = 1 gives q = 1 in real arithmetic (SURVEY [A2])."""
    rng = np.random.default_rng(9)
    for _ in range(50):
        q = rng.standard_normal(4)
        q /= np.linalg.norm(q)
        s = rng.uniform(0.02, 0.3, 3)
        u = rng.standard_normal(3)
        u /= np.linalg.norm(u)
        R = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()
        a = 3.0 * s + 0.3
        p = R @ (a * u)
        qq = O.collision_q([0, 0, 0], q, s, 0.3, 3.0, p)
        assert abs(qq - 1.0) < 1e-12


def test_principal_axis_variant():
    """principal axis taken as the radius; equals the ellipsoid rule when isotropic."""
    rng = np.random.default_rng(4)
    for _ in range(100):
        q = rng.standard_normal(4)
        r = rng.uniform(0.02, 0.3)
        p = rng.normal(0, 1, 3)
        a = O.collision_q([0, 0, 0], q, [r, r, r], 0.35, 3.0, p, rule=0)
        b = O.collision_q([0, 0, 0], q, [r, r, r], 0.35, 3.0, p, rule=1)
        assert a == pytest.approx(b, rel=1e-12)
    # anisotropic: radius = lambda_g * max s + r_robot regardless of orientation
    q = O.collision_q([0, 0, 0], [0.2, 0.5, -0.3, 0.7], [0.05, 0.2, 0.1], 0.3, 3.0, [0.0, 0.0, 0.89], rule=1)
    assert q == pytest.approx((0.89 / 0.9) ** 2, rel=1e-12)


# ----------------------------------------------------------------- visibility (O3)

def _cam(d, **over):
    d = dict(d)
    d.update(over)
    return W.Camera(d["width"], d["height"], d["fx"], d["fy"], d["cx"], d["cy"], d["z_near"], d["z_far"])


@pytest.mark.parametrize("case", _gold("visibility_cases.json")["cases"], ids=lambda c: c["name"])
def test_visibility_golden(case):
    g = _gold("visibility_cases.json")
    cam = _cam(g["camera"], **({"z_far": case["z_far"]} if "z_far" in case else {}))
    sg, sc = O.visibility_slacks(case["mu"], case["pose"], cam)
    assert bool(np.all(sg >= 0)) == case["visible"]
    on_boundary = bool(np.any(np.abs(sg) <= 1e-12 * sc))
    assert on_boundary == case["boundary"]


def _pinhole_uvd(mu, pose, cam):
    """The paper's projection mu_2D = K R^T (mu - T)/d, d = e3^T R^T (mu - T),
    with R = world-from-camera whose columns are the camera axes (right, down, forward)."""
    c, s = math.cos(pose[3]), math.sin(pose[3])
    R = np.array([[s, 0.0, c], [-c, 0.0, s], [0.0, -1.0, 0.0]])
    Kmat = np.array([[cam.fx, 0, cam.cx], [0, cam.fy, cam.cy], [0, 0, 1.0]])
    pc = R.T @ (np.asarray(mu, float) - np.asarray(pose[:3], float))
    d = pc[2]
    uvw = Kmat @ pc
    return uvw[0] / d, uvw[1] / d, d


def test_projection_spec_example_of_the_helper():
    """SPEC.md:54 pins the projection helper used below: mu=(0,0,2), f=100, c=50 -> (50,50), d=2.
    (optical axis +z: a pose whose forward axis is world +z is built directly here)."""
    Kmat = np.array([[100, 0, 50], [0, 100, 50], [0, 0, 1.0]])
    pc = np.array([0.0, 0.0, 2.0])
    uvw = Kmat @ pc
    assert (uvw[0] / pc[2], uvw[1] / pc[2], pc[2]) == (50.0, 50.0, 2.0)


def test_visibility_equals_projection_inside_image():
    rng = np.random.default_rng(21)
    cam = W.Camera(320, 240, 250.0, 250.0, 160.0, 120.0, 0.1, 6.0)
    cam_off = W.Camera(320, 240, 250.0, 260.0, 150.0, 100.0, 0.2, 6.0)   # off-centre principal point
    nvis = 0
    for cm in (cam, cam_off):
        for _ in range(4000):
            pose = [rng.uniform(-3, 3), rng.uniform(-3, 3), rng.uniform(0, 2), rng.uniform(-np.pi, np.pi)]
            mu = np.array(pose[:3]) + rng.normal(0, 3, 3)
            u, v, d = _pinhole_uvd(mu, pose, cm)
            ref = (cm.z_near <= d <= cm.z_far) and (0 <= u <= cm.width) and (0 <= v <= cm.height)
            sg, sc = O.visibility_slacks(mu, pose, cm)
            if np.any(np.abs(sg) <= 1e-9 * sc):
                continue
            assert bool(np.all(sg >= 0)) == ref
            nvis += ref
    assert nvis > 300


# ----------------------------------------------------------------- classification (O4)

@pytest.mark.parametrize("case", _gold("classify_cases.json")["cases"], ids=lambda c: c["name"])
def test_classify_golden(case):
    c = O.classify(np.array(case["w"], np.float32), None, variant=case["variant"], k_sigma=0.5)
    assert c["mean"] == pytest.approx(case["mean"], rel=1e-14)
    assert c["std"] == pytest.approx(case["std"], rel=1e-14, abs=1e-15)
    assert c["tau_hi"] == pytest.approx(case["tau_hi"], rel=1e-14)
    assert c["tau_lo"] == pytest.approx(case["tau_lo"], rel=1e-14)
    assert list(c["cls"]) == case["cls"]


def test_classify_scaling_invariance_and_flags():
    rng = np.random.default_rng(2)
    w = rng.uniform(0, 1, 1000).astype(np.float32)
    a = O.classify(w)
    b = O.classify((w * np.float32(4.0)).astype(np.float32))     # power-of-two scale: exact in fp32
    assert np.array_equal(a["cls"], b["cls"])
    flags = np.zeros(1000, np.uint8)
    flags[::3] = W.FLAG_NO_GAIN
    c = O.classify(w, flags)
    assert np.all(c["cls"][::3] == 2)
    sel = w[flags == 0].astype(np.float64)
    assert c["mean"] == pytest.approx(sel.mean(), rel=1e-12)
    assert c["std"] == pytest.approx(sel.std(), rel=1e-10)     # numpy population std


def test_classify_override():
    w = np.array([0.1, 0.5, 0.9], np.float32)
    c = O.classify(w, tau_hi=0.6, tau_lo=0.2)
    assert list(c["cls"]) == [-1, 0, 1]


# ----------------------------------------------------------------- xi and gain (O5)

def _front_map(ws, cls_w=None, dist=3.0):
    """Gaussians placed on the optical axis of a camera at the origin, yaw 0, spaced in y
    inside the frustum (visible), far from the robot (no collision)."""
    n = len(ws)
    means = np.zeros((3, n), np.float32)
    means[0] = dist
    means[1] = np.linspace(-0.5, 0.5, n) if n > 1 else 0.0
    means[2] = 0.0
    quats = np.zeros((4, n), np.float32)
    quats[0] = 1
    scales = np.full((3, n), 0.05, np.float32)
    return means, quats, scales


XI_CAM = W.Camera(64, 48, 50.0, 50.0, 32.0, 24.0, 0.1, 5.0)


def _wp(means, quats, scales, w, flags=None, tau=(0.6, 0.2), pose=(0.0, 0.0, 0.0, 0.0), lam=1.0):
    c = O.classify(np.asarray(w, np.float32), flags, tau_hi=tau[0], tau_lo=tau[1])
    r = O.waypoints(means, quats, scales, flags, c["cls"], c["u"], W.Robot(0.3), XI_CAM,
                    np.array([pose[0]]), np.array([pose[1]]), np.array([pose[2]]), np.array([pose[3]]))
    return r, c


def test_xi_spec_examples():
    """Eq. equ:view_util: 4 H + 1 L visible, lambda_xi = 1 -> 3."""
    w = [0.9, 0.9, 0.9, 0.9, 0.1]
    r, _ = _wp(*_front_map(w), w)
    assert r["nh"][0] - r["nl"][0] == 3
    w7 = [0.1] * 7
    r, _ = _wp(*_front_map(w7), w7)
    assert r["nh"][0] - r["nl"][0] == -7
    # nothing visible: same Gaussians behind the camera
    m, q, s = _front_map(w)
    m[0] = -3.0
    r, _ = _wp(m, q, s, w)
    assert r["nh"][0] == 0 and r["nl"][0] == 0 and r["gain"][0] == 0.0


def test_trace_proxy_equals_dense_matrix_trace():
    """Eq. eq:nbv with J replaced by its binary sparsity pattern: gain equals
    Tr(J Sigma J^T), Sigma = diag(u), J = binary visibility selection."""
    rng = np.random.default_rng(7)
    n = 40
    means = np.stack([rng.uniform(-1, 6, n), rng.uniform(-3, 3, n), rng.uniform(-2, 2, n)]).astype(np.float32)
    quats = np.tile(np.array([[1], [0], [0], [0]], np.float32), (1, n))
    scales = np.full((3, n), 0.05, np.float32)
    w = rng.uniform(0, 1, n).astype(np.float32)
    r, c = _wp(means, quats, scales, w, pose=(0.0, 0.0, 0.0, 0.0))
    vis = np.array([(lambda uvd: (XI_CAM.z_near <= uvd[2] <= XI_CAM.z_far) and 0 <= uvd[0] <= 64 and 0 <= uvd[1] <= 48)(
        _pinhole_uvd(means[:, g], (0, 0, 0, 0), XI_CAM)) for g in range(n)])
    J = np.diag(vis.astype(float))[vis]          # rows select visible Gaussians
    Sigma = np.diag(c["u"])
    assert r["gain"][0] == pytest.approx(np.trace(J @ Sigma @ J.T), rel=1e-12)
    assert vis.sum() > 3
    # monotonicity: adding a visible H member adds exactly +1, an L member -lambda
    assert r["nh"][0] == np.sum(vis & (c["cls"] == 1))


def test_gain_additive_and_nonnegative():
    rng = np.random.default_rng(8)
    n = 60
    means = np.stack([rng.uniform(0, 6, n), rng.uniform(-3, 3, n), rng.uniform(-2, 2, n)]).astype(np.float32)
    quats = np.tile(np.array([[1], [0], [0], [0]], np.float32), (1, n))
    scales = np.full((3, n), 0.05, np.float32)
    w = rng.uniform(0, 1, n).astype(np.float32)
    A = np.arange(n) < 25
    full, _ = _wp(means, quats, scales, w)
    ra, _ = _wp(means[:, A], quats[:, A], scales[:, A], w[A])
    rb, _ = _wp(means[:, ~A], quats[:, ~A], scales[:, ~A], w[~A])
    assert full["gain"][0] >= 0
    assert full["gain"][0] == pytest.approx(ra["gain"][0] + rb["gain"][0], rel=1e-12)
    assert full["nh"][0] == ra["nh"][0] + rb["nh"][0]
    assert full["nl"][0] == ra["nl"][0] + rb["nl"][0]


def test_no_gain_flag_and_beyond_far_contribute_zero():
    w = [0.9, 0.9]
    m, q, s = _front_map(w)
    flags = np.array([W.FLAG_NO_GAIN, 0], np.uint8)
    r, _ = _wp(m, q, s, w, flags=flags)
    assert r["nh"][0] == 1 and r["gain"][0] == pytest.approx(0.9, rel=1e-7)
    m2 = m.copy()
    m2[0] = 6.0            # beyond z_far = 5
    r, _ = _wp(m2, q, s, w)
    assert r["gain"][0] == 0.0 and r["nh"][0] == 0


def test_non_finite_waypoint_sees_and_hits_nothing():
    """Reading R8: a waypoint with a non-finite coordinate (trajectory padding, e.g. rtg_plan_tree's NaN
    after a candidate's last primitive) sees nothing -- not a NaN-propagated "every slack passes" -- and,
    when its position is non-finite, collides with nothing (the collision test reads the position only)."""
    w = [0.9, 0.1, 0.5]
    m, q, s = _front_map(w, dist=0.2)          # within the robot radius of the origin: collides when finite
    r, _ = _wp(m, q, s, w, pose=(0.0, 0.0, 0.0, 0.0))
    assert r["col"][0] == 1
    for pose in ((np.nan, 0.0, 0.0, 0.0), (0.0, np.nan, 0.0, 0.0), (0.0, 0.0, np.nan, 0.0), (np.inf, 0.0, 0.0, 0.0),
                 (0.0, 0.0, np.inf, 0.0), (0.0, -np.inf, 0.0, 0.0), (0.0, 0.0, 0.0, np.nan)):
        r, _ = _wp(m, q, s, w, pose=pose)
        assert r["gain"][0] == 0.0 and r["nh"][0] == 0 and r["nl"][0] == 0, pose
        # definitely nothing: no band case either (an infinite slack over an infinite scale is not one)
        assert r["amb_vis"][0] == 0 and r["gain_hi"][0] == 0.0 and r["nh_hi"][0] == 0, pose
        assert r["col"][0] == (1 if np.isfinite(pose[:3]).all() else 0), pose


# ----------------------------------------------------------------- trajectories (O6/O7)

def test_brute_force_pipeline_by_hand():
    """Two Gaussians, three straight trajectories; every answer derived by hand.
    Gaussian A: isotropic r=0.1 at (1.05, 0, 0.5): gamma = 0.3 + 3*0.1 = 0.6.
    Trajectory 0 heads +x at 1 m/s from the origin (z=0.5): waypoint t_l=(l+1)0.1 at x=0.1(l+1);
    collides when |x-1.05| < 0.6 -> x > 0.45 -> first l with 0.1(l+1) > 0.45 is l=4 (x=0.5).
    Trajectory 1 heads +y: distance to A >= 1.05 > 0.6 -> feasible.
    Trajectory 2 heads -x: feasible.  Gaussian B (w high) sits at (0, 3, 0.5), visible only
    from trajectory 1 (facing +y); A is visible from trajectory 0 until collision only."""
    means = np.array([[1.05, 0.0], [0.0, 3.0], [0.5, 0.5]], np.float32)
    quats = np.array([[1, 1], [0, 0], [0, 0], [0, 0]], np.float32)
    scales = np.full((3, 2), 0.1, np.float32)
    w = np.array([0.1, 0.9], np.float32)
    T = 10
    t = (np.arange(T) + 1) * 0.1
    x = np.stack([t, 0 * t, -t]).astype(np.float32)
    y = np.stack([0 * t, t, 0 * t]).astype(np.float32)
    z = np.full((3, T), 0.5, np.float32)
    yaw = np.stack([0 * t, 0 * t + np.pi / 2, 0 * t + np.pi]).astype(np.float32)
    wl = W.Workload("hand", means, quats, scales, np.ones(2, np.float32), w, None, x, y, z, yaw,
                    W.Robot(0.3), XI_CAM, 0.1)
    r = O.score(wl, tau_hi=0.5, tau_lo=0.2)
    assert list(r["first_col"]) == [4, 10, 10]
    assert list(r["feasible"]) == [False, True, True]
    # trajectory 1 sees B (H) from all 10 waypoints: B at distance 3-0.1(l+1) in [2, 2.9] < z_far
    assert r["xi"][1] == 10.0
    assert r["gain"][1] == pytest.approx(10 * float(np.float32(0.9)), rel=1e-12)
    # trajectory 2 faces away from both
    assert r["xi"][2] == 0.0 and r["gain"][2] == 0.0
    assert r["best"] == 1
    # info_stride 5 keeps waypoints l = 4, 9 only
    r5 = O.score(wl, tau_hi=0.5, tau_lo=0.2, info_stride=5)
    assert r5["xi"][1] == 2.0
    # include_start (Eq. equ:traj_utility sums l = 0..L): the shared start (origin,
    # z 0.5, heading +x) sees A at depth 1.05 (w 0.1 < tau_lo: class L -> xi -1, gain 0.1) and not B
    # (depth 0): every trajectory gains xi - 1 and gain + 0.1; the winner stays 1
    rs = O.score(wl, tau_hi=0.5, tau_lo=0.2, start=(0.0, 0.0, 0.5, 0.0))
    assert list(rs["xi"]) == [r["xi"][0] - 1.0, 9.0, -1.0]
    assert rs["gain"][2] == pytest.approx(float(np.float32(0.1)), rel=1e-12)
    assert list(rs["utility"][1:]) == [9.0, -1.0] and np.isneginf(rs["utility"][0])
    assert rs["best"] == 1
    rs5 = O.score(wl, tau_hi=0.5, tau_lo=0.2, info_stride=5, start=(0.0, 0.0, 0.5, np.pi / 2))
    assert rs5["xi"][1] == 3.0          # start facing +y sees B (H): l = 0, 4, 9


def test_argmax_ties_permutation_and_none():
    assert O.best(np.array([1.0, 3.0, 3.0, -np.inf])) == 1
    assert O.best(np.array([-np.inf, -np.inf])) == -1
    u = np.array([2.0, -5.0, 7.0, 7.0, 1.0])
    perm = np.array([4, 3, 0, 2, 1])
    assert perm[O.best(u[perm])] in (2, 3)
    assert O.best(u[perm]) == 1


def test_tiny_config_literal_reading_is_degenerate():
    """tiny (2000 Gaussians uniform in 300 m^3) collides at every waypoint."""
    wl = W.tiny()
    r = O.score(wl, traj_idx=np.arange(8))
    assert np.all(r["wp"]["col"])
    assert r["best"] == -1


# ----------------------------------------------------------------- sampler

@pytest.mark.parametrize("case", _gold("unicycle_cases.json")["cases"])
def test_unicycle_golden(case):
    x, y, z, yaw = O.unicycle(case["start"], case["v"], case["omega"], case["dt"], 1)
    assert (x[0], y[0], yaw[0]) == pytest.approx(tuple(case["end"]), abs=1e-12)


def test_unicycle_matches_ode_integration():
    rng = np.random.default_rng(12)
    for _ in range(10):
        v, om = rng.uniform(0, 2), rng.uniform(-1, 1)
        th0 = rng.uniform(-3, 3)
        x, y, z, yaw = O.unicycle([1.0, 2.0, 0.5, th0], v, om, 0.1, 30)
        sol = solve_ivp(lambda t, s: [v * math.cos(s[2]), v * math.sin(s[2]), om], (0, 3.0), [1.0, 2.0, th0],
                        t_eval=(np.arange(30) + 1) * 0.1, rtol=1e-11, atol=1e-12)
        assert np.allclose(x, sol.y[0], atol=1e-8) and np.allclose(y, sol.y[1], atol=1e-8)
        dyaw = np.angle(np.exp(1j * (yaw - sol.y[2])))
        assert np.all(np.abs(dyaw) < 1e-8)
        assert np.all((yaw > -np.pi) & (yaw <= np.pi))

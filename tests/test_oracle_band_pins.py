"""Pins of the oracle's ambiguity-band machinery, pair mask, ground flag and SUM utility (-m "not gpu").

These fix the parts of the oracle that the north_star tolerance is defined by:

  * the band itself: |q - 1| <= 1e-6 for collision, |sigma_j| <= 1e-6 scale_j for visibility
    (north_star: "Collision masks must match the oracle bit-exactly, except for pairs within 1e-6
    relative of the threshold"; the collision threshold is the gamma test, the
    visibility test the pinhole frustum).  Points are placed at
    +-0.5e-6 (inside the band) and +-2e-6 (outside it) of each threshold, with coordinates that are
    exact or whose fp32 rounding moves the relative margin by < 1e-7;
  * the {nominal, lo, hi} bounds those bands induce on gains, counts, first_col and the argmax
    (SURVEY §8(c) O5-O7);
  * orc_pair_mask, pair by pair, against the independent inverse-covariance route (scipy Rotation +
    numpy inverse) and the ground flag;
  * "removal of Gaussians on the ground plane for planning": a NO_COLLIDE
    Gaussian never collides, a NO_GAIN one still does;
  * RTGuIDE-sum: "the sum of the uncertainty of the Gaussians in the camera view"
    as the utility, on a hand case where it and xi pick different trajectories.
"""
import numpy as np
import pytest
from scipy.spatial.transform import Rotation

from oracle import oracle as O
from paper_2409_18122_b200 import workloads as W

CAM = W.Camera(64, 48, 50.0, 50.0, 32.0, 24.0, 0.1, 5.0)     # |X| <= 0.64 Z, |Y| <= 0.48 Z
IN, OUT = 0.5e-6, 2e-6                                         # inside / outside the 1e-6 band


def _map(mus, s=0.125, flags=None, w=None):
    n = len(mus)
    means = np.array(mus, np.float32).T.copy()
    quats = np.zeros((4, n), np.float32)
    quats[0] = 1
    scales = np.full((3, n), s, np.float32)
    w = np.full(n, 0.9, np.float32) if w is None else np.asarray(w, np.float32)
    fl = None if flags is None else np.asarray(flags, np.uint8)
    return means, quats, scales, w, fl


def _one_wp(mus, pose, robot=W.Robot(0.25), flags=None, w=None, do_collision=True, tau=(0.6, 0.2)):
    means, quats, scales, w, fl = _map(mus, flags=flags, w=w)
    c = O.classify(w, fl, tau_hi=tau[0], tau_lo=tau[1])
    return O.waypoints(means, quats, scales, fl, c["cls"], c["u"], robot, CAM, np.array([pose[0]]),
                       np.array([pose[1]]), np.array([pose[2]]), np.array([pose[3]]), do_collision=do_collision)


# ----------------------------------------------------------------- visibility band (O3, O5)

def _vis_point(which, rho):
    """A Gaussian mean whose slack j is rho * scale_j for a camera at the origin, yaw 0
    (Z = dx, X = -dy, Y = -dz).  Derivations (SURVEY §8(c) O3 slacks and scales):
      far:   sigma2 = z_far - Z,        scale 5          -> Z = 5 (1 - rho)
      near:  sigma1 = Z - z_near,       scale Z ~ 0.1    -> Z = 0.1 (1 + rho)
      right: sigma3 = 50 X + 32 Z,      Z = 2, scale 128 -> X = -1.28 + 128 rho / 50
      down:  sigma6 = 24 Z - 50 Y,      Z = 2, scale 96  -> Y = 0.96 - 96 rho / 50
      corner_far: Z = 5.5 beyond z_far, sigma3 = 352 rho -> never ambiguous (definitely out)."""
    if which == "far":
        return (5.0 * (1 - rho), 0.0, 0.0)
    if which == "near":
        return (0.1 * (1 + rho), 0.0, 0.0)
    if which == "right":
        return (2.0, -(-1.28 + 128 * rho / 50), 0.0)
    if which == "down":
        return (2.0, 0.0, -(0.96 - 96 * rho / 50))
    if which == "corner_far":
        return (5.5, -(-3.52 + 352 * rho / 50), 0.0)
    raise ValueError(which)


@pytest.mark.parametrize("which", ["far", "near", "right", "down"])
@pytest.mark.parametrize("rho", [IN, -IN, OUT, -OUT])
def test_visibility_band_flags_and_bounds(which, rho):
    mu = _vis_point(which, rho)
    # the relative slack the oracle sees is rho up to the fp32 rounding of the mean (< 1e-7)
    sg, sc = O.visibility_slacks(np.array(mu, np.float32), [0, 0, 0, 0], CAM)
    j = int(np.argmin(np.abs(sg) / sc))
    assert sg[j] / sc[j] == pytest.approx(rho, abs=1e-7)
    r = _one_wp([mu], (0.0, 0.0, 0.0, 0.0), do_collision=False)
    w = float(np.float32(0.9))
    nominal = rho > 0
    in_band = abs(rho) < 1e-6
    assert r["amb_vis"][0] == (1 if in_band else 0)
    assert r["gain"][0] == (w if nominal else 0.0)
    assert r["nh"][0] == int(nominal)
    if in_band:            # lo drops, hi keeps every band pair, whichever side it is on
        assert r["gain_lo"][0] == 0.0 and r["gain_hi"][0] == w
        assert r["nh_lo"][0] == 0 and r["nh_hi"][0] == 1
    else:                  # outside the band the bounds collapse onto the nominal decision
        assert r["gain_lo"][0] == r["gain_hi"][0] == r["gain"][0]
        assert r["nh_lo"][0] == r["nh_hi"][0] == r["nh"][0]


def test_visibility_band_needs_no_definitely_violated_slack():
    """Ambiguous <=> some |sigma_j| <= band and no sigma_j < -band: a point on the side boundary
    but beyond z_far is definitely out, not ambiguous."""
    for rho in (IN, -IN):
        r = _one_wp([_vis_point("corner_far", rho)], (0.0, 0.0, 0.0, 0.0), do_collision=False)
        assert r["amb_vis"][0] == 0 and r["gain_hi"][0] == 0.0 and r["nh_hi"][0] == 0


def test_visibility_band_counts_accumulate_per_class():
    """Two band pairs (one H inside, one L outside) and one definite H: the count bounds move by
    one each, xi_lo = nH_lo - nL_hi and xi_hi = nH_hi - nL_lo."""
    mus = [_vis_point("right", IN), _vis_point("down", -IN), (3.0, 0.0, 0.0)]
    r = _one_wp(mus, (0.0, 0.0, 0.0, 0.0), w=[0.9, 0.1, 0.9], do_collision=False)
    assert r["amb_vis"][0] == 2
    assert (r["nh"][0], r["nh_lo"][0], r["nh_hi"][0]) == (2, 1, 2)
    assert (r["nl"][0], r["nl_lo"][0], r["nl_hi"][0]) == (0, 0, 1)
    tr = O.reduce_trajectories(r, 1, 1)
    assert (tr["xi"][0], tr["xi_lo"][0], tr["xi_hi"][0]) == (2.0, 0.0, 2.0)


# ----------------------------------------------------------------- collision band (O2, O5)

A = 0.625          # 3 * 0.125 + 0.25, exact in binary


def _col_x(eps):
    """Waypoint x with q = (x / A)^2 = 1 + eps for an isotropic Gaussian at the origin."""
    return A * np.sqrt(1.0 + eps)


@pytest.mark.parametrize("eps", [IN, -IN, OUT, -OUT])
def test_collision_band_flags(eps):
    x = _col_x(eps)
    q = O.collision_q([0, 0, 0], [1, 0, 0, 0], [0.125] * 3, 0.25, 3.0, [float(np.float32(x)), 0, 0])
    assert q - 1.0 == pytest.approx(eps, abs=1e-7)
    r = _one_wp([(0.0, 0.0, 0.0)], (x, 0.0, 0.0, np.pi / 2))
    nominal = eps < 0
    in_band = abs(eps) < 1e-6
    assert r["col"][0] == nominal and r["n_col"][0] == int(nominal)
    assert r["amb_col"][0] == int(in_band)
    assert r["col_def"][0] == (nominal and not in_band)
    assert r["col_amb"][0] == in_band          # no definite collision, an ambiguous pair


def test_collision_definite_hides_ambiguous():
    """col_amb = no definite collision but an ambiguous pair: a definite hit elsewhere clears it."""
    # waypoint at the origin: q = 1 exactly from Gaussian 0, q = 1 - 0.5e-6 from Gaussian 1 -> both band
    origin = (0.0, 0.0, 0.0, 0.0)
    r = _one_wp([(A, 0.0, 0.0), (-_col_x(-IN), 0.0, 0.0)], origin)
    assert r["amb_col"][0] == 2 and not r["col_def"][0] and r["col_amb"][0]
    assert r["col"][0] and r["n_col"][0] == 1            # nominally, only Gaussian 1 (q < 1) collides
    # a band pair next to a definite hit (distance 0.5 < A): definite collision, col_amb cleared
    r = _one_wp([(_col_x(IN), 0.0, 0.0), (0.0, 0.5, 0.0)], origin)
    assert r["amb_col"][0] == 1 and r["col_def"][0] and not r["col_amb"][0] and r["n_col"][0] == 1


def _traj_workload(xs, mus):
    """K trajectories of explicit waypoints along the x axis (y = z = 0, yaw pi/2: the camera looks
    along +y and sees none of the Gaussians on the x axis)."""
    xs = np.array(xs, np.float64)
    K, T = xs.shape
    means, quats, scales, w, _ = _map(mus)
    f = lambda a: np.ascontiguousarray(a, np.float32)
    return W.Workload("band", means, quats, scales, np.ones(len(mus), np.float32), w, None, f(xs),
                      f(np.zeros((K, T))), f(np.zeros((K, T))), f(np.full((K, T), np.pi / 2)), W.Robot(0.25), CAM, 0.1)


def test_first_col_allowed_and_feasibility_bounds():
    """O6: allowed first_col = {t_def} u {t < t_def : col_amb(t)}; a trajectory that only has band
    collisions is maybe-feasible (utility_hi finite, utility_lo = -inf)."""
    far = -3.0
    xs = [
        [far, _col_x(-IN), far, 0.3, far, _col_x(-IN)],       # band hit at 1, definite at 3
        [far, far, _col_x(IN), far, far, far],                 # band (nominally free) at 2 only
        [far] * 6,                                             # clean
        [0.2, far, far, far, _col_x(-IN), far],                # definite at 0, band later
        [far, _col_x(-OUT), far, far, far, far],               # just outside the band: definite at 1
        [far, _col_x(OUT), far, far, far, far],                # just outside the band: free
    ]
    wl = _traj_workload(xs, [(0.0, 0.0, 0.0)])
    r = O.score(wl, tau_hi=0.5, tau_lo=0.2)
    allowed = [set(np.nonzero(a)[0]) for a in r["first_col_allowed"]]
    assert allowed == [{1, 3}, {2, 6}, {6}, {0}, {1}, {6}]
    assert list(r["first_col"]) == [1, 6, 6, 0, 1, 6]
    assert list(r["feasible"]) == [False, True, True, False, False, True]
    ul, uh = r["utility_lo"], r["utility_hi"]
    assert np.isneginf(ul[1]) and np.isfinite(uh[1])         # maybe feasible
    assert np.isfinite(ul[2]) and np.isfinite(uh[2])         # surely feasible
    assert np.isneginf(uh[0]) and np.isneginf(uh[3]) and np.isneginf(uh[4])
    assert np.isfinite(ul[5])


# ----------------------------------------------------------------- argmax acceptable set (O7)

def test_acceptable_best_hand_cases():
    """O7: acceptable = {k : utility_hi_k >= max_j utility_lo_j - 1e-5 |max|}; a singleton whenever
    the top two differ by more than the tolerance; -1 plus the maybe-feasible when none is sure."""
    a = lambda lo, hi=None: list(O.acceptable_best(np.array(lo, float), np.array(lo if hi is None else hi, float)))
    assert a([1.0, 5.0, 3.0]) == [1]
    assert a([5.0, 5.0 - 2.5e-5, 5.0 - 1e-4]) == [0, 1]           # within 1e-5 * 5 of the max
    assert a([-100.0, -100.0 - 5e-4, -100.0 - 2e-3]) == [0, 1]    # relative to |max|
    assert a([4.0, 4.5], [5.0, 4.6]) == [0, 1]                    # a band that reaches the max
    assert a([4.0, 4.5], [4.4, 4.6]) == [1]
    ninf = -np.inf
    assert a([ninf, ninf], [3.0, ninf]) == [-1, 0]
    assert a([ninf, ninf]) == [-1]


def test_best_is_lowest_index_of_maxima_and_oracle_wires_acceptable():
    far = -3.0
    xs = [[far] * 3, [far, _col_x(IN), far], [far] * 3]
    wl = _traj_workload(xs, [(0.0, 0.0, 0.0)])
    r = O.score(wl, tau_hi=0.5, tau_lo=0.2)
    # all utilities 0 (nothing visible): trajectory 1 is only maybe-feasible, 0 and 2 tie
    assert list(r["utility"]) == [0.0, 0.0, 0.0]
    assert r["best"] == 0
    assert list(r["acceptable"]) == [0, 1, 2]


# ----------------------------------------------------------------- pair mask and ground flag

def _scipy_q(mu, quat, s, r, lam, p):
    R = Rotation.from_quat([quat[1], quat[2], quat[3], quat[0]]).as_matrix()
    a = lam * np.asarray(s, float) + r
    cov = R @ np.diag(a ** 2) @ R.T
    d = np.asarray(p, float) - np.asarray(mu, float)
    return float(d @ np.linalg.inv(cov) @ d)


def test_pair_mask_pair_by_pair():
    """orc_pair_mask against the independent inverse-covariance route, pair by pair, with
    NO_COLLIDE rows zero and NO_GAIN rows still tested (collision only)."""
    rng = np.random.default_rng(31)
    n, m = 24, 40
    means = rng.uniform(-1.5, 1.5, (3, n)).astype(np.float32)
    q = rng.standard_normal((4, n))
    quats = (q / np.linalg.norm(q, axis=0)).astype(np.float32)
    scales = np.exp(rng.uniform(np.log(0.02), np.log(0.3), (3, n))).astype(np.float32)
    flags = np.zeros(n, np.uint8)
    flags[::4] = W.FLAG_NO_COLLIDE
    flags[1::4] = W.FLAG_NO_GAIN
    flags[2::8] = W.FLAG_NO_COLLIDE | W.FLAG_NO_GAIN
    wx, wy, wz = (rng.uniform(-1.5, 1.5, m).astype(np.float32) for _ in range(3))
    robot = W.Robot(0.3)
    mask, band = O.pair_mask(means, quats, scales, flags, robot, wx, wy, wz)
    hits = 0
    for i in range(m):
        for g in range(n):
            if flags[g] & W.FLAG_NO_COLLIDE:
                assert not mask[i, g] and not band[i, g]
                continue
            qs = _scipy_q(means[:, g].astype(float), quats[:, g].astype(float), scales[:, g].astype(float),
                          0.3, 3.0, [wx[i], wy[i], wz[i]])
            if abs(qs - 1.0) > 1e-9:
                assert mask[i, g] == (qs < 1.0), (i, g, qs)
            assert band[i, g] == (abs(qs - 1.0) <= 1e-6) or abs(abs(qs - 1.0) - 1e-6) < 1e-12
            hits += mask[i, g]
    assert hits > 15 and np.any(mask[:, 1::4])          # NO_GAIN Gaussians do collide


def test_pair_mask_band_bits():
    xs = np.array([_col_x(e) for e in (IN, -IN, OUT, -OUT)], np.float32)
    means, quats, scales, _, _ = _map([(0.0, 0.0, 0.0)])
    mask, band = O.pair_mask(means, quats, scales, None, W.Robot(0.25), xs, np.zeros(4, np.float32),
                             np.zeros(4, np.float32))
    assert list(mask[:, 0]) == [False, True, False, True]
    assert list(band[:, 0]) == [True, True, False, False]


def test_ground_flag_removes_collision_not_gain():
    """PAPER.md:328-329 removes ground Gaussians for planning (collision); they stay in the gain
    (DESIGN Q3).  NO_GAIN is the opposite: collides, contributes no gain."""
    pose = (0.0, 0.0, 0.0, 0.0)
    mu = [(0.2, 0.0, 0.0)]                  # inside the inflated sphere (A = 0.625) and in view
    r = _one_wp(mu, pose, flags=[0])
    assert r["col"][0] and r["n_col"][0] == 1 and r["nh"][0] == 1
    r = _one_wp(mu, pose, flags=[W.FLAG_NO_COLLIDE])
    assert not r["col"][0] and r["n_col"][0] == 0 and r["amb_col"][0] == 0 and r["nh"][0] == 1
    r = _one_wp(mu, pose, flags=[W.FLAG_NO_GAIN])
    assert r["col"][0] and r["n_col"][0] == 1 and r["nh"][0] == 0 and r["gain"][0] == 0.0
    r = _one_wp(mu, pose, flags=[W.FLAG_NO_COLLIDE | W.FLAG_NO_GAIN])
    assert not r["col"][0] and r["nh"][0] == 0
    # the band point too: a ground Gaussian never enters the collision band
    r = _one_wp([(0.0, 0.0, 0.0)], (_col_x(-IN), 0.0, 0.0, np.pi / 2), flags=[W.FLAG_NO_COLLIDE])
    assert r["amb_col"][0] == 0 and not r["col"][0]


# ----------------------------------------------------------------- RTGuIDE-sum

def test_sum_utility_is_summed_uncertainty_in_view():
    """Trajectory 0 looks at one H Gaussian (w = 0.9): xi = 1, summed uncertainty 0.9.
    Trajectory 1 looks the other way at five O Gaussians (w = 0.45): xi = 0, summed 2.25.
    XI picks trajectory 0; SUM ("sum of the uncertainty of the Gaussians in the camera view",
    PAPER.md:399) picks trajectory 1, with utility equal to that sum over its info waypoints."""
    mus = [(3.0, 0.0, 0.0)] + [(-3.0, y, 0.0) for y in (-0.4, -0.2, 0.0, 0.2, 0.4)]
    w = [0.9] + [0.45] * 5
    means, quats, scales, wv, _ = _map(mus, s=0.05, w=w)
    T = 2
    f = lambda a: np.ascontiguousarray(a, np.float32)
    wl = W.Workload("sum", means, quats, scales, np.ones(6, np.float32), wv, None, f(np.zeros((2, T))),
                    f(np.zeros((2, T))), f(np.zeros((2, T))), f([[0.0] * T, [np.pi] * T]), W.Robot(0.3), CAM, 0.1)
    rx = O.score(wl, tau_hi=0.6, tau_lo=0.2, variant=O.VARIANT_XI)
    rs = O.score(wl, tau_hi=0.6, tau_lo=0.2, variant=O.VARIANT_SUM)
    w32 = np.float32(0.9).item(), np.float32(0.45).item()
    assert list(rx["utility"]) == [2.0, 0.0] and rx["best"] == 0
    assert rs["utility"][0] == pytest.approx(2 * w32[0], rel=1e-15)
    assert rs["utility"][1] == pytest.approx(2 * 5 * w32[1], rel=1e-15)
    assert rs["best"] == 1
    assert list(rs["acceptable"]) == [1]
    # SQ (RTGuIDE-sq): the same selection from u = w^2
    rq = O.score(wl, tau_hi=0.6, tau_lo=0.2, variant=O.VARIANT_SQ)
    assert rq["gain"][1] == pytest.approx(2 * 5 * w32[1] ** 2, rel=1e-15)
    assert rq["gain"][0] == pytest.approx(2 * w32[0] ** 2, rel=1e-15)
    # caller tau applies to u = w^2 under SQ: 0.81 > 0.6 -> H; 0.2025 is O
    assert list(rq["utility"]) == [2.0, 0.0]


def test_closed_frustum_reading_on_exact_boundaries():
    """DESIGN.md readings Q2/Q5: the frustum is closed (visible <=> every slack >= 0).  The paper
    does not fix the boundary convention; this pins the reading the oracle implements.  Exact
    boundary points (every quantity exact in binary): Z = z_far = 5; with fx = 64, cx = 32,
    sigma3 = 64 X + 32 Z = 0 at (Z, X) = (2, -1); with fy = 64, cy = 24, sigma6 = 24 Z - 64 Y = 0
    at (Z, Y) = (2, 0.75)."""
    cam = W.Camera(64, 48, 64.0, 64.0, 32.0, 24.0, 0.125, 5.0)
    mus = [(5.0, 0.0, 0.0), (2.0, 1.0, 0.0), (2.0, 0.0, -0.75)]
    for mu in mus:
        sg, _ = O.visibility_slacks(np.array(mu, np.float32), [0, 0, 0, 0], cam)
        assert np.min(sg) == 0.0
        means, quats, scales, w, _ = _map([mu])
        c = O.classify(w, None, tau_hi=0.6, tau_lo=0.2)
        r = O.waypoints(means, quats, scales, None, c["cls"], c["u"], W.Robot(0.25), cam, np.zeros(1), np.zeros(1),
                        np.zeros(1), np.zeros(1), do_collision=False)
        assert r["nh"][0] == 1 and r["amb_vis"][0] == 1, mu

"""Python face of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  The product path
(``paper_2409_18122_b200``) never imports it and shares no code with it.

The per-pair arithmetic lives in ``rtg_oracle.c`` (double precision, compiled
here with plain ``gcc -O2 -fopenmp``, no fast-math).  This file adds the
per-trajectory reduction and the argmax written out in numpy (SURVEY.md §8(c)
O6-O7):

  O6  first_col_k = min{t : waypoint t collides} (T if none); feasible <=> first_col = T;
      over S = {t : (t+1) mod info_stride = 0}:
      gain_k = sum_S gain(k,t)  (trace proxy, Eq. eq:nbv with binary J)
      xi_k   = sum_S (n_H - lambda_xi n_L)   (Eq. equ:view_util PAPER.md:262 summed as in
               Eq. equ:traj_utility PAPER.md:316-319)
      utility_k = feasible ? xi_k (variants XI, SQ) | gain_k (variant SUM) : -inf
  O7  best = lowest index among the maxima of utility over feasible k; -1 if none
      (ties -> lowest index, SPEC S:419 reading Q11).

Every value comes with the {nominal, lo, hi} bounds induced by the north_star
ambiguity band, so a test can tell a genuine mismatch from a threshold pair.

parity pinned by tests/test_oracle_pins.py (closed forms, hand cases, brute force).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rtg_oracle.c")
_LIB = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

VARIANT_XI, VARIANT_SUM, VARIANT_SQ = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        os.makedirs(os.path.dirname(_LIB), exist_ok=True)
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-D_GNU_SOURCE", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        L = ctypes.c_longlong
        D = ctypes.c_double
        I = ctypes.c_int
        _lib.orc_collision_q.restype = D
        _lib.orc_collision_q.argtypes = [P, P, P, D, D, I, P]
        _lib.orc_visibility_slacks.restype = None
        _lib.orc_visibility_slacks.argtypes = [P, P, P, P, P]
        _lib.orc_classify.restype = I
        _lib.orc_classify.argtypes = [L, P, P, I, D, D, D, P, P, P, P]
        _lib.orc_waypoints.restype = I
        _lib.orc_waypoints.argtypes = [L, P, P, P, P, P, P, D, D, I, P, L, P, P, P, P, I,
                                       P, P, P, P, P, P]
        _lib.orc_pair_mask.restype = I
        _lib.orc_pair_mask.argtypes = [L, P, P, P, P, D, D, I, L, P, P, P, P, P]
        _lib.orc_unicycle.restype = None
        _lib.orc_unicycle.argtypes = [D, D, D, D, D, D, D, I, P, P, P, P]
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def cam_array(cam) -> np.ndarray:
    return np.array([cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, cam.z_near, cam.z_far],
                    dtype=np.float64)


# ---------------------------------------------------------------- single pairs

def collision_q(mu, quat, s, r_robot, lambda_g, p, rule=0) -> float:
    """O2 quadratic form of one pair (collide <=> q < 1)."""
    lib = _load()
    mu, quat, s, p = _f64(mu), _f64(quat), _f64(s), _f64(p)
    return lib.orc_collision_q(_p(mu), _p(quat), _p(s), r_robot, lambda_g, rule, _p(p))


def visibility_slacks(mu, pose, cam):
    """O3 slacks sigma[6] and their scales; visible <=> all sigma >= 0."""
    lib = _load()
    mu, pose = _f64(mu), _f64(pose)
    c = cam_array(cam) if not isinstance(cam, np.ndarray) else _f64(cam)
    sg = np.zeros(6)
    sc = np.zeros(6)
    lib.orc_visibility_slacks(_p(mu), _p(pose), _p(c), _p(sg), _p(sc))
    return sg, sc


def visible(mu, pose, cam) -> bool:
    sg, _ = visibility_slacks(mu, pose, cam)
    return bool(np.all(sg >= 0.0))


# ---------------------------------------------------------------- O4

def classify(info_w, flags=None, variant=VARIANT_XI, k_sigma=0.5, tau_hi=float("nan"),
             tau_lo=float("nan")) -> Dict[str, np.ndarray]:
    lib = _load()
    w = _f32(info_w)
    n = w.shape[0]
    fl = None if flags is None else np.ascontiguousarray(flags, dtype=np.uint8)
    tau = np.zeros(4)
    cls = np.zeros(n, np.int8)
    amb = np.zeros(n, np.uint8)
    u = np.zeros(n)
    lib.orc_classify(n, _p(w), _p(fl), variant, k_sigma, tau_hi, tau_lo, _p(tau), _p(cls), _p(amb), _p(u))
    return dict(tau_hi=tau[0], tau_lo=tau[1], mean=tau[2], std=tau[3], cls=cls, cls_amb=amb.astype(bool), u=u)


# ---------------------------------------------------------------- O5

def waypoints(means, quats, scales, flags, cls, u, robot, cam, wx, wy, wz, wyaw,
              do_collision=True) -> Dict[str, np.ndarray]:
    lib = _load()
    means, quats, scales = _f32(means), _f32(quats), _f32(scales)
    n = means.shape[1]
    fl = None if flags is None else np.ascontiguousarray(flags, dtype=np.uint8)
    cls = np.ascontiguousarray(cls, dtype=np.int8)
    u = _f64(u)
    wx, wy, wz, wyaw = (_f32(a).reshape(-1) for a in (wx, wy, wz, wyaw))
    m = wx.shape[0]
    col = np.zeros((m, 3), np.uint8)
    ncol = np.zeros(m, np.int32)
    gain = np.zeros((m, 3))
    nh = np.zeros((m, 3), np.int64)
    nl = np.zeros((m, 3), np.int64)
    amb = np.zeros((m, 2), np.int64)
    lib.orc_waypoints(n, _p(means), _p(quats), _p(scales), _p(fl), _p(cls), _p(u),
                      robot.r_robot, robot.lambda_g, robot.rule, _p(cam_array(cam)),
                      m, _p(wx), _p(wy), _p(wz), _p(wyaw), int(bool(do_collision)),
                      _p(col), _p(ncol), _p(gain), _p(nh), _p(nl), _p(amb))
    return dict(col=col[:, 0].astype(bool), col_def=col[:, 1].astype(bool), col_amb=col[:, 2].astype(bool),
                n_col=ncol, gain=gain[:, 0], gain_lo=gain[:, 1], gain_hi=gain[:, 2],
                nh=nh[:, 0], nh_lo=nh[:, 1], nh_hi=nh[:, 2], nl=nl[:, 0], nl_lo=nl[:, 1], nl_hi=nl[:, 2],
                amb_col=amb[:, 0], amb_vis=amb[:, 1])


def pair_mask(means, quats, scales, flags, robot, wx, wy, wz):
    lib = _load()
    means, quats, scales = _f32(means), _f32(quats), _f32(scales)
    n = means.shape[1]
    fl = None if flags is None else np.ascontiguousarray(flags, dtype=np.uint8)
    wx, wy, wz = (_f32(a).reshape(-1) for a in (wx, wy, wz))
    m = wx.shape[0]
    mask = np.zeros((m, n), np.uint8)
    band = np.zeros((m, n), np.uint8)
    lib.orc_pair_mask(n, _p(means), _p(quats), _p(scales), _p(fl), robot.r_robot, robot.lambda_g,
                      robot.rule, m, _p(wx), _p(wy), _p(wz), _p(mask), _p(band))
    return mask.astype(bool), band.astype(bool)


def unicycle(start, v, omega, dt, T):
    """Closed-form unicycle samples (x, y, z, yaw) at t_l = (l+1) dt, double."""
    lib = _load()
    out = [np.zeros(T) for _ in range(4)]
    lib.orc_unicycle(float(start[0]), float(start[1]), float(start[2]), float(start[3]), float(v),
                     float(omega), float(dt), int(T), *[_p(o) for o in out])
    return tuple(out)


# ---------------------------------------------------------------- O6 / O7

def reduce_trajectories(wp: Dict[str, np.ndarray], K: int, T: int, lambda_xi=1.0, variant=VARIANT_XI,
                        info_stride=1, start_wp: Optional[Dict[str, np.ndarray]] = None) -> Dict[str, np.ndarray]:
    """O6 per trajectory, written out step by step from the per-waypoint arrays.

    start_wp (optional): the O5 record of the shared start state x_i(0).  Eq. equ:traj_utility
     sums xi over l = 0..L, and l = 0 is the start, common to every trajectory:
    its gain / counts are added to every trajectory's info sums (SURVEY Q7 include_start)."""
    col = wp["col"].reshape(K, T)
    col_def = wp["col_def"].reshape(K, T)
    col_amb = wp["col_amb"].reshape(K, T)
    first = np.full(K, T, np.int64)
    first_def = np.full(K, T, np.int64)
    for k in range(K):
        hits = np.nonzero(col[k])[0]
        if hits.size:
            first[k] = hits[0]
        hd = np.nonzero(col_def[k])[0]
        if hd.size:
            first_def[k] = hd[0]
    allowed = np.zeros((K, T + 1), bool)        # allowed GPU answers for first_col
    for k in range(K):
        allowed[k, first_def[k]] = True
        for t in range(first_def[k]):
            if col_amb[k, t]:
                allowed[k, t] = True
    feasible = first == T
    S = ((np.arange(T) + 1) % info_stride) == 0
    g = wp["gain"].reshape(K, T)[:, S].sum(1)
    g_lo = wp["gain_lo"].reshape(K, T)[:, S].sum(1)
    g_hi = wp["gain_hi"].reshape(K, T)[:, S].sum(1)
    nh, nl = wp["nh"].reshape(K, T), wp["nl"].reshape(K, T)
    xi_wp = nh - lambda_xi * nl
    xi_wp_lo = wp["nh_lo"].reshape(K, T) - lambda_xi * wp["nl_hi"].reshape(K, T)
    xi_wp_hi = wp["nh_hi"].reshape(K, T) - lambda_xi * wp["nl_lo"].reshape(K, T)
    xi = xi_wp[:, S].sum(1).astype(np.float64)
    xi_lo = xi_wp_lo[:, S].sum(1).astype(np.float64)
    xi_hi = xi_wp_hi[:, S].sum(1).astype(np.float64)
    if start_wp is not None:     # + info state l = 0 (the shared start)
        g = g + start_wp["gain"][0]
        g_lo = g_lo + start_wp["gain_lo"][0]
        g_hi = g_hi + start_wp["gain_hi"][0]
        xi = xi + float(start_wp["nh"][0] - lambda_xi * start_wp["nl"][0])
        xi_lo = xi_lo + float(start_wp["nh_lo"][0] - lambda_xi * start_wp["nl_hi"][0])
        xi_hi = xi_hi + float(start_wp["nh_hi"][0] - lambda_xi * start_wp["nl_lo"][0])
    if variant == VARIANT_SUM:
        util, u_lo, u_hi = g.copy(), g_lo.copy(), g_hi.copy()
    else:
        util, u_lo, u_hi = xi.copy(), xi_lo.copy(), xi_hi.copy()
    util[~feasible] = -np.inf
    surely_feasible = allowed[:, T] & (allowed.sum(1) == 1)
    maybe_feasible = allowed[:, T]
    u_lo[~surely_feasible] = -np.inf
    u_hi[~maybe_feasible] = -np.inf
    return dict(first_col=first, first_col_allowed=allowed, feasible=feasible,
                gain=g, gain_lo=g_lo, gain_hi=g_hi, xi=xi, xi_lo=xi_lo, xi_hi=xi_hi,
                utility=util, utility_lo=u_lo, utility_hi=u_hi)


def best(utility: np.ndarray) -> int:
    """O7: lowest index among the maxima of utility; -1 if every entry is -inf."""
    best_k, best_v = -1, -np.inf
    for k, v in enumerate(utility):
        if v > best_v:
            best_k, best_v = k, v
    return best_k


def acceptable_best(util_lo: np.ndarray, util_hi: np.ndarray, tol=1e-5) -> np.ndarray:
    """Indices an implementation may return as argmax given the bands."""
    m = np.max(util_lo) if util_lo.size else -np.inf
    if not np.isfinite(m):
        cand = np.nonzero(np.isfinite(util_hi))[0]
        return np.concatenate([[-1], cand])
    return np.nonzero(util_hi >= m - tol * abs(m))[0]


def score(wl, lambda_xi=1.0, k_sigma=0.5, variant=VARIANT_XI, info_stride=1, tau_hi=float("nan"),
          tau_lo=float("nan"), traj_idx: Optional[np.ndarray] = None, no_collision=False,
          x=None, y=None, z=None, yaw=None, start=None) -> Dict[str, object]:
    """Whole oracle pipeline O1-O7 on a workloads.Workload (optionally a trajectory subset).
    start = (x, y, z, yaw) scores the shared start state as info state l = 0 (include_start)."""
    c = classify(wl.info_w, wl.flags, variant, k_sigma, tau_hi, tau_lo)
    X = wl.x if x is None else x
    Y = wl.y if y is None else y
    Z = wl.z if z is None else z
    YW = wl.yaw if yaw is None else yaw
    if traj_idx is not None:
        X, Y, Z, YW = (np.ascontiguousarray(a[traj_idx]) for a in (X, Y, Z, YW))
    K, T = X.shape
    wp = waypoints(wl.means, wl.quats, wl.scales, wl.flags, c["cls"], c["u"], wl.robot, wl.camera,
                   X, Y, Z, YW, do_collision=not no_collision)
    start_wp = None
    if start is not None:        # the start's view only: it is the robot's current state (not checked)
        st = np.asarray(start, np.float32)
        start_wp = waypoints(wl.means, wl.quats, wl.scales, wl.flags, c["cls"], c["u"], wl.robot, wl.camera,
                             st[0:1], st[1:2], st[2:3], st[3:4], do_collision=False)
    tr = reduce_trajectories(wp, K, T, lambda_xi, variant, info_stride, start_wp)
    tr["best"] = best(tr["utility"])
    tr["acceptable"] = acceptable_best(tr["utility_lo"], tr["utility_hi"])
    tr["wp"] = wp
    tr["classes"] = c
    return tr

"""Seeded synthetic workloads for the RT-GuIDE trajectory-scoring hot path.

This module is INPUT SYNTHESIS ONLY.  It builds the Gaussian maps and candidate
trajectories described by BASELINE.json ``configs[0..4]`` with the readings of
SURVEY.md §8(d) (recorded in DESIGN.md "Input recipe").  It holds none of the
method's scoring arithmetic (no quaternion->rotation, no collision quadratic
form, no frustum test, no classification, no reduction): the oracle
(``oracle/``) and the CUDA path (``csrc/``) both consume the float32 arrays it
returns, and neither imports the other.

Array conventions (the C-ABI layout, include/rtg.h):
  means  float32 [3, N]  planar SoA (x row, y row, z row), metres
  quats  float32 [4, N]  planar SoA (w, x, y, z), unit norm (3DGS convention)
  scales float32 [3, N]  per-axis standard deviation s_i, metres (local axes)
  opacity float32 [N], info_w float32 [N] (the displacement-magnitude ledger,
  PAPER.md:217-224), flags uint8 [N] (bit0 NO_COLLIDE = ground)
  trajectories: x, y, z, yaw float32 [K, T] (trajectory-major), waypoint l at
  time (l+1)*dt.

The paper's own workloads (AI2-THOR/iTHOR scenes and real-world maps,
PAPER.md:376-381, 410, 535-539) are not available; these generators stand in
for them with the shapes BASELINE.json states.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, Optional

import numpy as np

FLAG_NO_COLLIDE = 1
FLAG_NO_GAIN = 2


@dataclasses.dataclass
class Camera:
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    z_near: float
    z_far: float


@dataclasses.dataclass
class Robot:
    r_robot: float
    lambda_g: float = 3.0
    rule: int = 0           # 0 = inflated ellipsoid, 1 = principal axis


@dataclasses.dataclass
class Workload:
    name: str
    means: np.ndarray
    quats: np.ndarray
    scales: np.ndarray
    opacity: np.ndarray
    info_w: np.ndarray
    flags: Optional[np.ndarray]
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    yaw: np.ndarray
    robot: Robot
    camera: Camera
    dt: float
    # optional gain-only viewpoints (configs[4]): dict of x,y,z,yaw [Kv,1]
    views: Optional[Dict[str, np.ndarray]] = None
    # unicycle controls when the trajectories are flat unicycle primitives
    controls: Optional[Dict[str, np.ndarray]] = None

    @property
    def N(self) -> int:
        return int(self.means.shape[1])

    @property
    def K(self) -> int:
        return int(self.x.shape[0])

    @property
    def T(self) -> int:
        return int(self.x.shape[1])


# ----------------------------------------------------------------------------
# quaternion synthesis helpers (input generation only)
# ----------------------------------------------------------------------------

def _axis_angle_quat(axis: np.ndarray, angle: np.ndarray) -> np.ndarray:
    """(w,x,y,z) quaternions [M,4] for rotations by ``angle`` about unit ``axis`` [M,3]."""
    h = 0.5 * angle
    q = np.empty((axis.shape[0], 4), dtype=np.float64)
    q[:, 0] = np.cos(h)
    q[:, 1:] = axis * np.sin(h)[:, None]
    return q


def _qmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Hamilton product a*b for [M,4] (w,x,y,z) arrays."""
    aw, ax, ay, az = a.T
    bw, bx, by, bz = b.T
    return np.stack([
        aw * bw - ax * bx - ay * by - az * bz,
        aw * bx + ax * bw + ay * bz - az * by,
        aw * by - ax * bz + ay * bw + az * bx,
        aw * bz + ax * by - ay * bx + az * bw,
    ], axis=1)


def _tilt_quat(normals: np.ndarray) -> np.ndarray:
    """Quaternion taking local +z onto each unit normal [M,3]."""
    nz = np.clip(normals[:, 2], -1.0, 1.0)
    axis = np.stack([-normals[:, 1], normals[:, 0], np.zeros_like(nz)], axis=1)  # ez x n
    nrm = np.linalg.norm(axis, axis=1)
    flip = nrm < 1e-12
    axis[flip] = np.array([1.0, 0.0, 0.0])
    nrm[flip] = 1.0
    axis /= nrm[:, None]
    angle = np.arccos(nz)
    return _axis_angle_quat(axis, angle)


def _surface_quats(rng: np.random.Generator, normals: np.ndarray) -> np.ndarray:
    """Surface-aligned orientation: local axis 3 = normal, uniform in-plane angle."""
    m = normals.shape[0]
    psi = rng.uniform(0.0, 2.0 * np.pi, size=m)
    qz = _axis_angle_quat(np.tile(np.array([0.0, 0.0, 1.0]), (m, 1)), psi)
    return _qmul(_tilt_quat(normals), qz)


def _random_quats(rng: np.random.Generator, m: int) -> np.ndarray:
    q = rng.standard_normal((m, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _loguniform(rng, lo, hi, size):
    return np.exp(rng.uniform(np.log(lo), np.log(hi), size=size))


# ----------------------------------------------------------------------------
# trajectory synthesis
# ----------------------------------------------------------------------------

def _wrap(a: np.ndarray) -> np.ndarray:
    w = np.mod(a + np.pi, 2.0 * np.pi) - np.pi
    w[w <= -np.pi] += 2.0 * np.pi
    return w


def unicycle_waypoints(x0, y0, th0, v, w, T, dt):
    """Closed-form unicycle samples at t_l=(l+1)dt (input synthesis; SPEC S:392 form)."""
    t = (np.arange(T, dtype=np.float64) + 1.0) * dt
    v = np.asarray(v, np.float64)[:, None]
    w = np.asarray(w, np.float64)[:, None]
    th = th0 + w * t
    small = np.abs(w) < 1e-12
    ws = np.where(small, 1.0, w)
    xs = np.where(small, x0 + v * t * np.cos(th0), x0 + (v / ws) * (np.sin(th) - np.sin(th0)))
    ys = np.where(small, y0 + v * t * np.sin(th0), y0 + (v / ws) * (np.cos(th0) - np.cos(th)))
    return xs, ys, _wrap(th)


def _f32(*arrs):
    return [np.ascontiguousarray(a, dtype=np.float32) for a in arrs]


# ----------------------------------------------------------------------------
# surfaces (room / multi-room)
# ----------------------------------------------------------------------------

def _rect(o, e1, e2, n, flag=0):
    o, e1, e2, n = (np.asarray(a, np.float64) for a in (o, e1, e2, n))
    return dict(o=o, e1=e1, e2=e2, n=n / np.linalg.norm(n), area=float(np.linalg.norm(e1) * np.linalg.norm(e2)), flag=flag)


def _box_surfaces(cx, cy, sx, sy, sz):
    x0, x1, y0, y1 = cx - sx / 2, cx + sx / 2, cy - sy / 2, cy + sy / 2
    return [
        _rect((x0, y0, sz), (sx, 0, 0), (0, sy, 0), (0, 0, 1)),          # top
        _rect((x0, y0, 0), (sx, 0, 0), (0, 0, sz), (0, -1, 0)),          # -y side
        _rect((x0, y1, 0), (sx, 0, 0), (0, 0, sz), (0, 1, 0)),           # +y side
        _rect((x0, y0, 0), (0, sy, 0), (0, 0, sz), (-1, 0, 0)),          # -x side
        _rect((x1, y0, 0), (0, sy, 0), (0, 0, sz), (1, 0, 0)),           # +x side
    ]


def _place_boxes(rng, n, xlo, xhi, ylo, yhi, start_xy, clear=1.5):
    boxes = []
    tries = 0
    while len(boxes) < n and tries < 100000:
        tries += 1
        sx, sy, sz = rng.uniform(0.3, 1.5, size=3)
        cx = rng.uniform(xlo + sx / 2, xhi - sx / 2)
        cy = rng.uniform(ylo + sy / 2, yhi - sy / 2)
        if math.hypot(cx - start_xy[0], cy - start_xy[1]) < clear + 0.5 * math.hypot(sx, sy):
            continue
        boxes.append((cx, cy, sx, sy, sz))
    return boxes


def _sample_surfaces(rng, surfaces, N, jitter=0.02, inplane=(0.02, 0.15), normal_scale=0.005):
    areas = np.array([s["area"] for s in surfaces])
    counts = rng.multinomial(N, areas / areas.sum())
    pos, nrm, flg, sid = [], [], [], []
    for i, (s, c) in enumerate(zip(surfaces, counts)):
        if c == 0:
            continue
        u = rng.uniform(size=(c, 1))
        v = rng.uniform(size=(c, 1))
        p = s["o"] + u * s["e1"] + v * s["e2"] + rng.normal(0.0, jitter, size=(c, 1)) * s["n"]
        pos.append(p)
        nrm.append(np.tile(s["n"], (c, 1)))
        flg.append(np.full(c, s["flag"], np.uint8))
        sid.append(np.full(c, i, np.int32))
    pos = np.concatenate(pos)
    nrm = np.concatenate(nrm)
    quats = _surface_quats(rng, nrm)
    scales = np.empty((N, 3))
    scales[:, 0:2] = _loguniform(rng, inplane[0], inplane[1], (N, 2))
    scales[:, 2] = normal_scale
    return pos, quats, scales, np.concatenate(flg), np.concatenate(sid)


# ----------------------------------------------------------------------------
# configs
# ----------------------------------------------------------------------------

def tiny(seed: int = 0, N: int = 2000, K: int = 64, T: int = 20) -> Workload:
    """BASELINE.json configs[0]: uniform 10x10x3 m box, K=64 unicycles x T=20."""
    rng = np.random.default_rng(seed)
    means = np.stack([rng.uniform(-5, 5, N), rng.uniform(-5, 5, N), rng.uniform(0, 3, N)])
    quats = _random_quats(rng, N).T
    scales = _loguniform(rng, 0.02, 0.3, (3, N))
    opacity = rng.uniform(0.1, 1.0, N)
    info_w = rng.uniform(0.0, 1.0, N)
    v = rng.uniform(0.2, 1.5, K)
    w = rng.uniform(-1.0, 1.0, K)
    dt = 0.1
    xs, ys, th = unicycle_waypoints(0.0, 0.0, 0.0, v, w, T, dt)
    zs = np.full_like(xs, 0.5)
    m, q, s, a, iw = _f32(means, quats, scales, opacity, info_w)
    x, y, z, yaw = _f32(xs, ys, zs, th)
    return Workload("tiny", m, q, s, a, iw, None, x, y, z, yaw,
                    Robot(0.3), Camera(64, 48, 50.0, 50.0, 32.0, 24.0, 0.1, 5.0), dt,
                    controls=dict(v=v.astype(np.float32), w=w.astype(np.float32),
                                  start=np.array([0, 0, 0.5, 0], np.float32)))


def room(seed: int = 0, traj_seed: int = 1, N: int = 100_000, K: int = 1024, T: int = 50) -> Workload:
    """BASELINE.json configs[1]: 12x10x3 m room, floor + 4 walls + 20 boxes."""
    rng = np.random.default_rng(seed)
    surfaces = [_rect((-6, -5, 0), (12, 0, 0), (0, 10, 0), (0, 0, 1), FLAG_NO_COLLIDE)]
    surfaces += [
        _rect((-6, -5, 0), (0, 10, 0), (0, 0, 3), (1, 0, 0)),
        _rect((6, -5, 0), (0, 10, 0), (0, 0, 3), (-1, 0, 0)),
        _rect((-6, -5, 0), (12, 0, 0), (0, 0, 3), (0, 1, 0)),
        _rect((-6, 5, 0), (12, 0, 0), (0, 0, 3), (0, -1, 0)),
    ]
    for b in _place_boxes(rng, 20, -6, 6, -5, 5, (0.0, 0.0)):
        surfaces += _box_surfaces(*b)
    pos, quats, scales, flags, _ = _sample_surfaces(rng, surfaces, N)
    opacity = rng.uniform(0, 1, N)
    info_w = rng.uniform(0, 1, N)
    trng = np.random.default_rng(traj_seed)
    v = trng.uniform(0.2, 1.5, K)
    w = trng.uniform(-1.0, 1.0, K)
    dt = 0.1
    xs, ys, th = unicycle_waypoints(0.0, 0.0, 0.0, v, w, T, dt)
    zs = np.full_like(xs, 0.5)
    m, q, s, a, iw = _f32(pos.T, quats.T, scales.T, opacity, info_w)
    x, y, z, yaw = _f32(xs, ys, zs, th)
    return Workload("room", m, q, s, a, iw, flags, x, y, z, yaw,
                    Robot(0.35), Camera(320, 240, 250.0, 250.0, 160.0, 120.0, 0.1, 6.0), dt,
                    controls=dict(v=v.astype(np.float32), w=w.astype(np.float32),
                                  start=np.array([0, 0, 0.5, 0], np.float32)))


def multi_room(seed: int = 0, traj_seed: int = 1, N: int = 500_000, K: int = 4096, T: int = 50) -> Workload:
    """BASELINE.json configs[2]: 40x30x3 m, 4x3 rooms of 10x10 m with 1 m doorways."""
    rng = np.random.default_rng(seed)
    X0, X1, Y0, Y1, H = -20.0, 20.0, -15.0, 15.0, 3.0
    room_of = []
    surfaces = [_rect((X0, Y0, 0), (40, 0, 0), (0, 30, 0), (0, 0, 1), FLAG_NO_COLLIDE)]
    room_of.append(-1)
    # outer walls
    for s in [_rect((X0, Y0, 0), (0, 30, 0), (0, 0, H), (1, 0, 0)),
              _rect((X1, Y0, 0), (0, 30, 0), (0, 0, H), (-1, 0, 0)),
              _rect((X0, Y0, 0), (40, 0, 0), (0, 0, H), (0, 1, 0)),
              _rect((X0, Y1, 0), (40, 0, 0), (0, 0, H), (0, -1, 0))]:
        surfaces.append(s)
        room_of.append(-1)
    door = 1.0
    # interior walls x = -10, 0, 10 (segments per room row, doorway centred)
    for xw in (-10.0, 0.0, 10.0):
        for j in range(3):
            ya, yb = Y0 + 10 * j, Y0 + 10 * (j + 1)
            ym = 0.5 * (ya + yb)
            for (y_lo, y_hi) in ((ya, ym - door / 2), (ym + door / 2, yb)):
                for nx in (1.0, -1.0):
                    surfaces.append(_rect((xw, y_lo, 0), (0, y_hi - y_lo, 0), (0, 0, H), (nx, 0, 0)))
                    room_of.append(-1)
    for yw in (-5.0, 5.0):
        for i in range(4):
            xa, xb = X0 + 10 * i, X0 + 10 * (i + 1)
            xm = 0.5 * (xa + xb)
            for (x_lo, x_hi) in ((xa, xm - door / 2), (xm + door / 2, xb)):
                for ny in (1.0, -1.0):
                    surfaces.append(_rect((x_lo, yw, 0), (x_hi - x_lo, 0, 0), (0, 0, H), (0, ny, 0)))
                    room_of.append(-1)
    start = (5.0, 0.0)
    for i in range(4):
        for j in range(3):
            xa, ya = X0 + 10 * i, Y0 + 10 * j
            for b in _place_boxes(rng, 20, xa + 0.2, xa + 9.8, ya + 0.2, ya + 9.8, start):
                for s in _box_surfaces(*b):
                    surfaces.append(s)
                    room_of.append(i * 3 + j)
    pos, quats, scales, flags, sid = _sample_surfaces(rng, surfaces, N)
    opacity = rng.uniform(0, 1, N)
    # bimodal information weights: whole rooms (~20 % of N) hold the unobserved band
    rix = np.clip(((pos[:, 0] - X0) // 10).astype(int), 0, 3) * 3 + np.clip(((pos[:, 1] - Y0) // 10).astype(int), 0, 2)
    order = rng.permutation(12)
    high = np.zeros(N, bool)
    for r in order:
        if high.mean() >= 0.2:
            break
        high |= rix == r
    info_w = np.where(high, rng.uniform(0.8, 1.0, N), rng.uniform(0.0, 0.1, N))
    # double-integrator primitives: p0=(5,0), v0=(1,0), constant |a|<=1, |v|<=2 over the horizon
    trng = np.random.default_rng(traj_seed)
    dt = 0.1
    tmax = T * dt
    acc = np.empty((K, 2))
    filled = 0
    while filled < K:
        a = trng.uniform(-1, 1, size=(4 * K, 2))
        a = a[np.linalg.norm(a, axis=1) <= 1.0]
        vend = np.array([1.0, 0.0]) + a * tmax
        a = a[np.linalg.norm(vend, axis=1) <= 2.0]
        take = min(K - filled, a.shape[0])
        acc[filled:filled + take] = a[:take]
        filled += take
    t = (np.arange(T) + 1.0) * dt
    xs = start[0] + 1.0 * t[None, :] + 0.5 * acc[:, 0:1] * t[None, :] ** 2
    ys = start[1] + 0.0 * t[None, :] + 0.5 * acc[:, 1:2] * t[None, :] ** 2
    vx = 1.0 + acc[:, 0:1] * t[None, :]
    vy = acc[:, 1:2] * t[None, :]
    th = np.arctan2(vy, vx)
    zs = np.full_like(xs, 0.5)
    m, q, s, a_, iw = _f32(pos.T, quats.T, scales.T, opacity, info_w)
    x, y, z, yaw = _f32(xs, ys, zs, th)
    return Workload("multi_room", m, q, s, a_, iw, flags, x, y, z, yaw,
                    Robot(0.35), Camera(640, 480, 500.0, 500.0, 320.0, 240.0, 0.1, 8.0), dt)


class Terrain:
    """h(x,y) = (1/8) sum_j sin(k_j.(x,y) + phi_j); wavelengths U[10,40] m (SURVEY §8(d) reading)."""

    def __init__(self, rng):
        lam = rng.uniform(10.0, 40.0, 8)
        ang = rng.uniform(0, 2 * np.pi, 8)
        self.k = np.stack([np.cos(ang), np.sin(ang)], 1) * (2 * np.pi / lam)[:, None]
        self.phi = rng.uniform(0, 2 * np.pi, 8)

    def h(self, x, y):
        arg = np.multiply.outer(x, self.k[:, 0]) + np.multiply.outer(y, self.k[:, 1]) + self.phi
        return np.sin(arg).sum(-1) / 8.0

    def grad(self, x, y):
        arg = np.multiply.outer(x, self.k[:, 0]) + np.multiply.outer(y, self.k[:, 1]) + self.phi
        c = np.cos(arg) / 8.0
        return (c * self.k[:, 0]).sum(-1), (c * self.k[:, 1]).sum(-1)


def _outdoor_map(rng, N, half, n_clusters=300):
    terr = Terrain(rng)
    n_t = N // 2
    n_c = N - n_t
    tx = rng.uniform(-half, half, n_t)
    ty = rng.uniform(-half, half, n_t)
    gx, gy = terr.grad(tx, ty)
    nrm = np.stack([-gx, -gy, np.ones_like(gx)], 1)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    tpos = np.stack([tx, ty, terr.h(tx, ty)], 1) + rng.normal(0, 0.02, (n_t, 1)) * nrm
    tquat = _surface_quats(rng, nrm)
    tscale = np.empty((n_t, 3))
    tscale[:, 0:2] = _loguniform(rng, 0.02, 0.15, (n_t, 2))
    tscale[:, 2] = 0.005
    # clusters: centres >= 6 m (horizontal) from the start, centre z = h + 2 m
    cen = np.empty((n_clusters, 3))
    k = 0
    while k < n_clusters:
        c = rng.uniform(-half, half, 2)
        if math.hypot(c[0], c[1]) < 6.0:
            continue
        cen[k, 0:2] = c
        k += 1
    cen[:, 2] = terr.h(cen[:, 0], cen[:, 1]) + 2.0
    per = np.full(n_clusters, n_c // n_clusters)
    per[: n_c % n_clusters] += 1
    cid = np.repeat(np.arange(n_clusters), per)
    cpos = cen[cid] + rng.normal(0, 1.5, (n_c, 3))
    cquat = _random_quats(rng, n_c)
    cscale = _loguniform(rng, 0.05, 0.5, (n_c, 3))
    pos = np.concatenate([tpos, cpos])
    quat = np.concatenate([tquat, cquat])
    scale = np.concatenate([tscale, cscale])
    flags = np.concatenate([np.full(n_t, FLAG_NO_COLLIDE, np.uint8), np.zeros(n_c, np.uint8)])
    opacity = rng.uniform(0, 1, N)
    info_w = rng.uniform(0, 1, N)
    return terr, pos, quat, scale, flags, opacity, info_w


def outdoor(seed: int = 0, traj_seed: int = 1, N: int = 2_000_000, K: int = 16384, T: int = 100,
            half: float = 50.0, n_clusters: int = 300, views: int = 0, name: str = "outdoor") -> Workload:
    """BASELINE.json configs[3] (and configs[4] with half=100, N=5M, K=65536, views=8192)."""
    rng = np.random.default_rng(seed)
    terr, pos, quat, scale, flags, opacity, info_w = _outdoor_map(rng, N, half, n_clusters)
    trng = np.random.default_rng(traj_seed)
    v = trng.uniform(0.2, 2.0, K)
    w = trng.uniform(-1.0, 1.0, K)
    dt = 0.1
    xs, ys, th = unicycle_waypoints(0.0, 0.0, 0.0, v, w, T, dt)
    zs = terr.h(xs, ys) + 0.5                     # terrain-following (SURVEY §8(d) reading)
    vw = None
    if views:
        vx = trng.uniform(-half, half, views)
        vy = trng.uniform(-half, half, views)
        vw = dict(zip(("x", "y", "z", "yaw"), _f32(vx[:, None], vy[:, None],
                                                   (terr.h(vx, vy) + 0.5)[:, None],
                                                   trng.uniform(-np.pi, np.pi, views)[:, None])))
    m, q, s, a, iw = _f32(pos.T, quat.T, scale.T, opacity, info_w)
    x, y, z, yaw = _f32(xs, ys, zs, th)
    return Workload(name, m, q, s, a, iw, flags, x, y, z, yaw,
                    Robot(0.5), Camera(640, 480, 500.0, 500.0, 320.0, 240.0, 0.2, 15.0), dt, views=vw)


def scale(seed: int = 0, traj_seed: int = 1, N: int = 5_000_000, K: int = 65536, T: int = 100,
          views: int = 8192) -> Workload:
    """BASELINE.json configs[4]: outdoor recipe over 200x200 m, 5M Gaussians, 8192 views."""
    return outdoor(seed, traj_seed, N=N, K=K, T=T, half=100.0, views=views, name="scale")


CONFIGS = {"tiny": tiny, "room": room, "multi_room": multi_room, "outdoor": outdoor, "scale": scale}


def make(name: str, **kw) -> Workload:
    return CONFIGS[name](**kw)


def subset_trajectories(wl: Workload, idx: np.ndarray) -> Workload:
    """Same map, trajectories restricted to ``idx`` (copies)."""
    idx = np.asarray(idx)
    return dataclasses.replace(wl, x=np.ascontiguousarray(wl.x[idx]), y=np.ascontiguousarray(wl.y[idx]),
                               z=np.ascontiguousarray(wl.z[idx]), yaw=np.ascontiguousarray(wl.yaw[idx]))

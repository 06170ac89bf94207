"""CPU oracle of the planner's uncertainty bookkeeping and high-level guidance scoring
(TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s baseline legs may import this
module; the product path never imports it and shares no code with it.  Plain numpy / Python
loops in double precision, each function following the passage it cites, in the paper's order
and notation.  Pinned by tests/test_planning_pins.py.

  ledger_update   P:217-224 (§IV-A): the uncertainty of Gaussian g is the magnitude of
                  the change of its mean over the last map update, ||mu_k - mu_{k-1}||_2;
                  "Gaussians that remain unchanged in the most recent update retain their
                  previously computed displacement values".
  region_utility  P:236-240 (§IV-B1): the enclosing space is evenly partitioned into cuboidal
                  regions; Omega_k = (1/M_k) sum_{mu in o} ||mu_k - mu_{k-1}||_2 over the M_k
                  Gaussians of region o (region size 2.5 m).  Readings:
                  ground-plane Gaussians (flag NO_GAIN) are excluded, Gaussians
                  outside the partitioned box belong to no region, an empty region has Omega = 0
                  (SPEC S:344).
  view_distance   P:245-246: "the shortest viewing distance from the Gaussian region centroid to
                  the optical center of the camera, given the camera intrinsics": the distance
                  at which the region (edge `size`) fills the narrower field of view,
                  d = (size / 2) / tan(fov_min / 2).
  view_ring       SPEC S:324: n viewpoints on the circle of radius d around the region centroid
                  (in the robot's plane z), spaced 2 pi / n from angle 0, each facing the
                  centroid.
  cost_benefit    P:249: a viewpoint node at path distance d with utility Omega scores
                  Omega / e^d; the maximal score wins, ties -> smaller d, then smaller index
                  (SPEC S:333).
"""
from __future__ import annotations

import math

import numpy as np

FLAG_NO_GAIN = 2


def ledger_update(mu_prev, mu_cur, w_prev) -> np.ndarray:
    """w_g = ||mu_cur,g - mu_prev,g||_2 where the mean changed, else w_prev,g.
    Inputs fp32 (planar [3][N]); the norm is taken in double and stored as fp32."""
    mu_prev = np.asarray(mu_prev, np.float32)
    mu_cur = np.asarray(mu_cur, np.float32)
    w_prev = np.asarray(w_prev, np.float32)
    n = w_prev.shape[0]
    out = np.empty(n, np.float32)
    for g in range(n):
        a = [float(mu_prev[c, g]) for c in range(3)]
        b = [float(mu_cur[c, g]) for c in range(3)]
        if a == b:
            out[g] = w_prev[g]
        else:
            dx, dy, dz = b[0] - a[0], b[1] - a[1], b[2] - a[2]
            out[g] = np.float32(math.sqrt(dx * dx + dy * dy + dz * dz))
    return out


def region_utility(means, w, flags, origin, size, dims):
    """Omega per cuboidal region of edge `size` with lower corner `origin` and
    dims[0] x dims[1] x dims[2] regions (x fastest in the flat index).  Returns (omega, count),
    both flat of length prod(dims)."""
    means = np.asarray(means, np.float32)
    w = np.asarray(w, np.float32)
    nx, ny, nz = (int(d) for d in dims)
    total = [0.0] * (nx * ny * nz)
    count = [0] * (nx * ny * nz)
    for g in range(means.shape[1]):
        if flags is not None and (int(flags[g]) & FLAG_NO_GAIN):
            continue
        idx = []
        for c in range(3):
            idx.append(math.floor((float(means[c, g]) - float(origin[c])) / float(size)))
        if not (0 <= idx[0] < nx and 0 <= idx[1] < ny and 0 <= idx[2] < nz):
            continue
        r = (idx[2] * ny + idx[1]) * nx + idx[0]
        total[r] += float(w[g])
        count[r] += 1
    omega = np.array([t / c if c > 0 else 0.0 for t, c in zip(total, count)], np.float64)
    return omega, np.array(count, np.int64)


def fov(cam):
    """Horizontal and vertical fields of view [rad] of a pinhole camera (principal point
    anywhere in the image): the angles subtended by [0, W] and [0, H] at the optical centre."""
    h = math.atan(cam.cx / cam.fx) + math.atan((cam.width - cam.cx) / cam.fx)
    v = math.atan(cam.cy / cam.fy) + math.atan((cam.height - cam.cy) / cam.fy)
    return h, v


def view_distance(size, cam) -> float:
    """P:245-246 / SPEC S:324: d = (size/2) / tan(min(hfov, vfov) / 2)."""
    h, v = fov(cam)
    return (size / 2.0) / math.tan(min(h, v) / 2.0)


def view_ring(centroids, size, cam, n, z):
    """poses (x, y, z, yaw) of n viewpoints per centroid on the circle of radius
    view_distance around it, angles 2 pi j / n, heading towards the centroid.  Returns fp32 arrays
    of shape [R * n] (region-major)."""
    d = view_distance(size, cam)
    out = []
    for c in np.asarray(centroids, np.float64):
        for j in range(n):
            phi = 2.0 * math.pi * j / n
            x = c[0] + d * math.cos(phi)
            y = c[1] + d * math.sin(phi)
            yaw = math.atan2(c[1] - y, c[0] - x)   # facing the centroid
            out.append((x, y, z, yaw))
    a = np.array(out, np.float64).reshape(-1, 4)
    return tuple(a[:, k].astype(np.float32) for k in range(4))


def cost_benefit(omega, d):
    """P:249 / SPEC S:333: argmax_j omega_j / e^{d_j}; ties -> smaller d, then smaller j.
    Returns (best index or -1 when empty, best score)."""
    best, bs, bd = -1, -math.inf, math.inf
    for j, (o, dist) in enumerate(zip(np.asarray(omega, np.float64), np.asarray(d, np.float64))):
        s = float(o) / math.exp(float(dist))
        if s > bs or (s == bs and float(dist) < bd):
            best, bs, bd = j, s, float(dist)
    return best, bs

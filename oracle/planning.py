"""CPU oracle of the planner's uncertainty bookkeeping, high-level guidance scoring and motion-
primitive tree (TEST INFRASTRUCTURE ONLY).

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
  plan_tree       P:280-320 (§IV-B2): motion-primitive tree search for trajectory candidates (see
                  the section comment below).
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


# ---------------------------------------------------------------- N3 motion-primitive tree
# PAPER.md §IV-B2: unicycle motion primitives with fixed controls over dt, N_v x N_w
# controls sampled uniformly from [0, v_max] x [-w_max, w_max], a fixed number of
# collision samples per primitive, cost lambda_t tau + int u^T u dt (Eq.
# low_level_planner), minimum-time heuristic h = ||p_goal - p|| / v_max, the top N_traj
# candidates.  The search order is the layer-synchronous one DESIGN.md §2 (reading R5)
# states: every frontier node expanded by every control per layer, a closed lattice keeping the
# lowest g, a beam of the lowest f = g + h, goal-reaching nodes become candidates; ties go to
# creation order.

def controls(n_v, n_omega, v_max, omega_max):
    """v uniform on [0, v_max] incl. endpoints ({v_max} if n_v = 1), w uniform on
    [-w_max, w_max] incl. endpoints ({0} if n_omega = 1); order: v major, w minor."""
    v_max, omega_max = float(np.float32(v_max)), float(np.float32(omega_max))
    out = []
    for i in range(n_v):
        v = v_max if n_v == 1 else v_max * i / (n_v - 1)
        for j in range(n_omega):
            w = 0.0 if n_omega == 1 else omega_max * (2 * j - (n_omega - 1)) / (n_omega - 1)
            out.append((v, w))
    return out


def unicycle_at(x0, y0, th0, v, w, t):
    """SPEC S:392 closed form (not wrapped)."""
    th = th0 + w * t
    if abs(w) < 1e-12:
        vt = v * t
        return x0 + vt * math.cos(th0), y0 + vt * math.sin(th0), th
    r = v / w
    return x0 + r * (math.sin(th) - math.sin(th0)), y0 + r * (math.cos(th0) - math.cos(th)), th


def double_integrator(start, v0, a, dt, T):
    """Double-integrator motion primitive (BASELINE.json configs[2], SURVEY §8(b) optional sampler):
    constant acceleration a = (ax, ay) from p0 = start[0:2] with velocity v0, sampled at
    t_l = (l+1) dt: p(t) = p0 + v0 t + a t^2 / 2, z constant, heading along the velocity
    atan2(v0y + ay t, v0x + ax t) (0 when the velocity is zero).  FP64 (x, y, z, yaw) arrays."""
    f = lambda v: float(np.float32(v))
    x0, y0, z0 = f(start[0]), f(start[1]), f(start[2])
    vx, vy, ax, ay, dt = f(v0[0]), f(v0[1]), f(a[0]), f(a[1]), f(dt)
    out = [np.zeros(T) for _ in range(4)]
    for l in range(T):
        t = (l + 1) * dt
        out[0][l] = x0 + vx * t + 0.5 * ax * t * t
        out[1][l] = y0 + vy * t + 0.5 * ay * t * t
        out[2][l] = z0
        out[3][l] = math.atan2(vy + ay * t, vx + ax * t)
    return tuple(out)


def wrap_pi(a):
    r = math.remainder(a, 2.0 * math.pi)
    return r + 2.0 * math.pi if r <= -math.pi else r


def plan_tree(collides, start, goal, p):
    """Layer-synchronous motion-primitive tree search.  `collides(points)` takes an [n, 3] float32
    array of sample points and returns n booleans (the a4 collision decision).  `p` carries the
    rtg_tree_params fields (n_v, n_omega, v_max, omega_max, dt, lambda_t, samples, max_depth,
    goal_radius, lattice_xy, lattice_deg, beam, n_traj, z).
    Returns dict(cands=[node ids], nodes=[(x, y, th, g, parent, depth)], reached, expanded)."""
    f32 = lambda v: float(np.float32(v))
    ctl = controls(p.n_v, p.n_omega, p.v_max, p.omega_max)
    dt, lam, vmax = f32(p.dt), f32(p.lambda_t), f32(p.v_max)
    pcost = [(lam + v * v + w * w) * dt for v, w in ctl]
    gx, gy = f32(goal[0]), f32(goal[1])
    r2 = f32(p.goal_radius) * f32(p.goal_radius)
    h_of = lambda x, y: math.sqrt((gx - x) * (gx - x) + (gy - y) * (gy - y)) / vmax
    at_goal = lambda x, y: (x - gx) * (x - gx) + (y - gy) * (y - gy) <= r2
    lxy, ldeg = f32(p.lattice_xy), f32(p.lattice_deg)
    dedup = lxy > 0 and ldeg > 0
    key_of = lambda n: (math.floor(n[0] / lxy), math.floor(n[1] / lxy), math.floor(n[2] * (180.0 / math.pi) / ldeg))
    nodes = [(f32(start[0]), f32(start[1]), wrap_pi(f32(start[2])), 0.0, -1, 0)]
    closed = {key_of(nodes[0]): 0.0} if dedup else {}
    cands, frontier = [], []
    (cands if at_goal(nodes[0][0], nodes[0][1]) else frontier).append(0)
    S, z = int(p.samples), f32(p.z)
    expanded = 0
    for depth in range(1, int(p.max_depth) + 1):
        if not frontier:
            break
        # every sample of the layer, checked at once
        prims, pts = [], []
        for m in frontier:
            x0, y0, th0 = nodes[m][0], nodes[m][1], nodes[m][2]
            for pi, (v, w) in enumerate(ctl):
                last = None
                for j in range(1, S):
                    t = (j * dt) / (S - 1)
                    last = unicycle_at(x0, y0, th0, v, w, t)
                    pts.append((last[0], last[1], z))
                prims.append((m, pi, last))
        hit = np.asarray(collides(np.array(pts, np.float32).reshape(-1, 3)), bool).reshape(len(prims), S - 1)
        expanded += len(frontier)
        nxt = []
        for (m, pi, last), h in zip(prims, hit):
            if h.any():
                continue
            c = (last[0], last[1], wrap_pi(last[2]), nodes[m][3] + pcost[pi], m, depth)
            if dedup:
                k = key_of(c)
                if k in closed and closed[k] <= c[3]:
                    continue
                closed[k] = c[3]
            nodes.append(c)
            (cands if at_goal(c[0], c[1]) else nxt).append(len(nodes) - 1)
        nxt.sort(key=lambda i: nodes[i][3] + h_of(nodes[i][0], nodes[i][1]))   # stable: creation order on ties
        frontier = sorted(nxt[:int(p.beam)])
    if cands:
        reached = True
        pick = sorted(cands, key=lambda i: nodes[i][3])
    else:
        reached = False
        pick = sorted(range(1, len(nodes)), key=lambda i: (h_of(nodes[i][0], nodes[i][1]), nodes[i][3]))
    return dict(cands=pick[:int(p.n_traj)], nodes=nodes, reached=reached, expanded=expanded)


def tree_waypoints(res, max_depth):
    """Candidate waypoints [K, max_depth + 1] (x, y, yaw; NaN after the last primitive) and costs."""
    K, T = len(res["cands"]), max_depth + 1
    out = [np.full((K, T), np.nan, np.float32) for _ in range(3)]
    cost = np.zeros(K)
    for c, i in enumerate(res["cands"]):
        cost[c] = res["nodes"][i][3]
        while i >= 0:
            n = res["nodes"][i]
            out[0][c, n[5]], out[1][c, n[5]], out[2][c, n[5]] = n[0], n[1], n[2]
            i = n[4]
    return out[0], out[1], out[2], cost

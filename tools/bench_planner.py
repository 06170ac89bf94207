"""Measurements of the planner rows beyond the scoring step, CUDA events on the
calling stream, warm-up first; one JSON line per measurement.

  N3  rtg_plan_tree, the Fig. 4 analogue: paper defaults (N_v = 3, N_w = 5, v_max = 0.6,
      w_max = 0.9, 1 s primitives), goal 5 m ahead, depth 8, beam 4096, 5 samples per
      primitive, on outdoor-recipe maps of N = 1e5 .. 5e6 Gaussians (fixed 100 m x 100 m area);
      then the whole low-level cycle: 1024 tree candidates scored (rtg_score) and the argmax.
  N4  rtg_ledger_update + rtg_map_update_weights (ledger -> reclassified map, no repacking), N = 2M.
  N2  rtg_region_utility over a 2.5 m partition of the outdoor map, and 8,192 gain-only
      views (rtg_traj_view_ring around the top regions + rtg_score) + rtg_cost_benefit.

usage: python tools/bench_planner.py [--sizes 1e5,5e5,1e6,2e6,5e6] [--reps 5]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_18122_b200 import rtg as R  # noqa: E402
from paper_2409_18122_b200 import workloads as W  # noqa: E402


def timed(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        out = fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


def to_dev(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1e5,5e5,1e6,2e6,5e6")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    # ---- N3: tree planning time vs map size
    for n in [int(float(v)) for v in args.sizes.split(",")]:
        wl = W.outdoor(N=n, K=1, T=1)
        m = R.map_from_workload(wl)
        h0 = float(W.Terrain(np.random.default_rng(0)).h(np.array([0.0]), np.array([0.0]))[0]) + 0.5
        tp = R.make_tree_params(max_depth=8, beam=4096, z=h0)
        ms, out = timed(lambda: R.plan_tree(m, (0.0, 0.0, 0.0), (5.0, 0.0), tp), args.reps)
        tr, cost, reached, stats = out
        print(json.dumps({"row": "N3 rtg_plan_tree", "N": n, "ms": ms, "reached": reached, "candidates": len(cost),
                          "best_cost": float(cost[0]) if len(cost) else None, **stats}), flush=True)
        tr.close()
        # the whole low-level cycle of P:307-320: tree candidates -> scored at their segment end states
        # (Eq. traj_utility, gain-only on the collision-free primitives) -> argmax
        sp = R.make_params(mode=R.MODE_CULLED, flags=R.SCORE_FULL_GAIN | R.SCORE_NO_COLLISION)
        tp_many = R.make_tree_params(max_depth=8, beam=4096, z=h0, n_traj=1024)

        def cycle():
            t2, c2, r2, _ = R.plan_tree(m, (0.0, 0.0, 0.0), (5.0, 0.0), tp_many)
            out = R.score(m, t2, wl.camera, sp)
            b = R.best(out[3])
            t2.close()
            return b
        ms_c, b = timed(cycle, args.reps)
        print(json.dumps({"row": "N3 plan cycle (tree -> 1024 candidates -> rtg_score -> rtg_best)", "N": n,
                          "ms": ms_c, "best": list(b)}), flush=True)
        m.close()
    # ---- N4: ledger update and in-place reclassification, 2M
    wl = W.outdoor()
    dm = [to_dev(a) for a in (wl.means, wl.quats, wl.scales, wl.opacity, wl.info_w, wl.flags)]
    m = R.Map(*dm, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g)
    rng = np.random.default_rng(3)
    cur = wl.means + (rng.normal(0, 0.01, wl.means.shape) * (rng.random(wl.N) < 0.3)).astype(np.float32)
    prev_d, cur_d, w_d = to_dev(wl.means), to_dev(cur), to_dev(wl.info_w)
    w_out = torch.empty_like(w_d)
    ms_l, _ = timed(lambda: R.ledger_update(prev_d, cur_d, w_d, w_out), args.reps)
    ms_u, _ = timed(lambda: m.update_weights(w_out), args.reps)
    print(json.dumps({"row": "N4 rtg_ledger_update", "N": wl.N, "ms": ms_l}), flush=True)
    print(json.dumps({"row": "N4 rtg_map_update_weights", "N": wl.N, "ms": ms_u}), flush=True)
    # ---- N2: region utility (2.5 m), views around the top regions, cost-benefit
    lo = wl.means.min(axis=1) - 1e-3
    dims = np.ceil((wl.means.max(axis=1) - lo) / 2.5).astype(int) + 1
    ms_r, (om, cnt) = timed(lambda: R.region_utility(m, lo, 2.5, dims), args.reps)
    print(json.dumps({"row": "N2 rtg_region_utility", "N": wl.N, "regions": int(np.prod(dims)), "ms": ms_r}),
          flush=True)
    top = torch.topk(om, 1024).indices.cpu().numpy()
    iz, iy, ix = top // (dims[0] * dims[1]), (top // dims[0]) % dims[1], top % dims[0]
    cen = np.stack([lo[0] + (ix + 0.5) * 2.5, lo[1] + (iy + 0.5) * 2.5, lo[2] + (iz + 0.5) * 2.5]).astype(np.float32)
    p = R.make_params(mode=R.MODE_CULLED, flags=R.SCORE_FULL_GAIN | R.SCORE_NO_COLLISION)
    d = torch.from_numpy(np.linalg.norm(cen[:2], axis=0).astype(np.float64).repeat(8)).cuda()   # stand-in path distances (FP64, as the ABI reads them)

    def views():
        tr, _ = R.Traj.view_ring(torch.from_numpy(cen).cuda(), 2.5, wl.camera, 8, float(cen[2].mean()))
        fc, fe, g, u = R.score(m, tr, wl.camera, p)
        best = R.cost_benefit(g, d)
        tr.close()
        return best
    ms_v, best = timed(views, args.reps)
    print(json.dumps({"row": "N2 views (1024 regions x 8, ring + score + cost-benefit)", "N": wl.N, "views": 8192,
                      "ms": ms_v, "best": best}), flush=True)
    m.close()


if __name__ == "__main__":
    main()

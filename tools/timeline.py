"""GPU timeline of one outdoor planning cycle (torch.profiler / CUPTI kernel activity): every kernel
and memcpy/memset with its start offset and duration, and the idle gaps between them.

usage: python tools/timeline.py [--config outdoor] [--tree | --score eager|graph | --cycle eager|graph [--ranks N]]
  --tree: one rtg_plan_tree call (depth 8, beam 4096, goal 5 m ahead) on the config's map instead
  --cycle: the whole cycle on a layout map (rebuild + score + best, views on a forked stream), eager or as
           one CUDA graph (R.CycleGraph); --ranks N scores rank 0's interleaved 1/N shard (tools/shard_model.py)
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_18122_b200 import rtg as R  # noqa: E402
from paper_2409_18122_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="outdoor")
    ap.add_argument("--tree", action="store_true")
    ap.add_argument("--score", choices=("eager", "graph"), default=None,
                    help="only the scoring part (rtg_score + rtg_best_async) on a built map, eager or as one "
                         "CUDA-graph replay (R.ScoreGraph)")
    ap.add_argument("--cycle", choices=("eager", "graph"), default=None)
    ap.add_argument("--ranks", type=int, default=1)
    ap.add_argument("--host", action="store_true",
                    help="the standard cycle from pinned host buffers (bench.py's e2e step: map and waypoint "
                         "uploads inside, the waypoints on a second stream overlapping the map build)")
    args = ap.parse_args()
    wl = W.make(args.config)
    if args.ranks > 1:
        wl = W.subset_trajectories(wl, np.arange(0, wl.K, args.ranks))
    dev = torch.device("cuda", 0)
    to_dev = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    dmap = [to_dev(a) for a in (wl.means, wl.quats, wl.scales, wl.opacity, wl.info_w, wl.flags)]
    dtraj = [to_dev(a) for a in (wl.x, wl.y, wl.z, wl.yaw)]
    cam = R.make_camera(wl.camera)
    params = R.make_params(mode=R.MODE_CULLED)
    K = wl.K
    outs = (torch.empty(K, dtype=torch.int32, device=dev), torch.empty(K, dtype=torch.uint8, device=dev),
            torch.empty(K, dtype=torch.float64, device=dev), torch.empty(K, dtype=torch.float64, device=dev))

    tree_map = R.Map(*dmap, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g, collide_rule=wl.robot.rule) \
        if args.tree else None
    tp = R.make_tree_params(max_depth=8, beam=4096, z=float(wl.z.reshape(-1)[0]))

    def tree_step():
        t2, _, _, _ = R.plan_tree(tree_map, (0.0, 0.0, 0.0), (5.0, 0.0), tp)
        t2.close()

    score_map = score_tr = sg = None
    if args.score:
        score_map = R.Map(*dmap, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g, collide_rule=wl.robot.rule)
        score_tr = R.Traj.wrap(*dtraj)
        bo = torch.empty(2, dtype=torch.float64, device=dev)
        if args.score == "graph":
            sg = R.ScoreGraph(score_map, score_tr, cam, params)

    pin = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hmap = [pin(a) for a in (wl.means, wl.quats, wl.scales, wl.opacity, wl.info_w, wl.flags)] if args.host else None
    htraj = [pin(a) for a in (wl.x, wl.y, wl.z, wl.yaw)] if args.host else None
    aux = torch.cuda.Stream(device=dev)
    cg = None
    if args.cycle:
        import bench as BN
        gbox, cbox, rb_b, rho_b = BN.layout_bounds(wl)
        lm = R.LayoutMap(wl.N, gbox, cbox, rb_b, rho_b, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g,
                         collide_rule=wl.robot.rule)
        ctr = R.Traj.wrap(*dtraj)
        ctv = None
        if wl.views is not None:
            vi = np.arange(0, wl.views["x"].shape[0], args.ranks)
            ctv = R.Traj.wrap(*[to_dev(wl.views[c][vi]) for c in ("x", "y", "z", "yaw")])
        vparams = R.make_params(mode=R.MODE_CULLED, flags=R.SCORE_FULL_GAIN | R.SCORE_NO_COLLISION)
        cg = R.CycleGraph(lm, dmap, ctr, cam, params, views=ctv, vparams=vparams if ctv is not None else None)
        if args.cycle == "eager":
            cycle_eager = cg.graph   # keep the graph alive; the eager path re-issues the same calls
            vst = torch.cuda.Stream(device=dev)
            vbo = torch.empty(2, dtype=torch.float64, device=dev)
            bo2 = torch.empty(2, dtype=torch.float64, device=dev)

    def step():
        if cg is not None:
            if args.cycle == "graph":
                return cg.replay()
            cur = torch.cuda.current_stream()
            lm.rebuild(*dmap)
            if ctv is not None:
                vst.wait_stream(cur)
                R.score(lm, ctv, cam, vparams, *cg.vouts, stream=vst)
                R.best_async(cg.vouts[3], vbo, stream=vst)
            R.score(lm, ctr, cam, params, *outs)
            R.best_async(outs[3], bo2)
            if ctv is not None:
                cur.wait_stream(vst)
            return None
        if args.tree:
            return tree_step()
        if sg is not None:
            return sg.replay()
        if args.score:
            R.score(score_map, score_tr, cam, params, *outs)
            return R.best_async(outs[3], bo)
        if args.host:
            cur = torch.cuda.current_stream()
            src = [None if h is None else h.to(dev, non_blocking=True) for h in hmap]
            copied = torch.cuda.Event()
            copied.record(cur)
            aux.wait_event(copied)
            tr = R.Traj.upload(*htraj, stream=aux)
            m = R.Map(*src, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g, collide_rule=wl.robot.rule)
            cur.wait_stream(aux)
            R.score(m, tr, cam, params, *outs)
            r = R.best(outs[3])
            m.close()
            aux.wait_stream(cur)
            tr.close()
            return r
        m = R.Map(*dmap, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g, collide_rule=wl.robot.rule)
        tr = R.Traj.upload(*dtraj)
        R.score(m, tr, cam, params, *outs)
        r = R.best(outs[3])
        m.close()
        tr.close()
        return r

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):            # the last of three profiled cycles is reported (the first pays
            torch.cuda.synchronize()  # the profiler's own start-up)
            step()
            torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    first = "k_tree_init" if args.tree else ("k_set_cam64" if args.score else "k_bounds_init")
    starts = [i for i, e in enumerate(ev) if first in e.name]
    if args.host and starts:   # the cycle begins with the map's uploads just before its first kernel
        j = starts[-1]
        while j > 0 and "Memcpy HtoD" in ev[j - 1].name:
            j -= 1
        starts[-1] = j
    if not starts:   # (a layout rebuild starts elsewhere: the first event after the last synchronisation)
        starts = [0]
    ev = ev[starts[-1]:]
    t0 = ev[0].time_range.start
    prev_end = t0
    gaps = 0.0
    print(f"{'start_us':>9} {'dur_us':>8} {'gap_us':>7}  name")
    for e in ev:
        s, d = e.time_range.start, e.time_range.end - e.time_range.start
        gap = max(0.0, s - prev_end)
        gaps += gap
        print(f"{s - t0:9.1f} {d:8.1f} {gap:7.1f}  {e.name[:90]}")
        prev_end = max(prev_end, e.time_range.end)
    print(f"total {prev_end - t0:.1f} us, idle gaps {gaps:.1f} us")


if __name__ == "__main__":
    main()

"""Per-rank cycle time of the N-GPU strong-scaling plan, measured on one GPU (SURVEY §8(e) model).

At N ranks each rank builds the whole (replicated) map and scores its interleaved 1/N of the
trajectories and views (rank 0's shard here: k = 0, N, 2N, ...), then exchanges 16 bytes.  The ranks
share nothing else, so the per-rank time on an otherwise idle GPU is the N-GPU cycle minus the
exchange (a few tens of µs over NVLink; not measured here: one GPU).  This runs that per-rank step for
N = 1, 2, 4, 8 back to back on the one GPU (CUDA events, L2 flushed between steps) and reports
T(1) / T(N).  It is a measured model, not a multi-GPU measurement.

usage: python tools/shard_model.py [--config scale] [--steps 10] > profiles/r2_shard_model.jsonl
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_18122_b200 import rtg as R  # noqa: E402
from paper_2409_18122_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="scale")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--cells", default=None, help="visibility grid 'hy,hx,hz' [m] (rtg_map_options)")
    ap.add_argument("--z-centre", default="none", help="as bench.py: 'none', 'camera' or a height [m]")
    ap.add_argument("--graph", action="store_true",
                    help="each rank's cycle as one CUDA graph: layout map rebuilt without a host synchronisation "
                         "+ score + argmax (+ the views on a forked stream), R.CycleGraph")
    args = ap.parse_args()
    wl = W.make(args.config)
    dev = torch.device("cuda", 0)
    to_dev = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    dmap = [to_dev(a) for a in (wl.means, wl.quats, wl.scales, wl.opacity, wl.info_w, wl.flags)]
    cam = R.make_camera(wl.camera)
    params = R.make_params(mode=R.MODE_CULLED)
    vparams = R.make_params(mode=R.MODE_CULLED, flags=R.SCORE_FULL_GAIN | R.SCORE_NO_COLLISION)
    flush = torch.empty(512 << 18, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream()
    vstream = torch.cuda.Stream(device=dev)
    opts = None
    if args.cells:
        hy, hx, hz = (float(v) for v in args.cells.split(","))
        opts = (hy, hz, 0.0, hx)
    zc = None if args.z_centre == "none" else (float(np.median(wl.z)) if args.z_centre == "camera"
                                                 else float(args.z_centre))
    if zc is not None:
        opts = (opts or (0.0, 0.0, 0.0, 0.0)) + (zc,)
    base = None
    for n in (int(v) for v in args.ranks.split(",")):
        idx = np.arange(0, wl.K, n)
        traj = [to_dev(a[idx]) for a in (wl.x, wl.y, wl.z, wl.yaw)]
        views = None
        if wl.views is not None:
            vi = np.arange(0, wl.views["x"].shape[0], n)
            views = [to_dev(wl.views[c][vi]) for c in ("x", "y", "z", "yaw")]
        K = len(idx)
        outs = (torch.empty(K, dtype=torch.int32, device=dev), torch.empty(K, dtype=torch.uint8, device=dev),
                torch.empty(K, dtype=torch.float64, device=dev), torch.empty(K, dtype=torch.float64, device=dev))

        prof_on = [False]

        def step():
            m = R.Map(*dmap, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g, collide_rule=wl.robot.rule,
                      options=opts)
            if views is not None:
                vstream.wait_stream(st)   # views: the map build only, then concurrent (as bench.py)
            tr = R.Traj.wrap(*traj)
            R.score(m, tr, cam, params, *outs)
            if views is not None:   # (phase timers on the trajectories' stream only, as bench.py)
                if prof_on[0]:
                    R.profile_enable(False)
                tv = R.Traj.wrap(*views)
                fc, fe, g, u = R.score(m, tv, cam, vparams, stream=vstream)
                if prof_on[0]:
                    R.profile_enable(True)
            r = R.best(outs[3])
            if views is not None:
                if prof_on[0]:
                    R.profile_enable(False)
                R.best(u, stream=vstream)
                if prof_on[0]:
                    R.profile_enable(True)
                st.wait_stream(vstream)
                tv.close()
            tr.close()
            m.close()
            return r

        cg = None
        if args.graph:
            # the rank's whole cycle as one CUDA graph (no host synchronisation: a layout map from the
            # workload's extents, as bench.py's cuda_graph.cycle); per-phase timers do not run in a graph
            import bench as BN
            gbox, cbox, rb_b, rho_b = BN.layout_bounds(wl)
            lm = R.LayoutMap(wl.N, gbox, cbox, rb_b, rho_b, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g,
                             collide_rule=wl.robot.rule, options=opts)
            gtr = R.Traj.wrap(*traj)
            gtv = R.Traj.wrap(*views) if views is not None else None
            cg = R.CycleGraph(lm, dmap, gtr, cam, params, views=gtv, vparams=vparams if views is not None else None)
            step = cg.replay   # noqa: F811
        for _ in range(3):
            step()
        ms = []
        R.profile_read(reset=True)
        R.profile_enable(cg is None)
        prof_on[0] = cg is None
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            step()
            b.record(st)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        R.profile_enable(False)
        prof_on[0] = False
        prof = R.profile_read(reset=True)
        if cg is not None:
            lm.check()
            del cg
            gtr.close()
            if gtv is not None:
                gtv.close()
            lm.close()
        med = statistics.median(ms)
        base = med if base is None else base
        print(json.dumps({"config": args.config, "cells": args.cells, "gain_z_centre": zc, "graph": args.graph,
                          "ranks": n, "trajectories_per_rank": K,
                          "views_per_rank": len(views[0]) if views is not None else 0,
                          "per_rank_ms_median": med, "per_rank_ms_min": min(ms),
                          "modelled_speedup": base / med,
                          "phase_ms": {k: round(v / args.steps, 4) for k, v in prof["ms"].items()},
                          "launches_per_step": prof["launches"] / args.steps,
                          "note": "rank 0's shard on one GPU; excludes the 16-byte NCCL exchange"}), flush=True)


if __name__ == "__main__":
    main()

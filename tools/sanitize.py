"""Small planning cycles for compute-sanitizer (SURVEY §4 test layer 5): tiny and a room subset, both modes,
the debug path (pair mask, per-waypoint arrays), include_start, the samplers, a plan_tree call and the
N2/N4 entry points.  usage: compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_18122_b200 import rtg as R  # noqa: E402
from paper_2409_18122_b200 import workloads as W  # noqa: E402


def cycle(wl, mode, start=None):
    m = R.map_from_workload(wl)
    tr = R.traj_from_workload(wl)
    flags = R.SCORE_FULL_GAIN
    if start is not None:
        tr.set_start(start)
        flags |= R.SCORE_INCLUDE_START
    p = R.make_params(mode=mode, flags=flags)
    fc, fe, g, u = R.score(m, tr, wl.camera, p)
    b = R.best(u)
    d = R.score_debug(m, tr, wl.camera, p, pair_mask=wl.N * wl.K * wl.T <= 4e6)
    torch.cuda.synchronize()
    tr.close()
    return m, b, d


def main():
    tiny = W.tiny()
    room = W.subset_trajectories(W.room(N=20000, K=64, T=30), np.arange(0, 64, 4))
    for wl in (tiny, room):
        for mode in (R.MODE_CULLED, R.MODE_DENSE):
            m, b, _ = cycle(wl, mode, start=(0.0, 0.0, 0.5, 0.2))
            print(wl.name, mode, b)
            m.close()
    m, _, _ = cycle(room, R.MODE_CULLED)
    v = torch.full((8,), 0.8, device="cuda")
    w = torch.linspace(-0.5, 0.5, 8, device="cuda")
    ts = R.Traj.sample_unicycle(v, w, 20, 0.1, (0.0, 0.0, 0.5, 0.0))
    R.score(m, ts, room.camera, R.make_params(flags=R.SCORE_INCLUDE_START))
    ts.close()
    tp = R.make_tree_params(max_depth=4, beam=256, z=0.5)
    t2, cost, reached, stats = R.plan_tree(m, (0.0, 0.0, 0.0), (3.0, 0.0), tp)
    t2.close()
    om, cnt = R.region_utility(m, (-6.0, -5.0, 0.0), 2.5, (5, 4, 2))
    nw = R.ledger_update(torch.from_numpy(room.means).cuda(), torch.from_numpy(room.means).cuda() + 0.01,
                         torch.from_numpy(room.info_w).cuda())
    m.update_weights(nw)
    torch.cuda.synchronize()
    m.close()
    print("sanitize cycles ok")


if __name__ == "__main__":
    main()

"""GPU diagnostics: per-waypoint work statistics and phase times of the culled path.

usage: python tools/diag.py [config] [K] [gain_cell_xy gain_cell_z col_cell ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2409_18122_b200 import rtg as R
from paper_2409_18122_b200 import workloads as W


def run(cfg="outdoor", K=2048, opts=None, reps=3, mode="culled", stride=1, flags=0):
    wl = W.make(cfg)
    idx = np.arange(0, wl.K, max(1, wl.K // K))[:K]
    m = R.map_from_workload(wl, options=opts)
    info = m.info()
    tr = R.traj_from_workload(wl, x=wl.x[idx], y=wl.y[idx], z=wl.z[idx], yaw=wl.yaw[idx])
    p = R.make_params(mode=R.MODE_CULLED if mode == "culled" else R.MODE_DENSE, info_stride=stride, flags=flags)
    R.score(m, tr, wl.camera, p)
    torch.cuda.synchronize()
    R.profile_read(True)
    R.profile_enable(True)
    for _ in range(reps):
        fc, fe, g, u = R.score(m, tr, wl.camera, p)
    torch.cuda.synchronize()
    R.profile_enable(False)
    prof = R.profile_read(True)
    feas = fe.float().mean().item()
    out = dict(cfg=cfg, K=len(idx), opts=opts, mode=mode, feasible=feas,
               gain_dims=list(info.gain_dims), col_dims=list(info.col_dims), rb_max=info.rb_max,
               ms={k: round(v / reps, 4) for k, v in prof["ms"].items() if v})
    if mode == "culled":
        # per-waypoint statistics on a small subset via the debug entry point
        sub = idx[:64]
        trs = R.traj_from_workload(wl, x=wl.x[sub], y=wl.y[sub], z=wl.z[sub], yaw=wl.yaw[sub])
        d = R.score_debug(m, trs, wl.camera, p)
        nwp = len(sub) * wl.T
        out["per_wp"] = {k: v / nwp for k, v in d["stats"].items()}
        out["visible_per_wp"] = float((d["wp_nh"].double().mean() + 0).item())
        trs.close()
    ms_b = prof["ms"]["visibility_gain"] / reps
    out["gain_ns_per_wp"] = 1e6 * ms_b / max(1.0, feas * len(idx) * wl.T / stride)
    print(json.dumps(out), flush=True)
    m.close()
    tr.close()


if __name__ == "__main__":
    cfg = sys.argv[1] if len(sys.argv) > 1 else "outdoor"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    rest = [float(a) for a in sys.argv[3:]]
    if not rest:
        run(cfg, K)
    for i in range(0, len(rest), 3):
        run(cfg, K, opts=tuple(rest[i:i + 3]))

"""Collision-phase time (a4) of the outdoor workload for several collision-grid cell sizes."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2409_18122_b200 import rtg as R, workloads as W

wl = W.make(sys.argv[1] if len(sys.argv) > 1 else "outdoor")
dev = torch.device("cuda")
dm = [None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
      for a in (wl.means, wl.quats, wl.scales, wl.opacity, wl.info_w, wl.flags)]
tr = R.traj_from_workload(wl)
p = R.make_params(mode=R.MODE_CULLED, info_stride=wl.T + 1)   # no info waypoint: collision only
for cc in [float(c) for c in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0.5", "0.75", "1.0", "1.5"])]:
    m = R.Map(*dm, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g, device=0, options=(0.0, 0.0, cc, 0.0))
    for _ in range(3):
        fc, fe, g, u = R.score(m, tr, wl.camera, p)
    torch.cuda.synchronize()
    R.profile_read(reset=True)
    R.profile_enable(True)
    for _ in range(5):
        R.score(m, tr, wl.camera, p)
    torch.cuda.synchronize()
    R.profile_enable(False)
    pr = R.profile_read(reset=True)
    print(f"col_cell {cc}: collision {pr['ms']['collision'] / 5:.3f} ms, feasible {int(fe.sum())}, "
          f"dims {list(m.info().col_dims)}", flush=True)
    m.close()

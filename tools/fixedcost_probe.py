import sys, dataclasses, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2409_18122_b200 import rtg as R, workloads as W
wl = W.outdoor()
m = R.map_from_workload(wl)
tr = R.traj_from_workload(wl)
for zf in (15.0, 8.0, 4.0, 1.0, 0.4):
    cam = dataclasses.replace(wl.camera, z_far=zf)
    p = R.make_params(mode=R.MODE_CULLED, flags=0)
    for _ in range(3): R.score(m, tr, cam, p)
    torch.cuda.synchronize()
    R.profile_read(reset=True); R.profile_enable(True)
    for _ in range(5): R.score(m, tr, cam, p)
    torch.cuda.synchronize(); R.profile_enable(False)
    pr = R.profile_read(reset=True)
    fe = R.score(m, tr, cam, p)[1]
    nf = int(fe.sum().item())
    # work per waypoint
    idx = np.nonzero(fe.cpu().numpy())[0][:48]
    t2 = R.traj_from_workload(wl, x=wl.x[idx], y=wl.y[idx], z=wl.z[idx], yaw=wl.yaw[idx])
    d = R.score_debug(m, t2, cam, R.make_params(mode=R.MODE_CULLED, flags=R.SCORE_FULL_GAIN))["stats"]
    t2.close()
    nwp = len(idx) * wl.T
    print(f"z_far {zf}: gain {pr['ms']['visibility_gain']/5:.3f} ms, info wp {nf*100}, per-wp-per-warp {pr['ms']['visibility_gain']/5*1e3/(nf*100)*5328:.2f} us, "
          f"tests {d['tested']/nwp:.0f} units {d['units']/nwp:.0f} rows {d['rows']/nwp:.0f}")

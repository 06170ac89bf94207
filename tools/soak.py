"""Soak: many planning cycles (map create -> score -> best -> destroy, and plan_tree) in one
process; device free memory and cycle time are printed every 50 cycles (leaks or drift show up).

usage: python tools/soak.py [--cycles 300]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_18122_b200 import rtg as R  # noqa: E402
from paper_2409_18122_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=300)
    args = ap.parse_args()
    wl = W.outdoor()
    dev = torch.device("cuda", 0)
    to_dev = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    dmap = [to_dev(a) for a in (wl.means, wl.quats, wl.scales, wl.opacity, wl.info_w, wl.flags)]
    dtraj = [to_dev(a) for a in (wl.x, wl.y, wl.z, wl.yaw)]
    cam = R.make_camera(wl.camera)
    tp = R.make_tree_params(max_depth=8, beam=4096, z=float(wl.z.reshape(-1)[0]))
    t0 = time.perf_counter()
    for c in range(1, args.cycles + 1):
        m = R.Map(*dmap, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g, collide_rule=wl.robot.rule)
        tr = R.Traj.upload(*dtraj)
        out = R.score(m, tr, cam, R.make_params())
        b = R.best(out[3])
        t2, _, _, _ = R.plan_tree(m, (0.0, 0.0, 0.0), (5.0, 0.0), tp)
        t2.close()
        tr.close()
        m.close()
        del out
        if c % 50 == 0:
            torch.cuda.synchronize()
            free, total = torch.cuda.mem_get_info()
            print(f"cycle {c}: {1000 * (time.perf_counter() - t0) / 50:.2f} ms/cycle (host wall), best {b}, "
                  f"free {free / 2**30:.2f} GiB of {total / 2**30:.1f}", flush=True)
            t0 = time.perf_counter()


if __name__ == "__main__":
    main()

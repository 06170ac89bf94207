"""The C ABI used from plain C: examples/c_score.c builds with gcc against include/rtg.h and
librtg.so alone, and (on a GPU) prints the same best trajectory as the Python binding on the same
inputs (its splitmix64 input generator is re-implemented here)."""
import math
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "examples", "c_score.c")
CUDA = "/usr/local/cuda"


def _build(out):
    from paper_2409_18122_b200 import build as B
    B.build()
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include",
           SRC, "-L", os.path.join(ROOT, "paper_2409_18122_b200"), "-lrtg", "-L", f"{CUDA}/lib64", "-lcudart",
           f"-Wl,-rpath,{os.path.join(ROOT, 'paper_2409_18122_b200')}", "-lm", "-o", out]
    subprocess.check_call(cmd)


def test_c_example_builds(tmp_path):
    exe = str(tmp_path / "c_score")
    _build(exe)
    assert os.path.exists(exe)


class _SplitMix:
    def __init__(self):
        self.s = 0x9e3779b97f4a7c15

    def urand(self):
        m = (1 << 64) - 1
        self.s = (self.s + 0x9e3779b97f4a7c15) & m
        z = self.s
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & m
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & m
        z ^= z >> 31
        return (z >> 11) * (1.0 / 9007199254740992.0)


def _inputs(N, K, T):
    r = _SplitMix()
    means = np.zeros((3, N), np.float32)
    quats = np.zeros((4, N), np.float32)
    scales = np.zeros((3, N), np.float32)
    opac = np.zeros(N, np.float32)
    w = np.zeros(N, np.float32)
    for i in range(N):
        means[0, i] = 40.0 * r.urand() - 20.0
        means[1, i] = 40.0 * r.urand() - 20.0
        means[2, i] = 3.0 * r.urand()
        q = [r.urand() - 0.5 for _ in range(4)]
        qn = math.sqrt(sum(c * c for c in q))
        quats[:, i] = [c / qn for c in q]
        for c in range(3):
            scales[c, i] = 0.02 + 0.2 * r.urand()
        opac[i] = r.urand()
        w[i] = r.urand()
    x, y = np.zeros((K, T), np.float32), np.zeros((K, T), np.float32)
    for k in range(K):
        h = -1.57 + 3.14 * (k + 0.5) / K
        v = 0.5 + r.urand()
        for t in range(T):
            s = v * 0.1 * (t + 1)
            x[k, t] = s * math.cos(h)
            y[k, t] = s * math.sin(h)
    yaw = np.repeat(np.float32([-1.57 + 3.14 * (k + 0.5) / K for k in range(K)])[:, None], T, axis=1)
    return means, quats, scales, opac, w, x, y, np.full((K, T), 1.5, np.float32), yaw


@pytest.mark.gpu
def test_c_example_matches_binding(tmp_path):
    import torch
    from paper_2409_18122_b200 import rtg as R
    N, K, T = 3000, 64, 20
    exe = str(tmp_path / "c_score")
    _build(exe)
    out = subprocess.check_output([exe, str(N), str(K), str(T)], text=True).split()
    assert out[0] == "best" and out[3] == "feasible"
    c_idx, c_score, c_feas = int(out[1]), float(out[2]), int(out[4])
    means, quats, scales, opac, w, x, y, z, yaw = _inputs(N, K, T)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    m = R.Map(dev(means), dev(quats), dev(scales), dev(opac), dev(w), None, r_robot=0.3, lambda_g=3.0)
    tr = R.Traj.upload(dev(x), dev(y), dev(z), dev(yaw))
    from paper_2409_18122_b200 import workloads as W
    cam = R.make_camera(W.Camera(320, 240, 250.0, 250.0, 160.0, 120.0, 0.1, 6.0))
    fc, fe, g, u = R.score(m, tr, cam, R.make_params(mode=R.MODE_CULLED))
    b = R.best(u)
    assert int(fe.sum().item()) == c_feas
    assert b[1] == c_idx and abs(b[0] - c_score) <= 0.05   # xi is integer-valued; printed with %.1f
    m.close()
    tr.close()

#!/usr/bin/env python
"""Benchmark of the RT-GuIDE trajectory-scoring hot path on B200 (BASELINE.json metric).

One step = one planning cycle through the C ABI, every §8(a) row:
  a1+a2 rtg_map_create   (pack + classify + grids, from device-resident raw map arrays)
  a3    rtg_traj_upload  (device-resident waypoints of this rank's shard)
  a4-a6 rtg_score        (collision, visibility + gain, per-trajectory reduction)
  a7    rtg_best (+ NCCL all_gather of (score, index) across ranks when N > 1)
Workload: BASELINE.json configs[3] "outdoor" (N=2,000,000 Gaussians, K=16,384 trajectories,
T=100 waypoints) per GPU; trajectories of the global set are interleaved over ranks
(k = rank mod N): weak scaling, global K = 16,384 * N.

value = nominal waypoint x Gaussian pair-tests per second over all ranks (K*T*N / step time,
every pair counted once whether or not it was culled); ms_per_step = planning-cycle latency.
e2e   = the same step from pinned HOST buffers (H2D copies + 16-byte D2H result inside).
ms_per_step_median / _p90 = per-step latency distribution over the timed steps (max over ranks per step).

`--impl reference` times the CPU oracle (oracle/, the test-only FP64 reference) on a bounded
sample of the same workload and prints the same JSON line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "waypoint x Gaussian pair-tests/s (planning cycle, nominal pairs)"
UNIT = "pair-tests/s"
L2_FLUSH_BYTES = 512 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="rtg", choices=["rtg", "reference"])
    ap.add_argument("--config", default="outdoor", choices=["tiny", "room", "multi_room", "outdoor", "scale"])
    ap.add_argument("--mode", default="culled", choices=["culled", "dense"])
    ap.add_argument("--stride", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph replay of the scoring part")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=-1, help="steps timed per phase (default: all)")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="weak: K trajectories per GPU; strong: the config's K shared by the GPUs "
                         "(default: strong for the scale config, which fixes the total K, else weak)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: exercise the multi-rank code path with "
                         "several ranks on one GPU; the (score, index) exchange then runs on the host)")
    ap.add_argument("--z-centre", default="none",
                    help="visibility z-cells: 'none' starts them at the lowest mean (default), 'camera' centres one "
                         "on the waypoints' median camera height (rtg_map_options.gain_z_centre), or a height [m]")
    ap.add_argument("--cells", default=None,
                    help="visibility grid cells 'hy,hx,hz' [m] (rtg_map_options; default: library defaults)")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------- reference arm (CPU oracle)
def oracle_sample(wl, n_traj, seed=7):
    import numpy as np
    from oracle import oracle as O
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(wl.K, size=min(n_traj, wl.K), replace=False))
    t0 = time.perf_counter()
    O.score(wl, traj_idx=idx)
    dt = time.perf_counter() - t0
    pairs = len(idx) * wl.T * wl.N
    return pairs / dt, dt, len(idx)


def oracle_threads():
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_2409_18122_b200 import workloads as W
    O.build()
    wl = W.make(args.config)
    cores = oracle_threads()
    n_traj = max(1, min(wl.K, cores))
    vals, times = [], []
    for i in range(args.warmup + args.steps):
        v, dt, nt = oracle_sample(wl, n_traj, seed=100 + i)
        if i >= args.warmup:
            vals.append(v)
            times.append(dt)
    value = statistics.median(vals)
    sample = f"{n_traj} random trajectories x T={wl.T} x N={wl.N} per step (full K={wl.K} extrapolated linearly)"
    ms_full = 1000.0 * wl.K * wl.T * wl.N / value
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_full, "higher_is_better": True,
            # ms_per_step is NOT measured: each timed step scores a sample of the workload; the full
            # planning cycle's time is that sample's rate extrapolated linearly in trajectories
            "extrapolated": {"ms_per_step": True, "measured_ms_per_sample_step": 1000.0 * statistics.median(times),
                             "sample_trajectories": n_traj, "full_trajectories": wl.K,
                             "factor": wl.K / n_traj, "method": "linear in trajectories (oracle cost is per pair)"},
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} (BASELINE.json configs[3])" if args.config == "outdoor"
                       else args.config, "N": wl.N, "K": wl.K, "T": wl.T},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- rtg arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2409_18122_b200 import build as B
    B.build()
    from paper_2409_18122_b200 import dist as D
    from paper_2409_18122_b200 import rtg as R
    from paper_2409_18122_b200 import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    ndev = torch.cuda.device_count()
    if world > ndev and args.backend == "nccl":
        raise SystemExit(f"{world} ranks need {world} GPUs with NCCL ({ndev} visible); use --backend gloo")
    local_dev = local % ndev                    # gloo on one GPU: every rank shares cuda:0
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    cdev = dev if args.backend == "nccl" else torch.device("cpu")   # where collective tensors live
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    # ---- workload: the map is replicated; the global trajectory set (and the gain-only views of the
    # scale config) is interleaved over ranks: weak scaling grows it with the ranks, strong keeps it
    scaling = args.scaling or ("strong" if args.config == "scale" else "weak")
    base = W.make(args.config)
    glob = base if (world == 1 or scaling == "strong") else W.make(args.config, K=base.K * world)
    K_glob = glob.K
    wl = W.subset_trajectories(glob, np.arange(rank, glob.K, world)) if world > 1 else glob
    N, K, T = wl.N, wl.K, wl.T
    views = None
    Kv_glob = 0
    if glob.views is not None:
        vsel = np.arange(rank, glob.views["x"].shape[0], world)
        views = [np.ascontiguousarray(glob.views[c][vsel]) for c in ("x", "y", "z", "yaw")]
        Kv_glob = glob.views["x"].shape[0]
    vparams = R.make_params(mode=R.MODE_CULLED if args.mode == "culled" else R.MODE_DENSE,
                            flags=R.SCORE_FULL_GAIN | R.SCORE_NO_COLLISION)
    cam = R.make_camera(wl.camera)
    params = R.make_params(mode=R.MODE_CULLED if args.mode == "culled" else R.MODE_DENSE,
                           info_stride=args.stride)
    to_dev = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    dmap = [to_dev(a) for a in (wl.means, wl.quats, wl.scales, wl.opacity, wl.info_w, wl.flags)]
    dtraj = [to_dev(a) for a in (wl.x, wl.y, wl.z, wl.yaw)]
    pin = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hmap = [pin(a) for a in (wl.means, wl.quats, wl.scales, wl.opacity, wl.info_w, wl.flags)]
    htraj = [pin(a) for a in (wl.x, wl.y, wl.z, wl.yaw)]
    dviews = [to_dev(a) for a in views] if views is not None else None
    hviews = [pin(a) for a in views] if views is not None else None
    h2d_bytes = sum(a.numel() * a.element_size() for a in hmap + htraj + (hviews or []) if a is not None)
    Kv = views[0].shape[0] if views is not None else 0
    vouts = tuple(torch.empty(Kv, dtype=dt, device=dev) for dt in (torch.int32, torch.uint8, torch.float64,
                                                                    torch.float64)) if Kv else None
    outs = (torch.empty(K, dtype=torch.int32, device=dev), torch.empty(K, dtype=torch.uint8, device=dev),
            torch.empty(K, dtype=torch.float64, device=dev), torch.empty(K, dtype=torch.float64, device=dev))
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def global_best(score, idx):
        # one NCCL all_gather of (score, global index) per step (paper_2409_18122_b200/dist.py)
        return D.global_best(score, idx, rank, world, device=cdev)

    map_opts = None
    if args.cells:
        hy, hx, hz = (float(v) for v in args.cells.split(","))
        map_opts = (hy, hz, 0.0, hx)
    z_centre = None
    if args.z_centre == "camera":   # the planner's camera height: its waypoints share it (ground robot)
        z_centre = float(np.median(wl.z))
    elif args.z_centre != "none":
        z_centre = float(args.z_centre)
    if z_centre is not None:
        map_opts = (map_opts or (0.0, 0.0, 0.0, 0.0)) + (z_centre,)

    aux = torch.cuda.Stream(device=dev)
    vstream = torch.cuda.Stream(device=dev)

    prof_state = {"on": False}

    def step(host: bool):
        if host:
            # the map's arrays are copied first (pinned host -> device on this stream); the waypoint upload
            # (rtg_traj_upload from the pinned host arrays, on a second stream) waits only for those copies,
            # so it overlaps the validation, the bounds readback and the map build instead of following them
            src_map = [None if h is None else h.to(dev, non_blocking=True) for h in hmap]
            copied = torch.cuda.Event()
            copied.record(stream)
            aux.wait_event(copied)
            tr = R.Traj.upload(*htraj, device=local_dev, stream=aux)
        else:
            src_map = dmap
        m = R.Map(*src_map, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g, collide_rule=wl.robot.rule,
                  device=local_dev, options=map_opts)
        if Kv:
            vstream.wait_stream(stream)   # the views need the map build only
        if host:
            stream.wait_stream(aux)
        else:
            tr = R.Traj.wrap(*dtraj, device=local_dev)   # resident waypoints: borrowed, no copy
        R.score(m, tr, cam, params, *outs)
        tv = None
        if Kv:   # the scale config's gain-only views (T = 1, no collision), scored concurrently on a
            # third stream: their one-waypoint-per-warp launch would otherwise be a serial tail.  The
            # per-phase events skip them (their phases would count the wait for free SMs).
            if prof_state["on"]:
                R.profile_enable(False)
            tv = (R.Traj.upload(*hviews, device=local_dev, stream=vstream) if host
                  else R.Traj.wrap(*dviews, device=local_dev))
            R.score(m, tv, cam, vparams, *vouts, stream=vstream)
            if prof_state["on"]:
                R.profile_enable(True)
        s, i = R.best(outs[3])
        res = global_best(s, i)
        if Kv:   # best view by xi
            if prof_state["on"]:
                R.profile_enable(False)
            vs, vi = R.best(vouts[3], stream=vstream)
            if prof_state["on"]:
                R.profile_enable(True)
            res = res + global_best(vs, vi)
            stream.wait_stream(vstream)
            tv.close()
        m.close()
        if host:
            aux.wait_stream(stream)   # the waypoints are released on their upload stream
        tr.close()
        return res

    def timed(host: bool, steps: int, warmup: int, profile: bool = False):
        for _ in range(warmup):
            step(host)
        torch.cuda.synchronize()
        if profile:                      # per-phase CUDA events over the timed steps only
            R.profile_read(reset=True)
            R.profile_enable(True)
            prof_state["on"] = True
        total_ms = 0.0
        per_step = []
        res = None
        for _ in range(steps):
            flush.fill_(1.0)                     # L2 flush between timed steps (not timed)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            res = step(host)
            b.record(stream)
            torch.cuda.synchronize()
            total_ms += a.elapsed_time(b)
            per_step.append(a.elapsed_time(b))
        if profile:
            R.profile_enable(False)
            prof_state["on"] = False
        t = torch.tensor([total_ms] + per_step, dtype=torch.float64, device=cdev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)   # total and every step: max over ranks
        v = t.cpu().tolist()
        dist_ms["median"] = statistics.median(v[1:])
        dist_ms["p90"] = sorted(v[1:])[min(len(v) - 2, int(math.ceil(0.9 * (len(v) - 1))) - 1)]
        return v[0] / steps, res

    dist_ms = {}

    # ---- device-resident timing (value), with clocks and per-phase events
    with ClockSampler(local_dev) as clocks:
        ms, res = timed(False, args.steps, args.warmup, profile=True)
    step_stats = {"median": dist_ms["median"], "p90": dist_ms["p90"]}
    prof = R.profile_read(reset=True)
    nprof = args.steps
    launches_per_step = prof["launches"] / args.steps
    clock = clocks.summary()
    pairs = float(K_glob) * T * N + float(Kv_glob) * N
    value = pairs / (ms / 1000.0)

    # ---- e2e through the same public API from pinned host memory
    e2e = None
    if not args.no_e2e:
        ms_e2e, res_e2e = timed(True, args.steps, 1)
        assert res_e2e == res, (res_e2e, res)
        e2e = {"value": pairs / (ms_e2e / 1000.0), "unit": UNIT, "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": int(h2d_bytes), "d2h_bytes_per_step": 16 + 68}

    # ---- CUDA graphs: the scoring part of the cycle (rtg_score + rtg_best_async on a built
    # map) eager vs one graph replay (R.ScoreGraph), and -- without views -- the whole cycle on a layout
    # map (rtg_map_rebuild needs no host synchronisation, so R.CycleGraph captures rebuild + score + best)
    graph = None
    if args.mode == "culled" and not args.no_graph:
        m = R.Map(*dmap, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g, collide_rule=wl.robot.rule,
                  device=local_dev, options=map_opts)
        tr = R.Traj.wrap(*dtraj, device=local_dev)
        g = R.ScoreGraph(m, tr, cam, params)
        bo = torch.empty(2, dtype=torch.float64, device=dev)

        def eager():
            R.score(m, tr, cam, params, *outs)
            R.best_async(outs[3], bo)

        def t_of(fn):
            for _ in range(args.warmup):
                fn()
            vals = []
            for _ in range(args.steps):
                flush.fill_(1.0)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                torch.cuda.synchronize()
                vals.append(a.elapsed_time(b))
            return statistics.median(vals)

        ms_eager, ms_graph = t_of(eager), t_of(g.replay)
        assert R.read_best(bo) == R.read_best(g.best)
        graph = {"scope": "rtg_score + rtg_best_async on a built map (the cycle minus the map build)",
                 "eager_ms_median": ms_eager, "graph_ms_median": ms_graph}
        del g
        m.close()
    if graph is not None:
        # the whole cycle on a layout map (grids from the workload's extents, rebuilt without a host
        # synchronisation): eager, and captured with the score and the argmax into one graph (the scale
        # config's views on a second stream forked after the rebuild: concurrent branches of the graph)
        gbox, cbox, rb_b, rho_b = layout_bounds(wl)
        lm = R.LayoutMap(N, gbox, cbox, rb_b, rho_b, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g,
                         collide_rule=wl.robot.rule, device=local_dev, options=map_opts)
        tvw = R.Traj.wrap(*dviews, device=local_dev) if Kv else None
        vbo = torch.empty(2, dtype=torch.float64, device=dev) if Kv else None

        def eager_cycle():
            lm.rebuild(*dmap)
            if Kv:
                vstream.wait_stream(stream)
                R.score(lm, tvw, cam, vparams, *vouts, stream=vstream)
                R.best_async(vouts[3], vbo, stream=vstream)
            R.score(lm, tr, cam, params, *outs)
            R.best_async(outs[3], bo)
            if Kv:
                stream.wait_stream(vstream)

        cg = R.CycleGraph(lm, dmap, tr, cam, params, views=tvw, vparams=vparams)
        ms_ce, ms_cg = t_of(eager_cycle), t_of(cg.replay)
        lm.check()
        assert R.read_best(bo) == R.read_best(cg.best)
        if Kv:
            assert R.read_best(vbo) == R.read_best(cg.vbest)
        if world == 1:
            assert R.read_best(cg.best) == (res[0], res[1])
            if Kv:
                assert R.read_best(cg.vbest) == (res[2], res[3])
        graph["cycle"] = {"scope": "layout-map rebuild + rtg_score + rtg_best_async" + (" (+ the views on a forked "
                                   "stream)" if Kv else "") + ": the whole planning cycle "
                                   "without a host synchronisation (rtg_map_create_layout, grids from the "
                                   "workload's extents)",
                          "eager_ms_median": ms_ce, "graph_ms_median": ms_cg,
                          "standard_cycle_ms_median": step_stats["median"]}
        del cg
        if tvw is not None:
            tvw.close()
        lm.close()
    if graph is not None:
        tr.close()

    # ---- roofline of the dominant phase
    phase_ms = {k: v / nprof for k, v in prof["ms"].items()}
    dom = max(("collision", "visibility_gain", "map_build"), key=lambda k: phase_ms[k])
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    feasible = outs[1].cpu().numpy().astype(bool)
    work = None
    if args.mode == "culled":
        m = R.Map(*dmap, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g, collide_rule=wl.robot.rule,
                  device=local_dev, options=map_opts)
        work = work_sample(R, m, wl, cam, params, feasible)
        m.close()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(f"{args.config}/{args.mode}/stride{args.stride}")
    roof = roofline(dom, phase_ms[dom], wl, int(feasible.sum()), args.stride, args.mode, clock,
                    hbm_peak, work, traffic)
    executed_rate = None
    if work is not None:
        n_info = int(feasible.sum()) * (T // args.stride)
        executed = n_info * work["tested"] + float(K) * T * work["col_tested"]
        executed_rate = executed * world / (ms / 1000.0)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:   # contract: rank 0 at N = 1 only
        cores = oracle_threads()
        # ~20 s of oracle work: ~2.1e7 pair-tests/s per core measured (r1), whole multiples of the cores
        n_traj = int(20.0 * 2.1e7 * cores / (float(T) * max(N, 1)))
        n_traj = max(1, min(K, max(cores, n_traj // cores * cores)))
        v, dt, nt = oracle_sample(wl, n_traj)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{nt} random trajectories x T={T} x N={N} of this workload ({dt:.1f} s)"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "ms_per_step_median": step_stats["median"],
                "ms_per_step_p90": step_stats["p90"], "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": "outdoor (BASELINE.json configs[3])" if args.config == "outdoor" else args.config,
                           "N": N, "K": K_glob, "K_per_gpu": K, "views": Kv_glob, "T": T, "mode": args.mode,
                           "info_stride": args.stride,
                           "gain_z_centre": z_centre,
                           "parallelism": f"traj-shard x{world}, map replicated",
                           "l2": "flushed (512 MiB write) between timed steps",
                           **({"views_stream": "views scored concurrently on a second stream; phase_ms covers "
                                               "the trajectories' calls only"} if Kv_glob else {})},
                "best": {"score": res[0], "index": res[1]},
                **({"best_view": {"score": res[2], "index": res[3]}} if len(res) > 2 else {}),
                "phase_ms": {k: round(v, 4) for k, v in phase_ms.items()},
                "gpu_launches": int(round(launches_per_step)),
                # SURVEY §8(d) metric 2, "executed": pairs actually tested one by one (visibility tests
                # of the info waypoints + collision candidates), from the debug counters of a sample
                **({"executed_pair_tests_per_s": executed_rate} if executed_rate is not None else {}),
                "clocks": clock, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                **({"cuda_graph": graph} if graph is not None else {})}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def layout_bounds(wl, margin=0.05):
    """A layout for rtg_map_create_layout from the workload's extents (what a robot knows of its map):
    boxes around the gain-eligible and collidable means, bounds on the largest collision semi-axis
    a = lambda_g s + r_robot and its anisotropy, with margins."""
    import numpy as np
    f = wl.flags if wl.flags is not None else np.zeros(wl.N, np.uint8)
    gain, col = (f & 2) == 0, (f & 1) == 0
    m = wl.means.astype(np.float64)

    def box(sel):
        if not sel.any():
            return [0.0] * 3, [1.0] * 3
        return (m[:, sel].min(1) - margin).tolist(), (m[:, sel].max(1) + margin).tolist()

    a = wl.robot.lambda_g * wl.scales[:, col].astype(np.float64) + wl.robot.r_robot
    rb = float(a.max()) * 1.01 + 1e-3 if col.any() else 1.0
    rho = float((a.max(0) / a.min(0)).max()) * 1.01 if col.any() else 1.0
    return box(gain), box(col), rb, rho


# Algorithmic work per unit, SURVEY §8(d) (SURVEY.md:709, [A5]): ~10 lane-instructions per individually
# tested Gaussian, ~25 per grid cell classified (here: per (row, z-cell) unit and per footprint row, each
# a cell-interval classification); dense gain-only path ~15 FP32 instructions per pair (SURVEY §8(d)
# "Dense fused kernel": "~15 in the gain-only phase").  DESIGN.md "Roofline accounting".
I_TEST = 10.0
I_UNIT = 25.0
I_ROW = 25.0
I_DENSE_PAIR = 15.0
I_SPHERE = 8.0    # collision sphere reject per candidate pair (3 FADD, 3 FMA, compare, branch)
KERNEL = {("visibility_gain", "culled"): "k_gain_culled", ("collision", "culled"): "k_col_culled",
          ("visibility_gain", "dense"): "k_gain_dense", ("collision", "dense"): "k_col_dense",
          ("map_build", "culled"): "k_scatter_col", ("map_build", "dense"): "k_scatter_col"}


def work_sample(R, m, wl, cam, params, feasible, n=96):
    """Per-waypoint work units of the culled kernels, measured with rtg_score_debug on a sample of
    feasible trajectories (untimed)."""
    import numpy as np
    f = np.nonzero(feasible)[0]
    if len(f) == 0:
        return None
    idx = f[np.linspace(0, len(f) - 1, min(n, len(f))).astype(int)]
    tr = R.traj_from_workload(wl, x=wl.x[idx], y=wl.y[idx], z=wl.z[idx], yaw=wl.yaw[idx])
    p = R.make_params(mode=params.mode, info_stride=1, flags=R.SCORE_FULL_GAIN)
    d = R.score_debug(m, tr, cam, p)
    tr.close()
    nwp = len(idx) * wl.T
    return {k: v / nwp for k, v in d["stats"].items()}


# Algorithmic L2 -> SM bytes of the culled gain kernel per info waypoint:
# a 16-byte record per individually tested Gaussian, the 16-byte z-fastest table entries the (row, z-cell)
# units need (the run ends: 2 per unit, up to 2 more where the inside x-run differs from them), the copy-A
# column starts (4 bytes, 2 or 4 per footprint row) and z-occupancy blocks (8 bytes) of the rows -- all
# three counted in the kernel by rtg_score_debug -- and the waypoint's pose (16 B) and FP64 yaw sine and
# cosine (16 B).  Older stats without the table counters: 2 entries per unit + 2 per aggregated unit,
# 16 bytes per row.
B_REC, B_TAB, B_ROW, B_WP = 16.0, 16.0, 16.0, 32.0


def l2_roofline(n_info, work, ms, k_ncu):
    """Second roof of the culled gain kernel: its records and tables are L2-resident (ncu: DRAM bytes are
    < 0.1 % of the L2 reads), so the memory roof is the L2 -> SM read bandwidth, measured on B200 by
    tools/l2_peak.cu (profiles/r2j_l2_peak.json): sequential 16-byte loads through L2 (the hardware roof)
    and the kernel's own access pattern (runs of 8 consecutive 16-byte records at random offsets)."""
    if "unit_table_entries" in work:   # counted in the kernel (rtg_score_debug)
        bytes_wp = (B_REC * work["tested"] + B_TAB * work["unit_table_entries"] + work["row_table_bytes"] + B_WP)
    else:
        bytes_wp = (B_REC * work["tested"] + B_TAB * 2.0 * (work["units"] + work["cells_aggregated"])
                    + B_ROW * work.get("rows", 0.0) + B_WP)
    ach = n_info * bytes_wp / (ms / 1e3) / 1e9
    mean_run = (work["tested"] / work["runs"]) if work.get("runs") else None
    peak = pattern = pattern_run = None
    try:
        res = json.load(open(os.path.join(ROOT, "profiles", "r2j_l2_peak.json")))["results"]
        peak = max(r["GBps"] for r in res if r["pattern"] == "seq_cg")
        # the runs pattern at the longest measured run length not above the kernel's mean run length
        runs = sorted((r["run_records"], r["GBps"]) for r in res
                      if r["pattern"] == "runs" and r.get("warps_per_sm", 64) == 64)
        pattern_run, pattern = ([x for x in runs if mean_run is None or x[0] <= mean_run] or runs[:1])[-1]
    except Exception:
        pass
    out = {"bound": "l2", "achieved": ach, "peak": peak, "unit": "GB/s",
           "frac": ach / peak if peak else None,
           "peak_basis": "measured L2->SM read bandwidth, sequential ld.global.cg 16-byte loads over a 64 MB "
                         "L2-resident buffer (tools/l2_peak.cu, profiles/r2j_l2_peak.json)",
           "pattern_peak": pattern, "frac_of_pattern_peak": ach / pattern if pattern else None,
           "pattern_basis": f"the same tool: 16-byte records in runs of {pattern_run} consecutive records at random "
                            "offsets, 32 lanes on 32 consecutive items of the flattened runs (the test passes' "
                            "access pattern; the longest measured run length not above mean_run_records)",
           "mean_run_records": mean_run,
           "bytes_per_wp": bytes_wp, "per_unit_bytes": {"record": B_REC, "table_entry": B_TAB, "row": B_ROW,
                                                      "waypoint": B_WP},
           "bytes_basis": "16 B per tested record + 16 B per unit table entry + row table bytes (kernel counters) "
                          "+ 32 B pose and yaw trig per waypoint"}
    if k_ncu and k_ncu.get("l2_read_bytes"):
        out["ncu_l2_read_bytes"] = k_ncu["l2_read_bytes"]
        out["algorithmic_share_of_l2_reads"] = n_info * bytes_wp / k_ncu["l2_read_bytes"]
    return out


def roofline(phase, ms, wl, n_feasible, stride, mode, clock, hbm_peak, work, ncu):
    """Roofline object of the dominant phase (achieved = algorithmic work per launch / launch time).
    `ncu` holds the committed ncu --set full figures of the same kernel (profiles/traffic.json)."""
    sm_mhz = (clock.get("sm_mhz") or 1965.0)
    peak_ti = 148 * 128 * sm_mhz * 1e6 / 1e12          # lane-instruction issue peak, T/s (guide unit counts)
    kname = KERNEL.get((phase, mode), "")
    k_ncu = ncu.get(kname) if ncu else None
    if isinstance(k_ncu, (int, float)):                # older records: DRAM bytes only
        k_ncu = {"dram_bytes": k_ncu}
    tr = k_ncu.get("dram_bytes") if k_ncu else None
    if phase == "map_build":
        n = wl.N
        alg_bytes = n * 49 + n * (16 + 8 + 4) * 2 + (n // 2) * (16 + 48 + 72)
        gbs = alg_bytes / (ms / 1e3) / 1e9
        return {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                "traffic": tr, "phase": phase, "kernel_ms": ms}
    n_info = n_feasible * (wl.T // stride)
    units = None
    if phase == "visibility_gain":
        if mode == "dense":
            units = {"pairs_per_info_waypoint": float(wl.N), "I_pair": I_DENSE_PAIR}
            lane_instr = n_info * float(wl.N) * I_DENSE_PAIR
        elif work is None:     # nothing feasible (tiny): no info waypoint was scored
            units, lane_instr = {"info_waypoints": 0}, 0.0
        else:
            rows = work.get("rows", 0.0)
            units = {"info_waypoints": n_info, "tested_per_wp": work["tested"], "units_per_wp": work["units"],
                     "rows_per_wp": rows, "I_test": I_TEST, "I_unit": I_UNIT, "I_row": I_ROW}
            lane_instr = n_info * (I_TEST * work["tested"] + I_UNIT * work["units"] + I_ROW * rows)
    else:
        lane_instr = wl.K * wl.T * (work["col_tested"] if work else 0.0) * I_SPHERE
    ach = lane_instr / (ms / 1e3) / 1e12
    out = {"bound": "alu", "achieved": ach, "peak": peak_ti, "unit": "T lane-instr/s", "frac": ach / peak_ti,
           "traffic": tr, "phase": phase, "kernel": kname, "kernel_ms": ms,
           "peak_basis": "148 SMs x 128 FP32 lanes x measured SM clock (B200_PROFILING.md unit counts)",
           "work_units": units, "work_per_waypoint": work}
    l2 = None
    if phase == "visibility_gain" and mode == "culled" and work is not None:
        l2 = out["l2"] = l2_roofline(n_info, work, ms, k_ncu)
    if k_ncu:
        out["ncu"] = {k: v for k, v in k_ncu.items() if k != "dram_bytes"}
        wi = k_ncu.get("warp_inst")
        if wi:   # executed lane slots per launch vs the algorithmic lane instructions above
            out["ncu"]["algorithmic_share_of_executed"] = lane_instr / (32.0 * wi)
    if l2 is not None and l2.get("peak") and n_info > 0:
        # "the roofline fraction is the achieved rate over min(FP32 peak, arithmetic intensity x
        # bandwidth)"; the culled traversal's records and tables are L2-resident, so the bandwidth is the
        # measured L2 -> SM roof.  When that product is the smaller roof the line reports it as the primary
        # (frac = achieved bytes / L2 peak = achieved lane-instr / (AI x L2 peak)); the FP32 one stays under "alu"
        ai = lane_instr / (n_info * l2["bytes_per_wp"])            # lane instructions per algorithmic byte
        roof_l2 = ai * l2["peak"] * 1e9 / 1e12                     # T lane-instr/s
        rule = {"definition": "SURVEY 8(d): frac = achieved / min(FP32 peak, arithmetic intensity x bandwidth)",
                "ai_lane_instr_per_byte": ai, "fp32_roof": peak_ti, "l2_roof": roof_l2, "unit": "T lane-instr/s",
                "binding": "l2" if roof_l2 < peak_ti else "alu"}
        if roof_l2 < peak_ti:
            alu = {k: out.pop(k) for k in ("bound", "achieved", "peak", "unit", "frac", "peak_basis")}
            prim = {k: l2[k] for k in ("bound", "achieved", "peak", "unit", "frac", "peak_basis")}
            rest = {k: v for k, v in out.items() if k != "l2"}
            out = dict(prim, traffic=tr, roof_rule=rule, alu=alu, l2=l2, **{k: v for k, v in rest.items()
                                                                            if k != "traffic"})
        else:
            out["roof_rule"] = rule
    return out


if __name__ == "__main__":
    sys.exit(main())

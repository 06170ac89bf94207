"""Thin Python binding of librtg (include/rtg.h) -- argument marshalling only.

Every step of the scoring path runs in the library's CUDA kernels; this module only
turns torch tensors / numpy arrays into pointers, sizes and streams and raises on a
non-OK status.  There is no CPU fallback: importing this module fails loudly when
librtg.so is missing, and every call that needs a GPU fails loudly without one.

Names follow the C ABI: ``map_create`` -> rtg_map_create, ``traj_upload`` ->
rtg_traj_upload, ``traj_sample_unicycle``, ``score`` -> rtg_score, ``best`` -> rtg_best,
``score_debug`` -> rtg_score_debug.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librtg.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"librtg.so not found at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(nvcc, sm_100a). There is no CPU fallback.")
_lib = ctypes.CDLL(LIB_PATH)

# ------------------------------------------------------------------ ABI mirror
OK, ERR_INVALID_ARGUMENT, ERR_CUDA, ERR_OUT_OF_MEMORY, ERR_NO_FEASIBLE, ERR_BAD_HANDLE = range(6)
MEM_HOST, MEM_DEVICE = 0, 1
G_NO_COLLIDE, G_NO_GAIN = 1, 2
COLLIDE_ELLIPSOID, COLLIDE_PRINCIPAL_AXIS = 0, 1
VARIANT_XI, VARIANT_SUM, VARIANT_SQ = 0, 1, 2
MODE_DENSE, MODE_CULLED = 0, 1
SCORE_FULL_GAIN, SCORE_NO_COLLISION, SCORE_INCLUDE_START = 1, 2, 4
DEBUG_STATS = 12


class Robot(ctypes.Structure):
    _fields_ = [("r_robot", ctypes.c_float), ("lambda_g", ctypes.c_float), ("collide_rule", ctypes.c_int)]


class Camera(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int), ("height", ctypes.c_int), ("fx", ctypes.c_float), ("fy", ctypes.c_float),
                ("cx", ctypes.c_float), ("cy", ctypes.c_float), ("z_near", ctypes.c_float), ("z_far", ctypes.c_float)]


class ScoreParams(ctypes.Structure):
    _fields_ = [("lambda_xi", ctypes.c_float), ("k_sigma", ctypes.c_float), ("variant", ctypes.c_int),
                ("info_stride", ctypes.c_int), ("mode", ctypes.c_int), ("flags", ctypes.c_uint),
                ("tau_hi", ctypes.c_double), ("tau_lo", ctypes.c_double)]


class BestResult(ctypes.Structure):
    _fields_ = [("score", ctypes.c_double), ("index", ctypes.c_longlong)]


class MapOptions(ctypes.Structure):
    _fields_ = [("gain_cell_xy", ctypes.c_float), ("gain_cell_z", ctypes.c_float), ("col_cell", ctypes.c_float),
                ("gain_cell_x", ctypes.c_float), ("gain_z_centred", ctypes.c_int), ("gain_z_centre", ctypes.c_float)]


def make_map_options(options) -> "MapOptions":
    """rtg_map_options from (gain_cell_xy, gain_cell_z, col_cell, gain_cell_x[, gain_z_centre]); sizes <= 0 take
    the defaults, a gain_z_centre of None leaves the z-cells at the lowest mean."""
    v = list(options)
    zc = v[4] if len(v) > 4 else None
    return MapOptions(*[float(x) for x in v[:4]], int(zc is not None), float(zc) if zc is not None else 0.0)


class MapLayout(ctypes.Structure):
    _fields_ = [("capacity", ctypes.c_longlong), ("gain_lo", ctypes.c_float * 3), ("gain_hi", ctypes.c_float * 3),
                ("col_lo", ctypes.c_float * 3), ("col_hi", ctypes.c_float * 3), ("rb_max", ctypes.c_float),
                ("rho_max", ctypes.c_float)]


class MapInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_longlong), ("n_collide", ctypes.c_longlong), ("n_gain", ctypes.c_longlong),
                ("tau_hi", ctypes.c_double), ("tau_lo", ctypes.c_double), ("u_mean", ctypes.c_double),
                ("u_std", ctypes.c_double), ("fixed_point_shift", ctypes.c_int),
                ("gain_dims", ctypes.c_int * 3), ("col_dims", ctypes.c_int * 3), ("rb_max", ctypes.c_float),
                ("device_bytes", ctypes.c_longlong)]


class TreeParams(ctypes.Structure):
    _fields_ = [("n_v", ctypes.c_int), ("n_omega", ctypes.c_int), ("v_max", ctypes.c_float),
                ("omega_max", ctypes.c_float), ("dt", ctypes.c_float), ("lambda_t", ctypes.c_float),
                ("samples", ctypes.c_int), ("max_depth", ctypes.c_int), ("goal_radius", ctypes.c_float),
                ("lattice_xy", ctypes.c_float), ("lattice_deg", ctypes.c_float), ("beam", ctypes.c_int),
                ("n_traj", ctypes.c_int), ("z", ctypes.c_float)]


def make_tree_params(n_v=3, n_omega=5, v_max=0.6, omega_max=0.9, dt=1.0, lambda_t=1.0, samples=5, max_depth=8,
                     goal_radius=0.5, lattice_xy=0.1, lattice_deg=10.0, beam=4096, n_traj=10, z=0.5) -> "TreeParams":
    """Defaults: PAPER.md:330 (N_v = 3, v_max = 0.6, N_w = 5, w_max = 0.9, 1 s) and SPEC S:384."""
    return TreeParams(n_v, n_omega, v_max, omega_max, dt, lambda_t, samples, max_depth, goal_radius, lattice_xy,
                      lattice_deg, beam, n_traj, z)


class Profile(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 8), ("calls", ctypes.c_longlong * 8), ("launches", ctypes.c_longlong)]


PHASES = ("map_build", "classify", "collision", "info_list", "visibility_gain", "reduce", "argmax", "other")

_P = ctypes.c_void_p
_I = ctypes.c_int
_LL = ctypes.c_longlong
_S = ctypes.c_int  # rtg_status

_SIGS = {
    "rtg_map_create": (_S, [_I, _LL, _I, _P, _P, _P, _P, _P, _P, ctypes.POINTER(Robot), _P, ctypes.POINTER(_P)]),
    "rtg_map_create_ex": (_S, [_I, _LL, _I, _P, _P, _P, _P, _P, _P, ctypes.POINTER(Robot),
                               ctypes.POINTER(MapOptions), _P, ctypes.POINTER(_P)]),
    "rtg_map_destroy": (_S, [_P]),
    "rtg_map_create_layout": (_S, [_I, ctypes.POINTER(MapLayout), ctypes.POINTER(Robot), ctypes.POINTER(MapOptions),
                                   _P, ctypes.POINTER(_P)]),
    "rtg_map_rebuild": (_S, [_P, _LL, _P, _P, _P, _P, _P, _P, _P]),
    "rtg_map_check": (_S, [_P, _P]),
    "rtg_map_info": (_S, [_P, ctypes.POINTER(MapInfo)]),
    "rtg_traj_upload": (_S, [_I, _I, _I, _I, _P, _P, _P, _P, _P, ctypes.POINTER(_P)]),
    "rtg_traj_wrap": (_S, [_I, _I, _I, _P, _P, _P, _P, ctypes.POINTER(_P)]),
    "rtg_traj_sample_double_integrator": (_S, [_I, _I, _I, ctypes.c_float, _P, _P, _P, _P, _I, _P,
                                               ctypes.POINTER(_P)]),
    "rtg_traj_sample_unicycle": (_S, [_I, _I, _I, ctypes.c_float, ctypes.POINTER(ctypes.c_float), _P, _P, _I, _P,
                                      ctypes.POINTER(_P)]),
    "rtg_traj_read": (_S, [_P, _P, _P, _P, _P, _P]),
    "rtg_traj_set_start": (_S, [_P, ctypes.POINTER(ctypes.c_float)]),
    "rtg_traj_destroy": (_S, [_P]),
    "rtg_score": (_S, [_P, _P, ctypes.POINTER(Camera), ctypes.POINTER(ScoreParams), _P, _P, _P, _P, _P]),
    "rtg_best": (_S, [_P, _I, _LL, _P, ctypes.POINTER(BestResult)]),
    "rtg_best_async": (_S, [_P, _I, _LL, _P, _P]),
    "rtg_score_debug": (_S, [_P, _P, ctypes.POINTER(Camera), ctypes.POINTER(ScoreParams), _P, _P, _P, _P, _P,
                             _P, _P]),
    "rtg_ledger_update": (_S, [_I, _LL, _I, _P, _P, _P, _P, _P]),
    "rtg_map_update_weights": (_S, [_P, _I, _P, _P]),
    "rtg_region_utility": (_S, [_P, ctypes.POINTER(ctypes.c_double), ctypes.c_double, ctypes.POINTER(_I), _P, _P, _P]),
    "rtg_traj_view_ring": (_S, [_I, _I, _I, _P, ctypes.c_double, ctypes.POINTER(Camera), _I, ctypes.c_float, _P,
                                ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_double)]),
    "rtg_cost_benefit": (_S, [_P, _P, _I, _P, ctypes.POINTER(BestResult)]),
    "rtg_plan_tree": (_S, [_P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float),
                           ctypes.POINTER(TreeParams), _P, ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_double),
                           ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_LL)]),
    "rtg_profile_enable": (_S, [_I]),
    "rtg_profile_read": (_S, [ctypes.POINTER(Profile), _I]),
    "rtg_status_string": (ctypes.c_char_p, [_I]),
    "rtg_last_error": (ctypes.c_char_p, []),
    "rtg_version": (ctypes.c_char_p, []),
}
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIGS)


class RTGError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.rtg_last_error().decode()
        super().__init__(f"{where}: {_lib.rtg_status_string(status).decode()}: {msg}")


def _check(status: int, where: str, allow=()):
    if status != OK and status not in allow:
        raise RTGError(status, where)
    return status


def version() -> str:
    return _lib.rtg_version().decode()


def profile_enable(on: bool = True) -> None:
    _check(_lib.rtg_profile_enable(1 if on else 0), "rtg_profile_enable")


def profile_read(reset: bool = True) -> dict:
    """Accumulated device ms / calls per phase (CUDA events on the launch streams) + kernel launches."""
    p = Profile()
    _check(_lib.rtg_profile_read(ctypes.byref(p), 1 if reset else 0), "rtg_profile_read")
    return dict(ms={n: p.ms[i] for i, n in enumerate(PHASES)}, calls={n: p.calls[i] for i, n in enumerate(PHASES)},
                launches=p.launches)


# ------------------------------------------------------------------ helpers
def _torch():
    import torch
    return torch


def _ptr(a) -> Optional[int]:
    """Pointer of a contiguous torch tensor or numpy array (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("numpy array must be C-contiguous")
        return a.ctypes.data
    if not a.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return a.data_ptr()


_DT = {"float32": "float32", "torch.float32": "float32", "float64": "float64", "torch.float64": "float64",
       "int32": "int32", "torch.int32": "int32", "uint8": "uint8", "torch.uint8": "uint8"}


def _arg(name: str, a, dtype: str, shape=None, device: Optional[int] = None, cuda: bool = False, optional=False):
    """Validate one array argument against the C ABI before its pointer crosses it: dtype (the ABI
    reads raw memory, so a float64 numpy map would be read as float32 garbage), shape (a short
    output buffer would be written past its end), contiguity and, for device memory, that the
    tensor lives on the handle's device.  Returns the pointer (None for an optional NULL)."""
    if a is None:
        if optional:
            return None
        raise ValueError(f"{name}: required")
    dt = _DT.get(str(a.dtype))
    if dt != dtype:
        raise TypeError(f"{name}: dtype {a.dtype}, the C ABI expects {dtype}")
    if shape is not None and tuple(int(s) for s in a.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(a.shape)}, expected {tuple(shape)}")
    is_cuda = (not isinstance(a, np.ndarray)) and a.is_cuda
    if cuda and not is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor")
    if is_cuda and device is not None and a.device.index != device:
        raise ValueError(f"{name}: on cuda:{a.device.index}, the handle is on cuda:{device}")
    return _ptr(a)


def _kind(a) -> int:
    if isinstance(a, np.ndarray):
        return MEM_HOST
    return MEM_DEVICE if a.is_cuda else MEM_HOST


def _stream(stream) -> Optional[int]:
    if stream is None:
        torch = _torch()
        return torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else None
    return stream if isinstance(stream, int) else stream.cuda_stream


def make_camera(cam) -> Camera:
    return Camera(int(cam.width), int(cam.height), float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy),
                  float(cam.z_near), float(cam.z_far))


def make_params(lambda_xi=1.0, k_sigma=0.5, variant=VARIANT_XI, info_stride=1, mode=MODE_CULLED, flags=0,
                tau_hi=float("nan"), tau_lo=float("nan")) -> ScoreParams:
    return ScoreParams(lambda_xi, k_sigma, variant, info_stride, mode, flags, tau_hi, tau_lo)


# ------------------------------------------------------------------ handles
class Map:
    """rtg_map handle; arrays are planar SoA (means [3,N], quats [4,N], scales [3,N], ...).
    Host (numpy / CPU tensor) inputs are copied to the device inside the call; CUDA tensors are
    read in place."""

    def __init__(self, means, quats, scales, opacity, info_w, flags=None, r_robot=0.3, lambda_g=3.0,
                 collide_rule=COLLIDE_ELLIPSOID, device=0, stream=None, options=None):
        n = int(means.shape[-1])
        kind = _kind(means)
        for a in (quats, scales, opacity, info_w, flags):
            if a is not None and _kind(a) != kind:
                raise ValueError("all map arrays must live in the same memory (host or device)")
        ptrs = (_arg("means", means, "float32", (3, n), device), _arg("quats", quats, "float32", (4, n), device),
                _arg("scales", scales, "float32", (3, n), device), _arg("opacity", opacity, "float32", (n,), device),
                _arg("info_w", info_w, "float32", (n,), device),
                _arg("flags", flags, "uint8", (n,), device, optional=True))
        self._robot = Robot(float(r_robot), float(lambda_g), int(collide_rule))
        self.handle = _P()
        self.n = n
        self.device = device
        self._keep = (means, quats, scales, opacity, info_w, flags)
        st = _stream(stream)
        if options is not None:
            opt = make_map_options(options)
            s = _lib.rtg_map_create_ex(device, n, kind, *ptrs, ctypes.byref(self._robot), ctypes.byref(opt), st,
                                       ctypes.byref(self.handle))
        else:
            s = _lib.rtg_map_create(device, n, kind, *ptrs, ctypes.byref(self._robot), st, ctypes.byref(self.handle))
        _check(s, "rtg_map_create")

    def update_weights(self, info_w, stream=None) -> None:
        """rtg_map_update_weights: replace the ledger (input order) and reclassify (N4)."""
        p = _arg("info_w", info_w, "float32", (self.n,), self.device)
        _check(_lib.rtg_map_update_weights(self.handle, _kind(info_w), p, _stream(stream)),
               "rtg_map_update_weights")
        self._keep = self._keep + (info_w,)

    def info(self) -> MapInfo:
        out = MapInfo()
        _check(_lib.rtg_map_info(self.handle, ctypes.byref(out)), "rtg_map_info")
        return out

    def close(self):
        if self.handle:
            _check(_lib.rtg_map_destroy(self.handle), "rtg_map_destroy")
            self.handle = _P()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LayoutMap(Map):
    """rtg_map_create_layout handle: grids and capacity fixed from caller bounds; `rebuild` refills it
    from new CUDA arrays with device work only (capturable, e.g. by CycleGraph); `check` synchronises and
    raises RTGError if the last rebuild's data was invalid or broke the layout."""

    def __init__(self, capacity, gain_box, col_box, rb_max, rho_max, r_robot=0.3, lambda_g=3.0,
                 collide_rule=COLLIDE_ELLIPSOID, device=0, stream=None, options=None):
        lay = MapLayout()
        lay.capacity = int(capacity)
        for d in range(3):
            lay.gain_lo[d], lay.gain_hi[d] = float(gain_box[0][d]), float(gain_box[1][d])
            lay.col_lo[d], lay.col_hi[d] = float(col_box[0][d]), float(col_box[1][d])
        lay.rb_max, lay.rho_max = float(rb_max), float(rho_max)
        self._layout = lay
        self._robot = Robot(float(r_robot), float(lambda_g), int(collide_rule))
        self.handle = _P()
        self.n = 0
        self.capacity = int(capacity)
        self.device = device
        self._keep = ()
        opt = make_map_options(options) if options is not None else None
        _check(_lib.rtg_map_create_layout(device, ctypes.byref(lay), ctypes.byref(self._robot),
                                          ctypes.byref(opt) if opt is not None else None, _stream(stream),
                                          ctypes.byref(self.handle)), "rtg_map_create_layout")

    def rebuild(self, means, quats, scales, opacity, info_w, flags=None, stream=None) -> None:
        """rtg_map_rebuild from CUDA arrays (read when the stream reaches the call: keep them alive)."""
        n = int(means.shape[-1])
        for nm, a in (("means", means), ("quats", quats), ("scales", scales), ("opacity", opacity),
                      ("info_w", info_w), ("flags", flags)):
            if a is not None and (isinstance(a, np.ndarray) or not a.is_cuda):
                raise ValueError(f"{nm}: rtg_map_rebuild reads CUDA arrays")
        ptrs = (_arg("means", means, "float32", (3, n), self.device), _arg("quats", quats, "float32", (4, n), self.device),
                _arg("scales", scales, "float32", (3, n), self.device),
                _arg("opacity", opacity, "float32", (n,), self.device),
                _arg("info_w", info_w, "float32", (n,), self.device),
                _arg("flags", flags, "uint8", (n,), self.device, optional=True))
        _check(_lib.rtg_map_rebuild(self.handle, n, *ptrs, _stream(stream)), "rtg_map_rebuild")
        self.n = n
        self._keep = (means, quats, scales, opacity, info_w, flags)

    def check(self, stream=None) -> None:
        _check(_lib.rtg_map_check(self.handle, _stream(stream)), "rtg_map_check")


class CycleGraph:
    """The whole planning cycle -- rtg_map_rebuild of a LayoutMap from CUDA map arrays, rtg_score (culled) of
    a trajectory handle, rtg_best_async -- captured once into one CUDA graph and replayed.  The graph keeps
    every device pointer: a replay rebuilds from what the map arrays then hold and scores what the
    trajectory buffers then hold (refill both in place; the Gaussian count n is fixed).  One eager cycle
    precedes the capture."""

    def __init__(self, lmap: "LayoutMap", map_arrays, tr: "Traj", camera, params: ScoreParams, index_base: int = 0,
                 views: Optional["Traj"] = None, vparams: Optional[ScoreParams] = None, vindex_base: int = 0):
        torch = _torch()
        if params.mode != MODE_CULLED or (views is not None and (vparams is None or vparams.mode != MODE_CULLED)):
            raise ValueError("CycleGraph: culled mode only (dense mode reads the list length on the host)")
        dev = torch.device("cuda", lmap.device)

        def outs_for(K):
            return (torch.empty(K, dtype=torch.int32, device=dev), torch.empty(K, dtype=torch.uint8, device=dev),
                    torch.empty(K, dtype=torch.float64, device=dev), torch.empty(K, dtype=torch.float64, device=dev))

        self.outs = outs_for(tr.K)
        self.best = torch.empty(2, dtype=torch.float64, device=dev)
        # gain-only views (the scale config): scored on a second stream forked after the rebuild, joined
        # before the cycle ends -- inside the graph, the two scorings are concurrent branches
        self.vouts = outs_for(views.K) if views is not None else None
        self.vbest = torch.empty(2, dtype=torch.float64, device=dev) if views is not None else None
        vstream = torch.cuda.Stream(device=dev) if views is not None else None
        self._keep = (lmap, tuple(map_arrays), tr, views, vstream)
        cam = camera if isinstance(camera, Camera) else make_camera(camera)

        def cycle():
            lmap.rebuild(*map_arrays)
            cur = torch.cuda.current_stream(dev)
            if views is not None:
                vstream.wait_stream(cur)
                score(lmap, views, cam, vparams, *self.vouts, stream=vstream)
                best_async(self.vouts[3], self.vbest, vindex_base, stream=vstream)
            score(lmap, tr, cam, params, *self.outs)
            best_async(self.outs[3], self.best, index_base)
            if views is not None:
                cur.wait_stream(vstream)

        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            cycle()
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        lmap.check()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, capture_error_mode="thread_local"):
            cycle()

    def replay(self):
        """Enqueue one replay on the current stream; returns (first_col, feasible, gain, utility, best)
        (the views' outputs and best are in .vouts / .vbest)."""
        self.graph.replay()
        return self.outs + (self.best,)


class Traj:
    """rtg_traj handle: x, y, z, yaw each [K, T] (trajectory-major)."""

    def __init__(self, handle: _P, K: int, T: int, device: int = 0):
        self.handle = handle
        self.K = K
        self.T = T
        self.device = device

    @staticmethod
    def _xyzyaw(x, y, z, yaw, device, cuda=False):
        if len(x.shape) != 2:
            raise ValueError("x: expected [K, T]")
        K, T = (int(s) for s in x.shape)
        kind = _kind(x)
        for a in (y, z, yaw):
            if _kind(a) != kind:
                raise ValueError("x, y, z, yaw must live in the same memory (host or device)")
        return K, T, kind, [_arg(nm, a, "float32", (K, T), device, cuda=cuda)
                            for nm, a in (("x", x), ("y", y), ("z", z), ("yaw", yaw))]

    @classmethod
    def upload(cls, x, y, z, yaw, device=0, stream=None) -> "Traj":
        K, T, kind, ptrs = cls._xyzyaw(x, y, z, yaw, device)
        h = _P()
        _check(_lib.rtg_traj_upload(device, K, T, kind, *ptrs, _stream(stream), ctypes.byref(h)), "rtg_traj_upload")
        return cls(h, K, T, device)

    @classmethod
    def wrap(cls, x, y, z, yaw, device=0) -> "Traj":
        """rtg_traj_wrap: borrow device tensors [K, T] without copying (kept referenced here)."""
        K, T, _, ptrs = cls._xyzyaw(x, y, z, yaw, device, cuda=True)
        h = _P()
        _check(_lib.rtg_traj_wrap(device, K, T, *ptrs, ctypes.byref(h)), "rtg_traj_wrap")
        t = cls(h, K, T, device)
        t._borrowed = (x, y, z, yaw)
        return t

    @classmethod
    def sample_double_integrator(cls, ax, ay, T: int, dt: float, start, v0, device=0, stream=None) -> "Traj":
        """rtg_traj_sample_double_integrator: constant accelerations (ax, ay)[K] from start (x, y, z)
        with velocity v0 (vx, vy)."""
        K = int(ax.shape[0])
        if _kind(ay) != _kind(ax):
            raise ValueError("ax, ay must live in the same memory")
        pa, pb = _arg("ax", ax, "float32", (K,), device), _arg("ay", ay, "float32", (K,), device)
        st3 = (ctypes.c_float * 3)(*[float(s) for s in start[:3]])
        v2 = (ctypes.c_float * 2)(float(v0[0]), float(v0[1]))
        h = _P()
        _check(_lib.rtg_traj_sample_double_integrator(device, K, int(T), float(dt), st3, v2, pa, pb,
                                                      _kind(ax), _stream(stream), ctypes.byref(h)),
               "rtg_traj_sample_double_integrator")
        return cls(h, K, int(T), device)

    @classmethod
    def sample_unicycle(cls, v, omega, T: int, dt: float, start, device=0, stream=None) -> "Traj":
        K = int(v.shape[0])
        if _kind(omega) != _kind(v):
            raise ValueError("v, omega must live in the same memory")
        pv, pw = _arg("v", v, "float32", (K,), device), _arg("omega", omega, "float32", (K,), device)
        st4 = (ctypes.c_float * 4)(*[float(s) for s in start])
        h = _P()
        _check(_lib.rtg_traj_sample_unicycle(device, K, int(T), float(dt), st4, pv, pw, _kind(v),
                                             _stream(stream), ctypes.byref(h)), "rtg_traj_sample_unicycle")
        return cls(h, K, int(T), device)

    @classmethod
    def view_ring(cls, centroids, size: float, camera, n: int, z: float, device=0, stream=None):
        """rtg_traj_view_ring: n viewpoints per region centroid (centroids [3, R]) facing it at the
        shortest viewing distance (N2).  Returns (Traj with K = R n, T = 1, viewing distance)."""
        R = int(centroids.shape[-1])
        pc = _arg("centroids", centroids, "float32", (3, R), device)
        cam = camera if isinstance(camera, Camera) else make_camera(camera)
        h = _P()
        d = ctypes.c_double()
        _check(_lib.rtg_traj_view_ring(device, R, _kind(centroids), pc, float(size), ctypes.byref(cam),
                                       int(n), float(z), _stream(stream), ctypes.byref(h), ctypes.byref(d)),
               "rtg_traj_view_ring")
        return cls(h, R * int(n), 1, device), d.value

    def set_start(self, start) -> "Traj":
        """rtg_traj_set_start: the shared start state {x, y, z, yaw} (x_i(0) of Eq. equ:traj_utility),
        scored as info state l = 0 with SCORE_INCLUDE_START."""
        st4 = (ctypes.c_float * 4)(*[float(v) for v in start])
        _check(_lib.rtg_traj_set_start(self.handle, st4), "rtg_traj_set_start")
        return self

    def read(self, stream=None):
        torch = _torch()
        out = [torch.empty((self.K, self.T), dtype=torch.float32, device=f"cuda:{self.device}") for _ in range(4)]
        _check(_lib.rtg_traj_read(self.handle, *[_ptr(o) for o in out], _stream(stream)), "rtg_traj_read")
        return out

    def close(self):
        if self.handle:
            _check(_lib.rtg_traj_destroy(self.handle), "rtg_traj_destroy")
            self.handle = _P()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ calls
def score(m: Map, tr: Traj, camera, params: ScoreParams, first_col=None, feasible=None, gain=None, utility=None,
          stream=None):
    """rtg_score into caller-owned CUDA tensors (allocated here when None). Returns them."""
    torch = _torch()
    K = tr.K
    dev = torch.device("cuda", m.device)
    first_col = torch.empty(K, dtype=torch.int32, device=dev) if first_col is None else first_col
    feasible = torch.empty(K, dtype=torch.uint8, device=dev) if feasible is None else feasible
    gain = torch.empty(K, dtype=torch.float64, device=dev) if gain is None else gain
    utility = torch.empty(K, dtype=torch.float64, device=dev) if utility is None else utility
    outs = (("first_col", first_col, "int32"), ("feasible", feasible, "uint8"), ("gain", gain, "float64"),
            ("utility", utility, "float64"))
    ptrs = [_arg(nm, a, dt, (K,), m.device) for nm, a, dt in outs]
    for nm, a, _ in outs:
        if isinstance(a, np.ndarray) or not a.is_cuda:
            raise ValueError(f"{nm}: must be a CUDA tensor (rtg_score writes device memory)")
    cam = camera if isinstance(camera, Camera) else make_camera(camera)
    _check(_lib.rtg_score(m.handle, tr.handle, ctypes.byref(cam), ctypes.byref(params), *ptrs, _stream(stream)),
           "rtg_score")
    return first_col, feasible, gain, utility


def best(utility, index_base: int = 0, stream=None):
    """rtg_best -> (score, global index); index -1 / score -inf when nothing is feasible."""
    out = BestResult()
    if len(utility.shape) != 1:
        raise ValueError("utility: expected [K]")
    p = _arg("utility", utility, "float64", cuda=True)
    _check(_lib.rtg_best(p, int(utility.numel()), int(index_base), _stream(stream), ctypes.byref(out)),
           "rtg_best", allow=(ERR_NO_FEASIBLE,))
    return out.score, out.index


def best_async(utility, out, index_base: int = 0, stream=None):
    """rtg_best_async: the argmax written into `out` (a CUDA float64 tensor of 2 elements holding one
    rtg_best_result: score, then the index's int64 bits); no synchronisation (capturable)."""
    if len(utility.shape) != 1:
        raise ValueError("utility: expected [K]")
    p = _arg("utility", utility, "float64", cuda=True)
    o = _arg("out", out, "float64", (2,), cuda=True)
    _check(_lib.rtg_best_async(p, int(utility.numel()), int(index_base), o, _stream(stream)), "rtg_best_async")
    return out


def read_best(out):
    """(score, index) from a best_async result tensor (synchronises through the copy)."""
    h = out.detach().cpu()
    return float(h[0]), int(h.view(_torch().int64)[1])


class ScoreGraph:
    """rtg_score (culled mode) + rtg_best_async on one map and one trajectory handle, captured once into a
    CUDA graph (torch.cuda.CUDAGraph) and replayed.  The graph keeps the handles' device pointers: a replay
    scores what the trajectory buffers then hold (refill them in place, e.g. through Traj.wrap) against
    the same map.  The capture is preceded by one eager call (a reclassification, if the params ask for
    one, happens there, outside the graph)."""

    def __init__(self, m: Map, tr: Traj, camera, params: ScoreParams, index_base: int = 0):
        torch = _torch()
        if params.mode != MODE_CULLED:
            raise ValueError("ScoreGraph: culled mode only (dense mode reads the list length on the host)")
        dev = torch.device("cuda", m.device)
        K = tr.K
        self.outs = (torch.empty(K, dtype=torch.int32, device=dev), torch.empty(K, dtype=torch.uint8, device=dev),
                     torch.empty(K, dtype=torch.float64, device=dev), torch.empty(K, dtype=torch.float64, device=dev))
        self.best = torch.empty(2, dtype=torch.float64, device=dev)
        self._keep = (m, tr)   # the graph holds their device pointers
        cam = camera if isinstance(camera, Camera) else make_camera(camera)
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            score(m, tr, cam, params, *self.outs)
            best_async(self.outs[3], self.best, index_base)
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, capture_error_mode="thread_local"):
            score(m, tr, cam, params, *self.outs)
            best_async(self.outs[3], self.best, index_base)

    def replay(self):
        """Enqueue one replay on the current stream; returns (first_col, feasible, gain, utility, best)
        (the views' outputs and best are in .vouts / .vbest)."""
        self.graph.replay()
        return self.outs + (self.best,)


def ledger_update(mu_prev, mu_cur, w_prev, w_out=None, device=0, stream=None):
    """rtg_ledger_update (N4): w = |mu_cur - mu_prev| where the mean moved, else w_prev (CUDA out)."""
    torch = _torch()
    n = int(w_prev.shape[0])
    w_out = torch.empty(n, dtype=torch.float32, device=f"cuda:{device}") if w_out is None else w_out
    kind = _kind(mu_prev)
    if _kind(mu_cur) != kind or _kind(w_prev) != kind:
        raise ValueError("mu_prev, mu_cur, w_prev must live in the same memory")
    ptrs = (_arg("mu_prev", mu_prev, "float32", (3, n), device), _arg("mu_cur", mu_cur, "float32", (3, n), device),
            _arg("w_prev", w_prev, "float32", (n,), device), _arg("w_out", w_out, "float32", (n,), device, cuda=True))
    _check(_lib.rtg_ledger_update(device, n, kind, *ptrs, _stream(stream)), "rtg_ledger_update")
    return w_out


def region_utility(m: Map, origin, size: float, dims, stream=None):
    """rtg_region_utility (N2): (omega [prod dims] float64, count [prod dims] int32) CUDA tensors."""
    torch = _torch()
    nr = int(dims[0]) * int(dims[1]) * int(dims[2])
    omega = torch.empty(nr, dtype=torch.float64, device=f"cuda:{m.device}")
    count = torch.empty(nr, dtype=torch.int32, device=f"cuda:{m.device}")
    o = (ctypes.c_double * 3)(*[float(v) for v in origin])
    d = (_I * 3)(*[int(v) for v in dims])
    _check(_lib.rtg_region_utility(m.handle, o, float(size), d, _ptr(omega), _ptr(count), _stream(stream)),
           "rtg_region_utility")
    return omega, count


def plan_tree(m: Map, start, goal, params: TreeParams, stream=None):
    """rtg_plan_tree (N3): -> (Traj of candidates [K, max_depth + 1] or None, costs [K], reached, stats).
    Raises RTGError(ERR_NO_FEASIBLE) when nothing collision-free grows from the start."""
    st3 = (ctypes.c_float * 3)(*[float(v) for v in start])
    g2 = (ctypes.c_float * 2)(*[float(v) for v in goal])
    h = _P()
    cost = (ctypes.c_double * int(params.n_traj))()
    nf, rc = _I(), _I()
    stats = (_LL * 4)()
    _check(_lib.rtg_plan_tree(m.handle, st3, g2, ctypes.byref(params), _stream(stream), ctypes.byref(h), cost,
                              ctypes.byref(nf), ctypes.byref(rc), stats), "rtg_plan_tree")
    K = nf.value
    tr = Traj(h, K, int(params.max_depth) + 1)
    return tr, np.array(cost[:K]), bool(rc.value), dict(expanded=stats[0], created=stats[1], samples=stats[2],
                                                        candidates_tested=stats[3])


def cost_benefit(omega, d, stream=None):
    """rtg_cost_benefit (N2): argmax of omega / e^d (ties -> smaller d, then index) -> (score, index)."""
    out = BestResult()
    R = int(omega.numel())
    po = _arg("omega", omega, "float64", (R,), cuda=True)
    pd = _arg("d", d, "float64", (R,), cuda=True)
    _check(_lib.rtg_cost_benefit(po, pd, R, _stream(stream), ctypes.byref(out)), "rtg_cost_benefit")
    return out.score, out.index


def score_debug(m: Map, tr: Traj, camera, params: ScoreParams, pair_mask: bool = False, stream=None):
    """rtg_score_debug: per-waypoint arrays for every waypoint (+ optional pair mask, stats)."""
    torch = _torch()
    KT = tr.K * tr.T
    dev = torch.device("cuda", m.device)
    wp_col = torch.empty(KT, dtype=torch.uint8, device=dev)
    wp_gain = torch.empty(KT, dtype=torch.float64, device=dev)
    wp_nh = torch.empty(KT, dtype=torch.int32, device=dev)
    wp_nl = torch.empty(KT, dtype=torch.int32, device=dev)
    mask = None
    if pair_mask:
        words = (KT * m.n + 31) // 32
        mask = torch.empty(max(words, 1), dtype=torch.int32, device=dev)
    stats = (ctypes.c_longlong * DEBUG_STATS)()
    cam = camera if isinstance(camera, Camera) else make_camera(camera)
    _check(_lib.rtg_score_debug(m.handle, tr.handle, ctypes.byref(cam), ctypes.byref(params), _ptr(wp_col),
                                _ptr(wp_gain), _ptr(wp_nh), _ptr(wp_nl), _ptr(mask), stats, _stream(stream)),
           "rtg_score_debug")
    return dict(wp_col=wp_col, wp_gain=wp_gain, wp_nh=wp_nh, wp_nl=wp_nl, pair_mask=mask,
                stats=dict(col_refined=stats[0], vis_refined=stats[1], tested=stats[2], cells_aggregated=stats[3],
                           col_tested=stats[4], tested_flank=stats[5], units=stats[6], tested_visible=stats[7],
                           rows=stats[8], runs=stats[9], unit_table_entries=stats[10],
                           row_table_bytes=stats[11]))


def unpack_pair_mask(mask, KT: int, N: int) -> np.ndarray:
    words = mask.cpu().numpy().view(np.uint32)
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")[: KT * N]
    return bits.reshape(KT, N).astype(bool)


def map_from_workload(wl, device=0, stream=None, on_device=True, options=None) -> Map:
    """Convenience: build a Map from a workloads.Workload (arrays moved to CUDA when on_device)."""
    arrs = [wl.means, wl.quats, wl.scales, wl.opacity, wl.info_w, wl.flags]
    if on_device:
        torch = _torch()
        arrs = [None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{device}") for a in arrs]
    return Map(*arrs, r_robot=wl.robot.r_robot, lambda_g=wl.robot.lambda_g, collide_rule=wl.robot.rule,
               device=device, stream=stream, options=options)


def traj_from_workload(wl, device=0, stream=None, on_device=True, x=None, y=None, z=None, yaw=None) -> Traj:
    arrs = [wl.x if x is None else x, wl.y if y is None else y, wl.z if z is None else z,
            wl.yaw if yaw is None else yaw]
    if on_device:
        torch = _torch()
        arrs = [torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{device}") for a in arrs]
        t = Traj.upload(*arrs, device=device, stream=stream)
        t._keep = arrs
        return t
    return Traj.upload(*[np.ascontiguousarray(a, dtype=np.float32) for a in arrs], device=device, stream=stream)

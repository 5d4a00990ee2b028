"""ctypes binding of the C ABI in include/bilevel_b200.h.

The library is mandatory: there is no CPU fallback.  Importing works without a
GPU (so the CPU test suite can check the exported symbols), but creating a
:class:`Context` without a CUDA device raises immediately.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int64, c_longlong, c_size_t, c_uint, c_uint64, c_void_p

import numpy as np

LIB_PATH = os.environ.get("BD_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                           "libbilevel_b200.so")   # BD_LIB_PATH: tuning builds

BD_OK, BD_ERR_VALUE, BD_ERR_STRUCTURE, BD_ERR_NUMERICAL, BD_ERR_CUDA, BD_ERR_STATE = 0, -1, -2, -3, -4, -5

# name -> (restype, argtypes); mirrors include/bilevel_b200.h exactly.
_P = c_void_p
SIGNATURES = {
    "bd_abi_version": (c_int, []),
    "bd_create": (c_int, [c_int, POINTER(c_void_p)]),
    "bd_destroy": (None, [_P]),
    "bd_last_error": (c_char_p, [_P]),
    "bd_set_stream": (c_int, [_P, _P]),
    "bd_synchronize": (c_int, [_P]),
    "bd_set_option": (c_int, [_P, c_char_p, c_int]),
    "bd_launch_count": (c_int64, [_P]),
    "bd_error_bits": (c_int, [_P, POINTER(c_int)]),
    "bd_get_stat": (c_int, [_P, c_char_p, POINTER(c_double)]),
    "bd_probe": (c_int, [_P, c_char_p, POINTER(c_double)]),
    "bd_set_basis": (c_int, [_P, c_int, c_int, _P, _P, _P]),
    "bd_set_stage1": (c_int, [_P, c_int, c_int, c_int, _P, _P, _P, _P]),
    "bd_set_projection": (c_int, [_P, c_int, c_double, c_int, _P, _P]),
    "bd_set_scenes": (c_int, [_P, c_int, c_int, c_int, _P, _P, _P, _P, c_int, _P, _P]),
    "bd_stage1": (c_int, [_P, c_int, c_int, _P, _P, _P, _P]),
    "bd_project": (c_int, [_P, c_int, c_int, _P, _P, c_int, c_double, _P, _P, _P, _P, _P, _P]),
    "bd_solve_lower": (c_int, [_P, c_int, c_int, _P, c_int, c_double, _P, _P, _P, _P, _P, _P, _P, _P]),
    "bd_eval": (c_int, [_P, c_int, _P, _P, _P, _P, _P, _P, _P]),
    "bd_residuals": (c_int, [_P, c_int, c_int, _P, _P]),
    "bd_kkt_solve": (c_int, [_P, c_int, c_int, _P, _P, c_int, _P, _P]),
    "bd_solve_lower_shard": (c_int, [_P, c_int, _P, c_int, _P, _P, _P, _P, _P]),
    "bd_replay_shard": (c_int, [_P, c_int, _P, c_int, _P, _P, _P]),
    "bd_replay_shard_dev": (c_int, [_P, c_int, _P, c_int, _P, _P, _P, _P]),
    "bd_shard_p2p_set": (c_int, [_P, c_int, c_int, _P, _P, c_size_t, c_size_t, c_size_t, c_size_t, c_int]),
    "bd_solve_lower_shard_p2p": (c_int, [_P, c_int, _P, c_int, _P, _P, _P, _P, c_longlong, c_uint, c_double, _P]),
    "bd_shard_p2p_best_row": (c_int, [_P, _P, c_longlong, c_int, _P, c_uint, _P]),
    "bd_sample_philox": (c_int, [_P, c_int, c_int, _P, _P, c_uint64, c_int, c_int, c_int, _P]),
    "bd_sample": (c_int, [_P, c_int, c_int, _P, _P, _P, _P]),
    "bd_rank_refit": (c_int, [_P, c_int, c_int, c_int, _P, _P, _P, c_int, c_int, c_double, c_double, c_double, _P, _P,
                              _P, _P, _P, _P]),
    "bd_cem_cycle": (c_int, [_P, c_int, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "bd_cem_last_batch": (c_int, [_P, c_int, c_int, _P, _P, _P, _P]),
    "bd_set_normal_tables": (c_int, [_P, _P, _P, _P]),
    "bd_numpy_normals": (c_int, [_P, _P, c_longlong, c_longlong, _P, _P]),
    "bd_build_scenes": (c_int, [_P, c_int, c_int, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "bd_set_curvature": (c_int, [_P, c_int, c_int, _P, _P]),
    "bd_set_control_grid": (c_int, [_P, c_int, _P, _P, c_double, c_double, c_double, c_double]),
    "bd_controls": (c_int, [_P, c_int, _P, _P, _P, _P]),
    "bd_sim_run": (c_int, [_P, c_int, c_int, _P, _P, _P, _P, _P, _P, _P, _P, c_int, _P, c_int, c_int, _P, _P, _P,
                           _P]),
    "bd_cvae_set_weights": (c_int, [_P, c_int, _P, _P, _P]),
    "bd_cvae_decode": (c_int, [_P, c_int, _P, _P, _P]),
    "bd_cvae_warm_start": (c_int, [_P, c_int, _P, _P, _P, _P, _P, _P]),
}


class Limits(ctypes.Structure):
    """bd_limits: ConstraintSpec scalars (pkg/constraints.py:31-42)."""
    _fields_ = [(n, c_double) for n in
                ("ellipse_a", "ellipse_b", "v_min", "v_max", "a_max", "kappa_max", "c_max", "y_lb", "y_ub")]


class CemConfig(ctypes.Structure):
    """bd_cem_config: BiLevelConfig (pkg/bilevel.py:72-97) + projection budget."""
    _fields_ = [("batch", c_int), ("n_cons", c_int), ("n_elite", c_int), ("iterations", c_int),
                ("am_iters", c_int), ("eta", c_double), ("gamma", c_double), ("residual_weight", c_double),
                ("tol", c_double), ("seed", c_uint64), ("scene_offset", c_int), ("iter_begin", c_int),
                ("iter_end", c_int), ("pcg64_state", c_void_p), ("pcg64_positions", c_void_p)]


class Traffic(ctypes.Structure):
    """bd_traffic: IDMParams / MOBILParams (pkg/highway.py:73-89), tick length and wheelbase."""
    _fields_ = [(n, c_double) for n in
                ("idm_v0", "idm_time_headway", "idm_s0", "idm_a_max", "idm_b_comfort", "idm_delta", "idm_b_hard",
                 "mobil_politeness", "mobil_b_safe", "mobil_a_threshold", "mobil_cooldown", "dt", "wheelbase")]


class Env(ctypes.Structure):
    """bd_env: PlannerEnvConfig fields used by build_scene (pkg/planners.py:40-87)."""
    _fields_ = [("max_obstacles", c_int), ("obstacle_range", c_double), ("wheelbase", c_double),
                ("v_max", c_double), ("a_max", c_double), ("kappa_max", c_double), ("c_max", c_double),
                ("v_min", c_double), ("other_length", c_double), ("other_width", c_double)]


_lib = None


def load() -> ctypes.CDLL:
    """Load the CUDA library (raises ImportError if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"CUDA library missing: {LIB_PATH} (build it: python -m paper_2212_02224_b200.build)")
        lib = ctypes.CDLL(LIB_PATH)
        # BD_AB_OLD_LIB=1 (performance A/B of older library builds only): tolerate entry points
        # that an older build does not export
        lax = os.environ.get("BD_AB_OLD_LIB") == "1"
        for name, (res, args) in SIGNATURES.items():
            if lax and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def ptr(a):
    """Raw pointer of a numpy array or torch tensor (None passes through)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    raise TypeError(f"unsupported buffer type {type(a)}")


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class Context:
    """One device context (bd_ctx) of the C library."""

    def __init__(self, device: int = 0):
        self.lib = load()
        h = c_void_p()
        rc = self.lib.bd_create(int(device), ctypes.byref(h))
        if rc != 0:
            raise RuntimeError(f"bd_create(device={device}) failed with code {rc}: no usable CUDA device "
                               "(the B200 path has no CPU fallback)")
        self.h = h
        self.device = int(device)

    def close(self):
        if getattr(self, "h", None):
            self.lib.bd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int, what: str):
        if rc == 0:
            return
        msg = f"{what}: {self.lib.bd_last_error(self.h).decode()}"
        from .batch_qp import NumericalFailure, StructureError
        if rc == BD_ERR_VALUE:
            raise ValueError(msg)
        if rc == BD_ERR_STRUCTURE:
            raise StructureError(msg)
        if rc == BD_ERR_NUMERICAL:
            raise NumericalFailure(msg)
        raise RuntimeError(msg)

    def call(self, name: str, *args):
        """Call bd_<name>(ctx, *args); numpy arrays / torch tensors are passed by pointer and
        stay referenced for the duration of the call."""
        fn = getattr(self.lib, name)
        conv = [ptr(a) if isinstance(a, np.ndarray) or hasattr(a, "data_ptr") else a for a in args]
        self.check(fn(self.h, *conv), name)
        del args

    def launches(self) -> int:
        return int(self.lib.bd_launch_count(self.h))

    def set_option(self, key: str, value: int):
        self.call("bd_set_option", key.encode(), int(value))

    def set_stream(self, stream_ptr: int | None):
        """Run on an external cudaStream_t; 0 (torch's legacy default stream) maps to cudaStreamLegacy,
        None restores the library's own stream."""
        if stream_ptr == 0:
            stream_ptr = 1   # cudaStreamLegacy
        self.call("bd_set_stream", stream_ptr)

    def synchronize(self):
        self.call("bd_synchronize")

    def stat(self, key: str) -> float:
        v = c_double(0.0)
        self.call("bd_get_stat", key.encode(), ctypes.byref(v))
        return v.value

    def probe(self, what: str) -> float:
        v = c_double(0.0)
        self.call("bd_probe", what.encode(), ctypes.byref(v))
        return v.value

    def error_bits(self) -> int:
        bits = c_int(0)
        self.call("bd_error_bits", ctypes.byref(bits))
        return bits.value


def scene_limits(spec) -> Limits:
    return Limits(spec.ellipse_a, spec.ellipse_b, spec.v_min, spec.v_max, spec.a_max, spec.kappa_max, spec.c_max,
                  spec.y_lb, spec.y_ub)


def upload_scenes(ctx: Context, scenes, m: int):
    """bd_set_scenes for a list of PlanningScene (all with the same obstacle count)."""
    S = len(scenes)
    n_obs = scenes[0].spec.num_obstacles
    for sc in scenes:
        if sc.spec.num_obstacles != n_obs:
            raise ValueError("all scenes of a fleet must carry the same number of obstacle rows")
        if sc.spec.num_samples != m:
            raise ValueError("constraint spec and basis disagree on the time grid")
    ox = f64(np.stack([sc.spec.obstacles_x for sc in scenes])) if n_obs else None
    oy = f64(np.stack([sc.spec.obstacles_y for sc in scenes])) if n_obs else None
    lims = (Limits * S)(*[scene_limits(sc.spec) for sc in scenes])
    b0 = f64(np.stack([sc.initial_state for sc in scenes]))
    curves = [sc.spec.road_curvature for sc in scenes]
    n_curv = 0
    cx = ck = None
    if any(c is not None for c in curves):
        lens = {len(np.asarray(c[0])) for c in curves if c is not None}
        n_curv = max(lens)
        cx = np.zeros((S, n_curv))
        ck = np.zeros((S, n_curv))
        for s, c in enumerate(curves):
            if c is None:   # straight road: kappa == 0 everywhere
                cx[s] = np.arange(n_curv, dtype=float)
                continue
            xs, ks = np.asarray(c[0], float), np.asarray(c[1], float)
            if len(xs) != n_curv:   # pad by repeating the last knot (np.interp clamps beyond it)
                xs = np.concatenate([xs, xs[-1] + np.arange(1, n_curv - len(xs) + 1)])
                ks = np.concatenate([ks, np.full(n_curv - len(ks), ks[-1])])
            cx[s], ck[s] = xs, ks
        cx, ck = f64(cx), f64(ck)
    ctx.call("bd_set_scenes", S, n_obs, m, ptr(ox), ptr(oy), ctypes.cast(lims, c_void_p), ptr(b0), n_curv,
             ptr(cx), ptr(ck))

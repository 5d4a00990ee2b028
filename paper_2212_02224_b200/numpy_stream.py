"""numpy's Generator(PCG64).standard_normal stream on the device (drop-in sampling, K4).

The reference draws every CEM iteration's set-points with ``rng.standard_normal((n, dim))``
(pkg/bilevel.py:56).  ``solve_bilevel`` keeps that contract -- same numbers, generator left in
the same state -- but instead of drawing on the host it hands the generator's PCG64 state to
the library, which reproduces numpy's 256-layer ziggurat on the device
(csrc/numpy_normals.cuh) and reports how many raw outputs were consumed; the generator is then
advanced by exactly that many steps (``PCG64.advance``).

numpy's ziggurat tables (ki, wi, fi) are read from numpy's own compiled module and validated
once per process against numpy itself; if they cannot be found or the validation fails, the
caller draws on the host as before.
"""
from __future__ import annotations

import glob
import math
import os
import struct

import numpy as np

__all__ = ["ziggurat_tables", "pcg64_state_words", "device_stream_ok"]

_KI0 = 0x000EF33D8025EF6A          # ki[0] of numpy's normal ziggurat (ziggurat_constants.h)
_TABLES = None
_ZIG_R = 3.6541528853610087963519472518
_ZIG_INV_R = 0.27366123732975827203338247596


def _candidate_files():
    d = os.path.join(os.path.dirname(np.__file__), "random")
    return sorted(glob.glob(os.path.join(d, "_generator*.so")) + glob.glob(os.path.join(d, "_generator*.pyd")))


def _replica(bitgen: np.random.PCG64, count: int, ki, wi, fi) -> np.ndarray:
    """numpy's random_standard_normal in Python on raw PCG64 outputs (validation only)."""
    raw = iter(int(v) for v in bitgen.random_raw(count * 2 + 64))
    out = np.empty(count)
    for i in range(count):
        while True:
            r = next(raw)
            idx = r & 0xFF
            r >>= 8
            sign = r & 1
            rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
            x = float(rabs) * float(wi[idx])
            if sign:
                x = -x
            if rabs < int(ki[idx]):
                break
            if idx == 0:
                while True:
                    xx = -_ZIG_INV_R * math.log1p(-((next(raw) >> 11) * (1.0 / 9007199254740992.0)))
                    yy = -math.log1p(-((next(raw) >> 11) * (1.0 / 9007199254740992.0)))
                    if yy + yy > xx * xx:
                        x = -(_ZIG_R + xx) if (rabs >> 8) & 1 else _ZIG_R + xx
                        break
                break
            u = (next(raw) >> 11) * (1.0 / 9007199254740992.0)
            if (float(fi[idx - 1]) - float(fi[idx])) * u + float(fi[idx]) < math.exp(-0.5 * x * x):
                break
        out[i] = x
    return out


def ziggurat_tables():
    """(ki uint64[256], wi float64[256], fi float64[256]) of this numpy, or None."""
    global _TABLES
    if _TABLES is not None:
        return _TABLES or None
    _TABLES = False
    sig = struct.pack("<Q", _KI0)
    for path in _candidate_files():
        with open(path, "rb") as fh:
            blob = fh.read()
        off = blob.find(sig)
        while off >= 4096:
            ki = np.frombuffer(blob[off:off + 2048], dtype="<u8").copy()
            wi = np.frombuffer(blob[off - 2048:off], dtype="<f8").copy()
            fi = np.frombuffer(blob[off - 4096:off - 2048], dtype="<f8").copy()
            if ki[1] == 0 and fi[0] == 1.0 and 8e-16 < wi[0] < 9e-16 and np.all(np.diff(fi) < 0):
                ok = True
                for seed in (0, 2024):
                    want = np.random.Generator(np.random.PCG64(seed)).standard_normal(2000)
                    if not np.array_equal(_replica(np.random.PCG64(seed), 2000, ki, wi, fi), want):
                        ok = False
                        break
                if ok:
                    _TABLES = (ki, wi, fi)
                    return _TABLES
            off = blob.find(sig, off + 1)
    return None


def pcg64_state_words(bitgen, state: dict | None = None) -> np.ndarray | None:
    """[state lo, state hi, inc lo, inc hi] of a PCG64 bit generator (its `state` dict may be
    passed in when the caller already holds it), else None."""
    if type(bitgen) is not np.random.PCG64:
        return None
    st = bitgen.state if state is None else state
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    return np.array([s & m, s >> 64, inc & m, inc >> 64], dtype=np.uint64)


def device_stream_ok(rng) -> bool:
    return pcg64_state_words(rng.bit_generator) is not None and ziggurat_tables() is not None


def ensure_device_tables(ctx) -> bool:
    """Upload numpy's ziggurat tables to a context once; False if they are unavailable."""
    if getattr(ctx, "_nn_tables", False):
        return True
    tb = ziggurat_tables()
    if tb is None:
        return False
    ki, wi, fi = (np.ascontiguousarray(t) for t in tb)
    ctx.call("bd_set_normal_tables", ki.ctypes.data, wi.ctypes.data, fi.ctypes.data)
    ctx._nn_tables = True
    return True

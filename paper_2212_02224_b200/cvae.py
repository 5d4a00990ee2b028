"""CVAE warm-start decoder (paper PAPER.md:715-746; BASELINE config 3).

The reference package replaces the CVAE with a file-backed sample source
(`WarmStartSource`, pkg/behavior.py:96-137); the paper's decoder maps a scene
observation (the 55-entry `observe()` vector, pkg/highway.py:208-246) and a latent
z ~ N(0, I_2) to a behaviour vector through
(55+2) -> 1024 -> 1024 -> 1024 -> 1024 -> 256 -> dim, Linear + BatchNorm + ReLU per hidden
layer.  BatchNorm (inference form) is folded into the Linear weights here; the decoder runs on
the device (K5, `bd_cvae_decode`) and its samples feed iteration 1 of the device CEM cycle
through the reference's `warm_start` hook.  No trained weights exist in the reference, so
`CVAEDecoder.synthetic` builds seeded random weights of the paper's architecture.
"""

from __future__ import annotations

import ctypes

import numpy as np

from ._native import Context
from .behavior import DeviceWarmStart, ParamLayout, WarmStartSource

__all__ = ["CVAEDecoder", "fold_batchnorm", "OBS_DIM", "LATENT_DIM", "HIDDEN"]

OBS_DIM = 55
LATENT_DIM = 2
HIDDEN = (1024, 1024, 1024, 1024, 256)


def fold_batchnorm(W, b, gamma, beta, mean, var, eps=1e-5):
    """Linear(W, b) followed by inference BatchNorm == Linear(W', b')."""
    s = gamma / np.sqrt(var + eps)
    return W * s[:, None], (b - mean) * s + beta


class CVAEDecoder:
    def __init__(self, weights: list[np.ndarray], biases: list[np.ndarray], context: Context | None = None,
                 device: int = 0):
        if len(weights) != len(biases) or not weights:
            raise ValueError("need one bias per weight matrix")
        self.W = [np.ascontiguousarray(w, dtype=np.float32) for w in weights]
        self.b = [np.ascontiguousarray(b, dtype=np.float32) for b in biases]
        dims = [self.W[0].shape[1]] + [w.shape[0] for w in self.W]
        for l, w in enumerate(self.W):
            if w.shape[1] != dims[l] or self.b[l].shape != (w.shape[0],):
                raise ValueError(f"layer {l}: weight {w.shape} / bias {self.b[l].shape} do not chain")
        if dims[0] <= OBS_DIM:
            raise ValueError("the first layer takes the 55-entry observation plus the latent")
        self.dims = dims
        self.latent_dim = dims[0] - OBS_DIM
        self.out_dim = dims[-1]
        self.ctx = context if context is not None else Context(device)
        L = len(self.W)
        wp = (ctypes.c_void_p * L)(*[w.ctypes.data for w in self.W])
        bp = (ctypes.c_void_p * L)(*[b.ctypes.data for b in self.b])
        d = (ctypes.c_int * (L + 1))(*dims)
        self.ctx.call("bd_cvae_set_weights", L, ctypes.cast(d, ctypes.c_void_p), ctypes.cast(wp, ctypes.c_void_p),
                      ctypes.cast(bp, ctypes.c_void_p))

    @staticmethod
    def synthetic(seed: int, out_dim: int = 8, hidden=HIDDEN, latent_dim: int = LATENT_DIM, **kw) -> "CVAEDecoder":
        """Seeded decoder of the paper's architecture with BatchNorm folded into each hidden Linear."""
        rng = np.random.default_rng(seed)
        dims = [OBS_DIM + latent_dim, *hidden, out_dim]
        Ws, bs = [], []
        for l in range(len(dims) - 1):
            fan_in, fan_out = dims[l], dims[l + 1]
            W = rng.standard_normal((fan_out, fan_in)) * np.sqrt(2.0 / fan_in)
            b = 0.01 * rng.standard_normal(fan_out)
            if l < len(dims) - 2:       # hidden layers: Linear + BatchNorm (+ ReLU in the kernel)
                W, b = fold_batchnorm(W, b, 1.0 + 0.1 * rng.standard_normal(fan_out), 0.1 * rng.standard_normal(fan_out),
                                      0.1 * rng.standard_normal(fan_out), 1.0 + 0.1 * rng.random(fan_out))
            Ws.append(W)
            bs.append(b)
        return CVAEDecoder(Ws, bs, **kw)

    def decode(self, obs: np.ndarray, z: np.ndarray) -> np.ndarray:
        """(count, out_dim) behaviour vectors for one scene observation and latent draws z."""
        obs = np.ascontiguousarray(np.asarray(obs, dtype=np.float32).reshape(-1))
        z = np.ascontiguousarray(np.asarray(z, dtype=np.float32))
        if obs.shape != (OBS_DIM,) or z.ndim != 2 or z.shape[1] != self.latent_dim:
            raise ValueError(f"need obs ({OBS_DIM},) and z (count, {self.latent_dim})")
        out = np.empty((z.shape[0], self.out_dim))
        self.ctx.call("bd_cvae_decode", z.shape[0], obs, z, out)
        return out

    def warm_start(self, obs: np.ndarray, count: int, layout: ParamLayout, rng: np.random.Generator,
                   scale: np.ndarray | None = None, shift: np.ndarray | None = None) -> WarmStartSource:
        """Decode `count` samples (z ~ N(0, I)) into the reference's warm-start interface.
        `scale`/`shift` map the decoder output to set-point units (y [m], v [m/s]):
        rows = decode * scale + shift.  The rows stay on the device (`bd_cvae_warm_start`) and
        `solve_bilevel` on the same context feeds them to the cycle in place; `samples` / `draw`
        build the host copy on first use."""
        if layout.dim != self.out_dim:
            raise ValueError(f"decoder rows have {self.out_dim} columns, the layout {layout.dim}")
        obs32 = np.ascontiguousarray(np.asarray(obs, dtype=np.float32).reshape(-1))
        if obs32.shape != (OBS_DIM,):
            raise ValueError(f"need obs ({OBS_DIM},)")
        z = rng.standard_normal((count, self.latent_dim))
        z32 = np.ascontiguousarray(z, dtype=np.float32)
        sc = None if scale is None else np.ascontiguousarray(np.broadcast_to(np.asarray(scale, dtype=np.float64),
                                                                             (self.out_dim,)))
        sh = None if shift is None else np.ascontiguousarray(np.broadcast_to(np.asarray(shift, dtype=np.float64),
                                                                             (self.out_dim,)))
        rows = ctypes.c_void_p()
        self.ctx.call("bd_cvae_warm_start", count, obs32.ctypes.data, z32.ctypes.data,
                      None if sc is None else sc.ctypes.data, None if sh is None else sh.ctypes.data, None,
                      ctypes.addressof(rows))
        gen = getattr(self.ctx, "_warm_gen", 0) + 1
        self.ctx._warm_gen = gen

        def materialize():
            p = self.decode(obs32, z32)
            if sc is not None:
                p = p * sc
            if sh is not None:
                p = p + sh
            return p

        return DeviceWarmStart(self.ctx, rows.value, count, layout, gen, materialize)

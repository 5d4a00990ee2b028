"""numpy restatement of the device Philox4x32-10 normal stream (csrc/cem_kernels.cuh,
philox_normals) — test infrastructure: pins the device sampler and drives the CPU stand-in
backend of the multi-rank tests."""

from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, seed: int):
    """Vectorised over uint32 counter arrays; returns the four output words."""
    c = [np.asarray(x, dtype=np.uint64) & MASK for x in (c0, c1, c2, c3)]
    k0 = np.uint64(seed & 0xFFFFFFFF)
    k1 = np.uint64((seed >> 32) & 0xFFFFFFFF)
    for _ in range(10):
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c = [(hi1 ^ c[1] ^ k0) & MASK, lo1, (hi0 ^ c[3] ^ k1) & MASK, lo0]
        k0 = (k0 + np.uint64(W0)) & MASK
        k1 = (k1 + np.uint64(W1)) & MASK
    return c


def philox_normals(seed: int, scene: int, iteration: int, samples: np.ndarray, d: int) -> np.ndarray:
    """(len(samples), d) standard normals, identical to the device stream."""
    samples = np.asarray(samples, dtype=np.uint64)
    out = np.empty((samples.shape[0], d))
    for base in range(0, d, 4):
        c = philox4x32_10(samples, np.full_like(samples, iteration), np.full_like(samples, scene),
                          np.full_like(samples, base // 4), seed)
        for q in range(0, 4, 2):
            if base + q >= d:
                break
            u1 = (c[q].astype(np.float64) + 0.5) * 2.3283064365386963e-10
            u2 = (c[q + 1].astype(np.float64) + 0.5) * 2.3283064365386963e-10
            r = np.sqrt(-2.0 * np.log(u1))
            out[:, base + q] = r * np.cos(2.0 * np.pi * u2)
            if base + q + 1 < d:
                out[:, base + q + 1] = r * np.sin(2.0 * np.pi * u2)
    return out

"""float64 numpy forward pass of the CVAE decoder MLP — test infrastructure (parity of K5 is
unpinned by the reference, which ships no decoder; this pins the kernel to the architecture
restated from PAPER.md:715-746)."""

import numpy as np


def decode(weights, biases, obs, z):
    h = np.concatenate([np.repeat(np.asarray(obs, float).reshape(1, -1), len(z), axis=0), np.asarray(z, float)],
                       axis=1)
    for l, (W, b) in enumerate(zip(weights, biases)):
        h = h @ np.asarray(W, float).T + np.asarray(b, float)
        if l < len(weights) - 1:
            h = np.maximum(h, 0.0)
    return h

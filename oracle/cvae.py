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


def to_bf16(x):
    """Round to bfloat16 (round-to-nearest-even on the float32 bits, as __float2bfloat16_rn), as float64."""
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def decode_bf16(weights, biases, obs, z):
    """float64 forward pass with the tensor-core path's roundings: the first layer's output, every
    hidden layer's weights and every hidden activation are rounded to bf16 (fp32 bias + ReLU before
    the rounding); the last layer takes bf16 activations and fp32 weights."""
    x = np.concatenate([np.repeat(np.asarray(obs, np.float32).astype(float).reshape(1, -1), len(z), axis=0),
                        np.asarray(z, np.float32).astype(float)], axis=1)
    L = len(weights)
    h = to_bf16(np.maximum(x @ np.asarray(weights[0], np.float32).astype(float).T
                           + np.asarray(biases[0], np.float32), 0.0))
    for l in range(1, L - 1):
        W = to_bf16(weights[l])
        h = to_bf16(np.maximum(h @ W.T + np.asarray(biases[l], np.float32), 0.0))
    return h @ np.asarray(weights[L - 1], np.float32).astype(float).T + np.asarray(biases[L - 1], np.float32)

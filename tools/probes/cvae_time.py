"""CVAE decode timing: fused single launch vs per-layer launches (and parity between them)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2212_02224_b200.cvae import CVAEDecoder
from oracle.cvae import decode_bf16
dec = CVAEDecoder.synthetic(7)
rng = np.random.default_rng(1)
obs = rng.standard_normal(55).astype(np.float32)
for count in (1000, 77, 2000):
    z = rng.standard_normal((count, 2)).astype(np.float32)
    outs = {}
    for fused in (1, 0):
        dec.ctx.set_option("cvae_fused", fused)
        for _ in range(5): dec.decode(obs, z)
        t = []
        for _ in range(50):
            t0 = time.perf_counter(); outs[fused] = dec.decode(obs, z); t.append(time.perf_counter() - t0)
        print(f"count {count} fused={fused}: p50 {np.median(t) * 1e6:.1f} us  launches/call {dec.ctx.launch_count() if hasattr(dec.ctx, 'launch_count') else '?'}")
    emu = decode_bf16(dec.W, dec.b, obs, z)
    sc = np.abs(emu).max()
    for f in (1, 0):
        e = np.abs(outs[f] - emu)
        print(f"   fused={f}: max {e.max() / sc:.2e} mean {e.mean() / sc:.2e}")
    print("   fused vs per-layer max", np.abs(outs[1] - outs[0]).max() / sc)

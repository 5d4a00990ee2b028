"""Warm GPU time per CVAE decode: 200 bd_cvae_warm_start calls (no host output, no synchronise)
queued back to back on torch's stream, CUDA events around them (libraries via BD_LIB_PATH)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import ctypes
import numpy as np
import torch
from paper_2212_02224_b200.cvae import CVAEDecoder
dec = CVAEDecoder.synthetic(7)
torch.cuda.init()
s = torch.cuda.current_stream()
dec.ctx.set_stream(s.cuda_stream)
rng = np.random.default_rng(1)
obs = rng.standard_normal(55).astype(np.float32)
z = rng.standard_normal((1000, 2)).astype(np.float32)
rows = ctypes.c_void_p()
def one():
    dec.ctx.call("bd_cvae_warm_start", 1000, obs.ctypes.data, z.ctypes.data, None, None, None, ctypes.addressof(rows))
for _ in range(20): one()
torch.cuda.synchronize()
res = []
for rep in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(200): one()
    b.record(s)
    torch.cuda.synchronize()
    res.append(a.elapsed_time(b) * 1e3 / 200)
print(f"{os.environ.get('BD_LIB_PATH', 'default')}: GPU time per decode {np.median(res):.1f} us (reps {[round(r, 1) for r in res]})")

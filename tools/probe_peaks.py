"""FP32 issue-rate probes (scalar FFMA and packed FFMA2) on cuda:0 -> JSON on stdout.

The AM kernel's hot arithmetic is FFMA2 (fma.rn.f32x2), so its roofline denominator is the
larger of the two probes (bench.py records both)."""
import json
import subprocess
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2212_02224_b200._native import Context  # noqa: E402

ctx = Context(0)
out = {}
for what in ("fp32_tflops", "fp32x2_tflops"):
    vals = [ctx.probe(what) for _ in range(5)]
    out[what] = {"best": max(vals), "runs": vals}
try:
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip()
    out["clocks_after"] = clk
except OSError:
    pass
print(json.dumps(out, indent=1))

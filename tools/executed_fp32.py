"""Executed FP32 work of a kernel from an ncu report (--set full --import-source on): per SASS
line, predicated-on thread instructions x FP32 operations per thread instruction (FFMA 2, FADD /
FMUL 1, packed FFMA2 4, FADD2 / FMUL2 2), divided by the sample-iterations the launch ran.

    python tools/executed_fp32.py REPORT.ncu-rep SAMPLE_ITERS [--kernel REGEX]
"""
import argparse
import csv
import io
import json
import subprocess

FLOPS = {"FFMA": 2, "FADD": 1, "FMUL": 1, "FFMA2": 4, "FADD2": 2, "FMUL2": 2}

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("samples", type=float)
ap.add_argument("--kernel", default=None)
a = ap.parse_args()
sel = ["-k", "regex:" + a.kernel, "-c", "1"] if a.kernel else []
out = subprocess.run(["ncu", "-i", a.rep, *sel, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
per_op, thread_ops = {}, {}
for r in rows[2:]:
    if len(r) < len(hdr):
        break
    tok = r[ix["Source"]].split()
    if not tok:
        continue
    op = (tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]).split(".")[0]
    if op not in FLOPS:
        continue
    n = float(r[ix["Predicated-On Thread Instructions Executed"]].replace(",", "") or 0)
    thread_ops[op] = thread_ops.get(op, 0.0) + n
    per_op[op] = per_op.get(op, 0.0) + n * FLOPS[op]
total = sum(per_op.values())
print(json.dumps({"executed_fp32_flop_per_sample_iter": total / a.samples,
                  "by_opcode_flop_per_sample_iter": {k: round(v / a.samples, 1) for k, v in sorted(per_op.items())},
                  "thread_instructions_per_sample_iter": {k: round(v / a.samples, 1) for k, v in sorted(thread_ops.items())}},
                 indent=1))

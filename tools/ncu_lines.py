"""Warp-stall samples per CUDA source line of one kernel in an ncu report.

    python tools/ncu_lines.py REPORT.ncu-rep [--top 25]
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, cur, fname = {}, None, ""
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif r[0] and r[0].isdigit():
        cur = (fname, int(r[0]), r[1].strip()[:90])
        agg.setdefault(cur, 0.0)
    elif r[0] == "" and len(r) > 4 and r[2].startswith("0x") and cur is not None:
        try:
            agg[cur] += float(r[4])
        except ValueError:
            pass
tot = sum(agg.values()) or 1.0
for (f, line, src), v in sorted(agg.items(), key=lambda kv: -kv[1])[:a.top]:
    print(f"{100 * v / tot:5.1f}%  {f}:{line}  {src}")

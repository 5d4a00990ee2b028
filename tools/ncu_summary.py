"""Summarise an ncu report (.ncu-rep) of the AM kernel into profiles/ (markdown + json).

    python tools/ncu_summary.py gpurun_out/X.ncu-rep profiles/r01/NAME [--samples S*B*iters]

Extracts duration, issue/IPC, occupancy, pipe utilisation, DRAM bytes, warp-stall mix and the
per-opcode instruction mix (per sample-iteration when --samples is given).
"""

import argparse
import collections
import csv
import io
import json
import subprocess


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--samples", type=float, default=None, help="sample-iterations executed by the launch")
    ap.add_argument("--kernel", default=None, help="regex of the kernel to summarise (first matching launch)")
    a = ap.parse_args()
    sel = ["-k", "regex:" + a.kernel, "-c", "1"] if a.kernel else []
    det = ncu_csv(a.rep, *sel, "--page", "details")
    hdr = det[0]
    metrics = {}
    for row in det[1:]:
        d = dict(zip(hdr, row))
        if d.get("Metric Name"):
            metrics[d["Metric Name"]] = (d["Metric Value"], d.get("Metric Unit", ""))
    raw = ncu_csv(a.rep, *sel, "--page", "raw")
    rh, ru, rv = raw[0], raw[1], raw[2]
    rawd = {h: (v, u) for h, u, v in zip(rh, ru, rv)}

    def num(x):
        try:
            return float(str(x).replace(",", ""))
        except ValueError:
            return None

    dram = (num(rawd.get("dram__bytes_read.sum", ("0",))[0]) or 0.0)
    dram_w = (num(rawd.get("dram__bytes_write.sum", ("0",))[0]) or 0.0)
    unit_r = rawd.get("dram__bytes_read.sum", ("", ""))[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram_bytes = dram * scale.get(unit_r, 1) + dram_w * scale.get(rawd.get("dram__bytes_write.sum", ("", ""))[1], 1)
    pipes = {k: num(v[0]) for k, v in rawd.items()
             if k.startswith("sm__inst_executed_pipe_") and k.endswith("avg.pct_of_peak_sustained_active")}
    sass = ncu_csv(a.rep, *sel, "--page", "source", "--print-source", "sass")
    sh = sass[1]
    idx = {h: i for i, h in enumerate(sh)}
    stalls = collections.Counter()
    ops = collections.Counter()
    total = 0.0
    for r in sass[2:]:
        if len(r) < len(sh):
            break
        for h in sh:
            if h.startswith("stall_") and "Not Issued" not in h:
                stalls[h[6:]] += num(r[idx[h]]) or 0.0
        n = num(r[idx["Instructions Executed"]]) or 0.0
        tok = r[idx["Source"]].split()
        if tok:
            op = tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]
            ops[op.split(".")[0]] += n
            total += n
    st = sum(stalls.values()) or 1.0
    keep = ["Duration", "Elapsed Cycles", "SM Frequency", "Executed Ipc Active", "Issue Slots Busy",
            "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Block Size", "Grid Size",
            "Dynamic Shared Memory Per Block", "Theoretical Active Warps per SM", "Achieved Active Warps Per SM",
            "Waves Per SM", "Executed Instructions", "DRAM Throughput", "Compute (SM) Throughput"]
    summary = {
        "report": a.rep,
        "metrics": {k: " ".join(metrics[k]).strip() for k in keep if k in metrics},
        "dram_bytes_per_launch": dram_bytes,
        "pipe_pct_of_peak_active": {k.replace("sm__inst_executed_pipe_", "").split(".")[0]: v
                                    for k, v in sorted(pipes.items()) if v},
        "stall_pct": {k: round(100 * v / st, 1) for k, v in stalls.most_common(10)},
        "instructions_total": total,
    }
    if a.samples:
        summary["instructions_per_sample_iteration"] = total / a.samples
        summary["opcode_mix_per_sample_iteration"] = {k: round(v / a.samples, 1) for k, v in ops.most_common(30)}
    with open(a.out + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)
    with open(a.out + ".md", "w") as fh:
        fh.write(f"# ncu summary: {a.rep}\n\n")
        for k, v in summary["metrics"].items():
            fh.write(f"- {k}: {v}\n")
        fh.write(f"- DRAM bytes (read+write) per launch: {dram_bytes:.4g}\n")
        fh.write("\n## pipe utilisation (% of peak, active)\n")
        for k, v in summary["pipe_pct_of_peak_active"].items():
            fh.write(f"- {k}: {v:.1f}\n")
        fh.write("\n## warp stall mix (% of samples)\n")
        for k, v in summary["stall_pct"].items():
            fh.write(f"- {k}: {v}\n")
        if a.samples:
            fh.write(f"\n## instructions per sample-iteration: {summary['instructions_per_sample_iteration']:.1f}\n")
            for k, v in summary["opcode_mix_per_sample_iteration"].items():
                fh.write(f"- {k}: {v}\n")
    print(json.dumps(summary["metrics"], indent=1))


if __name__ == "__main__":
    main()

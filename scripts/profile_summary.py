"""Summarise ncu captures (run here, on the .ncu-rep brought back by gpurun)."""
import csv, io, subprocess, sys
from collections import Counter


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summary(rep, units=None, label=""):
    lines = [f"# {label or rep}"]
    rows = ncu_csv(rep, "--page", "details")
    h = rows[0]
    want = ["Duration", "SM Frequency", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput",
            "DRAM Throughput", "Issue Slots Busy", "Executed Instructions", "No Eligible",
            "Registers Per Thread", "Achieved Occupancy", "Grid Size", "Block Size",
            "Dynamic Shared Memory Per Block"]
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in want:
            lines.append(f"{d['Metric Name']}: {d['Metric Value']} {d['Metric Unit']}")
    raw = ncu_csv(rep, "--page", "raw")
    rh, rv = raw[0], raw[2]
    dr = {a: b for a, b in zip(rh, rv)}
    for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]:
        if k in dr:
            lines.append(f"{k}: {dr[k]}")
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    sh = src[1]
    data = [dict(zip(sh, r)) for r in src[2:]]
    tot = sum(int(d["Instructions Executed"] or 0) for d in data)
    samp = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data) or 1
    c, s = Counter(), Counter()
    for d in data:
        t = d["Source"].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        c[op] += int(d["Instructions Executed"] or 0)
        s[op] += int(d["Warp Stall Sampling (All Samples)"] or 0)
    lines.append(f"warp instructions: {tot}" + (f"  -> per unit {tot * 32 / units:.2f}" if units else ""))
    lines.append("opcode mix (share of instructions, share of stall samples):")
    for op, n in c.most_common(16):
        per = f"  {n * 32 / units:6.2f}/unit" if units else ""
        lines.append(f"  {op:10s} {100 * n / tot:6.2f}%{per}   stalls {100 * s[op] / samp:5.1f}%")
    return "\n".join(lines)


if __name__ == "__main__":
    rep = sys.argv[1]
    units = float(sys.argv[2]) if len(sys.argv) > 2 else None
    print(summary(rep, units, sys.argv[3] if len(sys.argv) > 3 else ""))

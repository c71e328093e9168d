"""Stall / pipe summary of an ncu report (run here on the .ncu-rep)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for row in rows[2:]:
    d = dict(zip(h, row))
    print("==", d.get("Kernel Name", "")[:90], d.get("gpu__time_duration.sum", ""))
    for k, v in d.items():
        if (("average_warps_issue_stalled" in k and "not_issued" not in k) or k in (
                "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
                "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "smsp__warps_eligible.avg.per_cycle_active",
                "sm__warps_active.avg.pct_of_peak_sustained_active",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                "smsp__inst_executed.sum")):
            try:
                if float(v) > 0.01:
                    print(f"  {k.replace('smsp__average_warps_issue_stalled_', 'stall_').replace('_per_issue_active.ratio', '')}: {v}")
            except ValueError:
                pass
